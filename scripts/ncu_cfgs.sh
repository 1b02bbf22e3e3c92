# ncu source-level captures of the search kernel on anchor subsets of (21,8) and (23,9)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/search_21_8_s10 -f \
  python scripts/profile_run.py 21 8 0 1 10 > gpurun_out/ncu_21_8.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/search_23_9_s20 -f \
  python scripts/profile_run.py 23 9 0 1 20 > gpurun_out/ncu_23_9.log 2>&1
