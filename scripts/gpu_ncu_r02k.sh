# ncu --set full (source-level) of the current search kernel: (21,8) every-10th S1 l-mer
# subset, whole (17,6) instance; per-config profile_run counters (clock split)
mkdir -p gpurun_out
for cfg in "21 8 0 1 10" "17 6 0 1 1" "50 21 0 1 50"; do timeout 300 python scripts/profile_run.py $cfg > gpurun_out/prof_$(echo $cfg | cut -d' ' -f1-2 | tr ' ' _).txt 2>&1; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02k_search_21_8_s10 -f \
  python scripts/profile_run.py 21 8 0 1 10 > gpurun_out/ncu_21_8.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02k_search_17_6 -f \
  python scripts/profile_run.py 17 6 0 1 1 > gpurun_out/ncu_17_6.log 2>&1
echo done
