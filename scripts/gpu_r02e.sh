# timings of the current build per config (+ t=3 consensus experiment); ncu (50,21)
mkdir -p gpurun_out
{
for cfg in "50 21 0 1 50" "21 8 0 1 10" "23 9 0 1 20" "17 6 0 2" "13 4 0 2"; do
  timeout 300 python scripts/profile_run.py $cfg | grep -v histogram
done
PMS8G_CONS3=1 timeout 300 python scripts/profile_run.py 17 6 0 2 | grep -v histogram
PMS8G_CONS3=1 timeout 300 python scripts/profile_run.py 13 4 3 2 | grep -v histogram
timeout 300 python scripts/profile_run.py 13 4 3 2 | grep -v histogram
} > gpurun_out/prof.txt 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02e_search_50_21_s200 -f \
  python scripts/profile_run.py 50 21 0 1 200 > gpurun_out/ncu_50.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
echo done
