# GPU tests + per-config timings + default bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
{
for cfg in "50 21 0 1 50" "50 21 0 1 50" "21 8 0 1 10" "23 9 0 1 20" "17 6 0 2" "13 4 0 2"; do
  timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -3 | grep -v histogram
done
PMS8G_GLOBAL_TABLE=1 timeout 300 python scripts/profile_run.py 17 6 0 2 2>&1 | head -1
} > gpurun_out/prof.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo done
