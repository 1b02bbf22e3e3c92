# Round-2 pass: GPU tests, per-config timings of the current build, ncu of
# the (50,21) search kernel on three S1 l-mers, the default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
{
timeout 300 python scripts/profile_run.py 50 21 0 1 50
timeout 300 python scripts/profile_run.py 21 8 0 1 10
timeout 300 python scripts/profile_run.py 23 9 0 1 20
timeout 300 python scripts/profile_run.py 17 6 0 2
} > gpurun_out/prof.txt 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02b_search_50_21_s200 -f \
  python scripts/profile_run.py 50 21 0 1 200 > gpurun_out/ncu_50.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo done
