# Round-2 baseline pass: GPU tests, (50,21) stride-50 line, ncu --set full of the
# (50,21) and (21,8) search kernels on anchor subsets (final round-1 build).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --config 50_21 --sample-stride 50 --steps 3 --no-cpu-baseline > gpurun_out/b50_s50.json 2> gpurun_out/b50_s50.err
timeout 300 python scripts/profile_run.py 50 21 0 1 50 > gpurun_out/prof50.txt 2>&1
timeout 300 python scripts/profile_run.py 21 8 0 1 10 > gpurun_out/prof21.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02base_search_50_21_s50 -f \
  python scripts/profile_run.py 50 21 0 1 50 > gpurun_out/ncu_50.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02base_search_21_8_s10 -f \
  python scripts/profile_run.py 21 8 0 1 10 > gpurun_out/ncu_21.log 2>&1
echo done
