# Round-2 re-entry pass: GPU tests, default bench line, per-config lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_50_21.json 2> gpurun_out/bench_50_21.err
for c in 21_8 23_9; do timeout 900 python bench.py --config $c --steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in 17_6 13_4; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
echo done
