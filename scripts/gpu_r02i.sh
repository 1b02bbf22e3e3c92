# Measurement pass on the current build: default bench line (50,21), the launch
# list of the same command, ncu --set full of its search kernel, per-config lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_50_21.json 2> gpurun_out/bench_50_21.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_50_21.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_search_50_21_bench -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
for c in 21_8 23_9; do timeout 900 python bench.py --config $c --steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in 17_6 13_4; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
echo done
