# Round-2 final pass (session 4): GPU tests, default bench line (whole (50,21) instance) + reference arm,
# per-config lines, launch list of the default bench command, ncu --set full of the (50,21) search kernel on
# the 56-S1-l-mer subset and the quoted metrics on the whole-instance launch
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/p_smoke.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/p_bench_50_21_nocpu.json 2> gpurun_out/p_bench_50_21.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k regex:search_kernel -c 1 --csv --page raw --log-file gpurun_out/p_ncu_50_21_whole.csv \
  python scripts/profile_run.py 50 21 0 1 1 > gpurun_out/p_ncu_50_21_whole.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02p_search_50_21 -f \
  python scripts/profile_run.py 50 21 0 1 10 > gpurun_out/p_ncu_50_21.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches_50_21.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p_ncu_launches.log 2>&1
timeout 900 python bench.py --config 50_21 --sample-stride 10 --no-cpu-baseline > gpurun_out/p_bench_50_21_s10.json 2>> gpurun_out/p_bench_50_21.err
for c in 21_8 23_9; do timeout 900 python bench.py --config $c --steps 3 > gpurun_out/p_bench_$c.json 2> gpurun_out/p_bench_$c.err; done
for c in 17_6 13_4; do timeout 600 python bench.py --config $c > gpurun_out/p_bench_$c.json 2> gpurun_out/p_bench_$c.err; done
echo done
