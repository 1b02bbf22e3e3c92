# Round-2 (session 3) pass: GPU tests, default bench line + reference arm, per-config lines,
# launch list of the default bench command, ncu --set full of its search kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_50_21.json 2> gpurun_out/bench_50_21.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_50_21.json 2> gpurun_out/bench_ref_50_21.err
for c in 21_8 23_9; do timeout 900 python bench.py --config $c --steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in 17_6 13_4; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_50_21.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02m_search_50_21 -f \
  python scripts/profile_run.py 50 21 0 1 10 > gpurun_out/ncu_50_21.log 2>&1  # the bench step's workload (every 10th S1 offset)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02m_search_21_8_s10 -f \
  python scripts/profile_run.py 21 8 0 1 10 > gpurun_out/ncu_21_8.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02m_search_17_6 -f \
  python scripts/profile_run.py 17 6 0 1 1 > gpurun_out/ncu_17_6.log 2>&1
for cfg in "21 8 0 1 10" "17 6 0 1 1" "23 9 0 1 20" "50 21 0 1 1"; do timeout 300 python scripts/profile_run.py $cfg > gpurun_out/prof_$(echo $cfg | cut -d' ' -f1-2 | tr ' ' _).txt 2>&1; done
PMS8G_LIB=$PWD/paper_1307_0571_b200/lib_diag/libpms8g.so timeout 300 python scripts/profile_run.py 50 21 0 1 10 2>&1 | grep -v histogram > gpurun_out/levels.txt  # -DPMS8G_LEVELSTATS build (make EXTRA=-DPMS8G_LEVELSTATS LIB=.../lib_diag)
echo done
