# Round-2 (session 4) pass: whole-instance (50,21) bench (the new default), reference arm,
# launch list of the default bench command, ncu --set full of its search kernel
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/n_bench_50_21.json 2> gpurun_out/n_bench_50_21.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/n_bench_ref_50_21.json 2> gpurun_out/n_bench_ref_50_21.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/n_launches_50_21.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/n_ncu_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02n_search_50_21 -f \
  python scripts/profile_run.py 50 21 0 1 1 > gpurun_out/n_ncu_50_21.log 2>&1
echo done
