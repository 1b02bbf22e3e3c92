# End-of-round measurement: tests, smoke, bench lines for every config, the
# reference arm, launch list, (50,21) branch comparison.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 bash scripts/bench_all.sh ${TAG:-r01f} > gpurun_out/bench_all.log 2>&1
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_17_6.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 python bench.py --config 50_21 --steps 2 > gpurun_out/bench_${TAG:-r01f}_50_21.json 2> gpurun_out/bench_50.err
timeout 900 python scripts/branch_compare_50_21.py 0,1,2,3 > gpurun_out/bc50.json 2> gpurun_out/bc50.err
echo done
