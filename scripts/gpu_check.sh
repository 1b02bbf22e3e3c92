# GPU pass after a change: scanner tests, then an ncu --set full capture of
# the (17,6) search kernel (one launch) for the roofline's traffic figure.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py -x -q > gpurun_out/gpu_scan.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_scan.log
timeout 300 python scripts/scan_bench.py > gpurun_out/scan_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -c 1 \
  -o gpurun_out/search_17_6_full -f python bench.py --steps 1 --warmup 0 > gpurun_out/ncu_full.log 2>&1
echo done
