mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "deep_switch or threshold_invariance or 50_21" > gpurun_out/pytest_t7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t7.log
{
for t in 6 7; do
  timeout 300 python scripts/profile_run.py 50 21 $t 1 10 2>&1 | grep -v "histogram\|long task" | cut -c1-400
done
timeout 300 python scripts/profile_run.py 50 21 7 1 50 2>&1 | grep -v "histogram\|long task" | cut -c1-400
} > gpurun_out/t7.txt 2>&1
