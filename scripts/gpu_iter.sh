# Iteration pass: profile_run timings for the 4 bench configs (with and
# without row tracking), then the full GPU test suite.
mkdir -p gpurun_out
{
for cfg in "13 4" "17 6" "21 8" "23 9"; do
  timeout 300 python scripts/profile_run.py $cfg 0 2 2>&1 | head -2
  PMS8G_NO_ROWTRACK=1 timeout 300 python scripts/profile_run.py $cfg 0 2 2>&1 | head -2
done
} > gpurun_out/iter.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
