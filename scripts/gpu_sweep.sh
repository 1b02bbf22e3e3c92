# donation-parameter sweep on the (50,21) every-10th-S1 subset (and one (23,9) line each)
mkdir -p gpurun_out
{
for dg in 1 8; do for dp in 32 4; do
  echo "== PMS8G_DON_GEN=$dg PMS8G_DON_PUSHES=$dp"
  PMS8G_DON_GEN=$dg PMS8G_DON_PUSHES=$dp timeout 300 python scripts/profile_run.py 50 21 0 1 10 2>&1 | grep -v "histogram\|long task" | cut -c1-300
done; done
for dp in 4; do
  echo "== PMS8G_DON_PUSHES=$dp"
  PMS8G_DON_PUSHES=$dp timeout 300 python scripts/profile_run.py 23 9 0 1 20 2>&1 | grep -v "histogram\|long task" | cut -c1-300
  PMS8G_DON_PUSHES=$dp timeout 300 python scripts/profile_run.py 21 8 0 1 10 2>&1 | grep -v "histogram\|long task" | cut -c1-300
  PMS8G_DON_PUSHES=$dp timeout 300 python scripts/profile_run.py 17 6 0 1 1 2>&1 | grep -v "histogram\|long task" | cut -c1-300
done
} > gpurun_out/sweep.txt 2>&1
