# A/B: DSMEM cluster table vs global table for W=2; switch-depth sweeps with consensus rows
mkdir -p gpurun_out
{
for i in 1 2 3; do
  timeout 300 python scripts/profile_run.py 50 21 0 1 50 | head -1
  PMS8G_GLOBAL_TABLE=1 timeout 300 python scripts/profile_run.py 50 21 0 1 50 | head -1
done
for t in 5 6; do timeout 300 python scripts/profile_run.py 50 21 $t 1 50 | head -1; done
for t in 4 5; do timeout 300 python scripts/profile_run.py 21 8 $t 1 10 | head -1; done
for t in 4 5; do timeout 300 python scripts/profile_run.py 23 9 $t 1 20 | head -1; done
for t in 3 4; do timeout 300 python scripts/profile_run.py 17 6 $t 2 | head -1; done
timeout 300 python scripts/profile_run.py 21 8 4 1 10 | head -1
PMS8G_GLOBAL_TABLE=1 timeout 300 python scripts/profile_run.py 21 8 4 1 10 | head -1
} > gpurun_out/ab.txt 2>&1
echo done
