# donation-parameter sweep on WHOLE instances (the earlier sweeps ran subsets, whose tails differ)
mkdir -p gpurun_out
{
for dp in 4 2 8 16; do
  for cfg in "50 21" "21 8" "23 9"; do
    echo "== PMS8G_DON_PUSHES=$dp ($cfg)"
    PMS8G_DON_PUSHES=$dp timeout 300 python scripts/profile_run.py $cfg 0 2 1 2>&1 | grep -v "histogram\|long task" | cut -c1-200 | head -3
  done
done
for dg in 4 16; do
  echo "== PMS8G_DON_GEN=$dg (50 21)"
  PMS8G_DON_GEN=$dg timeout 300 python scripts/profile_run.py 50 21 0 2 1 2>&1 | grep -v "histogram\|long task" | cut -c1-200 | head -1
done
for cc in 1 8; do
  echo "== PMS8G_CLAIM_CHUNK=$cc (50 21)"
  PMS8G_CLAIM_CHUNK=$cc timeout 300 python scripts/profile_run.py 50 21 0 2 1 2>&1 | grep -v "histogram\|long task" | cut -c1-200 | head -1
done
} > gpurun_out/sweep_whole.txt 2>&1
