# A/B of two builds on the per-config subsets: lib/ (current) vs lib_base/ (saved previous build)
mkdir -p gpurun_out
{
for i in 1 2; do
for cfg in "50 21 0 1 50" "21 8 0 1 10" "23 9 0 1 20"; do
  timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -1 | sed 's/^/NEW /'
  PMS8G_LIB=$PWD/paper_1307_0571_b200/lib_base/libpms8g.so timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -1 | sed 's/^/OLD /'
done
done
} > gpurun_out/ab.txt 2>&1
echo done
