# A/B timing of two builds on per-config subsets: A = lib_base (saved previous
# build), B = lib (current). usage: bash scripts/ab2.sh  -> gpurun_out/ab2.txt
mkdir -p gpurun_out
A=paper_1307_0571_b200/lib_base/libpms8g.so
B=paper_1307_0571_b200/lib/libpms8g.so
{
for rep in 1 2; do
for cfg in "21 8 0 2 10" "23 9 0 2 20" "17 6 0 3 1" "50 21 0 2 50" "13 4 0 5 1"; do
  PMS8G_LIB=$A timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -1 | sed 's/^/A /' | cut -c1-100
  PMS8G_LIB=$B timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -1 | sed 's/^/B /' | cut -c1-100
done
done
} > gpurun_out/ab2.txt 2>&1
echo done
