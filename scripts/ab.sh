# A/B timing of two builds: LIBA (default lib/libpms8g_base.so) against LIBB
# (default lib/libpms8g.so). usage: bash scripts/ab.sh "17 6" "13 4" ...
mkdir -p gpurun_out
A=${LIBA:-paper_1307_0571_b200/lib/libpms8g_base.so}
B=${LIBB:-paper_1307_0571_b200/lib/libpms8g.so}
for cfg in "$@"; do
  for rep in 1 2; do
    PMS8G_LIB=$A timeout 300 python scripts/profile_run.py $cfg 0 2 2>&1 | head -1 | sed 's/^/A /' | cut -c1-90
    PMS8G_LIB=$B timeout 300 python scripts/profile_run.py $cfg 0 2 2>&1 | head -1 | sed 's/^/B /' | cut -c1-90
  done
done
