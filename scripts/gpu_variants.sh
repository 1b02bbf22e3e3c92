# A/B of build variants (lib_<name>/) against lib/ on the configs in CFGS
mkdir -p gpurun_out
{
for i in 1 2; do
IFS=";" read -ra CF <<< "${CFGS:-21 8 0 1 10;23 9 0 1 20}"; for cfg in "${CF[@]}"; do
  for v in "" $VARIANTS; do
    L=$PWD/paper_1307_0571_b200/lib${v:+_$v}/libpms8g.so
    PMS8G_LIB=$L timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -2 | cut -c1-200 | sed "s/^/[${v:-base}] /"
  done
done
done
} > gpurun_out/variants.txt 2>&1
