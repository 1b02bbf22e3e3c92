# A/B of builds on whole instances: lib/ = new, lib_base/ = previous, optional VARIANTS="lib_g ..." = extra variants
# (make EXTRA=-D... LIB=.../lib_g BIN=.../bin_g) + parity of the affected paths through lib/
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTS:-50_21 or deep_switch or long_motifs or large_instances or whole_heavy or more_than_32}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
{
for i in 1 2 3; do
for cfg in "50 21 0 1 1" "50 21 0 1 10"; do
  timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -1 | sed 's/^/NEW /'
  for v in $VARIANTS lib_base; do
    PMS8G_LIB=$PWD/paper_1307_0571_b200/$v/libpms8g.so timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -1 | sed "s/^/$v /"
  done
done
done
} > gpurun_out/ab.txt 2>&1
echo done
