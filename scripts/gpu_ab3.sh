# A/B of two builds (lib/ = new, lib_base/ = previous) + parity of the affected paths (+ ncu of the (50,21) subset with NCU50=1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTS:-50_21 or deep_switch or long_motifs or large_instances or threshold_invariance or small_random or wraparound or 17_6 or 21_8 or jitter or shared_queue}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
{
for i in 1 2; do
for cfg in "50 21 0 1 50" "50 21 0 1 10" "21 8 0 1 10" "23 9 0 1 20" "17 6 0 1 1"; do
  timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -3 | sed 's/^/NEW /'
  if [ -z "$NOBASE" ]; then PMS8G_LIB=$PWD/paper_1307_0571_b200/lib_base/libpms8g.so timeout 300 python scripts/profile_run.py $cfg 2>&1 | head -1 | sed 's/^/OLD /'; fi
done
done
} > gpurun_out/ab.txt 2>&1
if [ -n "$NCU50" ]; then
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02n_search_50_21_s50 -f \
  python scripts/profile_run.py 50 21 0 1 50 > gpurun_out/ncu_50_21.log 2>&1
fi
echo done
