# Round-2 (session 4): whole-instance (50,21) search kernel under ncu with the few metrics the
# bench line quotes (a --set full replay of the 2.3 s kernel exceeds 20 min: 37 passes with
# save/restore of the scratch), whole-instance counters of (21,8)/(23,9), ncu --set full of (23,9)
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k regex:search_kernel -c 1 --csv --page raw --log-file gpurun_out/o_ncu_50_21_whole.csv \
  python scripts/profile_run.py 50 21 0 1 1 > gpurun_out/o_ncu_50_21_whole.log 2>&1
for cfg in "21 8 0 1 1" "23 9 0 1 1"; do timeout 300 python scripts/profile_run.py $cfg 2>&1 | grep -v "long task" > gpurun_out/o_prof_$(echo $cfg | cut -d' ' -f1-2 | tr ' ' _).txt; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 1 -o gpurun_out/r02o_search_23_9_s20 -f \
  python scripts/profile_run.py 23 9 0 1 20 > gpurun_out/o_ncu_23_9.log 2>&1
echo done
