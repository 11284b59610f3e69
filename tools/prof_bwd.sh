# ncu evidence for the GRPO backward (tools/bwd_perf.py, one warm-up call, no
# timed reps): the launch list of the whole call at c2 (per-kernel durations)
# and one --set full capture of each attention-backward kernel.
mkdir -p gpurun_out
W=${WORKLOAD:-c2}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -c 4000 --csv --log-file gpurun_out/ncu_bwd_launches_$W.csv \
  env WORKLOAD=$W REPS=0 python tools/bwd_perf.py > gpurun_out/ncu_bwd_run.log 2>&1
echo "launch list rc=$?"
python tools/ncu_summary.py gpurun_out/ncu_bwd_launches_$W.csv > gpurun_out/ncu_bwd_summary_$W.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_d -c 2 \
  -o gpurun_out/attn_bwd_full_$W -f env WORKLOAD=$W REPS=0 python tools/bwd_perf.py > gpurun_out/ncu_bwd_full.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/attn_bwd_full_$W.ncu-rep --page raw --csv > gpurun_out/attn_bwd_full_raw_$W.csv 2>/dev/null
