# Round-2 evidence: bench lines for the other configs (N = 1), the ncu launch
# list of one c4 step, and one --set full capture of the c4 attention launch.
mkdir -p gpurun_out
for wl in c2 c3 c5; do
  timeout 900 python bench.py --workload $wl --no-cpu --no-gen --no-bwd > gpurun_out/bench_$wl.log 2>&1
  echo "bench $wl rc=$?"; tail -1 gpurun_out/bench_$wl.log | cut -c1-200
done
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -c 2500 --csv --log-file gpurun_out/r2_launches_c4_step.csv \
  python tools/step_probe.py c4 1 > gpurun_out/ncu_step.log 2>&1
echo "launch list rc=$?"
python tools/ncu_summary.py gpurun_out/r2_launches_c4_step.csv 20 > gpurun_out/r2_launches_c4_step_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 1 \
  -o gpurun_out/attn_full_r2 -f python tools/ncu_kernels.py attn > gpurun_out/ncu_attn_full_r2.log 2>&1
echo "attn full rc=$?"
ncu -i gpurun_out/attn_full_r2.ncu-rep --page raw --csv > gpurun_out/r2_ncu_attention_c4_raw.csv 2>/dev/null
cat gpurun_out/r2_launches_c4_step_summary.txt
