# ncu of the HBM-bound kernels of one c4 step (pack = the pad/sequence pack,
# norms, RoPE, patchify, log-prob combine / gather) — per-launch duration and
# DRAM bytes, for profiles/r1_hbm_kernels.md
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size \
  --clock-control none -k "regex:pack_kernel|rmsnorm|rope_kernel|combine|patchify|scatter3|broadcast_rows|grpo_stats" \
  -c 320 --csv --log-file gpurun_out/ncu_hbm.csv python tools/step_probe.py c4 1 > gpurun_out/ncu_hbm_run.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_hbm_run.log; wc -l gpurun_out/ncu_hbm.csv
