# ncu of one c4-shaped attention launch per kernel generation (dev tool)
for impl in 2 4; do
  MRSP_ATTN_IMPL=$impl MRSP_ATTN_POLY=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:attn_fwd -c 1 --csv python tools/ncu_kernels.py attn > gpurun_out/ncu_impl$impl.csv 2>&1
  grep -E "attn_fwd" gpurun_out/ncu_impl$impl.csv | awk -F'","' '{print $(NF-3), $(NF-2), $(NF-1), $NF}'
done
