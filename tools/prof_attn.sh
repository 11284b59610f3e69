# Attention profiling pass: MUFU microbench, CUDA-event throughput, one
# source-level ncu capture of the c4-shaped attention launch.
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mufu tools/ubench/mufu.cu && ./gpurun_out/mufu
timeout 600 python tools/attn_perf.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 1 \
  -o gpurun_out/attn_src -f python tools/ncu_kernels.py attn > gpurun_out/ncu_attn.log 2>&1
tail -3 gpurun_out/ncu_attn.log
