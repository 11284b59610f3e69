# round-end evidence: ncu --set full of the c4 attention launch and of the
# SwiGLU GEMM, plus the HBM-kernel launch list (tools/prof_hbm.sh)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 1 \
  -o gpurun_out/attn_full -f python tools/ncu_kernels.py attn > gpurun_out/ncu_attn_full.log 2>&1
ncu -i gpurun_out/attn_full.ncu-rep --page raw --csv > gpurun_out/attn_full_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:gemm_bf16 -c 1 \
  -o gpurun_out/gemm_full -f python tools/ncu_kernels.py gemm > gpurun_out/ncu_gemm_full.log 2>&1
ncu -i gpurun_out/gemm_full.ncu-rep --page raw --csv > gpurun_out/gemm_full_raw.csv 2>/dev/null
bash tools/prof_hbm.sh
ls -la gpurun_out
