# ncu --set full of the decode-step kernels of a c4 generation (dev tool): the
# two-stream tcgen05 decode attention, the gate/up G-row GEMM and the residual
# reduction + RMSNorm cluster kernel, from the first graph-replayed step.
bash tools/prof_gen_graph.sh >/dev/null 2>&1 || true   # writes /tmp/gen4.py
for spec in "dec_attn_tc:28:attn" "splitk_reduce_resid_norm:56:resid_norm"; do
  IFS=: read k skip tag <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip $skip -c 1 \
    -o gpurun_out/dec_$tag -f python /tmp/gen4.py > gpurun_out/ncu_dec_$tag.log 2>&1
  ncu -i gpurun_out/dec_$tag.ncu-rep --page raw --csv > gpurun_out/dec_${tag}_raw.csv 2>/dev/null
done
# gate/up GEMM of a decode step: grid 148, after the prefill's launches
timeout 900 ncu --set full --clock-control none -k "regex:gemm_bf16_tcgen05" --launch-skip 500 -c 6 \
  -o gpurun_out/dec_gemm -f python /tmp/gen4.py > gpurun_out/ncu_dec_gemm.log 2>&1
ncu -i gpurun_out/dec_gemm.ncu-rep --page raw --csv > gpurun_out/dec_gemm_raw.csv 2>/dev/null
ls -la gpurun_out/ | grep dec_
