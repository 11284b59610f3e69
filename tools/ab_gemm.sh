# same-box A/B of the GEMM kernel choice on the c4 step (dev tool)
for impl in 1 3 1 3; do
  MRSP_GEMM_IMPL=$impl timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/ab_$impl.log 2>&1
  python - "$impl" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("gemm impl", sys.argv[1], "tok/s", round(d["value"]), "attn_ms", d["kernel_ms"]["llm_attention"],
      "gemm_ms", d["kernel_ms"]["llm_gemm"], "clk", d["clocks"]["sm_mhz"])
PY
done
