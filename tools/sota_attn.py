"""Same-box comparison of the attention kernel against NVIDIA's trtllm-gen
FMHA (flashinfer's precompiled sm100a cubins) — dev tool, not product code.

Plain causal self-attention, 28 query / 4 KV heads, head dim 128, bf16, one
sequence of L tokens (the MR-SP prefix is plain causal: 94% of c4's attention
FLOPs). The two kernels run interleaved (A B A B ...) so they see the same
clocks; each line reports CUDA-event time and causal FLOP rate, plus the
max |difference| of the outputs.

  python tools/sota_attn.py [L ...]
  python tools/sota_attn.py --power [L ...]   # ~6 s sustained per kernel, NVML
                                              # SM clock / power, TFLOP/s per GHz
"""
import json
import math
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch

from paper_2507_07966_b200 import ops

NQ, NKV, HD = 28, 4, 128


def timed(f, iters):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def run(L, rounds=3):
    import flashinfer
    torch.manual_seed(0)
    qkv = torch.randn(L, (NQ + 2 * NKV) * HD, device="cuda").bfloat16()
    scale = 1 / math.sqrt(HD)
    out = torch.empty(L, NQ * HD, device="cuda", dtype=torch.bfloat16)
    ours = lambda: ops.attention(qkv, 0, qkv, NQ * HD, qkv, (NQ + NKV) * HD, L, NQ, NQ // NKV,
                                 scale, 0, L, 0, 0, out=out)
    # trtllm-gen: query [L, H, D]; K/V paged HND [pages, kv_heads, page, D]
    page = 64
    n_pages = (L + page - 1) // page
    q = qkv[:, : NQ * HD].reshape(L, NQ, HD).contiguous()

    def paged(col0):
        x = qkv[:, col0 : col0 + NKV * HD].reshape(L, NKV, HD)
        pad = torch.zeros(n_pages * page, NKV, HD, device="cuda", dtype=torch.bfloat16)
        pad[:L] = x
        return pad.reshape(n_pages, page, NKV, HD).permute(0, 2, 1, 3).contiguous()

    kc, vc = paged(NQ * HD), paged((NQ + NKV) * HD)
    ws = torch.zeros(256 << 20, device="cuda", dtype=torch.uint8)
    bt = torch.arange(n_pages, device="cuda", dtype=torch.int32).reshape(1, n_pages)
    sl = torch.tensor([L], device="cuda", dtype=torch.int32)
    cu = torch.tensor([0, L], device="cuda", dtype=torch.int32)
    o2 = torch.empty(L, NQ, HD, device="cuda", dtype=torch.bfloat16)
    trt = lambda: flashinfer.prefill.trtllm_batch_context_with_kv_cache(
        q, (kc, vc), ws, bt, sl, L, L, scale, 1.0, 1, cu, cu, out=o2, kv_layout="HND",
        causal=True)
    ours()
    trt()
    torch.cuda.synchronize()
    diff = (out.float().reshape(L, NQ, HD) - o2.float()).abs().max().item()
    flops = 4 * HD * NQ * L * L / 2
    iters = 2 if L > 65536 else 5
    res = {"ours": [], "trtllm_gen": []}
    for _ in range(rounds):
        res["ours"].append(timed(ours, iters))
        res["trtllm_gen"].append(timed(trt, iters))
    line = {"L": L, "max_abs_diff": diff}
    for k, v in res.items():
        ms = min(v)
        line[k] = {"ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1),
                   "all_ms": [round(x, 3) for x in v]}
    line["ratio_ours_over_trtllm"] = round(line["trtllm_gen"]["ms"] / line["ours"]["ms"], 3)
    print(json.dumps(line), flush=True)


def sustained(f, flops, seconds=6.0):
    """Run f back to back for ~`seconds` while NVML samples SM clock and board
    power: TFLOP/s, median clock, median power, and TFLOP/s per GHz (the
    per-clock efficiency, separating power-cap clock loss from scheduling)."""
    import statistics
    import threading
    import time
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.02)
    ms1 = timed(f, 2)
    n = max(3, int(seconds * 1000 / ms1))
    th = threading.Thread(target=sampler)
    th.start()
    ms = timed(f, n)
    stop.set()
    th.join()
    clk = statistics.median(c for c, _ in samples)
    pw = statistics.median(p for _, p in samples)
    tf = flops / ms / 1e9
    return {"ms": round(ms, 3), "tflops": round(tf, 1), "sm_mhz": clk, "power_w": round(pw, 1),
            "tflops_per_ghz": round(tf / (clk / 1000.0), 1), "iters": n}


def run_power(L):
    import flashinfer
    torch.manual_seed(0)
    qkv = torch.randn(L, (NQ + 2 * NKV) * HD, device="cuda").bfloat16()
    scale = 1 / math.sqrt(HD)
    out = torch.empty(L, NQ * HD, device="cuda", dtype=torch.bfloat16)
    ours = lambda: ops.attention(qkv, 0, qkv, NQ * HD, qkv, (NQ + NKV) * HD, L, NQ, NQ // NKV,
                                 scale, 0, L, 0, 0, out=out)
    page = 64
    n_pages = (L + page - 1) // page
    q = qkv[:, : NQ * HD].reshape(L, NQ, HD).contiguous()

    def paged(col0):
        x = qkv[:, col0 : col0 + NKV * HD].reshape(L, NKV, HD)
        pad = torch.zeros(n_pages * page, NKV, HD, device="cuda", dtype=torch.bfloat16)
        pad[:L] = x
        return pad.reshape(n_pages, page, NKV, HD).permute(0, 2, 1, 3).contiguous()

    kc, vc = paged(NQ * HD), paged((NQ + NKV) * HD)
    ws = torch.zeros(256 << 20, device="cuda", dtype=torch.uint8)
    bt = torch.arange(n_pages, device="cuda", dtype=torch.int32).reshape(1, n_pages)
    sl = torch.tensor([L], device="cuda", dtype=torch.int32)
    cu = torch.tensor([0, L], device="cuda", dtype=torch.int32)
    o2 = torch.empty(L, NQ, HD, device="cuda", dtype=torch.bfloat16)
    trt = lambda: flashinfer.prefill.trtllm_batch_context_with_kv_cache(
        q, (kc, vc), ws, bt, sl, L, L, scale, 1.0, 1, cu, cu, out=o2, kv_layout="HND",
        causal=True)
    flops = 4 * HD * NQ * L * L / 2
    for rnd in range(2):
        for name, f in (("ours", ours), ("trtllm_gen", trt)):
            r = sustained(f, flops)
            r.update(L=L, kernel=name, round=rnd)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--power":
        for L in [int(x) for x in args[1:]] or [16384, 32768, 131109]:
            run_power(L)
    else:
        for L in [int(x) for x in args] or [16384, 32768, 131109]:
            run(L)
