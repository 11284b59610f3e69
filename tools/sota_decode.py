"""Decode attention of G rollouts that share one long prompt: NVIDIA's
trtllm-gen decode kernel (flashinfer's precompiled sm100a cubins) with every
row's page table pointing at the same prompt pages — the best case of a paged
serving engine with prefix caching — for comparison with the engine's
shared-prefix decode attention (dev tool, not product code).

One layer of c4: 131,109 prompt keys, 28 query / 4 KV heads, hd 128, bf16,
G = 8 rows. Prints CUDA-event time per call; run it under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none`
to compare with the engine's decode launch list (tools/prof_gen_graph.sh).

  python tools/sota_decode.py [G] [Lp]
"""
import json
import math
import sys

import torch

NQ, NKV, HD = 28, 4, 128


def main(G=8, Lp=131109, iters=20):
    import flashinfer
    torch.manual_seed(0)
    page = 64
    n_pages = (Lp + page - 1) // page
    k = torch.randn(n_pages, NKV, page, HD, device="cuda").bfloat16()
    v = torch.randn(n_pages, NKV, page, HD, device="cuda").bfloat16()
    q = torch.randn(G, NQ, HD, device="cuda").bfloat16()
    bt = torch.arange(n_pages, device="cuda", dtype=torch.int32).repeat(G, 1)  # shared prompt pages
    sl = torch.full((G,), Lp, device="cuda", dtype=torch.int32)
    ws = torch.zeros(256 << 20, device="cuda", dtype=torch.uint8)
    out = torch.empty(G, NQ, HD, device="cuda", dtype=torch.bfloat16)
    call = lambda: flashinfer.decode.trtllm_batch_decode_with_kv_cache(
        q, (k, v), ws, bt, sl, Lp, bmm1_scale=1 / math.sqrt(HD), bmm2_scale=1.0, out=out,
        kv_layout="HND")
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        call()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / iters * 1e3
    kv_bytes = 2 * Lp * NKV * HD * 2
    print(json.dumps({"kernel": "trtllm-gen decode, shared prompt pages", "G": G, "prompt_keys": Lp,
                      "us_per_layer": round(us, 1), "prompt_kv_bytes": kv_bytes,
                      "unique_kv_TBps": round(kv_bytes / us / 1e6, 2)}), flush=True)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
