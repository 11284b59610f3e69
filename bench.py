#!/usr/bin/env python
"""MR-SP encode+prefill benchmark (BASELINE.json metric) on 1..8 B200.

One step = Stage 1 (a fresh video: sharded SigLIP-shaped encode + all-gather
into the device cache; the G rollout fetches then hit the cache) + Stage 2
(policy and reference Ulysses prefill of the packed GRPO group + fused LM-head
log-probs). Workload c4 of BASELINE.json (512 frames x 256 tokens, 28-layer
Qwen2.5-7B-shaped LLM, G = 8) split over N GPUs as SP = N (strong scaling).

  python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload c4]

Prints ONE JSON line on rank 0. Multi-GPU: one process per GPU under
torch.distributed.run (`--gpus N` without WORLD_SIZE re-executes itself that
way); the engine's exchanges go over CUDA-IPC peer memory (MRSP_COMM=nccl:
NCCL), the torch process group is host plumbing only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MR-SP step tokens/s (encode+prefill), 512 frames, 1/2/4/8 B200; % roofline"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled during the timed region."""

    def __init__(self, device_index: int, period: float = 0.2):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.dev, self._stop = period, device_index, threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for n, bit in names.items():
                    if mask & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        load = [s for s in self.samples if s > 300] or self.samples
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------- CPU baseline
def cpu_port_timing(w, group, budget_s: float = 20.0):
    """Time the CPU port (oracle/transformer.py, fp64 numpy over bf16-valued
    tensors, all host threads via BLAS) on a bounded sample of the same
    workload and extrapolate to one step with the algorithmic FLOP table."""
    import numpy as np
    from oracle import transformer as T
    c = T.Cfg.from_any(w.cfg)
    fl = T.step_flops(c, w.frames, w.n_question, group.lengths)
    rng = np.random.default_rng(0)
    timings = {}
    # (1) one SigLIP-shaped frame through the full tower + projector
    # weight VALUES do not change the port's arithmetic cost: fast random tensors
    # of the exact SigLIP-shaped shapes stand in for the counter-based init
    Wv = {}
    for k_, v_ in vision_shapes(c).items():
        Wv[k_] = (rng.random(v_, dtype=np.float32) - np.float32(0.5)) * np.float32(0.05)
        if k_.endswith("_w") and len(v_) == 1:
            Wv[k_] += np.float32(1.0)
    pix = rng.uniform(-1, 1, size=(1, 3 * c.image_size ** 2)).astype(np.float32)
    t = time.perf_counter()
    T.vision_forward(c, Wv, pix)
    timings["vision_frame_s"] = time.perf_counter() - t
    del Wv
    # (2) one 7B-shaped decoder layer (linear part) over a 512-token slice
    n = 512
    d, hd, nq, nkv = c.dim, c.head_dim, c.n_q_heads, c.n_kv_heads
    rnd = lambda *shape: rng.random(shape, dtype=np.float32) - np.float32(0.5)
    x = rnd(n, d)
    wq, wo = rnd((nq + 2 * nkv) * hd, d), rnd(d, nq * hd)
    wg, wu, wd = rnd(c.mlp, d), rnd(c.mlp, d), rnd(d, c.mlp)
    t = time.perf_counter()
    xn = T.rmsnorm(x, np.ones(d, np.float32), 1e-6)
    T.linear(xn, wq)
    h = x + T.linear(T.bf16_round(rnd(n, nq * hd)), wo)
    xn = T.rmsnorm(h, np.ones(d, np.float32), 1e-6)
    act = T.bf16_round((T.silu(T.linear(xn, wg)) * T.linear(xn, wu)).astype(np.float32))
    T.linear(act, wd)
    timings["layer_linear_512tok_s"] = time.perf_counter() - t
    lin_flops = 2 * (d * (nq + 2 * nkv) * hd + nq * hd * d + 3 * d * c.mlp) * n
    del wq, wo, wg, wu, wd
    # (3) attention: 28 heads, 256 queries x 4096 keys
    q = rng.standard_normal((nq, 256, hd))
    k = rng.standard_normal((nkv, 4096, hd))
    mask = np.ones((256, 4096), dtype=bool)
    t = time.perf_counter()
    T.attention(q, k, k, mask, 1 / np.sqrt(hd))
    timings["attention_28h_256x4096_s"] = time.perf_counter() - t
    attn_flops = 4 * nq * 256 * 4096 * hd
    # (4) LM head block: 32 tokens x V
    xs = T.bf16_round(rnd(32, d))
    wl = rnd(c.vocab, d)
    t = time.perf_counter()
    T.linear(xs, wl)
    timings["lm_head_32tok_s"] = time.perf_counter() - t
    lm_flops = 2 * 32 * d * c.vocab
    del wl
    vis_per_flop = timings["vision_frame_s"] / (fl["encode"] / w.frames)
    lin_per_flop = timings["layer_linear_512tok_s"] / lin_flops
    attn_per_flop = timings["attention_28h_256x4096_s"] / attn_flops
    lm_per_flop = timings["lm_head_32tok_s"] / lm_flops
    step_s = (fl["encode"] * vis_per_flop + 2 * fl["linear"] * lin_per_flop
              + 2 * (fl["attn_prefix"] + fl["attn_resp"]) * attn_per_flop
              + 2 * fl["lm_head"] * lm_per_flop)
    cores = os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        cores = max((i.get("num_threads") or 0) for i in threadpool_info()) or cores
    except Exception:
        pass
    return {
        "value": fl["tokens"] / step_s, "unit": "tokens/s", "cores": cores, "kind": "port",
        **cpu_host(),
        "sample": ("oracle/transformer.py (fp64 numpy over bf16 tensors): 1 SigLIP-shaped frame "
                   "(27 layers + projector), 1 Qwen2.5-7B-shaped decoder layer (linear) on 512 "
                   "tokens, attention 28 heads x 256 q x 4096 k, LM head 32 tokens; extrapolated "
                   "to the full step by the SURVEY §8d FLOP table"),
        "extrapolated_step_s": step_s, "timings_s": timings,
    }


def vision_shapes(c):
    vd, kreal = c.v_dim, 3 * c.patch * c.patch
    sh = {"patch_w": (vd, kreal), "patch_b": (vd,), "pos": (c.T, vd), "post_w": (vd,),
          "post_b": (vd,), "p1_w": (c.dim, vd), "p1_b": (c.dim,), "p2_w": (c.dim, c.dim),
          "p2_b": (c.dim,)}
    for l in range(c.v_layers):
        p = f"vision.{l}."
        sh.update({p + "ln1_w": (vd,), p + "ln1_b": (vd,), p + "wqkv": (3 * vd, vd),
                   p + "bqkv": (3 * vd,), p + "wo": (vd, vd), p + "bo": (vd,), p + "ln2_w": (vd,),
                   p + "ln2_b": (vd,), p + "w1": (c.v_mlp, vd), p + "b1": (c.v_mlp,),
                   p + "w2": (vd, c.v_mlp), p + "b2": (vd,)})
    return sh


def reference_toy_engine():
    """The literal reference CPU engine (lvrl mrsp::bench, toy model) if built."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe, "512", "8", "1", "5", "2"], capture_output=True, text=True,
                             timeout=120, env={**os.environ, "OMP_NUM_THREADS": "8"})
        cell = json.loads(out.stdout.strip().splitlines()[-1])
        cell["note"] = ("reference lvrl mrsp::bench, toy model (1 token/frame, d 128), "
                        "512 frames sp 8 cache on, OpenMP threads = sp")
        return cell
    except Exception as e:  # informational only
        return {"error": str(e)}


def self_launch(n: int) -> int:
    """Re-executes this command as N ranks (torch.distributed.run, 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    return subprocess.call(cmd + sys.argv[1:])


def cpu_host():
    """Host CPU model (lscpu 'Model name') and logical core count."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.strip().startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# -------------------------------------------------------------- the bench
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gen", action="store_true", help="skip the rollout-generation side line")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-bwd", action="store_true", help="skip the GRPO-backward side line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        # `bench.py --gpus N` without a launcher: one process per GPU under
        # torch.distributed.run (rank 0 prints the line)
        sys.exit(self_launch(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "b200" and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")

    from paper_2507_07966_b200 import engine as E
    from oracle import transformer as T  # FLOP accounting (the algorithmic numerator)

    w = E.workloads()[args.workload]
    group = E.make_group(w, seed=3)
    fl = T.step_flops(T.Cfg.from_any(w.cfg), w.frames, w.n_question, group.lengths)
    peaks, peak_src = load_peaks()

    if args.impl == "reference":
        if rank != 0:
            return
        t0 = time.perf_counter()
        # each step is one bounded sample of the workload (cpu_port_timing:
        # ~8 s of the port's work on all host threads); W untimed samples, then
        # K timed ones. value = the step's tokens over the full-step time the
        # sample implies (FLOP table); ms_per_step = the sample's own wall time
        for _ in range(args.warmup):
            cpu_port_timing(w, group)
        times, walls = [], []
        base = None
        for _ in range(max(args.steps, 1)):
            ts = time.perf_counter()
            b = cpu_port_timing(w, group)
            walls.append(time.perf_counter() - ts)
            times.append(b["extrapolated_step_s"])
            base = base or b
        step_s = statistics.median(times)
        val = fl["tokens"] / step_s
        base["value"] = val
        base["extrapolated_step_s"] = step_s
        line = {
            "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(walls) * 1e3,
            "ms_per_step_note": "wall time of one bounded sample per step (cpu_baseline.sample); "
                                "value = the step's tokens over the full-step time the sample "
                                "implies by the SURVEY 8d FLOP table (cpu_baseline.extrapolated_step_s)",
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 (over bf16-valued tensors)",
            "data": "synthetic", "config": workload_config(w, group, fl, args.gpus),
            "cpu_baseline": base,
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "reference_toy_engine": reference_toy_engine(),
            "wall_s": time.perf_counter() - t0,
        }
        print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    # MRSP_BENCH_SAME_DEVICE=1 (tests): every rank on device 0 and a gloo host
    # group, so the multi-process flow runs on a one-GPU box
    same_dev = os.environ.get("MRSP_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    # Engine data path for N > 1: peer memory over NVLink (CUDA IPC, fused
    # QKV / attention scatters, device barrier) by default; MRSP_COMM=nccl
    # selects the NCCL all-gather / all-to-all path instead. The torch process
    # group is host plumbing only (blob exchange, barrier, max-over-ranks).
    comm = os.environ.get("MRSP_COMM", "p2p")
    nccl_id = None
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        if comm == "nccl":
            if same_dev:  # NCCL refuses two ranks on one GPU of one host: a host id
                # per rank puts them on its socket transport over loopback
                os.environ["NCCL_HOSTID"] = f"mrsp-bench-{rank}"
                os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
                os.environ.setdefault("NCCL_IB_DISABLE", "1")
            obj = [E.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
    from paper_2507_07966_b200 import _lib
    eng = E.Engine(w.cfg, sp=world, rank=rank, n_procs=world, vision_seed=2, policy_seed=3,
                   ref_seed=4, with_ref=True, nccl_id=nccl_id)
    if world > 1 and nccl_id is None:
        L = w.frames * w.cfg.tokens_per_frame + len(group.question) + group.resp.shape[0] * group.Lmax
        blob = eng.p2p_export(w.frames, L, group.scored)
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        eng.p2p_import(blobs)
    eng.cache_capacity(2)
    S = w.cfg.image_size
    pix_host = torch.from_numpy(E.gen_video(1, w.frames, 3 * S * S)).pin_memory()
    pix = pix_host.cuda()
    n_scored = group.scored
    lp_dev = tuple(torch.empty(n_scored, device="cuda") for _ in range(3))  # lp_policy, lp_ref, kl
    stream = torch.cuda.ExternalStream(eng.stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if same_dev else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    step_no = [0]

    def one_step(dev_inputs=True):
        vid = E.video_id(1000 + step_no[0], w.frames)  # fresh video -> Stage 1 runs every step
        step_no[0] += 1
        if dev_inputs:
            eng.step(vid, pix, group, out=lp_dev)
            return None
        return eng.step(vid, pix_host.numpy(), group, with_kl=True)  # host in, host out

    for _ in range(args.warmup):
        one_step()
    eng.stats(reset=True)

    # ---- device-resident timed region
    barrier()
    launches0 = int(_lib.lib().mrsp_launch_count())
    eng.profile(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            one_step(True)
        ev1.record(stream)
        ev1.synchronize()
        barrier()
    prof = eng.profile(False)
    launches = int(_lib.lib().mrsp_launch_count()) - launches0
    rank_ms = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(rank_ms)
    # per-rank device time by kernel class (imbalance across SP ranks)
    mine = {"rank": rank, "ms_per_step": round(rank_ms, 3),
            **{k: round(v[0] / args.steps, 2) for k, v in prof.items()}}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
        launches = int(max_over_ranks(float(launches)))
    stats = eng.stats(reset=True)
    value = fl["tokens"] / (ms / 1e3)

    # ---- end to end: host pixels (pinned) in, host log-probs out, copies timed
    e2e = None
    if not args.no_e2e:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_wall = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            lp_p, lp_r, kl = one_step(False)
        e1.record(stream)
        e1.synchronize()
        wall = (time.perf_counter() - t_wall) / args.steps * 1e3
        e2e_ms = max_over_ranks(max(e0.elapsed_time(e1) / args.steps, wall))
        frame_bytes = 3 * S * S * 4
        tok_bytes = 4 * (len(group.question) + group.resp.size + group.lengths.size)
        e2e = {"value": fl["tokens"] / (e2e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": w.frames * frame_bytes + 2 * world * tok_bytes,
               "d2h_bytes_per_step": 3 * world * n_scored * 4,
               "ms_per_step": e2e_ms,
               "note": "mrsp_engine_step with pinned host pixels in; host log-probs (policy, ref) and exact KL out"}

    # ---- roofline of the dominant kernel (LLM attention), live CUDA events
    attn_ms, attn_n = prof["llm_attention"]
    attn_flops_total = args.steps * 2 * (fl["attn_prefix"] + fl["attn_resp"]) / world
    per_launch_flops = attn_flops_total / max(attn_n, 1)
    achieved = per_launch_flops / (attn_ms / max(attn_n, 1) / 1e3) / 1e12 if attn_n else 0.0
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "attention_dram_bytes.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            # the capture is one launch of a given workload at SP = 1
            if tj.get("workload") == w.name and tj.get("world", 1) == world:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": "attn_fwd_tcgen05 (LLM layer attention)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": f"{peak_src} bf16_tflops_sustained",
                "launches": attn_n, "avg_launch_ms": attn_ms / max(attn_n, 1),
                "algorithmic_flops_per_launch": per_launch_flops,
                "share_of_step": attn_ms / (ms * args.steps)}
    step_tflops = fl["step"] / (ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": workload_config(w, group, fl, world),
        "comm": (("nccl" if nccl_id else "p2p: CUDA-IPC peer memory, fused QKV/attention "
                  "scatters") if world > 1 else "none (SP=1)"),
        "roofline": roofline,
        "step_roofline": {"flops_per_step": fl["step"], "achieved_tflops": step_tflops,
                          "frac_of_sustained": step_tflops / world / peak},
        "kernel_ms": {k: round(v[0] / args.steps, 2) for k, v in prof.items()},
        "kernel_launches": {k: v[1] for k, v in prof.items()},
        "kernel_ms_per_rank": per_rank if world > 1 else None,
        "e2e": e2e, "gpu_launches": launches, "counters_per_step":
            {k: v // args.steps for k, v in stats.items()},
    }
    if rank == 0:
        clocks = clk.summary()
        line["clocks"] = clocks
        if world == 1 and not args.no_cpu:
            try:
                line["cpu_baseline"] = cpu_port_timing(w, group)
            except Exception as e:
                line["cpu_baseline"] = {"error": str(e)}
        line["reference_toy_engine"] = reference_toy_engine() if world == 1 else None
        if world == 1 and not args.no_gen:
            try:
                line["rollout_generation"] = generation_side_line(eng, w, group, peaks, pix)
            except Exception as e:
                line["rollout_generation"] = {"error": str(e)}
    eng.close()
    if rank == 0:
        if world == 1 and not args.no_bwd:
            try:
                line["grpo_backward"] = backward_side_line(w, peaks)
            except Exception as e:
                line["grpo_backward"] = {"error": str(e)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def backward_side_line(w, peaks):
    """SURVEY §8f rank 3, not the metric: one GRPO gradient through the
    prefill (mrsp_engine_grpo_backward: reference + policy passes keeping the
    layer inputs, fused dual LM head, then the backward of the LM head and of
    every decoder layer recomputed from its kept input), on the same workload
    when its SP = 1 working set fits next to the gradients (c1-c4), else on c4
    (c5's 108 GB of fp32 layer inputs need SP > 1 across GPUs). Wall time of the call, device time of the
    backward kernels, and the attention-backward kernels' algorithmic TFLOP/s
    (2.5x the forward attention FLOPs: S, dP, dQ, dK, dV)."""
    import numpy as np
    from oracle import transformer as T
    from paper_2507_07966_b200 import engine as E
    name = w.name if w.name in ("c1", "c2", "c3", "c4") else "c4"
    wb = E.workloads()[name]
    c = T.Cfg.from_any(wb.cfg)
    eng = E.Engine(wb.cfg, sp=1)
    try:
        pix = E.gen_video(1, wb.frames, 3 * c.image_size ** 2)
        grp = E.make_group(wb, seed=3)
        vid = E.video_id(1, wb.frames)
        eng.encode(vid, pix)
        lp = eng.prefill_logprobs(vid, grp, 0)
        rng = np.random.default_rng(0)
        old = lp - rng.normal(0, 0.1, size=lp.shape).astype(np.float32)
        adv = rng.normal(0, 1, size=wb.G).astype(np.float32)
        eng.grpo_backward(vid, grp, old, adv)  # warm-up: allocations
        eng.profile(True)
        t0 = time.perf_counter()
        st, _ = eng.grpo_backward(vid, grp, old, adv)
        wall = time.perf_counter() - t0
        prof = eng.profile(False)
    finally:
        eng.close()
    fl = T.step_flops(c, wb.frames, len(grp.question), list(grp.lengths), passes=1)
    attn = fl["attn_prefix"] + fl["attn_resp"]
    bwd_ms, attn_ms = prof["backward"][0], prof["attention_backward"][0]
    # algorithmic: dgrad + wgrad of every linear layer, the attention backward
    # (2.5x its forward) and the LM head's two products — the checkpointing
    # recompute of the linear layers is not counted (the attention is not
    # recomputed when the policy pass keeps its outputs, MRSP_BWD_STASH_ATTN)
    bwd_flops = 2 * fl["linear"] + 2.5 * attn + 2 * fl["lm_head"]
    return {"workload": name, "tokens": fl["tokens"], "wall_ms": round(wall * 1e3, 1),
            "tokens_per_s": round(fl["tokens"] / wall, 1),
            "backward_kernels_ms": round(bwd_ms, 1),
            "backward_algorithmic_tflops": round(bwd_flops / (bwd_ms / 1e3) / 1e12, 1),
            "attention_backward_ms": round(attn_ms, 1),
            "attention_backward_tflops": round(2.5 * attn / (attn_ms / 1e3) / 1e12, 1),
            "forward_passes_ms": round(prof["llm_attention"][0] + prof["llm_gemm"][0]
                                       + prof["lm_head"][0] + prof["misc"][0], 1),
            "objective": st["objective"],
            "note": "policy-LLM gradients of the GRPO objective (exact KL, beta 0.04, clip 0.2); "
                    "vision tower frozen; backward FLOPs exclude the checkpointing recompute; "
                    "parity in tests/test_backward_transformer_gpu.py"}


def generation_side_line(eng, w, group, peaks, pix):
    """SURVEY §8f rank 2, not the metric: G rollouts of the same workload's
    prompt (cached video + question) sampled by the engine (Engine::generate).
    Device time per decode step from two runs 64 steps apart (the prompt
    prefill cancels), against the HBM bound of a step (policy weights + the
    prompt K/V read once)."""
    import numpy as np
    c = w.cfg
    G = int(group.resp.shape[0])
    q = np.asarray(group.question, dtype=np.int32)
    vid = "rollout-gen"
    eng.encode(vid, pix)
    eng.generate(vid, q, G, 4, seed=1)  # warm
    dev = {}
    n1, n2 = 8, 72
    for n in (n1, n2):
        eng.profile(True)
        eng.generate(vid, q, G, n, temperature=1.0, seed=2)
        prof = eng.profile(False)
        dev[n] = sum(v[0] for v in prof.values())
    step_ms = (dev[n2] - dev[n1]) / (n2 - n1)
    L, d, nq, nkv, mlp, V = c.layers, c.dim, c.n_q_heads, c.n_kv_heads, c.mlp, c.vocab
    weights = 2 * (L * (d * (nq + 2 * nkv) * 128 + nq * 128 * d + 3 * d * mlp) + V * d)
    Lp = w.frames * c.tokens_per_frame + len(q)
    kv = 2 * L * Lp * 2 * nkv * 128
    bound_ms = (weights + kv) / (peaks.get("hbm_gbs", 7000.0) * 1e9) * 1e3
    return {"rows": G, "prompt_tokens": Lp, "decode_step_ms_device": round(step_ms, 3),
            "tokens_per_s_device": round(G / (step_ms / 1e3), 1),
            "hbm_bytes_per_step": weights + kv, "hbm_bound_step_ms": round(bound_ms, 3),
            "hbm_frac": round(bound_ms / step_ms, 3),
            "note": "device time per decode step (engine profile classes: steps t >= 1 are one CUDA-graph replay each), 64-step difference"}


def workload_config(w, group, fl, n):
    return {"workload": f"{w.name}: {w.desc}", "frames": w.frames,
            "tokens_per_frame": w.cfg.tokens_per_frame, "prefix_tokens": fl["Lp"],
            "G": w.G, "scored_tokens": int(group.scored), "Lmax": group.Lmax,
            "total_tokens": fl["tokens"], "sp_degree": n, "parallelism": f"sp{n} (Ulysses)",
            "model": "SigLIP-shaped 27L tower + 2-layer projector; Qwen2.5-7B-shaped 28L LLM "
                     "(policy + reference, V 152064)",
            "l2": "inputs larger than L2 (~31 GB of weights streamed per step)"}


if __name__ == "__main__":
    main()
