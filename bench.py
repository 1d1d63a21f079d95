#!/usr/bin/env python
"""MoE-layer fwd+bwd tokens/s on B200 — the FlexMoE (arXiv 2304.03946) hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0 (driver contract). Workload at N=1 is BASELINE.json
configs[1]: one MoE layer, 16 experts, top-2, d_model 1024, d_ff 4096, 65,536
tokens, Zipf(1.25)-skewed routing produced by the real gate, static placement.

* value  : device-timed (CUDA events on the launching stream) tokens/s of the
           full layer step (gate, route, dispatch, expert FFN fwd+bwd, combine,
           all gradients) with inputs resident in HBM. Per-step working set is
           several GB (> 126 MB L2), so no extra L2 flush is inserted.
* e2e    : same metric through the public API (MoELayer) with x and dy copied
           from pinned host memory every step (prefetched one step ahead on a
           copy stream) and the step's expert histogram — the input of the
           host placement policy — read back to the host every step.
* roofline: dominant kernel = the tcgen05 grouped GEMM (six launches per
           step), achieved = 12*U*d*f FLOP (U = tokens*k units, padding not
           counted) / summed CUDA-event time of those launches, against the
           measured sustained bf16 peak (MEASURED_PEAKS.json).
* cpu_baseline: the CPU oracle port (numpy, float64) of the same layer step
           on a bounded token sample, rank 0 at N=1 only.
`--impl reference` times the reference's own CPU path (oracle/_ref: the
unmodified moesim route() on the step's demand) plus the oracle port of the
layer math, on the host cores, same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG2 = dict(workload="BASELINE configs[1]: single B200 MoE layer, 16 experts top-2, d_model 1024, "
            "d_ff 4096, 64K tokens, Zipf-skewed routing, static placement",
            N=16, k=2, d=1024, f=4096, T=65536, zipf=1.25)
METRIC = "MoE-layer fwd+bwd tokens/sec"


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j["bf16_tflops_sustained"],
                    source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, source="fallback")


def zipf_log_popularity(N, s, seed):
    rng = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, N + 1) ** s
    p = p / p.sum()
    return np.log(p)[rng.permutation(N)]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.dev)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU legs
def cpu_layer_sample(cfg, tokens, seed=0):
    """One oracle fwd+bwd over `tokens` tokens; returns seconds."""
    from oracle import layer as OL

    rng = np.random.default_rng(seed)
    N, k, d, f = cfg["N"], cfg["k"], cfg["d"], cfg["f"]
    x = OL.bf16(rng.standard_normal((tokens, d)))
    x[:, 0] = 1.0
    wg = OL.bf16(rng.standard_normal((N, d)) * d**-0.5)
    wg[:, 0] = zipf_log_popularity(N, cfg["zipf"], seed)
    w1 = OL.bf16(rng.standard_normal((N, f, d)) * d**-0.5)
    w2 = OL.bf16(rng.standard_normal((N, d, f)) * f**-0.5)
    b1 = np.zeros((N, f))
    b2 = np.zeros((N, d))
    dy = OL.bf16(rng.standard_normal((tokens, d)))
    t0 = time.perf_counter()
    st = OL.forward(x, wg, w1, b1, w2, b2, k)
    OL.backward(st, dy)
    return time.perf_counter() - t0, st["hist"]


def host_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=1)
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, budget_s=12.0):
    t_small, _ = cpu_layer_sample(cfg, 512)
    tokens = int(min(16384, max(512, 512 * budget_s / max(t_small, 1e-3))))
    tokens = max(512, tokens // 512 * 512)
    secs, hist = cpu_layer_sample(cfg, tokens)
    out = {"value": tokens / secs, "unit": "tokens/s", "cores": host_threads(), "kind": "port",
           "sample": f"oracle/layer.py float64 numpy fwd+bwd of {tokens} tokens of the bench "
                     f"workload ({secs:.1f} s); host nproc={os.cpu_count()}"}
    try:
        import oracle

        if oracle.Reference.available():
            ref = oracle.Reference()
            D = np.asarray(hist, np.int64).reshape(cfg["N"], 1) * (cfg["T"] // tokens)
            cnt = np.ones((cfg["N"], 1), np.int32)
            out["reference_route_us"] = ref.time_route(D, cnt, iters=2000) * 1e6
    except Exception as exc:  # reference shim optional on the box
        out["reference_route_error"] = str(exc)[:100]
    return out


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's CPU path on the host cores."""
    if rank != 0:
        return
    import oracle

    cfg = dict(CFG2)
    # whole run bounded to ~2 minutes of host work: per-step sample sized to it
    budget = max(0.25, 120.0 / max(1, args.steps + args.warmup))
    t_small, hist = cpu_layer_sample(cfg, 256)
    tokens = max(128, int(256 * budget / max(t_small, 1e-3)) // 128 * 128)
    tokens = min(tokens, 16384)
    ref = oracle.Reference() if oracle.Reference.available() else None
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        secs, hist = cpu_layer_sample(cfg, tokens, seed=i)
        if ref is not None:  # the reference's own per-step count path on the step demand
            D = np.asarray(hist, np.int64).reshape(cfg["N"], 1)
            ref.route(D, np.ones((cfg["N"], 1), np.int32), 2 * cfg["N"])
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    step = statistics.mean(times)
    value = tokens / step
    kind = "port"
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["workload"], "tokens_per_step_sampled": tokens,
                       "global_batch": cfg["T"], "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": host_threads(),
                             "kind": kind,
                             "sample": f"{tokens} tokens/step: reference route() "
                                       f"({'oracle/_ref' if ref else 'unavailable'}) + oracle "
                                       "port of gate/FFN/combine fwd+bwd (float64 numpy)"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args, world, rank, local_rank):
    import torch

    from paper_2304_03946_b200.layer import MoELayer

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    cfg = dict(CFG2)
    N, k, d, f, T = cfg["N"], cfg["k"], cfg["d"], cfg["f"], cfg["T"]
    dev = torch.device("cuda", local_rank)
    # Each rank runs the single-GPU layer on its own shard of tokens
    # (replicas; the multi-GPU exchange path is exercised by the phase API).
    layer = MoELayer(N, k, d, f, max_tokens=T)
    params = layer.init_params(seed=1234)
    gen = torch.Generator(device="cpu").manual_seed(100 + rank)
    logp = torch.tensor(zipf_log_popularity(N, cfg["zipf"], 42), dtype=torch.float32)
    params["wg"][:, 0] = (logp * 2).to(params["wg"].dtype).to(dev)  # skew through the gate
    x_host = torch.randn(T, d, generator=gen).to(torch.bfloat16)
    x_host[:, 0] = 0.5
    dy_host = (torch.randn(T, d, generator=gen) * 0.1).to(torch.bfloat16)
    x = x_host.to(dev)
    dy = dy_host.to(dev)
    P = (params["wg"], params["w1"], params["b1"], params["w2"], params["b2"])
    grads = None
    stream = torch.cuda.current_stream()

    def step():
        nonlocal grads
        layer.forward(x, *P)
        grads = layer.backward(dy, grads)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---------------- device-timed region (value) with live per-phase timing
    layer.set_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    phases = layer.read_timing()
    layer.set_timing(False)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    hist = layer.read("hist", N)
    units = int(hist.sum())

    # ---------------- e2e through the public API, pinned host inputs
    xh = [x_host.pin_memory(), torch.randn(T, d, generator=gen).to(torch.bfloat16).pin_memory()]
    dyh = [dy_host.pin_memory(), dy_host.clone().pin_memory()]
    xb = [torch.empty_like(x), torch.empty_like(x)]
    dyb = [torch.empty_like(dy), torch.empty_like(dy)]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    hist_host = None

    def e2e_run(n):
        nonlocal grads, hist_host
        with torch.cuda.stream(copy_stream):
            xb[0].copy_(xh[0], non_blocking=True)
            dyb[0].copy_(dyh[0], non_blocking=True)
            copied[0].record(copy_stream)
        for i in range(n):
            cur, nxt = i % 2, (i + 1) % 2
            if i + 1 < n:  # prefetch next step's inputs while this one computes
                with torch.cuda.stream(copy_stream):
                    copy_stream.wait_stream(stream)
                    xb[nxt].copy_(xh[nxt], non_blocking=True)
                    dyb[nxt].copy_(dyh[nxt], non_blocking=True)
                    copied[nxt].record(copy_stream)
            stream.wait_event(copied[cur])
            layer.forward(xb[cur], *P)
            grads = layer.backward(dyb[cur], grads)
            hist_host = layer.read("hist", N)  # host policy input, every step

    e2e_run(2)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    gemm_names = ["ffn1_fwd", "ffn2_fwd", "ffn2_dgrad", "ffn1_dgrad", "ffn2_wgrad", "ffn1_wgrad"]
    gemm_ms = sum(phases[n][0] for n in gemm_names) / args.steps
    gemm_launches = sum(phases[n][1] for n in gemm_names) / args.steps
    flop_step = 12.0 * units * d * f
    achieved = flop_step / (gemm_ms * 1e-3) / 1e12
    traffic = None
    tp = ROOT / "profiles" / "gemm_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("bytes_per_launch")
    # HBM kernels: algorithmic bytes per step
    hbm_bytes = {
        "gate": T * d * 2 + N * d * 2 + units * 12,
        "dispatch": T * d * 2 + units * d * 2 + units * 4,
        "combine_fwd": units * (d * 2 + 8) + T * d * 2,
        "combine_bwd": T * d * 2 + units * (d * 2 * 2 + 12),
        "unpermute": units * (d * 2 + 12) + T * d * 2,
        "bias_grad": units * (f + d) * 2,
    }
    kernels = {}
    for name, (pms, n) in phases.items():
        if n == 0:
            continue
        per = pms / args.steps
        ent = {"ms_per_step": round(per, 4), "launches_per_step": n / args.steps}
        if name in hbm_bytes and per > 0:
            gbs = hbm_bytes[name] / (per * 1e-3) / 1e9
            ent.update({"achieved_GBps": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm"], 3)})
        if name in gemm_names and per > 0:
            tf = 2.0 * units * d * f / (per * 1e-3) / 1e12
            ent.update({"achieved_TFLOPs": round(tf, 1), "frac_bf16": round(tf / peaks["bf16_sus"], 3)})
        kernels[name] = ent
    kernels_per_step = 9 + 9 + (1 if k > 1 else 0)
    line = {
        "metric": METRIC,
        "value": T * world / (ms_step * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights of the configs[1] architecture; skew via the gate)",
        "config": {"workload": cfg["workload"], "model": "MoE layer N16 k2 d1024 f4096",
                   "global_batch": T * world, "tokens_per_gpu": T, "seq_len": None,
                   "parallelism": "ep1" if world == 1 else f"replicas x{world}",
                   "zipf": cfg["zipf"], "units_per_step": units,
                   "expert_load_max_over_mean": float(hist.max() / hist.mean()),
                   "l2": "per-step working set > L2 (no flush)"},
        "e2e": {"value": T * world / (e2e_ms * 1e-3 / args.steps), "unit": "tokens/s",
                "h2d_bytes_per_step": int(2 * T * d * 2), "d2h_bytes_per_step": int(N * 8)},
        "gpu_launches": kernels_per_step * args.steps,
        "roofline": {"bound": "tensor", "kernel": "grouped_gemm (tcgen05, 6 launches/step)",
                     "achieved": round(achieved, 1), "peak": peaks["bf16_sus"],
                     "unit": "TFLOP/s", "frac": round(achieved / peaks["bf16_sus"], 4),
                     "traffic": traffic, "peak_source": f"{peaks['source']} bf16 sustained",
                     "gemm_ms_per_step": round(gemm_ms, 4), "gemm_launches_per_step": gemm_launches},
        "kernels": kernels,
        "clocks": clocks.summary(),
        "balance_ratio": 1.0,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as exc:
            line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
    else:
        run_ours(args, world, rank, local_rank)


if __name__ == "__main__":
    main()
