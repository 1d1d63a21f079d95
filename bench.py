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
           measured burst bf16 peak (MEASURED_PEAKS.json; frac_sustained
           beside it against the sustained peak, with this run's SM clock).
* cpu_baseline: the CPU oracle port of the same layer step in float32
           (numpy on multithreaded OpenBLAS + the C oracle's OpenMP bf16
           rounding, all host cores) on a bounded token sample, rank 0 at N=1.
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
                    sus_mhz=j.get("clocks_under_load", {}).get("sm_mhz_median"), source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, sus_mhz=None, source="fallback")


def zipf_log_popularity(N, s, seed):
    rng = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, N + 1) ** s
    p = p / p.sum()
    return np.log(p)[rng.permutation(N)]


def bench_inputs(cfg, rank=0):
    """The bench's synthetic inputs on the host: gate weight [N, d] f32 (random
    init of the architecture; column 0 = 2 * Zipf log-popularity, so the skew
    is produced by the real gate — x[:, 0] = 0.5), x and dy [T, d] bf16 for
    `rank`, and the generator that drew them (the e2e leg draws its second
    input buffer from it). tests/test_gate_real_gpu.py uses the same inputs."""
    import torch

    N, d, T = cfg["N"], cfg["d"], cfg["T"]
    g = torch.Generator(device="cpu").manual_seed(1234)
    wg = torch.randn(N, d, generator=g) * d**-0.5
    wg[:, 0] = torch.tensor(zipf_log_popularity(N, cfg["zipf"], 42) * 2, dtype=torch.float32)
    gen = torch.Generator(device="cpu").manual_seed(100 + rank)
    x = torch.randn(T, d, generator=gen).to(torch.bfloat16)
    x[:, 0] = 0.5
    dy = (torch.randn(T, d, generator=gen) * 0.1).to(torch.bfloat16)
    return wg, x, dy, gen


def line_config(cfg, world, multi):
    """The `config` object of the JSON line — identical for both arms (the
    reference arm runs the same workload on a bounded token sample per step,
    described in its cpu_baseline.sample)."""
    N, k, d, f, T = cfg["N"], cfg["k"], cfg["d"], cfg["f"], cfg["T"]
    return {"workload": cfg["workload"],
            "model": f"MoE layer N{N} k{k} d{d} f{f}",
            "global_batch": T * world, "tokens_per_gpu": T, "seq_len": None,
            "parallelism": f"ep{world}" + ("+replicas" if multi else ""),
            "zipf": cfg["zipf"],
            "placement": "dynamic" if multi else "static",
            "l2": "per-step working set > L2 (no flush)",
            "step": ("gate top-k + histogram, route + plan, dispatch, expert FFN, combine; backward "
                     "of all of it incl. dx and every weight / bias / gate-weight gradient"
                     + (", replica-group gradient all-reduce" if multi else "")
                     + " (the BASELINE metric is the layer's fwd+bwd; the optimizer is outside it)")}


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
_CPU_WEIGHTS: dict = {}


def cpu_layer_sample(cfg, tokens, seed=0):
    """One oracle fwd+bwd over `tokens` tokens; returns (seconds of the
    fwd+bwd alone, histogram). The synthetic weights are generated once per
    model shape; tokens and gradients per seed."""
    from oracle import layer as OL

    N, k, d, f = cfg["N"], cfg["k"], cfg["d"], cfg["f"]
    key = (N, d, f, cfg["zipf"])
    f32 = np.float32
    if key not in _CPU_WEIGHTS:  # bf16-valued weights, held in float32
        wr = np.random.default_rng(0)
        wg = OL.bf16(wr.standard_normal((N, d)) * d**-0.5)
        wg[:, 0] = zipf_log_popularity(N, cfg["zipf"], 0)
        _CPU_WEIGHTS[key] = (wg.astype(f32),
                             OL.bf16_f32(wr.standard_normal((N, f, d), dtype=f32) * f32(d**-0.5)),
                             OL.bf16_f32(wr.standard_normal((N, d, f), dtype=f32) * f32(f**-0.5)))
    wg, w1, w2 = _CPU_WEIGHTS[key]
    rng = np.random.default_rng(seed)
    x = OL.bf16_f32(rng.standard_normal((tokens, d), dtype=f32))
    x[:, 0] = 1.0
    b1 = np.zeros((N, f), f32)
    b2 = np.zeros((N, d), f32)
    dy = OL.bf16_f32(rng.standard_normal((tokens, d), dtype=f32))
    t0 = time.perf_counter()  # fp32 on multithreaded BLAS (all host cores)
    st = OL.forward(x, wg, w1, b1, w2, b2, k, dtype=f32)
    OL.backward(st, dy)
    return time.perf_counter() - t0, st["hist"]


def host_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=1)
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# BASELINE configs as the reference engine sees them: (N, G, k, tokens per GPU,
# zipf, PolicyMode (0 Dynamic, 1 FixedInterval, 2 Static), interval)
REF_CONFIGS = {
    "configs[0]": (8, 4, 2, 1024, 1.25, 0, 10),
    "configs[1]": (16, 1, 2, 65536, 1.25, 2, 10),
    "configs[2]": (64, 8, 1, 65536, 1.25, 0, 10),
    "configs[3]": (32, 8, 2, 65536, 1.25, 1, 100),
    "configs[4]": (128, 8, 1, 32768, 2.0, 0, 10),
}


def reference_count_path(which=None, min_seconds=0.05):
    """the reference's own count-level per-step path, timed
    on ONE host thread from oracle/_ref (the unmodified moesim sources):
    route (+balance_ratio), step_cost, make_scheduling_plan, plan_migrations
    and one SimEngine step, per BASELINE config, in microseconds per call."""
    import oracle

    ref = oracle.Reference()
    out = {}
    for name, (N, G, k, T, z, mode, iv) in REF_CONFIGS.items():
        if which is not None and name != which:
            continue
        trace = ref.generate_trace(N, G, T * k * G, zipf=z, steps=50)
        slots = 2 * -(-N // G)
        t = ref.time_count_path(trace, slots, mode, iv, min_seconds)
        out[name] = {kk: round(v * 1e6, 2) for kk, v in t.items()}
    return out


def cpu_baseline(cfg, budget_s=12.0):
    t_small, _ = cpu_layer_sample(cfg, 512)
    tokens = int(min(16384, max(512, 512 * budget_s / max(t_small, 1e-3))))
    tokens = max(512, tokens // 512 * 512)
    secs, hist = cpu_layer_sample(cfg, tokens)
    out = {"value": tokens / secs, "unit": "tokens/s", "cores": host_threads(), "kind": "port",
           "sample": f"oracle/layer.py float32 fwd+bwd (multithreaded BLAS, OpenMP rounding) of {tokens} "
                     f"tokens of the bench workload ({secs:.1f} s); host nproc={os.cpu_count()}, {cpu_model()}"}
    try:
        import oracle

        if oracle.Reference.available():
            out["reference_count_path_us"] = reference_count_path()
            out["reference_count_path_threads"] = 1
    except Exception as exc:  # reference shim optional on the box
        out["reference_count_path_error"] = str(exc)[:100]
    return out


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's CPU path on the host cores."""
    if rank != 0:
        return
    import oracle

    # the same workload our arm runs at this N (configs[1] at 1 GPU, configs[2..4] otherwise)
    multi = world > 1 or args.workload in WORKLOADS
    cfg = dict(WORKLOADS[args.workload or "cfg3"] if multi else CFG2)
    if cfg.get("scaling") == "strong":
        cfg["T"] = cfg["T"] // world
    # whole run bounded to ~3 minutes of host work: the per-step sample is the
    # largest that fits, from a two-point fit t(n) = a + b*n (the port has a
    # per-step cost that does not shrink with n: every expert's weights are read)
    budget = max(0.5, 180.0 / max(1, args.steps + args.warmup))
    cpu_layer_sample(cfg, 256)  # warm the weights cache
    t1, _ = cpu_layer_sample(cfg, 256)
    t2, _ = cpu_layer_sample(cfg, 1024)
    b = max((t2 - t1) / 768.0, 1e-7)
    a_fixed = max(t1 - 256 * b, 0.0)
    tokens = int((budget - a_fixed) / b) // 128 * 128
    tokens = min(max(tokens, 256), 16384)
    # the reference's own per-step count path (route, cost, policy, migration
    # pass, queue drain: one SimEngine step) at this config, one thread
    ref_name = {"cfg3": "configs[2]", "cfg4": "configs[3]", "cfg5": "configs[4]"}.get(
        args.workload or "cfg3") if multi else "configs[1]"
    count_path = reference_count_path(ref_name)[ref_name] if oracle.Reference.available() else {}
    engine_s = count_path.get("engine_step", 0.0) * 1e-6
    times = []
    for i in range(args.warmup + args.steps):
        # timed: the layer math (cpu_layer_sample times its fwd+bwd only, not the
        # synthetic input generation) + the reference's engine step
        secs, _ = cpu_layer_sample(cfg, tokens, seed=i)
        if i >= args.warmup:
            times.append(secs + engine_s)
    step = statistics.mean(times)
    value = tokens / step
    full_step_s = a_fixed + cfg["T"] * b + engine_s
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
            "higher_is_better": True, "scaling": cfg.get("scaling", "weak"), "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": line_config(cfg, world, multi),
            "sample": {"tokens_per_step": tokens, "tokens_per_gpu_in_config": cfg["T"],
                       "extrapolation": (f"tokens/s measured on {tokens} of the config's {cfg['T']} tokens per "
                                         f"step; the layer math is linear in tokens (two-point fit: "
                                         f"{a_fixed * 1e3:.1f} ms fixed + {b * 1e6:.1f} us/token), so the full "
                                         f"step would take {full_step_s:.1f} s = "
                                         f"{cfg['T'] / full_step_s:.0f} tokens/s"),
                       "full_step_tokens_per_s_estimate": cfg["T"] / full_step_s},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": host_threads(),
                             "kind": "port",
                             "sample": f"{tokens} tokens/step of {cfg['T']}: the reference's own SimEngine step "
                                       f"({'oracle/_ref' if count_path else 'unavailable'}, 1 thread, "
                                       f"{count_path.get('engine_step', 0):.1f} us) + the oracle port of the "
                                       "gate/FFN/combine fwd+bwd (float32: multithreaded OpenBLAS + OpenMP "
                                       "bf16 rounding, all host threads); "
                                       f"host nproc={os.cpu_count()}, {cpu_model()}",
                             "reference_count_path_us": {ref_name: count_path} if count_path else None},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
CFG3 = dict(workload="BASELINE configs[2]: GPT-MoE layer, 64 experts top-1, d_model 1024, d_ff 4096, "
            "65,536 tokens per GPU (weak scaling), drifting Zipf traffic",
            N=64, k=1, d=1024, f=4096, T=65536, zipf=1.25, policy_mode=0, interval=10, scaling="weak")
CFG4 = dict(workload="BASELINE configs[3]: BERT-MoE layer, 32 experts top-2, d_model 768, d_ff 3072, "
            "65,536 tokens per GPU, expand/shrink/migrate every 100 steps with P2P weight+optimizer "
            "migration", N=32, k=2, d=768, f=3072, T=65536, zipf=1.25, policy_mode=1, interval=100,
            scaling="weak")
CFG5 = dict(workload="BASELINE configs[4]: Swin-MoE-scale layer, 128 experts top-1, d_model 1024, "
            "d_ff 4096, 256K tokens in total (strong scaling), severe imbalance (Zipf 2.0), migration "
            "cost included", N=128, k=1, d=1024, f=4096, T=262144, zipf=2.0, policy_mode=0, interval=10,
            scaling="strong")
WORKLOADS = {"cfg3": CFG3, "cfg4": CFG4, "cfg5": CFG5}


class FusedArm:
    """configs[1] on one GPU: the fused single-GPU step (no host sync)."""

    def __init__(self, cfg, dev, rank):
        import torch

        from paper_2304_03946_b200.layer import MoELayer

        N, k, d, f, T = cfg["N"], cfg["k"], cfg["d"], cfg["f"], cfg["T"]
        self.layer = MoELayer(N, k, d, f, max_tokens=T)
        p = self.layer.init_params(seed=1234)
        p["wg"] = bench_inputs(dict(cfg, T=1))[0].to(dev).to(p["wg"].dtype)  # skew through the real gate
        self.P = (p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
        self.grads = None
        self.N, self.G = N, 1

    def step(self, x, dy):
        self.layer.forward(x, *self.P)
        self.grads = self.layer.backward(dy, self.grads)

    def set_timing(self, on):
        self.layer.set_timing(on)

    def timing(self):
        return self.layer.read_timing(), {}

    def flows(self):
        return self.layer.read("flows", self.N).reshape(self.N, 1, 1)

    def hist(self):
        return self.layer.read("hist", self.N)

    def hist_async(self, host):
        return self.layer.copy_out_async("hist", host)

    def check(self):
        """Raise if a device-side P2P arrival wait gave up during the run."""
        if getattr(self, "transport", None) == "p2p" and self.dl.p2p_timed_out():
            raise RuntimeError("P2P arrival wait timed out: the measured steps are invalid")


def measured_tps(N, k, d, f):
    """(TPS, source): the committed B200 measurement for this model shape, if any."""
    for path in sorted(Path(__file__).resolve().parent.glob("profiles/b200_profile_*.json")):
        m = json.loads(path.read_text())["measurement"]
        if m["model"] == {"num_experts": N, "top_k": k, "d_model": d, "d_ff": f}:
            return float(m["tps"]), f"measured ({path.name})"
    return 1.2e15 / (12.0 * d * f), "assumed 1.2 PFLOP/s grouped GEMM"


class DistArm:
    """configs[2]: one process per GPU, NCCL all-to-all / all-reduce between phases,
    drifting Zipf traffic, dynamic expand/shrink/migrate by the host scheduler with
    peer-to-peer migration of expert state inside the timed region."""

    def __init__(self, cfg, dev, rank, world):
        import torch

        from paper_2304_03946_b200 import scheduler as S
        from paper_2304_03946_b200.distributed import LoopbackHub, TorchExchange
        from paper_2304_03946_b200.runtime import FlexMoERuntime

        N, k, d, f, T = cfg["N"], cfg["k"], cfg["d"], cfg["f"], cfg["T"]
        G = world
        slots = 2 * ((N + G - 1) // G)  # vExpert budget 2*ceil(N/G) (moesim.cpp:141-146)
        # B200 profile (paper_2304_03946_b200/profile.py): NVLink 5 link / NCCL bus
        # bandwidth (B200_PROFILING.md), f32 gradients, 14 B/param of state, and the
        # per-GPU TPS MEASURED on a B200 for this model shape (profiles/b200_profile_*.json;
        # without one, the grouped GEMM's 12*d*f FLOP per unit at 1.2 PFLOP/s).
        from paper_2304_03946_b200.profile import b200_profile
        self.tps, self.tps_source = measured_tps(N, k, d, f)
        prof = b200_profile(G, slots, self.tps, d, f)
        import torch.distributed as tdist

        ex = TorchExchange() if tdist.is_initialized() else LoopbackHub(1).endpoint(0)
        wg = bench_inputs(dict(cfg, T=1))[0]
        self.logp = zipf_log_popularity(N, cfg["zipf"], 42)
        sched_cfg = S.SchedulerConfig.defaults(policy_mode=cfg["policy_mode"], interval_steps=cfg["interval"])
        self.transport = cfg.get("transport", "p2p")
        # placement flips on completed state copies, policy on the scheduler's worker thread
        # (include/flexmoe_b200.h fm_scheduler_config); --flip modelled = the reference's drain
        self.flip = cfg.get("flip", "copy")
        self.rt = FlexMoERuntime(N, k, d, f, ex, prof, sched_cfg=sched_cfg, max_tokens=T, gate_weight=wg,
                                 optimizer=False, transport=self.transport, flip=self.flip,
                                 async_policy=self.flip == "copy")
        self.layer, self.dl = self.rt.layer, self.rt.dl
        self.drift = np.random.default_rng(42)  # same walk on every rank
        self.N, self.G = N, G
        self.reset_stats()

    def reset_stats(self):
        self.mig_bytes = 0
        self.mig0 = self.rt.migration_stats()
        self.applied = 0
        self.accepted = 0
        self.ratios = []

    def step(self, x, dy):
        import torch

        # drifting popularity (workload.cpp:164-170: p *= exp(U[-0.02, 0.02]), renormalised),
        # applied through the gate's skew column. The walk is host-side and
        # independent of the device, so it is generated 256 steps at a time and
        # staged on the device once (no per-step pageable copy / host sync).
        if not getattr(self, "_walk", None) or self._walk_i == self._walk[1].shape[0]:
            cols = []
            for _ in range(256):
                self.logp = self.logp + self.drift.uniform(-0.02, 0.02, self.N)
                self.logp -= np.log(np.exp(self.logp).sum())
                cols.append(self.logp * 2)
            dev_walk = torch.tensor(np.stack(cols), dtype=torch.float32).to(self.rt.wg.device).to(self.rt.wg.dtype)
            self._walk, self._walk_i = (None, dev_walk), 0
        self.rt.wg[:, 0] = self._walk[1][self._walk_i]
        self._walk_i += 1
        out = self.rt.step(x, dy)
        self.mig_bytes += out.migration_bytes
        self.applied += len(out.applied)
        self.accepted += len(out.accepted)
        self.ratios.append(out.balance_ratio)

    def set_timing(self, on):
        self.layer.set_timing(on)
        self.dl.set_timing(on)
        if on:
            self.reset_stats()

    def timing(self):
        return self.layer.read_timing(), self.dl.read_timing()

    def flows(self):
        return self.layer.read("flows", self.N * self.G * self.G).reshape(self.N, self.G, self.G)

    def hist(self):
        return self.layer.read("hist", self.N)

    def hist_async(self, host):
        return self.layer.copy_out_async("hist", host)

    def check(self):
        """Raise if a device-side P2P arrival wait gave up during the run."""
        if getattr(self, "transport", None) == "p2p" and self.dl.p2p_timed_out():
            raise RuntimeError("P2P arrival wait timed out: the measured steps are invalid")

    def summary(self, steps):
        return {"placement": "dynamic (host scheduler: expand/shrink/migrate, B200 profile)",
                "token_transport": ("P2P: rows written/read in the expert GPU's permuted buffers inside "
                                    "dispatch/combine/un-permute (CUDA IPC, NVLink), device-side flags")
                if self.transport == "p2p" else "NCCL all-to-all of staging buffers",
                "profile_tps": self.tps, "profile_tps_source": self.tps_source,
                "balance_ratio_mean": float(np.mean(self.ratios)) if self.ratios else None,
                "balance_ratio_last": self.ratios[-1] if self.ratios else None,
                "ops_accepted": self.accepted, "ops_applied": self.applied,
                "migration_bytes_per_step": self.mig_bytes / steps,
                "migration_copy_ms_per_step": (self.rt.migration_stats()["copy_ms"] - self.mig0["copy_ms"]) / steps,
                "migration_transport": "P2P cudaMemcpyAsync of pool slots on a side stream (CUDA IPC)",
                "placement_flip": ("copy: ops issued at one boundary, state pulled during that step (the "
                                   "receiver joins the replica group with zero rows and waits for the copy "
                                   "only before the group all-reduce), effective at the next boundary; "
                                   "policy on the scheduler's worker thread; table-only placement switch "
                                   "(no allocation, no host sync)") if self.flip == "copy" else
                                  ("modelled: ops effective when their modelled bytes drain (reference); "
                                   "the expert FFN waits for the pull in the same step"),
                "replica_counts": self.rt.history[-1].replica_counts.tolist() if self.rt.history else None}


def run_ours(args, world, rank, local_rank):
    import torch

    from paper_2304_03946_b200 import _lib as L
    from paper_2304_03946_b200 import routing

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1 or "RANK" in os.environ:  # launched by torchrun: NCCL transport even at N=1
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    multi = world > 1 or args.workload in WORKLOADS
    cfg = dict(WORKLOADS[args.workload or "cfg3"] if multi else CFG2)
    cfg["transport"] = args.transport
    cfg["flip"] = args.flip
    if cfg.get("scaling") == "strong":  # fixed total tokens, split over the GPUs
        cfg["T"] = cfg["T"] // world
    N, k, d, f, T = cfg["N"], cfg["k"], cfg["d"], cfg["f"], cfg["T"]
    arm = DistArm(cfg, dev, rank, world) if multi else FusedArm(cfg, dev, rank)

    _, x_host, dy_host, gen = bench_inputs(cfg, rank)
    x, dy = x_host.to(dev), dy_host.to(dev)
    stream = torch.cuda.current_stream()

    for _ in range(max(args.warmup, 3)):
        arm.step(x, dy)
    torch.cuda.synchronize()

    # ---------------- device-timed region (value), live per-phase timing
    # The timed region runs the plain steps; the per-phase CUDA events (two
    # records per kernel, ~1.4 % of a configs[1] step) are recorded in a
    # second pass of the same K steps right after it, which feeds `kernels`
    # and the roofline's per-launch durations.
    arm.set_timing(False)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.lib().fm_kernel_launches()
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            arm.step(x, dy)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = L.lib().fm_kernel_launches() - launches0  # this library's kernels in the timed region
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    dyn = arm.summary(args.steps) if multi else None
    # ---------------- kernel-timing pass: K more steps with per-phase events
    arm.set_timing(True)
    kev0, kev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    kev0.record(stream)
    for _ in range(args.steps):
        arm.step(x, dy)
    kev1.record(stream)
    torch.cuda.synchronize()
    ms_instr = kev0.elapsed_time(kev1) / args.steps
    phases, comm = arm.timing()
    arm.set_timing(False)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    hist = arm.hist()
    side = arm.layer.side_jobs if hasattr(arm.layer, "side_jobs") else 0
    flows = arm.flows()
    units = int(hist.sum())  # this GPU's demand units (T * k)
    recv_units = int(flows[:, :, rank].sum())  # units this GPU's experts processed
    balance = routing.balance_ratio(flows)

    # ---------------- e2e through the public API, pinned host inputs
    xh = [x_host.pin_memory(), torch.randn(T, d, generator=gen).to(torch.bfloat16).pin_memory()]
    dyh = [dy_host.pin_memory(), dy_host.clone().pin_memory()]
    xb = [torch.empty_like(x), torch.empty_like(x)]
    dyb = [torch.empty_like(dy), torch.empty_like(dy)]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    hist_h = [torch.empty(N, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    hist_read = [torch.cuda.Event(), torch.cuda.Event()]
    seen_units = []

    def e2e_run(n):
        with torch.cuda.stream(copy_stream):
            xb[0].copy_(xh[0], non_blocking=True)
            dyb[0].copy_(dyh[0], non_blocking=True)
            copied[0].record(copy_stream)
        for i in range(n):
            cur, nxt = i % 2, (i + 1) % 2
            if i + 1 < n:  # prefetch the next step's inputs while this one computes
                with torch.cuda.stream(copy_stream):
                    copy_stream.wait_stream(stream)
                    xb[nxt].copy_(xh[nxt], non_blocking=True)
                    dyb[nxt].copy_(dyh[nxt], non_blocking=True)
                    copied[nxt].record(copy_stream)
            stream.wait_event(copied[cur])
            arm.step(xb[cur], dyb[cur])
            # the step's expert histogram to the host (placement-policy input):
            # enqueued behind the step, read one step later, so the host never
            # drains the device between steps
            arm.hist_async(hist_h[cur])
            hist_read[cur].record(stream)
            if i > 0:
                hist_read[nxt].synchronize()
                seen_units.append(int(hist_h[nxt].sum()))
        hist_read[(n - 1) % 2].synchronize()
        seen_units.append(int(hist_h[(n - 1) % 2].sum()))

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
    arm.check()
    if any(u != units for u in seen_units):  # every step's histogram read back holds T*k units
        raise RuntimeError(f"e2e: histogram read-back {seen_units[:4]}... != {units} units per step")
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
    flop_step = 12.0 * recv_units * d * f  # algorithmic: real (unpadded) units on this GPU
    achieved = flop_step / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    traffic = None
    tp = ROOT / "profiles" / "gemm_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("bytes_per_launch")
    hbm_bytes = {  # algorithmic bytes per step
        "gate": T * d * 2 + N * d * 2 + units * 12,
        # expert scan: per-128-token-tile expert counts in, tile bases out (+ histogram)
        "scan": 2 * (-(-T // 128)) * N * 4 + N * 8,
        "dispatch": T * d * 2 + units * d * 2 + units * 4,
        "combine_fwd": units * (d * 2 + 8) + T * d * 2,
        "combine_bwd": T * d * 2 + units * (d * 2 * 2 + 12),
        "unpermute": units * (d * 2 + 12) + T * d * 2,
        # fused path: per-tile column sums of dY_perm (db2) and dl-weighted X_perm (dWg)
        # + the db1/db2/dWg partial reduces; the reduces alone when the sums ran
        # beside the FFN2 weight-gradient GEMM (side_jobs bit 0)
        "bias_grad": (None if multi else 4 * (units // 128) * (f + 2 * d) * 2 if side & 1 else
                      units * (2 * d * 2 + 4) + 4 * (units // 128) * (f + 2 * d) * 2),
        "relayout": 4 * recv_units * d * 2,
    }
    side_bytes = {"ffn2_wgrad": (1, "db2 / dWg tile column sums", units * (2 * d * 2 + 4)),
                  "ffn1_wgrad": (2, "un-permute" + (" + bias / gate-weight partial reduce" if side & 4 else ""),
                                 units * (d * 2 + 12) + T * d * 2)}
    kernels = {}
    for name, (pms, n) in phases.items():
        if n == 0:
            continue
        per = pms / args.steps
        ent = {"ms_per_step": round(per, 4), "launches_per_step": n / args.steps}
        if hbm_bytes.get(name) and per > 0:
            gbs = hbm_bytes[name] / (per * 1e-3) / 1e9
            ent.update({"achieved_GBps": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm"], 3)})
        if name in gemm_names and per > 0:
            tf = 2.0 * recv_units * d * f / (per * 1e-3) / 1e12
            ent.update({"achieved_TFLOPs": round(tf, 1), "frac_bf16": round(tf / peaks["bf16"], 3)})
            if name in side_bytes and side & side_bytes[name][0]:
                ent["side_job"] = {"what": side_bytes[name][1] + " on the launch's spare CTA pairs",
                                   "hbm_bytes_per_step": side_bytes[name][2]}
        kernels[name] = ent
    for name, (cms, n) in comm.items():
        kernels["comm_" + name] = {"ms_per_step": round(cms / args.steps, 4),
                                   "calls_per_step": n / args.steps}
    line = {
        "metric": METRIC,
        "value": T * world / (ms_step * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": cfg.get("scaling", "weak"),
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights of the configs architecture; Zipf skew via the gate)",
        "config": line_config(cfg, world, multi),
        "workload_stats": {"units_per_step_rank0": units,
                           "expert_load_max_over_mean": float(hist.max() / max(hist.mean(), 1e-9))},
        "e2e": {"value": T * world / (e2e_ms * 1e-3 / args.steps), "unit": "tokens/s",
                "h2d_bytes_per_step": int(2 * T * d * 2), "d2h_bytes_per_step": int(N * 8),
                "what": ("x and dy copied H2D from pinned host memory every step (prefetched one step "
                         "ahead on a copy stream); the step's result read back D2H is the expert "
                         "histogram (TokenDemand column, the placement policy's input), one step behind"),
                "outputs_on_device": ("y and dx stay in HBM: in training they are the next layer's input "
                                      "and the previous layer's output gradient, and the weight gradients "
                                      "feed the on-device optimizer; copying them to the host would time "
                                      "PCIe, not the layer")},
        "gpu_launches": int(launches),
        "timing": {"value": "CUDA events around the K timed steps, no per-phase events inside",
                   "kernels": "a second pass of K steps with two CUDA events per kernel on the launching "
                              "stream (roofline achieved, kernels.*)",
                   "ms_per_step_instrumented": round(ms_instr, 4)},
        "roofline": {"bound": "tensor", "kernel": "grouped_gemm (tcgen05, 6 launches/step)",
                     "achieved": round(achieved, 1), "peak": peaks["bf16"],
                     "unit": "TFLOP/s", "frac": round(achieved / peaks["bf16"], 4),
                     "traffic": traffic, "peak_source": f"{peaks['source']} bf16 burst (MEASURED_PEAKS.json)",
                     "frac_sustained": round(achieved / peaks["bf16_sus"], 4),
                     "peak_sustained": peaks["bf16_sus"],
                     "peak_note": ("frac is against the burst peak (cuBLAS at full clock); the sustained peak "
                                   f"was measured at a {peaks.get('sus_mhz')} MHz median SM clock, this run's "
                                   "median is in clocks.sm_mhz"),
                     "gemm_ms_per_step": round(gemm_ms, 4), "gemm_launches_per_step": gemm_launches,
                     **({"side_jobs": "the weight-gradient launches also run memory-bound backward work on "
                                      "their spare CTA pairs (kernels.*.side_job); their durations include it"}
                        if side else {})},
        "kernels": kernels,
        "clocks": clocks.summary(),
        "balance_ratio": balance,
    }
    if multi:
        line["dynamic_placement"] = dyn
    if world == 1 and not multi and not args.no_cpu_baseline:
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
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="multi-GPU token transport (configs[2..4] workloads)")
    ap.add_argument("--flip", default="copy", choices=["copy", "modelled"],
                    help="dynamic placement: ops become effective when their state copies complete "
                         "(copy, default) or when their modelled bytes drain (the reference's rule)")
    ap.add_argument("--workload", default=None, choices=[None, "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="default: cfg2 at 1 GPU, cfg3 (multi-GPU runtime) at N > 1; "
                         "cfg3-5 run the multi-GPU runtime at any N")
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
