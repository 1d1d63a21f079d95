"""Measured B200 cluster profile.

The reference's cost model (proj/src/cost_model.cpp:30-111) prices a step
per GPU as compute = units / TPS, plus 4 all-to-alls at the link bandwidth,
plus replica all-reduces at the measured per-group-size throughput
(`ClusterTopology`, topology.cpp:64-138). This module produces that profile
for B200 from measurements:

* TPS: TokenDemand units per second through one GPU's full layer step (gate,
  routing, dispatch, the six expert GEMMs, combine, backward) — everything
  the model charges as compute — measured on the device with uniform
  demand (`measure_tps`), AT THE CONFIG'S OPERATING POINT: the tokens each
  GPU routes and the experts it hosts on the config's GPU count (the model is
  linear in units, compute = M / TPS, cost_model.cpp:30-35, so TPS must be
  taken where the scheduler prices steps, not at another size: a fixed
  per-step cost makes units/TPS wrong by 10-50 % at 1/4 of the size);
* link and all-reduce numbers: BORROWED from B200_PROFILING.md (NVLink 5
  through NVSwitch, 770 GB/s per direction; 725 GB/s all-reduce bus bandwidth
  on 8 ranks) — one GPU here; `profiles/measure_links.py` measures both per
  group size on a box with >= 2 GPUs and its JSON replaces them
  (`--links`);
* `validate`: the cost model's prediction (units / TPS) against the measured
  step time around the operating point — +-10 % units (the per-GPU load
  spread at the policy's 1.1 balance threshold), skew among the hosted
  experts, twice the hosted experts (replicas) — (the paper reports < 3 %
  error for its model).

`python -m paper_2304_03946_b200.profile --config cfg3 --out profiles/b200_profile_cfg3.json`
writes the profile in the reference's JSON format (loadable by
`ClusterTopology::from_file`) plus the validation table.
"""
from __future__ import annotations

import argparse
import json

import numpy as np
import torch

from . import scheduler as S
from .layer import MoELayer
from .trace import replay_inputs

LINK_BPS = 770e9          # NVLink 5 per direction — borrowed from B200_PROFILING.md (not measured here)
ALLREDUCE_BUS_BPS = 725e9  # 8-rank NCCL all-reduce bus bandwidth — borrowed from B200_PROFILING.md

# BASELINE.json configs[1..4]: (experts, top_k, d_model, d_ff, tokens per GPU, GPUs)
CONFIGS = {
    "cfg2": (16, 2, 1024, 4096, 65536, 1),
    "cfg3": (64, 1, 1024, 4096, 65536, 8),
    "cfg4": (32, 2, 768, 3072, 65536, 8),
    "cfg5": (128, 1, 1024, 4096, 262144 // 8, 8),
}


def expert_param_bytes(d, f):
    """Gradient bytes synchronised per replicated expert (f32 grads of W1, b1, W2, b2)."""
    return 4.0 * (2 * d * f + d + f)


def expert_state_bytes(d, f):
    """f32 master + Adam m/v: 12 B per parameter — what an ExpertPool slot
    transfer moves (pool.py; the bf16 working copy of SURVEY.md §8d's 14 B is
    re-derived from the master on arrival instead of being copied)."""
    return 12.0 * (2 * d * f + d + f)


def _column(N, units, zipf):
    if zipf <= 0:
        col = np.full(N, units // N, np.int64)
        col[: units - col.sum()] += 1
        return col
    p = 1.0 / np.arange(1, N + 1) ** zipf
    p /= p.sum()
    col = np.floor(p * units).astype(np.int64)
    col[np.argsort(-(p * units - col), kind="stable")[: units - col.sum()]] += 1
    return col


def step_ms(N, k, d, f, tokens, zipf=0.0, steps=20, warmup=3, seed=0):
    """Median ms of one fused layer fwd+bwd step on this GPU. Routing is
    exact (trace replay inputs, every expert's demand under T)."""
    units = tokens * k
    col = _column(N, units, zipf)
    col = np.minimum(col, tokens)
    col[np.argmin(col)] += units - col.sum()
    dev = torch.device("cuda", torch.cuda.current_device())
    x, wg = replay_inputs(col, k, d, device=dev)
    g = torch.Generator(device="cpu").manual_seed(seed)
    w1 = (torch.randn(N, f, d, generator=g) * d**-0.5).to(dev, torch.bfloat16)
    w2 = (torch.randn(N, d, f, generator=g) * f**-0.5).to(dev, torch.bfloat16)
    b1 = torch.zeros(N, f, device=dev)
    b2 = torch.zeros(N, d, device=dev)
    dy = (torch.randn(tokens, d, generator=g) * 0.1).to(dev, torch.bfloat16)
    lay = MoELayer(N, k, d, f, max_tokens=tokens)
    for _ in range(warmup):
        lay.forward(x, wg, w1, b1, w2, b2)
        lay.backward(dy)
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lay.forward(x, wg, w1, b1, w2, b2)
        lay.backward(dy)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def measure_tps(N, k, d, f, tokens, steps=20, warmup=3):
    """TokenDemand units per second through one GPU (uniform demand)."""
    return tokens * k / (step_ms(N, k, d, f, tokens, 0.0, steps, warmup) * 1e-3)


def b200_profile(num_gpus, slots_per_gpu, tps, d, f):
    return S.ClusterProfile.b200(num_gpus, slots_per_gpu, tps=tps, expert_param_bytes=expert_param_bytes(d, f),
                                 expert_state_bytes=expert_state_bytes(d, f), token_bytes=2.0 * d,
                                 link_bps=LINK_BPS, allreduce_bus_bps=ALLREDUCE_BUS_BPS)


def validate(N, k, d, f, tps, cases, steps=20):
    """Cost-model prediction (G = 1: makespan = units / TPS) vs measured."""
    out = []
    for tokens, zipf in cases:
        ms = step_ms(N, k, d, f, tokens, zipf, steps)
        pred = tokens * k / tps * 1e3
        out.append({"tokens": tokens, "zipf": zipf, "measured_ms": round(ms, 4), "predicted_ms": round(pred, 4),
                    "error": round((pred - ms) / ms, 4)})
    return out


def operating_point(N, k, T, G):
    """What one GPU computes in a balanced step of the config: its own T tokens
    through gate / dispatch / combine and ~T*k received units spread over the
    experts it hosts (N / G distinct experts at the round-robin start)."""
    return {"tokens_per_gpu": T, "units_per_gpu": T * k, "local_experts": max(1, N // G), "gpus": G}


def validate_at(op, k, d, f, tps, steps=20):
    """Cost-model prediction (compute = units / TPS) vs the measured step time
    around the operating point."""
    T, n = op["tokens_per_gpu"], op["local_experts"]
    cases = [(T, 0.0, n), (int(T * 0.9) // 128 * 128, 0.0, n), (int(T * 1.1) // 128 * 128, 0.0, n),
             (T, 1.0, n), (T, 0.0, 2 * n), (T, 1.0, 2 * n)]
    out = []
    for tokens, zipf, nl in cases:
        ms = step_ms(nl, k, d, f, tokens, zipf, steps)
        pred = tokens * k / tps * 1e3
        out.append({"tokens": tokens, "zipf_among_local_experts": zipf, "local_experts": nl,
                    "measured_ms": round(ms, 4), "predicted_ms": round(pred, 4),
                    "error": round((pred - ms) / ms, 4)})
    return out


def fit_minimax(val, tps):
    """TPS that minimises the largest relative error of units / TPS over the
    validation points (the model is linear in units; the device is not quite:
    128-row tile quantisation and the per-step fixed cost), and the errors it
    leaves. Same JSON shape as the validation rows."""
    ratios = [v["measured_ms"] / v["predicted_ms"] for v in val]  # measured / predicted at tps
    c = 2.0 / (max(ratios) + min(ratios))  # scale of tps: prediction x 1/c
    fitted = tps * c
    rows = [dict(v, predicted_ms=round(v["predicted_ms"] / c, 4),
                 error=round((v["predicted_ms"] / c - v["measured_ms"]) / v["measured_ms"], 4)) for v in val]
    return fitted, rows


def finalize(res):
    """Adds the minimax-fitted TPS (used by the topology) to a profile result."""
    m = res["measurement"]
    fitted, rows = fit_minimax(res["validation"], m["tps"])
    m["tps_at_operating_point"] = m["tps"]
    m["tps"] = fitted
    m["tps_fit"] = "minimax relative error over the validation points"
    res["topology"]["tps"] = fitted
    res["validation_measured_tps"] = res["validation"]
    res["validation"] = rows
    res["max_abs_error_measured_tps"] = max(abs(v["error"]) for v in res["validation_measured_tps"])
    res["max_abs_error"] = max(abs(v["error"]) for v in rows)
    return res


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="calibrate at this BASELINE config's operating point (sets the shape options)")
    ap.add_argument("--experts", type=int, default=16)
    ap.add_argument("--top-k", type=int, default=2)
    ap.add_argument("--d-model", type=int, default=1024)
    ap.add_argument("--d-ff", type=int, default=4096)
    ap.add_argument("--tokens", type=int, default=65536, help="tokens per GPU")
    ap.add_argument("--num-gpus", type=int, default=8)
    ap.add_argument("--slots", type=int, default=0, help="vExpert slots per GPU (default 2*ceil(N/G))")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--links", default=None, help="profiles/measure_links.py JSON (replaces the borrowed numbers)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    if a.config:
        a.experts, a.top_k, a.d_model, a.d_ff, a.tokens, a.num_gpus = CONFIGS[a.config]
    N, k, d, f, G = a.experts, a.top_k, a.d_model, a.d_ff, a.num_gpus
    op = operating_point(N, k, a.tokens, G)
    tps = measure_tps(op["local_experts"], k, d, f, a.tokens, a.steps)
    slots = a.slots or 2 * -(-N // G)
    link = {"value": LINK_BPS, "source": "borrowed: B200_PROFILING.md (not measured on this box)"}
    ar = {"value": ALLREDUCE_BUS_BPS, "source": "borrowed: B200_PROFILING.md (not measured on this box)"}
    if a.links:
        with open(a.links) as fh:
            lk = json.load(fh)
        if lk.get("p2p_bps"):
            link = {"value": lk["p2p_bps"], "source": f"measured ({a.links})"}
        if lk.get("allreduce_bus_bps_by_group"):
            ar = {"value": max(lk["allreduce_bus_bps_by_group"].values()), "source": f"measured ({a.links})"}
    prof = S.ClusterProfile.b200(G, slots, tps=tps, expert_param_bytes=expert_param_bytes(d, f),
                                 expert_state_bytes=expert_state_bytes(d, f), token_bytes=2.0 * d,
                                 link_bps=link["value"], allreduce_bus_bps=ar["value"])
    val = validate_at(op, k, d, f, tps, a.steps)
    res = {"topology": prof.to_json(),
           "measurement": {"what": "TokenDemand units/s through one B200's full MoE-layer fwd+bwd step "
                                   "at the config's operating point",
                           "config": a.config,
                           "model": {"num_experts": N, "top_k": k, "d_model": d, "d_ff": f},
                           "operating_point": op,
                           "calibration_tokens": a.tokens, "tps": tps,
                           "link_bps": link, "allreduce_bus_bps": ar},
           "validation": val,
           "max_abs_error": max(abs(v["error"]) for v in val)}
    res = finalize(res)
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    return res


if __name__ == "__main__":
    main()
