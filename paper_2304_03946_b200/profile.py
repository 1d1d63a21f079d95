"""Measured B200 cluster profile.

The reference's cost model (proj/src/cost_model.cpp:30-111) prices a step
per GPU as compute = units / TPS, plus 4 all-to-alls at the link bandwidth,
plus replica all-reduces at the measured per-group-size throughput
(`ClusterTopology`, topology.cpp:64-138). This module produces that profile
for B200 from measurements:

* TPS: TokenDemand units per second through one GPU's full layer step (gate,
  routing, dispatch, the six expert GEMMs, combine, backward) — everything
  the model charges as compute — measured on the device with uniform
  demand (`measure_tps`);
* link and all-reduce numbers: NVLink 5 through NVSwitch as measured in
  B200_PROFILING.md (770 GB/s per direction, 725 GB/s all-reduce bus
  bandwidth on 8 ranks) — one GPU here, so these are recorded, not
  re-measured (`b200_profile`);
* `validate`: the cost model's prediction (units / TPS on one GPU) against
  the measured step time at other token counts and routing skews (the paper
  reports < 3 % error for its model).

`python -m paper_2304_03946_b200.profile --out profiles/b200_profile.json`
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

LINK_BPS = 770e9          # NVLink 5 per direction, B200_PROFILING.md (measured)
ALLREDUCE_BUS_BPS = 725e9  # 8-rank NCCL all-reduce bus bandwidth, B200_PROFILING.md (measured)


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


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--experts", type=int, default=16)
    ap.add_argument("--top-k", type=int, default=2)
    ap.add_argument("--d-model", type=int, default=1024)
    ap.add_argument("--d-ff", type=int, default=4096)
    ap.add_argument("--tokens", type=int, default=65536, help="calibration tokens per GPU")
    ap.add_argument("--num-gpus", type=int, default=8)
    ap.add_argument("--slots", type=int, default=0, help="vExpert slots per GPU (default 2*ceil(N/G))")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    N, k, d, f = a.experts, a.top_k, a.d_model, a.d_ff
    tps = measure_tps(N, k, d, f, a.tokens, a.steps)
    slots = a.slots or 2 * -(-N // a.num_gpus)
    prof = b200_profile(a.num_gpus, slots, tps, d, f)
    cases = [(a.tokens // 4, 0.0), (a.tokens // 2, 0.0), (a.tokens * 2, 0.0),
             (a.tokens, 1.25), (a.tokens, 2.0), (a.tokens // 2, 1.25)]
    val = validate(N, k, d, f, tps, cases, a.steps)
    res = {"topology": prof.to_json(),
           "measurement": {"what": "TokenDemand units/s through one B200's full MoE-layer fwd+bwd step",
                           "model": {"num_experts": N, "top_k": k, "d_model": d, "d_ff": f},
                           "calibration_tokens": a.tokens, "tps": tps,
                           "link_bps": {"value": LINK_BPS, "source": "B200_PROFILING.md (measured, not re-measured here)"},
                           "allreduce_bus_bps": {"value": ALLREDUCE_BUS_BPS,
                                                 "source": "B200_PROFILING.md (measured, not re-measured here)"}},
           "validation": val,
           "max_abs_error": max(abs(v["error"]) for v in val)}
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    return res


if __name__ == "__main__":
    main()
