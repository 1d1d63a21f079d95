"""Modelled configs[2] scaling on 1/2/4/8 B200 (no multi-GPU box in this pool).

The reference's cost model (Eqs. 5, 8-10: cost_model.cpp:30-111) with the
B200 cluster profile of profiles/b200_profile_cfg3.json — expert throughput
MEASURED through the whole layer step at configs[2]'s operating point, NVLink
and all-reduce bandwidths BORROWED from B200_PROFILING.md — drives the
product's scheduler (fm_scheduler_*, the reference's policy and step driver)
over a drifting Zipf(1.25) TokenDemand trace of 64 experts, top-1, 65,536
tokens per GPU (weak scaling), as bench.py's multi-GPU workload. Reports the
modelled per-step makespan after the placement settles (FlexMoE dynamic vs the
static round-robin placement) and the implied tokens/s. A model, not a
measurement: bench.py --gpus N is the measurement on a multi-GPU box.

usage: python profiles/model_scaling.py [steps] > profiles/r02_model_scaling.json
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2304_03946_b200 import scheduler as S  # noqa: E402
from paper_2304_03946_b200.profile import b200_profile  # noqa: E402

N, k, d, f, T, ZIPF = 64, 1, 1024, 4096, 65536, 1.25
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
prof_json = json.loads((ROOT / "profiles" / "b200_profile_cfg3.json").read_text())
tps = prof_json["measurement"]["tps_at_operating_point"]


def trace(G, steps, seed=42):
    """Per step D[e][g]: each GPU's T*k units split over the experts by a
    Zipf popularity that drifts (p *= exp(U[-0.02, 0.02]) per step, as
    workload.cpp:164-170), rounded by largest remainder per GPU."""
    rng = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, N + 1) ** ZIPF
    p = p[rng.permutation(N)]
    out = []
    for _ in range(steps):
        p = p * np.exp(rng.uniform(-0.02, 0.02, N))
        q = p / p.sum()
        D = np.zeros((N, G), np.int64)
        for g in range(G):
            x = q * T * k
            base = np.floor(x).astype(np.int64)
            rem = T * k - base.sum()
            order = np.argsort(-(x - base), kind="stable")
            base[order[:rem]] += 1
            D[:, g] = base
        out.append(D)
    return out


rows = []
for G in (1, 2, 4, 8):
    E = 2 * ((N + G - 1) // G)  # slots per GPU: room for replicas
    prof = b200_profile(G, E, tps, d, f)
    tr = trace(G, steps)
    res = {}
    for mode in ("dynamic", "static"):
        cfg = S.SchedulerConfig.defaults()
        if mode == "static":
            cfg.policy_mode = 2
        sch = S.Scheduler(prof, N, cfg)
        ms = []
        for D in tr:
            ms.append(sch.step(D).report.makespan_s * 1e3)
        tail = ms[steps // 4:]
        res[mode] = {"makespan_ms_mean": round(float(np.mean(tail)), 4),
                     "tokens_per_s": round(G * T / (float(np.mean(tail)) * 1e-3), 1)}
    rows.append({"gpus": G, "slots_per_gpu": E, **res})

base = rows[0]["dynamic"]["tokens_per_s"]
for r in rows:
    r["weak_scaling_efficiency_dynamic"] = round(r["dynamic"]["tokens_per_s"] / (r["gpus"] * base), 3)
print(json.dumps({"what": __doc__.strip().splitlines()[0], "model_inputs": {
    "tps_units_per_s": tps, "tps_source": "measured (profiles/b200_profile_cfg3.json)",
    "link_bps": prof_json["measurement"]["link_bps"], "allreduce_bus_bps": prof_json["measurement"]["allreduce_bus_bps"],
    "workload": f"N={N} k={k} d={d} f={f}, {T} tokens/GPU, Zipf {ZIPF} drifting, {steps} steps (mean of the last 3/4)"},
    "rows": rows}, indent=1))
