"""Generates tests/golden/*.json from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
The fixtures pin the oracle (and through it the product) to outputs of the
reference itself: oracle/_ref/libmoesim_ref.so compiled from
/root/reference/proj/src by oracle/Makefile.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def random_instance(rng, N, G, slots, max_demand=200):
    """Every expert on >= 1 GPU, plus extra replicas; demand uniform in [0, max)."""
    cnt = np.zeros((N, G), np.int32)
    used = np.zeros(G, np.int32)
    for e in range(N):
        while True:
            g = int(rng.integers(G))
            if used[g] < slots:
                cnt[e, g] += 1
                used[g] += 1
                break
    for _ in range(int(rng.integers(G * slots // 2 + 1))):
        e, g = int(rng.integers(N)), int(rng.integers(G))
        if used[g] < slots:
            cnt[e, g] += 1
            used[g] += 1
    D = rng.integers(0, max_demand, size=(N, G)).astype(np.int64)
    return D, cnt


def main():
    ref = oracle.Reference()
    golden = {}

    # Config 1 of BASELINE.json: N=8, G=4, k=2, 4096 tokens -> 8192 units, seed 42.
    trace = ref.generate_trace(8, 4, 8192, zipf=1.25, drift=0.02, seed=42, steps=4)
    cnt0 = np.zeros((8, 4), np.int32)
    for e in range(8):
        cnt0[e, e % 4] = 1
    cnt1 = cnt0.copy()
    cnt1[0, 1] += 1
    cnt1[0, 2] += 1
    golden["config1"] = {
        "trace": trace.tolist(),
        "placements": {"initial": cnt0.tolist(), "expand_e0_g1_g2": cnt1.tolist()},
        "flows_initial": ref.route(trace[0], cnt0, 4).tolist(),
        "flows_expanded": ref.route(trace[0], cnt1, 4).tolist(),
        "balance_initial": ref.balance_ratio(trace[0], cnt0, 4),
        "balance_expanded": ref.balance_ratio(trace[0], cnt1, 4),
    }

    # Random routing instances (the style of proj/tests/test_router.cpp:128-153).
    rng = np.random.default_rng(2304_03946)
    cases = []
    for _ in range(300):
        N = int(rng.integers(1, 9))
        G = int(rng.integers(1, 9))
        slots = int(rng.integers(1, 4))
        if N > G * slots:
            continue
        D, cnt = random_instance(rng, N, G, slots)
        cases.append({"D": D.tolist(), "cnt": cnt.tolist(), "slots": slots,
                      "flows": ref.route(D, cnt, slots).tolist()})
    golden["route_random"] = cases

    # Largest-remainder rounding, including ties and drift cases.
    lrr = []
    for n in (1, 2, 3, 5, 8, 16):
        for _ in range(20):
            exact = rng.random(n) * 50
            total = int(round(exact.sum())) + int(rng.integers(-2, 3))
            total = max(total, 0)
            lrr.append({"exact": exact.tolist(), "total": total,
                        "out": ref.largest_remainder_round(exact, total).tolist()})
    lrr.append({"exact": [0.5, 0.5, 0.5, 0.5], "total": 2,
                "out": ref.largest_remainder_round([0.5] * 4, 2).tolist()})
    golden["largest_remainder_round"] = lrr

    # StaticEP capacity drops (baselines.cpp:89-122) on skewed traces.
    sep = []
    for (N, G, tokens, zipf, cf) in [(8, 4, 8192, 1.25, 1.0), (16, 1, 131072, 1.25, 1.0),
                                     (32, 8, 65536 * 8 * 2, 1.25, 1.25), (64, 8, 65536 * 8, 1.5, 1.0),
                                     (128, 8, 262144, 2.0, 2.0)]:
        tr = ref.generate_trace(N, G, tokens, zipf=zipf, drift=0.02, seed=42, steps=3)
        dropped, ratio = ref.static_ep(tr, cf)
        sep.append({"N": N, "G": G, "tokens": tokens, "zipf": zipf, "cf": cf,
                    "trace": tr.tolist(), "dropped": dropped.tolist(), "ratio": ratio.tolist()})
    golden["static_ep"] = sep

    # Policy: one scheduling round on the 2x2 skewed case (test_policy.cpp:138-158 shape).
    D = np.array([[1500, 1500], [500, 500]], np.int64)
    cnt = np.array([[1, 0], [0, 1]], np.int32)
    golden["policy_2x2"] = {"D": D.tolist(), "cnt": cnt.tolist(), "slots": 2,
                            "ops": ref.make_scheduling_plan(D, cnt, 2).tolist()}

    # Dynamic engine on config-1-like traffic (expand/shrink counts, balance path).
    tr = ref.generate_trace(8, 4, 8192, zipf=1.25, drift=0.02, seed=42, steps=100)
    ratio, replicas, ops = ref.engine_run(tr, slots=4)
    golden["engine_cfg1"] = {"steps": 100, "slots": 4, "ratio_first": float(ratio[0]),
                             "ratio_last": float(ratio[-1]), "ops": ops.tolist(),
                             "replicas_last": replicas[-1].tolist()}

    path = OUT / "reference_golden.json"
    path.write_text(json.dumps(golden))
    print(f"wrote {path} ({path.stat().st_size / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
