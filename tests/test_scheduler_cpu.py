"""Host placement scheduler (C ABI) vs the reference library (CPU).

Exact equality throughout (the scheduler routes with the same integer
route() and evaluates the cost model in the reference's operation order):
step_cost per GPU, make_scheduling_plan / plan_migrations op lists, and the
Alg. 1 step driver over whole traces — per-step modelled makespan, adjust
bytes and the ops accepted — for Dynamic / FixedInterval / Static modes, the
variance trigger, and a two-node (16-GPU) profile.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2304_03946_b200 import scheduler as S
from paper_2304_03946_b200 import InvalidArgument

REF = oracle.Reference() if oracle.Reference.available() else None
needs_ref = pytest.mark.skipif(REF is None, reason="reference shim not built")
GOLD = json.loads((Path(__file__).parent / "golden" / "reference_golden.json").read_text())


def random_placement(rng, N, G, E):
    cnt = np.zeros((N, G), np.int32)
    used = np.zeros(G, int)
    for e in range(N):
        while True:
            g = int(rng.integers(G))
            if used[g] < E:
                cnt[e, g] += 1
                used[g] += 1
                break
    for _ in range(int(rng.integers(G * E // 2 + 1))):
        e, g = int(rng.integers(N)), int(rng.integers(G))
        if used[g] < E:
            cnt[e, g] += 1
            used[g] += 1
    return cnt


def test_engine_golden_config1():
    g = GOLD["engine_cfg1"]
    tr = oracle.Oracle().generate_trace(8, 4, 8192, seed=42, steps=g["steps"])
    sch = S.Scheduler(S.ClusterProfile.reference_default(4, g["slots"]), 8)
    ratios, totals = [], [0, 0, 0]
    for s in range(g["steps"]):
        r = sch.step(tr[s])
        ratios.append(r.report.balance_ratio)
        for op in r.accepted:
            totals[op[0]] += 1
    assert ratios[0] == g["ratio_first"] and ratios[-1] == g["ratio_last"]
    assert totals == g["ops"]
    assert sch.placement()[1].sum(axis=1).tolist() == g["replicas_last"]


def test_policy_golden_2x2():
    g = GOLD["policy_2x2"]
    prof = S.ClusterProfile.reference_default(2, g["slots"])
    slots = S.slots_from_counts(g["cnt"], g["slots"])
    ops = S.make_scheduling_plan(np.array(g["D"]), slots, prof)
    assert [list(o) for o in ops] == g["ops"]


def test_placement_ops_and_errors():
    prof = S.ClusterProfile.reference_default(4, 2)
    slots = S.slots_from_counts(np.eye(4, dtype=np.int32), 2)
    s2, t = S.apply_op(slots, 4, prof, (S.EXPAND, 0, 1, -1, -1, -1, -1))
    assert s2[1].tolist() == [1, 0] and t == [(0, 1, 150e6)]
    s3, t = S.apply_op(s2, 4, prof, (S.EXPAND, 0, 0, -1, -1, -1, -1))  # same GPU: shared weights
    assert t == [] and s3[0].tolist() == [0, 0]
    s4, t = S.apply_op(s3, 4, prof, (S.SHRINK, 0, 1, -1, -1, -1, -1))
    assert s4[1].tolist() == [1, -1]
    with pytest.raises(InvalidArgument, match="last replica"):
        S.apply_op(slots, 4, prof, (S.SHRINK, 2, 2, -1, -1, -1, -1))
    s5, t = S.apply_op(slots, 4, prof, (S.MIGRATE, -1, -1, 0, 0, 3, 0))
    assert s5[0, 0] == 3 and s5[3, 0] == 0 and len(t) == 2


@needs_ref
def test_step_cost_matches_reference():
    rng = np.random.default_rng(1)
    for _ in range(150):
        G = int(rng.choice([2, 4, 8, 16]))
        E = int(rng.integers(1, 5))
        N = int(rng.integers(1, G * E + 1))
        cnt = random_placement(rng, N, G, E)
        D = rng.integers(0, 5000, size=(N, G))
        prof = S.ClusterProfile.reference_default(G, E)
        mk, per = S.step_cost(D, S.slots_from_counts(cnt, E), prof)
        mk_r, per_r = REF.step_cost(D, cnt, E)
        assert mk == mk_r and (per == per_r).all()


@needs_ref
def test_policy_plans_match_reference():
    rng = np.random.default_rng(2)
    nonempty = 0
    for _ in range(300):
        G = int(rng.choice([2, 3, 4, 8, 16]))
        E = int(rng.integers(1, 5))
        N = int(rng.integers(2, G * E + 1))
        cnt = random_placement(rng, N, G, E)
        p = 1.0 / np.arange(1, N + 1) ** float(rng.uniform(0.5, 2.0))
        D = np.outer(rng.permutation(p) / p.sum(), np.ones(G)) * float(rng.integers(1000, 100000))
        D = np.floor(D).astype(np.int64)
        prof = S.ClusterProfile.reference_default(G, E)
        slots = S.slots_from_counts(cnt, E)
        ours = S.make_scheduling_plan(D, slots, prof, horizon=50)
        ref = [tuple(o) for o in REF.make_scheduling_plan(D, cnt, E, 50)]
        assert ours == ref
        nonempty += bool(ours)
        assert S.plan_migrations(slots, N, prof) == [tuple(o) for o in REF.plan_migrations(cnt, E)]
    assert nonempty > 50


ENGINE_CASES = [
    # (N, G, E, tokens, zipf, steps, policy_mode, interval, metric)
    (8, 4, 4, 8192, 1.25, 80, 0, 10, 0),
    (64, 8, 16, 65536 * 8, 1.25, 60, 0, 10, 0),      # configs[2] shape
    (32, 8, 8, 65536 * 8 * 2, 1.25, 120, 1, 100, 0),  # configs[3]: FixedInterval(100)
    (128, 8, 32, 262144, 2.0, 40, 0, 10, 0),          # configs[4]: severe skew
    (16, 16, 2, 32768, 1.5, 50, 0, 10, 0),            # two nodes: inter-node links, migrations
    (16, 4, 8, 16384, 1.25, 50, 0, 10, 1),            # variance trigger
    (16, 4, 8, 16384, 1.25, 20, 2, 10, 0),            # static
]


@needs_ref
@pytest.mark.parametrize("case", ENGINE_CASES)
def test_engine_matches_reference(case):
    N, G, E, tokens, zipf, steps, mode, interval, metric = case
    tr = REF.generate_trace(N, G, tokens, zipf=zipf, drift=0.02, seed=42, steps=steps)
    mk_r, ab_r, ops_r = REF.engine_detail(tr, E, policy_mode=mode, interval=interval, metric=metric)
    cfg = S.SchedulerConfig.defaults(policy_mode=mode, interval_steps=interval, metric=metric)
    sch = S.Scheduler(S.ClusterProfile.reference_default(G, E), N, cfg)
    n_ops = 0
    for s in range(steps):
        r = sch.step(tr[s])
        assert r.report.makespan_s == mk_r[s], s
        assert r.report.adjust_bytes == ab_r[s], s
        assert r.accepted == [tuple(o) for o in ops_r[s]], s
        n_ops += len(r.accepted)
    if mode != 2:
        assert n_ops > 0


def test_split_step_equals_step():
    tr = oracle.Oracle().generate_trace(16, 4, 16384, zipf=1.5, seed=3, steps=40)
    a = S.Scheduler(S.ClusterProfile.reference_default(4, 8), 16)
    b = S.Scheduler(S.ClusterProfile.reference_default(4, 8), 16)
    for s in range(40):
        ra = a.step(tr[s])
        applied = b.begin_step()
        rb = b.finish_step(tr[s])
        assert applied == ra.applied == rb.applied
        assert ra.accepted == rb.accepted
        assert ra.report.makespan_s == rb.report.makespan_s
