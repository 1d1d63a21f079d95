"""Comparison baselines step by step against the
reference's run_baseline (proj/src/baselines.cpp:81-276) on reference traces:
StaticEP (capacity drops), FullReplicate (hot-expert shadowing),
StrictRebalance (loads rewritten to B/G). Every StepReport field that the
reference produces must match exactly (doubles included).
"""
import numpy as np
import pytest

import oracle
from paper_2304_03946_b200 import scheduler as S

pytestmark = pytest.mark.skipif(not oracle.Reference.available(), reason="oracle/_ref not built")

KIND_REF = {S.STATIC_EP: 0, S.FULL_REPLICATE: 1, S.STRICT_REBALANCE: 2}  # BaselineKind order

CASES = [
    # kind, N, G, E, units, zipf, steps, cf, top, metric
    (S.STATIC_EP, 8, 4, 2, 8192, 1.25, 20, 1.0, 1, 0),
    (S.STATIC_EP, 64, 8, 8, 65536, 1.5, 20, 1.25, 1, 1),
    (S.STATIC_EP, 16, 1, 16, 131072, 1.25, 5, 2.0, 1, 0),
    (S.STATIC_EP, 32, 8, 4, 65536, 1.25, 10, float("inf"), 1, 0),
    (S.FULL_REPLICATE, 8, 4, 3, 8192, 1.25, 20, 1.0, 1, 0),
    (S.FULL_REPLICATE, 64, 8, 10, 65536, 1.25, 30, 1.0, 2, 0),
    (S.FULL_REPLICATE, 128, 8, 20, 262144, 1.8, 20, 1.0, 4, 1),
    (S.FULL_REPLICATE, 32, 8, 6, 65536, 1.0, 20, 1.0, 32, 0),  # top clamps to N
    (S.STRICT_REBALANCE, 8, 4, 2, 8192, 1.25, 20, 1.0, 1, 0),
    (S.STRICT_REBALANCE, 64, 8, 8, 65536, 1.5, 20, 1.0, 1, 1),
    (S.STRICT_REBALANCE, 32, 8, 4, 65536, 1.25, 10, 1.0, 1, 0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c[:3] + c[6:9])))
def test_baseline_matches_reference(case):
    kind, N, G, E, units, zipf, steps, cf, top, metric = case
    ref = oracle.Reference()
    tr = ref.generate_trace(N, G, units, zipf=zipf, drift=0.02, seed=42, steps=steps)
    r = ref.baseline_run(KIND_REF[kind], tr, E, cf=cf, replicate_top=top, metric=metric)
    b = S.Baseline(S.ClusterProfile.reference_default(G, E), N,
                   S.BaselineConfig.make(kind, capacity_factor=cf, replicate_top=top, metric=metric))
    for s in range(steps):
        o = b.step(tr[s])
        rep = o.report
        assert rep.balance_ratio == r["ratio"][s], s
        assert rep.metric_value == r["metric"][s], s
        assert rep.makespan_s == r["makespan"][s], s
        assert rep.group_misses == r["misses"][s], s
        assert rep.tokens_dropped == r["dropped"][s], s
        assert rep.tokens_reassigned == r["reassigned"][s], s
        assert rep.slot_utilization == r["util"][s], s
        np.testing.assert_array_equal(o.counts.sum(axis=1), r["replicas"][s])
        assert o.demand.sum() == tr[s].sum() - rep.tokens_dropped
        # flows conserve the routed demand
        np.testing.assert_array_equal(o.flows.sum(axis=2), o.demand)


def test_full_replicate_shadows_hottest_everywhere():
    ref = oracle.Reference()
    tr = ref.generate_trace(16, 4, 16384, zipf=1.5, drift=0.02, seed=3, steps=3)
    b = S.Baseline(S.ClusterProfile.reference_default(4, 6), 16, S.BaselineConfig.make("full-replicate", replicate_top=2))
    for s in range(3):
        o = b.step(tr[s])
        hot = np.argsort(-tr[s].sum(axis=1), kind="stable")[:2]
        assert (o.counts[hot] > 0).all()
        cold = np.setdiff1d(np.arange(16), hot)
        assert (o.counts[cold].sum(axis=1) == 1).all()
        slots, counts = b.placement()
        np.testing.assert_array_equal(counts, o.counts)


def test_baseline_errors():
    prof = S.ClusterProfile.reference_default(4, 2)
    from paper_2304_03946_b200 import _lib as L
    with pytest.raises(L.InvalidArgument, match="replicate_top"):
        S.Baseline(prof, 8, S.BaselineConfig.make("full-replicate", replicate_top=0))
    b = S.Baseline(prof, 8, S.BaselineConfig.make("strict-rebalance"))
    D = np.zeros((8, 4), np.int64)
    D[0, 0] = 5  # 5 tokens over 4 GPUs
    with pytest.raises(L.InvalidArgument, match="not divisible"):
        b.step(D)
