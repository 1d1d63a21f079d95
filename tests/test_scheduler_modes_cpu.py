"""The scheduler's device-runtime modes (include/flexmoe_b200.h, fm_scheduler_config):

* async_policy: the policy half of finish_step runs on a worker thread over a
  snapshot of the target placement. Joined right after finish_step it must
  reproduce the inline (reference) scheduler exactly — the snapshot logic is
  the only thing that differs; left running it enters the queue one step
  later, deterministically.
* flip_mode 1: ops become effective one boundary after they were issued, in
  queue order; each boundary issues a non-empty queue prefix when the queue is
  non-empty; target = effective + the queued ops.
"""
import numpy as np
import pytest

import oracle
from paper_2304_03946_b200 import scheduler as S

CASES = [
    # (N, G, E, tokens, zipf, steps)
    (8, 4, 4, 8192, 1.25, 60),
    (64, 8, 16, 65536 * 8, 1.25, 40),
    (128, 8, 32, 262144, 2.0, 25),
]


def trace(N, G, tokens, zipf, steps):
    return oracle.Oracle().generate_trace(N, G, tokens, zipf=zipf, drift=0.02, seed=42, steps=steps)


@pytest.mark.parametrize("case", CASES)
def test_async_policy_joined_equals_inline(case):
    N, G, E, tokens, zipf, steps = case
    tr = trace(N, G, tokens, zipf, steps)
    prof = S.ClusterProfile.reference_default(G, E)
    ref = S.Scheduler(prof, N)
    asy = S.Scheduler(prof, N, S.SchedulerConfig.defaults(async_policy=1))
    n_ops = 0
    for s in range(steps):
        r = ref.step(tr[s])
        applied = asy.begin_step()
        a = asy.finish_step(tr[s])
        late = asy.join_policy()
        assert applied == r.applied, s
        assert a.report.makespan_s == r.report.makespan_s, s
        assert a.report.balance_ratio == r.report.balance_ratio, s
        assert late == r.accepted, s
        n_ops += len(late)
        for which in ("effective", "target"):
            assert np.array_equal(asy.placement(which)[0], ref.placement(which)[0]), (s, which)
    assert n_ops > 0


@pytest.mark.parametrize("case", CASES[:2])
def test_async_policy_lags_one_step_deterministically(case):
    N, G, E, tokens, zipf, steps = case
    tr = trace(N, G, tokens, zipf, steps)
    prof = S.ClusterProfile.reference_default(G, E)
    runs = []
    for _ in range(2):
        sch = S.Scheduler(prof, N, S.SchedulerConfig.defaults(async_policy=1))
        log = []
        for s in range(steps):
            applied = sch.begin_step()
            r = sch.finish_step(tr[s])
            log.append((applied, r.accepted, r.report.makespan_s))
        runs.append(log)
    assert runs[0] == runs[1]
    assert runs[0][0][1] == []  # nothing can be accepted before the first worker finishes
    assert sum(len(a) for _, a, _ in runs[0]) > 0


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("async_policy", [0, 1])
def test_flip_mode_issue_then_effective(case, async_policy):
    N, G, E, tokens, zipf, steps = case
    tr = trace(N, G, tokens, zipf, steps)
    prof = S.ClusterProfile.reference_default(G, E)
    sch = S.Scheduler(prof, N, S.SchedulerConfig.defaults(flip_mode=1, async_policy=async_policy))
    prev_issued = []
    queue = []  # our model of the adjustment queue
    n_flips = 0
    for s in range(steps):
        before = sch.placement("effective")[0]
        applied = sch.begin_step()
        assert applied == prev_issued, s  # exactly last boundary's batch, in order
        expect = before
        for op in applied:  # the effective placement moves by exactly these ops
            expect, _ = S.apply_op(expect, N, prof, op)
        assert np.array_equal(sch.placement("effective")[0], expect), s
        queue = queue[len(applied):]
        issued = sch.issued
        assert issued == queue[: len(issued)], s  # a queue prefix
        if queue:
            assert issued, s  # never stalls a non-empty queue
        r = sch.finish_step(tr[s])
        queue += r.accepted
        prev_issued = issued
        n_flips += len(applied)
    assert n_flips > 0
    # target = effective + every queued op
    tgt = sch.placement("effective")[0]
    if async_policy:
        queue += sch.join_policy()
    for op in queue:
        tgt, _ = S.apply_op(tgt, N, prof, op)
    assert np.array_equal(sch.placement("target")[0], tgt)
