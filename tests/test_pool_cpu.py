"""Slot bookkeeping of the expert state pool (host logic, no GPU).

Every rank keeps every rank's slot table and applies the same placement
changes; the pull list derived from it must be identical everywhere, never
reuse a slot vacated in the same step (a peer may still be reading it), and
always name the source's current slot."""
import numpy as np

from paper_2304_03946_b200 import scheduler as S
from paper_2304_03946_b200.pool import SlotAllocator, apply_placement_change, state_moves


def test_state_moves_lowest_holder():
    old = np.array([[1, 0, 1], [0, 1, 0]])
    new = np.array([[1, 1, 1], [1, 0, 1]])
    # expert 0 gains GPU 1 (from GPU 0); expert 1 moves from GPU 1 to GPUs 0 and 2
    assert state_moves(old, new) == [(0, 0, 1), (1, 1, 0), (1, 1, 2)]


def test_vacated_slot_not_reused_in_same_step():
    dirs = [SlotAllocator(2) for _ in range(2)]
    old = np.array([[1, 0], [1, 0]])  # experts 0 and 1 on GPU 0
    for e in (0, 1):
        dirs[0].host(e)
    # expert 0 migrates GPU0 -> GPU1 while expert 1 stays (GPU0's two slots were both in use)
    new = np.array([[0, 1], [1, 0]])
    pulls = apply_placement_change(dirs, old, new)
    assert pulls == [(0, 0, 0, 1, 0)]  # GPU1 pulls GPU0's slot 0 into its slot 0
    assert 0 not in dirs[0].slot_of and dirs[0].slot_of[1] == 1
    # same step: GPU0 may not take slot 0 back -> only after begin_step
    assert dirs[0]._free == [] and dirs[0]._vacated == [0]
    old, new2 = new, np.array([[1, 1], [1, 0]])  # next step: expert 0 expands back onto GPU 0
    pulls = apply_placement_change(dirs, old, new2)
    assert pulls == [(0, 1, 0, 0, 0)]  # now slot 0 is free again


def test_directory_identical_on_all_ranks_random_ops():
    rng = np.random.default_rng(5)
    N, G, E = 12, 4, 6
    prof = S.ClusterProfile.reference_default(G, E)
    sched_slots = S.slots_from_counts(np.eye(N, G, dtype=np.int32) + np.eye(N, G, -G, dtype=np.int32)
                                      + np.eye(N, G, -2 * G, dtype=np.int32), E)
    dirs_per_rank = [[SlotAllocator(2 * E) for _ in range(G)] for _ in range(G)]
    counts = S.counts_from_slots(sched_slots, N)
    for dirs in dirs_per_rank:
        for g in range(G):
            for e in range(N):
                if counts[e, g] > 0:
                    dirs[g].host(e)
    slots = sched_slots.copy()
    for step in range(60):
        old = S.counts_from_slots(slots, N)
        # random legal expand/shrink ops
        e, g = int(rng.integers(N)), int(rng.integers(G))
        if old[e, g] == 0 and (slots[g] < 0).any():
            op = (S.EXPAND, e, g, -1, -1, -1, -1)
        elif old[e].astype(bool).sum() > 1 and old[e, g] > 0:
            op = (S.SHRINK, e, g, -1, -1, -1, -1)
        else:
            continue
        slots, _ = S.apply_op(slots, N, prof, op)
        new = S.counts_from_slots(slots, N)
        pulls = [apply_placement_change(dirs, old, new) for dirs in dirs_per_rank]
        assert all(p == pulls[0] for p in pulls[1:])
        for e_, src, ss, dst, ds in pulls[0]:
            assert old[e_, src] > 0 and new[e_, dst] > 0 and old[e_, dst] == 0
        for g in range(G):  # hosted experts == placement, distinct slots
            d = dirs_per_rank[0][g]
            assert set(d.slot_of) == set(np.nonzero(new[:, g] > 0)[0].tolist())
            assert len(set(d.slot_of.values())) == len(d.slot_of)
