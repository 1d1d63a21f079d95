"""Host-side multi-GPU logic on CPU: LRU communicator cache, collective order,
and — with torch.distributed gloo, world_size 2 — the replica-group gradient
sync and the all-to-all layout contract of the dispatch (peer-major send
buffers, src-major receive order, canonical expert segments).

Goldens follow proj/tests/test_sim_engine.cpp:235-294 (collective order, LRU).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_03946_b200.distributed import (
    LruGroupCache,
    TorchExchange,
    collective_order,
    collective_order_deadlock_free,
    sync_replica_grads,
)


def _initial(N, G):
    c = np.zeros((N, G), np.int32)
    c[np.arange(N), np.arange(N) % G] = 1
    return c


# ------------------------------------------------------------- reference goldens
def test_lru_group_cache_goldens():
    c = LruGroupCache(2)
    assert not c.touch((0, 1)) and c.touch((0, 1)) and c.misses == 1
    c = LruGroupCache(2)
    c.touch((0, 1)), c.touch((2, 3)), c.touch((4, 5))  # C evicts A
    assert not c.touch((0, 1)) and c.misses == 4
    c = LruGroupCache(4)
    for _ in range(100):
        c.touch((0, 1))
        c.touch((2, 3, 4))
    assert c.misses == 2
    destroyed = []
    c = LruGroupCache(1, create=lambda k: ("pg", k), destroy=destroyed.append)
    c.get((1, 0))
    c.get((2, 3))
    assert destroyed == [("pg", (0, 1))]


def test_collective_order_goldens():
    p = _initial(8, 8)
    p[5, 0] += 1
    p[2, 0] += 1  # GPU 0 hosts {0, 2, 5}; 2 and 5 replicated
    order = collective_order(p)
    assert order[0] == [2, 5] and order[1] == []
    assert all(o == [] for o in collective_order(_initial(8, 8)))
    rng = np.random.default_rng(13)
    for _ in range(100):
        p = _initial(8, 8)
        for _ in range(8):
            e, g = int(rng.integers(8)), int(rng.integers(8))
            if p[:, g].sum() < 3:
                p[e, g] += 1
        assert collective_order_deadlock_free(p)


# ------------------------------------------------------------- gloo, world 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except BaseException as exc:  # report, don't hang the parent
        q.put((rank, exc))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        if isinstance(v, BaseException):
            raise v
    return [res[r] for r in range(world)]


class _Grads:
    def __init__(self, nl, N, d, f, seed):
        g = torch.Generator().manual_seed(seed)
        self.dw1 = torch.randn(nl, f, d, generator=g)
        self.db1 = torch.randn(nl, f, generator=g)
        self.dw2 = torch.randn(nl, d, f, generator=g)
        self.db2 = torch.randn(nl, d, generator=g)
        self.dwg = torch.randn(N, d, generator=g)


CNT = np.array([[1, 1], [1, 0], [0, 1], [2, 1]], np.int32)  # experts 0 and 3 replicated


def _sync_body(rank, world):
    ex = TorchExchange()
    local = [e for e in range(CNT.shape[0]) if CNT[e, rank] > 0]
    g = _Grads(len(local), CNT.shape[0], 8, 16, seed=100 + rank)
    before = {k: getattr(g, k).clone() for k in ("dw1", "db1", "dw2", "db2", "dwg")}
    sync_replica_grads(ex, CNT, local, g)
    return local, before, {k: getattr(g, k) for k in before}, ex.groups.misses


@pytest.mark.timeout(300)
def test_replica_grad_sync_gloo():
    (l0, b0, a0, m0), (l1, b1, a1, m1) = _spawn(_sync_body)
    assert l0 == [0, 1, 3] and l1 == [0, 2, 3]
    for e in (0, 3):  # replicated: SUM over the group on both members
        i0, i1 = l0.index(e), l1.index(e)
        for k in ("dw1", "db1", "dw2", "db2"):
            s = b0[k][i0] + b1[k][i1]
            assert torch.allclose(a0[k][i0], s) and torch.allclose(a1[k][i1], s)
    assert torch.equal(a0["dw1"][1], b0["dw1"][1])  # expert 1 only on GPU 0: untouched
    assert torch.equal(a1["dw1"][1], b1["dw1"][1])  # expert 2 only on GPU 1
    assert torch.allclose(a0["dwg"], b0["dwg"] + b1["dwg"])
    assert m0 == m1 == 1  # both groups are {0, 1}: one communicator, cached


def _layout_body(rank, world):
    """Dispatch layout contract through real collectives: each rank sends token
    ids (rank, t) in its canonical send order; the receiver's relayout must
    produce segments ordered by (src ascending, canonical rank)."""
    import oracle
    from oracle import layer as OL

    ex = TorchExchange()
    N, k, T = 6, 2, 50
    cnt = np.array([[1, 1], [1, 0], [0, 1], [1, 0], [0, 1], [1, 1]], np.int32)
    rng = np.random.default_rng(rank)
    logits = rng.standard_normal((T, N)) + np.array([2, 1, 0, 0, -1, 1.5])
    idx = np.argsort(-logits, axis=1, kind="stable")[:, :k].astype(np.int32)
    hist = torch.tensor(OL.histogram(idx, N))
    D = ex.all_gather(hist).numpy().T  # [N, G]
    flows = oracle.Oracle().route(D, cnt)
    rows, dsts = OL.dispatch_rows(idx, OL.unit_ranks(idx, N), flows, rank, world, N)
    send = torch.zeros(T * k, 2)
    for t in range(T):
        for j in range(k):
            send[rows[t, j]] = torch.tensor([rank, t * k + j], dtype=torch.float32)
    send_rows = [int(flows[:, rank, d].sum()) for d in range(world)]
    recv_rows = [int(flows[:, s, rank].sum()) for s in range(world)]
    recv = torch.zeros(sum(recv_rows), 2)
    ex.all_to_all(recv, send, recv_rows, send_rows)
    # relayout: receive order is (src, local expert ascending, rank order)
    local = [e for e in range(N) if cnt[e, rank] > 0]
    segs = {e: [] for e in local}
    o = 0
    for s in range(world):
        for e in local:
            c = int(flows[e, s, rank])
            segs[e].extend(tuple(map(int, r)) for r in recv[o:o + c].tolist())
            o += c
    return segs, idx, flows


@pytest.mark.timeout(300)
def test_dispatch_layout_gloo():
    import oracle  # noqa: F401
    from oracle import layer as OL

    (segs0, idx0, fl0), (segs1, idx1, fl1) = _spawn(_layout_body)
    assert (fl0 == fl1).all()
    idx = [idx0, idx1]
    N, k = idx0.shape[1] * 3, idx0.shape[1]
    for me, segs in enumerate([segs0, segs1]):
        for e, got in segs.items():
            assert len(got) == fl0[e, :, me].sum()
            # expected: src ascending; within a src, the units this dst got, in rank order
            exp = []
            for s in range(2):
                units = [u for u in range(idx[s].size) if idx[s].reshape(-1)[u] == e]
                lo = 0
                order = [s] + [g for g in range(2) if g != s]
                for dst in order:
                    c = int(fl0[e, s, dst])
                    if dst == me:
                        exp.extend((s, u) for u in units[lo:lo + c])
                    lo += c
            assert got == exp, (me, e)


def _p2p_body(rank, world):
    """Migration transport: batched send/recv pairs matched per (src, dst) in order."""
    ex = TorchExchange()
    a = torch.full((4, 3), float(rank + 1))
    b = torch.arange(5, dtype=torch.float32) + 10 * rank
    sends = [(1 - rank, a), (1 - rank, b)]
    ra, rb = torch.empty(4, 3), torch.empty(5)
    ex.p2p(sends, [(1 - rank, ra), (1 - rank, rb)])
    ex.p2p([], [])  # empty rounds are legal (every rank calls p2p every step)
    return ra, rb


@pytest.mark.timeout(300)
def test_p2p_migration_transport_gloo():
    (ra0, rb0), (ra1, rb1) = _spawn(_p2p_body)
    assert torch.equal(ra0, torch.full((4, 3), 2.0)) and torch.equal(ra1, torch.full((4, 3), 1.0))
    assert torch.equal(rb0, torch.arange(5.0) + 10) and torch.equal(rb1, torch.arange(5.0))


# three GPUs, four distinct replica groups ({0,1}, {1,2}, {0,2}, {0,1,2}): with a
# two-entry communicator cache every step evicts groups that some ranks are not
# members of (torch hands non-members a placeholder, not a process group)
CNT3 = np.array([[1, 1, 0], [0, 1, 1], [1, 0, 1], [1, 1, 1], [1, 0, 0]], np.int32)


def _evict_body(rank, world):
    ex = TorchExchange(max_live_groups=2)
    local = [e for e in range(CNT3.shape[0]) if CNT3[e, rank] > 0]
    outs = []
    for step in range(2):
        g = _Grads(len(local), CNT3.shape[0], 4, 8, seed=10 * step + rank)
        before = {k: getattr(g, k).numpy().copy() for k in ("dw1", "db1", "dw2", "db2")}
        sync_replica_grads(ex, CNT3, local, g)
        outs.append((before, {k: getattr(g, k).numpy().copy() for k in before}))
    return local, outs, ex.groups.misses  # numpy: tensors in the queue outlive the worker


@pytest.mark.timeout(300)
def test_replica_grad_sync_group_eviction_gloo():
    res = _spawn(_evict_body, world=3)
    for step in range(2):
        for e in range(CNT3.shape[0]):
            members = [r for r in range(3) if CNT3[e, r] > 0]
            if len(members) < 2:
                continue
            for k in ("dw1", "db1", "dw2", "db2"):
                s = sum(res[r][1][step][0][k][res[r][0].index(e)] for r in members)
                for r in members:
                    assert np.allclose(res[r][1][step][1][k][res[r][0].index(e)], s, atol=1e-5)
    assert all(m == 8 for _, _, m in res)  # 4 groups x 2 steps, cache of 2: every touch misses
