"""Multi-GPU layer path on one B200: G virtual ranks (threads) drive the real
phase kernels (gate, route over the all-gathered demand, dispatch into
peer-major send buffers, relayout, expert FFN, combine, and the backward
mirror) with an in-process loopback transport, then the replica-group
gradient sync. Checked against the CPU oracle:

* bit-exact: all-gathered TokenDemand, flows (= reference route()), every
  rank's dispatch rows (canonical permutation), per-peer row counts;
* bf16 tolerance (see test_layer_gpu.py): y and dx per rank equal the
  single-GPU oracle on the same tokens (replicas hold identical weights);
* after the SUM all-reduce over each replica group, every replica's weight
  gradients equal the oracle's full-batch gradients (rel. error <= 1e-2).
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import layer as OL  # noqa: E402
from paper_2304_03946_b200.distributed import (  # noqa: E402
    DistributedMoELayer,
    LoopbackHub,
    collective_order_deadlock_free,
)
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402

from tests.test_layer_gpu import close_bf16, close_f32  # noqa: E402


def run_ranks(G, fn):
    errs, outs = [None] * G, [None] * G

    def body(r):
        try:
            outs[r] = fn(r)
        except BaseException as exc:  # surface in the main thread
            errs[r] = exc

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for e in errs:
        if e is not None:
            raise e
    return outs


PLACEMENTS = {
    # config-1 shape: 8 experts on 4 GPUs, expert 0 expanded onto GPUs 1 and 2
    "cfg1_expanded": (8, 4, [(e, e % 4) for e in range(8)] + [(0, 1), (0, 2)]),
    # hot expert replicated everywhere, two slots of expert 3 on GPU 0
    "replicated": (8, 4, [(e, e % 4) for e in range(8)] + [(5, 0), (5, 2), (5, 3), (3, 0)]),
    "two_gpus": (16, 2, [(e, e % 2) for e in range(16)] + [(1, 0), (2, 1)]),
    # configs[2]-like width: N*G = 512 > the plan kernel's 256 threads (multi-
    # element scans), a hot expert on four GPUs
    "wide_8gpus": (64, 8, [(e, e % 8) for e in range(64)] + [(0, 1), (0, 2), (0, 3), (5, 0), (9, 7)]),
    # a GPU that hosts no expert: it only sends its tokens and receives outputs
    "idle_gpu": (8, 4, [(e, e % 3) for e in range(8)] + [(0, 1)]),
}


def p2p_rows(idx, flows, me, G, N, cnt):
    """P2P: row of each unit in its destination GPU's X_perm (that GPU's padded
    expert segments, sources ascending inside a segment, then rank)."""
    ranks = OL.unit_ranks(idx, N)
    starts = {}
    for dst in range(G):
        local = [e for e in range(N) if cnt[e, dst] > 0]
        for e, (s0, _, _) in zip(local, OL.segments(flows, local, dst)):
            starts[(e, dst)] = s0 + int(flows[e, :me, dst].sum())
    order = [me] + [g for g in range(G) if g != me]
    rows = np.zeros(idx.shape, np.int64)
    for t in range(idx.shape[0]):
        for j in range(idx.shape[1]):
            e, r, lo = idx[t, j], ranks[t, j], 0
            for dst in order:
                c = flows[e, me, dst]
                if r < lo + c:
                    rows[t, j] = starts[(e, dst)] + r - lo
                    break
                lo += c
    return rows


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("name", sorted(PLACEMENTS))
def test_multigpu_loopback_parity(name, transport):
    """transport "nccl": staging buffers + all-to-alls (loopback copies here);
    "p2p": rows written / read directly in the peers' permuted buffers inside
    the dispatch / combine / un-permute kernels, device-side arrival flags."""
    N, G, pairs = PLACEMENTS[name]
    k, d, f, T = 2, 256, 512, 600
    cnt = np.zeros((N, G), np.int32)
    for e, g in pairs:
        cnt[e, g] += 1
    assert collective_order_deadlock_free(cnt)
    rng = np.random.default_rng(7)
    p = 1.0 / np.arange(1, N + 1) ** 1.25
    skew = np.log(p / p.sum())[rng.permutation(N)] + 3
    X, wg, w1, b1, w2, b2 = OL.exact_inputs(rng, T * G, d, N, f, skew=skew)
    dY = OL.bf16(rng.standard_normal((T * G, d)) * 0.5)
    st = OL.forward(X, wg, w1, b1, w2, b2, k)  # full batch, single-GPU math
    gr = OL.backward(st, dY)

    hub = LoopbackHub(G)
    bf = torch.bfloat16
    dev = lambda a, dt=bf: torch.tensor(np.asarray(a), dtype=dt, device="cuda")

    def rank_fn(r):
        torch.cuda.set_device(0)
        lay = MoELayer(N, k, d, f, replica_counts=cnt, num_gpus=G, rank=r, max_tokens=T)
        loc = lay.local_experts
        dl = DistributedMoELayer(lay, hub.endpoint(r), transport=transport)
        xs = slice(r * T, (r + 1) * T)
        y = dl.forward(dev(X[xs]), dev(wg), dev(w1[loc]), dev(b1[loc], torch.float32),
                       dev(w2[loc]), dev(b2[loc], torch.float32))
        g = dl.backward(dev(dY[xs]))
        torch.cuda.synchronize()
        idx = lay.read("topk_idx", T * k).reshape(T, k)
        pos = lay.read("unit_pos", T * k).reshape(T, k)
        flows = lay.read("flows", N * G * G).reshape(N, G, G)
        D = dl.last_demand.cpu().numpy()
        if transport == "p2p":
            assert not dl.p2p_timed_out(), "a P2P arrival wait timed out"
        st_ = dl._st
        return dict(loc=loc, y=y.float().cpu().numpy(), idx=idx, pos=pos, flows=flows, D=D,
                    send_rows=st_.send_rows if st_ else None, recv_rows=st_.recv_rows if st_ else None,
                    dx=g.dx.float().cpu().numpy(), dw1=g.dw1.cpu().numpy(), dw2=g.dw2.cpu().numpy(),
                    db1=g.db1.cpu().numpy(), db2=g.db2.cpu().numpy(), dwg=g.dwg.cpu().numpy())

    outs = run_ranks(G, rank_fn)

    # ---- routing state, bit-exact
    hist = np.stack([OL.histogram(st["idx"][r * T:(r + 1) * T], N) for r in range(G)])  # [G, N]
    flows_ref = oracle.Oracle().route(hist.T, cnt)
    for r, o in enumerate(outs):
        assert (o["D"] == hist).all(), "all-gathered demand differs"
        assert (o["flows"] == flows_ref).all(), "flows differ from route()"
        idx_r = st["idx"][r * T:(r + 1) * T]
        assert (o["idx"] == idx_r).all()
        if transport == "p2p":
            rows = p2p_rows(idx_r, flows_ref, r, G, N, cnt)
            assert (o["pos"] == rows).all(), f"rank {r}: X_perm rows on the expert GPUs differ"
            continue
        rows, _ = OL.dispatch_rows(idx_r, OL.unit_ranks(idx_r, N), flows_ref, r, G, N)
        assert (o["pos"] == rows).all(), f"rank {r}: dispatch rows differ"
        assert o["send_rows"] == [int(flows_ref[:, r, dst].sum()) for dst in range(G)]
        assert o["recv_rows"] == [int(flows_ref[:, src, r].sum()) for src in range(G)]

    # ---- outputs and gradients
    for r, o in enumerate(outs):
        xs = slice(r * T, (r + 1) * T)
        close_bf16(o["y"], st["y"][xs], f"y[rank {r}]")
        close_bf16(o["dx"], gr["dx"][xs], f"dx[rank {r}]")
        for i, e in enumerate(o["loc"]):
            close_f32(o["dw1"][i], gr["dw1"][e], f"dw1[e{e}@{r}]")
            close_f32(o["dw2"][i], gr["dw2"][e], f"dw2[e{e}@{r}]")
            close_f32(o["db1"][i], gr["db1"][e], f"db1[e{e}@{r}]")
            close_f32(o["db2"][i], gr["db2"][e], f"db2[e{e}@{r}]")
        close_f32(o["dwg"], gr["dwg"], f"dwg[{r}]", tol=2e-2)


def test_phase_api_single_gpu_matches_fused():
    """G == 1 through the phase API (identity exchange) equals the fused step."""
    N, k, d, f, T = 8, 2, 256, 256, 1000
    rng = np.random.default_rng(11)
    x, wg, w1, b1, w2, b2 = OL.exact_inputs(rng, T, d, N, f)
    dy = OL.bf16(rng.standard_normal((T, d)))
    bf = torch.bfloat16
    dev = lambda a, dt=bf: torch.tensor(np.asarray(a), dtype=dt, device="cuda")
    P = [dev(wg), dev(w1), dev(b1, torch.float32), dev(w2), dev(b2, torch.float32)]
    fused = MoELayer(N, k, d, f, max_tokens=T)
    y1 = fused.forward(dev(x), *P)
    g1 = fused.backward(dev(dy))
    hub = LoopbackHub(1)
    phased = DistributedMoELayer(MoELayer(N, k, d, f, max_tokens=T), hub.endpoint(0))
    y2 = phased.forward(dev(x), *P)
    g2 = phased.backward(dev(dy))
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(g1.dx, g2.dx)
    for a, b in [(g1.dw1, g2.dw1), (g1.dw2, g2.dw2), (g1.db1, g2.db1)]:
        assert torch.allclose(a, b, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_multigpu_rank_without_tokens(transport):
    """Ragged ranks: GPU 1 contributes no tokens this step but hosts experts —
    it still receives GPU 0's units, computes them and returns the outputs;
    GPU 0's y / dx equal the single-GPU step on its tokens (bit-identical),
    GPU 1's are empty."""
    N, k, d, f, G = 8, 2, 256, 512, 2
    Ts = [700, 0]
    cnt = np.zeros((N, G), np.int32)
    for e in range(N):
        cnt[e, e % G] = 1
    cnt[0, 1] = 1
    rng = np.random.default_rng(21)
    x, wg, w1, b1, w2, b2 = OL.exact_inputs(rng, Ts[0], d, N, f)
    dY = OL.bf16(rng.standard_normal((Ts[0], d)) * 0.5)
    bf = torch.bfloat16
    dev = lambda a, dt=bf: torch.tensor(np.asarray(a), dtype=dt, device="cuda")
    single = MoELayer(N, k, d, f, max_tokens=Ts[0])
    y1 = single.forward(dev(x), dev(wg), dev(w1), dev(b1, torch.float32), dev(w2), dev(b2, torch.float32))
    g1 = single.backward(dev(dY))
    torch.cuda.synchronize()
    hub = LoopbackHub(G)

    def rank_fn(r):
        torch.cuda.set_device(0)
        lay = MoELayer(N, k, d, f, replica_counts=cnt, num_gpus=G, rank=r, max_tokens=max(Ts))
        loc = lay.local_experts
        dl = DistributedMoELayer(lay, hub.endpoint(r), transport=transport)
        xr = dev(x) if r == 0 else torch.empty(0, d, dtype=bf, device="cuda")
        dyr = dev(dY) if r == 0 else torch.empty(0, d, dtype=bf, device="cuda")
        y = dl.forward(xr, dev(wg), dev(w1[loc]), dev(b1[loc], torch.float32), dev(w2[loc]),
                       dev(b2[loc], torch.float32))
        g = dl.backward(dyr)
        torch.cuda.synchronize()
        if transport == "p2p":
            assert not dl.p2p_timed_out()
        return y.clone(), g.dx.clone()

    outs = run_ranks(G, rank_fn)
    assert torch.equal(outs[0][0], y1) and torch.equal(outs[0][1], g1.dx)
    assert outs[1][0].shape == (0, d) and outs[1][1].shape == (0, d)


@pytest.mark.parametrize("N,G", [(256, 64), (64, 32)])
def test_plan_large_world_matches_route(N, G):
    """Flows beyond the plan kernel's shared-memory staging (N*G*G int32 >
    200 KB: 256 experts on 64 GPUs, 64 on 32) are read from global memory:
    the device route + plan of rank 0 still equal the host route() bit for bit,
    and the per-peer row counts equal the flows' sums."""
    from paper_2304_03946_b200 import _lib as L
    from paper_2304_03946_b200 import routing

    k, d, f, T = 2, 256, 256, 256
    rng = np.random.default_rng(N + G)
    cnt = np.zeros((N, G), np.int32)
    cnt[np.arange(N), np.arange(N) % G] = 1
    cnt[0, :] = 1  # one expert on every GPU
    cnt[1, G // 2] += 1
    D = np.zeros((N, G), np.int64)
    for g in range(G):  # each GPU's column sums to T * k
        D[:, g] = np.bincount(rng.integers(0, N, T * k), minlength=N)
    lay = MoELayer(N, k, d, f, replica_counts=cnt, num_gpus=G, rank=0, max_tokens=T)
    gathered = torch.tensor(D.T.copy(), device="cuda")
    send = np.zeros(G, np.int32)
    recv = np.zeros(G, np.int32)
    L.check(L.lib().fm_layer_route(lay._h, gathered.data_ptr(), send.ctypes.data, recv.ctypes.data,
                                   L.stream_ptr()))
    flows = lay.read("flows", N * G * G).reshape(N, G, G)
    ref = routing.route(D, cnt)
    assert (flows == ref).all()
    assert (send == ref[:, 0, :].sum(axis=0)).all()
    assert (recv == ref[:, :, 0].sum(axis=0)).all()
