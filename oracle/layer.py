"""TEST INFRASTRUCTURE ONLY — numpy restatement of the MoE-layer math.

The reference has no implementation of the gate, token permutation, expert
FFN or combine ("parity for these is unpinned by the
reference"); this module restates them from the paper and the SPEC:

* gate      g(x) = softmax(TopK(x . W_g))          PAPER.md:219-223 (Eq. 3)
             TopK ties -> lower expert id           SPEC.md:436 convention
             one demand unit per (token, k-slot)
* FFN       W2 . ReLU(W1 . x + b1) + b2            PAPER.md:206-210 (Eq. 2)
* combine   y = sum_i g(x)_i e_i(x)                 PAPER.md:225-229 (Eq. 4)
* counts    route()                                 proj/src/router.cpp:57-169
            (via the C oracle, itself pinned to the reference)
* layout    canonical permutation of DESIGN.md §2.

Arithmetic: float64 with the product's bf16 storage points mirrored
(activations after ReLU, expert outputs, dY rows, dH, dX rows, y, dx are
rounded to bf16 exactly where the device stores bf16), so remaining
differences are f32-vs-f64 accumulation order only. `dtype=np.float32` runs
the same math in float32 on multithreaded BLAS (all host cores): that is the
CPU layer baseline bench.py times, checked against the
float64 path in tests/test_oracle_layer_cpu.py.
"""
from __future__ import annotations

import numpy as np

from . import Oracle

ROW_ALIGN = 128


def bf16(a) -> np.ndarray:
    """Round to bfloat16 (round-to-nearest-even), returned as float64."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def bf16_f32(a) -> np.ndarray:
    """bf16 rounding (RNE) of a float32 array, kept in float32 (in place;
    finite inputs). Large arrays go through the C oracle's OpenMP loop."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.size >= (1 << 20):
        return Oracle().bf16_round_f32(a)
    u = a.view(np.uint32)
    u += np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    u &= np.uint32(0xFFFF0000)
    return u.view(np.float32)


def _bf16(a, dt):
    """bf16 storage rounding in the working precision."""
    return bf16(a) if dt == np.float64 else bf16_f32(np.asarray(a, np.float32))


def gate(x, wg, k, dt=np.float64):
    """Returns (idx [T,k] int32, w [T,k], logits [T,N])."""
    logits = np.asarray(x, dt) @ np.asarray(wg, dt).T
    order = np.argsort(-logits, axis=1, kind="stable")  # equal logits keep ascending id
    idx = order[:, :k].astype(np.int32)
    kept = np.take_along_axis(logits, idx, axis=1)
    ex = np.exp(kept - kept[:, :1])
    w = ex / ex.sum(axis=1, keepdims=True)
    return idx, w, logits


def histogram(idx, N):
    return np.bincount(idx.reshape(-1), minlength=N).astype(np.int64)


def unit_ranks(idx, N):
    """Rank of each unit among units of the same expert, ascending token order
    (units are in (token, slot) order; a stable sort by expert keeps it)."""
    T, k = idx.shape
    flat = idx.reshape(-1).astype(np.int64)
    order = np.argsort(flat, kind="stable")
    start = np.concatenate([[0], np.cumsum(np.bincount(flat, minlength=N))[:-1]])
    ranks = np.empty(flat.shape[0], np.int64)
    ranks[order] = np.arange(flat.shape[0]) - start[flat[order]]
    return ranks.reshape(T, k)


def dispatch_rows(idx, ranks, flows, me, G, N):
    """Row of each unit in the source's dispatch buffer (dst-major, expert-minor).

    Chunk order within (me, e): me first, then ascending dst != me.
    """
    T, k = idx.shape
    send_off = np.zeros((N, G), np.int64)
    off = 0
    for dst in range(G):
        for e in range(N):
            send_off[e, dst] = off
            off += flows[e, me, dst]
    rows = np.zeros((T, k), np.int64)
    dsts = np.zeros((T, k), np.int64)
    order = [me] + [g for g in range(G) if g != me]
    for t in range(T):
        for j in range(k):
            e, r = idx[t, j], ranks[t, j]
            lo = 0
            for dst in order:
                c = flows[e, me, dst]
                if r < lo + c:
                    rows[t, j] = send_off[e, dst] + r - lo
                    dsts[t, j] = dst
                    break
                lo += c
    return rows, dsts


def segments(flows, local_experts, me):
    """(seg_start, seg_real, seg_rows) of the padded expert segments on `me`."""
    start, out = 0, []
    for e in local_experts:
        real = int(flows[e, :, me].sum())
        rows = (real + ROW_ALIGN - 1) // ROW_ALIGN * ROW_ALIGN
        out.append((start, real, rows))
        start += rows
    return out


def single_gpu_positions(idx, N, capacity_factor=0.0):
    """G == 1: X_perm row of each unit (-1 = dropped) and the segment table.

    With capacity_factor > 0 (StaticEP, baselines.cpp:89-122) the demand is
    first cut to static_ep_kept (C oracle, pinned to the reference); the
    units dropped are the last ones of each expert in canonical order."""
    ranks = unit_ranks(idx, N)
    hist = histogram(idx, N)
    routed = hist.reshape(N, 1)
    if capacity_factor > 0 and np.isfinite(capacity_factor):
        routed, _ = Oracle().static_ep_kept(routed, capacity_factor)
    flows = Oracle().route(routed, np.ones((N, 1), np.int32))
    segs = segments(flows, list(range(N)), 0)
    seg_start = np.array([s[0] for s in segs], np.int64)
    keep = ranks < routed[idx, 0]
    pos = np.where(keep, seg_start[idx] + ranks, -1)
    return pos, segs, flows, hist


def forward(x, wg, w1, b1, w2, b2, k, capacity_factor=0.0, dtype=np.float64):
    """Single-GPU layer forward. Weights [N,...] in expert order. Returns a state dict."""
    dt = dtype
    x = np.asarray(x, dt)
    T, d = x.shape
    N = wg.shape[0]
    idx, w, logits = gate(x, wg, k, dt)
    pos, segs, flows, hist = single_gpu_positions(idx, N, capacity_factor)
    rows = sum(s[2] for s in segs)
    f = w1.shape[1]
    x_perm = np.zeros((rows, d), dt)
    for j in range(k):
        kept = pos[:, j] >= 0
        x_perm[pos[kept, j]] = x[kept]
    act = np.zeros((rows, f), dt)
    y_perm = np.zeros((rows, d), dt)
    for e, (s0, real, r) in enumerate(segs):
        if r == 0:
            continue
        seg = slice(s0, s0 + r)
        act[seg] = _bf16(np.maximum(x_perm[seg] @ np.asarray(w1[e], dt).T + np.asarray(b1[e], dt), 0), dt)
        y_perm[seg] = _bf16(act[seg] @ np.asarray(w2[e], dt).T + np.asarray(b2[e], dt), dt)
    live = (pos >= 0).astype(dt)  # dropped units contribute nothing
    y = _bf16(np.einsum("tk,tkd->td", w.astype(np.float32).astype(dt) * live, y_perm[np.maximum(pos, 0)]), dt)
    return dict(x=x, wg=np.asarray(wg, dt), w1=w1, w2=w2, idx=idx, w=w, logits=logits,
                pos=pos, segs=segs, flows=flows, hist=hist, x_perm=x_perm, act=act,
                y_perm=y_perm, y=y, k=k, dt=dt)


def backward(st, dy):
    dt = st.get("dt", np.float64)
    dy = np.asarray(dy, dt)
    idx, w, pos, segs = st["idx"], st["w"], st["pos"], st["segs"]
    x_perm, act, y_perm = st["x_perm"], st["act"], st["y_perm"]
    T, k = idx.shape
    N, d = st["wg"].shape
    f = act.shape[1]
    wf = w.astype(np.float32).astype(dt)
    dy_perm = np.zeros_like(y_perm)
    live = pos >= 0
    for j in range(k):
        dy_perm[pos[live[:, j], j]] = _bf16(wf[live[:, j], j : j + 1] * dy[live[:, j]], dt)
    dw = np.einsum("td,tkd->tk", dy, y_perm[np.maximum(pos, 0)]) * live
    dl = wf * (dw - (wf * dw).sum(axis=1, keepdims=True))
    dh = np.zeros((x_perm.shape[0], f), dt)
    dx_perm = np.zeros_like(x_perm)
    dw1 = np.zeros((N, f, d), dt)
    dw2 = np.zeros((N, d, f), dt)
    db1 = np.zeros((N, f), dt)
    db2 = np.zeros((N, d), dt)
    for e, (s0, real, r) in enumerate(segs):
        if r == 0:
            continue
        seg = slice(s0, s0 + r)
        da = dy_perm[seg] @ np.asarray(st["w2"][e], dt)
        dh[seg] = _bf16(da * (act[seg] > 0), dt)
        dx_perm[seg] = _bf16(dh[seg] @ np.asarray(st["w1"][e], dt), dt)
        dw1[e] = dh[seg].T @ x_perm[seg]
        dw2[e] = dy_perm[seg].T @ act[seg]
        db1[e] = dh[seg].sum(axis=0)
        db2[e] = dy_perm[seg].sum(axis=0)
    gate_in = np.einsum("tk,tkd->td", dl, st["wg"][idx]) if k > 1 else 0.0
    dx = _bf16((dx_perm[np.maximum(pos, 0)] * live[:, :, None]).sum(axis=1) + gate_in, dt)
    dwg = np.zeros((N, d), dt)
    if k > 1:  # sum over units of expert e of dl * x: one [N, T] x [T, d] product per k-slot
        for j in range(k):
            sel = np.zeros((N, T), dt)
            sel[idx[:, j], np.arange(T)] = dl[:, j]
            dwg += sel @ st["x"]
    return dict(dx=dx, dwg=dwg, dw1=dw1, dw2=dw2, db1=db1, db2=db2, dl=dl, dy_perm=dy_perm,
                dh=dh, dx_perm=dx_perm)


def exact_inputs(rng, T, d, N, f, skew=None, wdtype=np.float64):
    """Exact-arithmetic parity inputs: x in {j/8}, Wg in {j/64}
    (|j| <= 8), so every logit is a multiple of 2^-9 with |logit| <= d/8 and is
    computed exactly in f32 in any order -> top-k comparable bit for bit.
    `skew` (log-popularity per expert) is added through a constant feature
    column, quantised to multiples of 1/64 and then to bf16 (|v| >= 4 keeps
    only 1/32 steps), as in the bench's Zipf gate: the device multiplies the
    bf16 value, so the oracle must too. `wdtype=np.float32` keeps the expert
    weights (bf16 values, exact in f32) at half the host memory — for the
    128-expert d1024/f4096 shape (a different random stream than float64)."""
    x = rng.integers(-8, 9, size=(T, d)) / 8.0
    wg = rng.integers(-8, 9, size=(N, d)) / 64.0
    if skew is not None:
        x[:, 0] = 1.0
        wg[:, 0] = bf16(np.clip(np.round(np.asarray(skew) * 64) / 64, -8, 8))
    if wdtype == np.float32:
        w1 = bf16_f32(rng.standard_normal((N, f, d), dtype=np.float32) * np.float32(d**-0.5))
        w2 = bf16_f32(rng.standard_normal((N, d, f), dtype=np.float32) * np.float32(f**-0.5))
    else:
        w1 = bf16(rng.standard_normal((N, f, d)) * d**-0.5)
        w2 = bf16(rng.standard_normal((N, d, f)) * f**-0.5)
    b1 = (rng.standard_normal((N, f)) * 0.1).astype(np.float32).astype(np.float64)
    b2 = (rng.standard_normal((N, d)) * 0.1).astype(np.float32).astype(np.float64)
    return x, wg, w1, b1, w2, b2
