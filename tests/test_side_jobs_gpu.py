"""Side jobs: the db2 / dWg tile column sums and the un-permute
run on spare CTA pairs of the weight-gradient GEMM launches when the shape
leaves spare pairs (64 output tiles per expert: d 1024, f 4096). Their code is
the standalone kernels' arithmetic, so every output of the backward must be
bit-identical with the side jobs on and off — checked here at the configs[1]
shape (where both side jobs run) and at a d 768 / f 3072 shape (where the
launcher declines them and the standalone kernels run in both modes).
"""
from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")

from paper_2304_03946_b200.layer import MoELayer  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = {
    # N, k, d, f, T, expected side_jobs mask with the side jobs enabled
    "configs1": (16, 2, 1024, 4096, 65536, 0b111),
    "top1_d1024": (64, 1, 1024, 4096, 32768, 0b111),
    "d768": (32, 2, 768, 3072, 32768, 0b00),
}


def _step(layer, x, dy, params, side):
    layer.set_side_jobs(side)
    y = layer.forward(x, *params)
    g = layer.backward(dy)
    torch.cuda.synchronize()
    return y.clone(), {k: v.clone() for k, v in vars(g).items() if torch.is_tensor(v)}, layer.side_jobs


@pytest.mark.parametrize("name", list(SHAPES))
def test_side_jobs_bit_identical(name):
    N, k, d, f, T, mask = SHAPES[name]
    torch.manual_seed(7)
    dev = torch.device("cuda", 0)
    layer = MoELayer(N, k, d, f, max_tokens=T)
    p = layer.init_params(seed=11)
    params = (p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
    x = torch.randn(T, d, device=dev).to(torch.bfloat16)
    dy = (torch.randn(T, d, device=dev) * 0.5).to(torch.bfloat16)
    y_on, g_on, m_on = _step(layer, x, dy, params, True)
    y_off, g_off, m_off = _step(layer, x, dy, params, False)
    assert m_on == mask, f"side jobs ran: {m_on:#b}, expected {mask:#b}"
    assert m_off == 0
    assert torch.equal(y_on, y_off)
    assert set(g_on) == set(g_off) and len(g_on) >= 5
    for key in g_on:
        assert torch.equal(g_on[key], g_off[key]), f"{key} differs between side jobs on and off"


def test_p2p_world1_side_jobs_bit_identical():
    """The P2P phase path at world 1 (what torchrun --nproc-per-node 1 runs):
    with fm_layer_p2p_bind_dx the un-permute rides beside the FFN1 weight
    gradients and waits on the arena's own "dX ready" flag; every output must
    match the standalone kernels bit for bit, and no P2P wait may time out."""
    from paper_2304_03946_b200.distributed import DistributedMoELayer, LoopbackHub

    N, k, d, f, T = 16, 2, 1024, 4096, 32768
    torch.manual_seed(3)
    dev = torch.device("cuda", 0)
    lay = MoELayer(N, k, d, f, max_tokens=T)
    p = lay.init_params(seed=5)
    dl = DistributedMoELayer(lay, LoopbackHub(1).endpoint(0), transport="p2p")
    x = torch.randn(T, d, device=dev).to(torch.bfloat16)
    dy = (torch.randn(T, d, device=dev) * 0.5).to(torch.bfloat16)
    runs = []
    for side in (True, False):
        lay.set_side_jobs(side)
        y = dl.forward(x, p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
        g = dl.backward(dy)
        torch.cuda.synchronize()
        assert not dl.p2p_timed_out()
        runs.append((y.clone(), {key: v.clone() for key, v in vars(g).items() if torch.is_tensor(v)},
                     lay.side_jobs))
    (y_on, g_on, m_on), (y_off, g_off, m_off) = runs
    assert m_on == 0b111 and m_off == 0
    assert torch.equal(y_on, y_off)
    for key in g_on:
        assert torch.equal(g_on[key], g_off[key]), f"{key} differs between side jobs on and off"


@pytest.mark.parametrize("T,cf", [(1000, 0.0), (3333, 0.0), (4096, 1.0), (2500, 1.25)])
def test_side_jobs_edge_shapes(T, cf):
    """Ragged token counts (partial 128-token gate tiles, experts with no
    rows, pair-tail tiles) and StaticEP capacity drops (cf > 0: dropped units
    carry no dispatch row, their gate gradient goes through the drop kernel):
    side jobs on and off stay bit-identical."""
    N, k, d, f = 16, 2, 1024, 4096
    torch.manual_seed(T)
    dev = torch.device("cuda", 0)
    layer = MoELayer(N, k, d, f, max_tokens=T)
    if cf:
        layer.set_capacity_factor(cf)
    p = layer.init_params(seed=T)
    params = (p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
    x = torch.randn(T, d, device=dev).to(torch.bfloat16)
    dy = (torch.randn(T, d, device=dev) * 0.5).to(torch.bfloat16)
    y_on, g_on, _ = _step(layer, x, dy, params, True)
    y_off, g_off, m_off = _step(layer, x, dy, params, False)
    assert m_off == 0
    assert torch.equal(y_on, y_off)
    for key in g_on:
        assert torch.equal(g_on[key], g_off[key]), f"{key} differs between side jobs on and off"


def test_nccl_transport_deterministic():
    """NCCL transport (staging all-to-alls), 2 loopback ranks: the gate-weight
    gradient is summed piece by piece over the send buffer in a fixed order, so
    two runs of the same step give bit-identical gradients (StaticEP drops on)."""
    import threading

    from paper_2304_03946_b200.distributed import DistributedMoELayer, LoopbackHub

    N, k, d, f, T, G = 8, 2, 256, 512, 3000, 2
    cnt = torch.zeros(N, G, dtype=torch.int32)
    for e in range(N):
        cnt[e, e % G] = 1
    cnt[0, 1] = 1  # expert 0 replicated
    torch.manual_seed(9)
    xs = [torch.randn(T, d).to(torch.bfloat16) for _ in range(G)]
    dys = [(torch.randn(T, d) * 0.5).to(torch.bfloat16) for _ in range(G)]

    def run():
        hub = LoopbackHub(G)
        outs = [None] * G

        def body(r):
            torch.cuda.set_device(0)
            lay = MoELayer(N, k, d, f, replica_counts=cnt.numpy(), num_gpus=G, rank=r, max_tokens=T)
            lay.set_capacity_factor(1.0)
            p = lay.init_params(seed=4)
            dl = DistributedMoELayer(lay, hub.endpoint(r), transport="nccl")
            dev = torch.device("cuda", 0)
            y = dl.forward(xs[r].to(dev), p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
            g = dl.backward(dys[r].to(dev))
            torch.cuda.synchronize()
            outs[r] = (y.cpu(), g.dwg.cpu(), g.dx.cpu())

        th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        return outs

    a, b = run(), run()
    for r in range(G):
        for i, name in enumerate(("y", "dwg", "dx")):
            assert torch.equal(a[r][i], b[r][i]), f"rank {r}: {name} differs between two runs"
