"""configs[2]'s layer (64 experts, top-1, d 1024, f 4096) at its full per-GPU
size, 65,536 tokens on each of two ranks, through the P2P token transport
(loopback ranks sharing one B200), against the fused single-GPU step on the
concatenated batch — a size-independent property of the path: moving units to
other GPUs must not change any token's math.

* y and dx per rank: bit-identical to the single-GPU rows (every output row is
  one GEMM row with the same K order, top-1 combine weight 1.0);
* weight gradients of experts hosted once: rows reach the expert GPU in the
  same (source, token) order as in the concatenated batch — equal to the
  single-GPU gradients within 1e-5 relative;
* the replicated hot expert: the replica-group SUM all-reduce of the two
  partial gradients equals the single-GPU gradient within 1e-2 relative (the
  sum is split at a different row), identical on both replicas.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import layer as OL  # noqa: E402
from paper_2304_03946_b200.distributed import DistributedMoELayer, LoopbackHub  # noqa: E402
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402

from tests.test_multigpu_gpu import run_ranks  # noqa: E402


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def test_configs2_full_size_p2p_matches_single_gpu():
    N, k, d, f, T, G = 64, 1, 1024, 4096, 65536, 2
    rng = np.random.default_rng(99)
    p = 1.0 / np.arange(1, N + 1) ** 1.25
    skew = np.log(p / p.sum())[rng.permutation(N)] + 2.0
    x, wg, w1, b1, w2, b2 = OL.exact_inputs(rng, T * G, d, N, f, skew=skew)
    hot = int(np.argmax(skew))
    cnt = np.zeros((N, G), np.int32)
    for e in range(N):
        cnt[e, e % G] = 1
    cnt[hot, 1 - hot % G] = 1  # the hottest expert replicated on the other GPU
    bf, f32 = torch.bfloat16, torch.float32
    dev = lambda a, dt=bf: torch.tensor(np.asarray(a), dtype=f32).to("cuda").to(dt)
    X, WG = dev(x), dev(wg)
    W1, B1, W2, B2 = dev(w1), dev(b1, f32), dev(w2), dev(b2, f32)
    DY = (torch.randn(T * G, d, device="cuda", generator=torch.Generator("cuda").manual_seed(3)) * 0.1).to(bf)

    single = MoELayer(N, k, d, f, max_tokens=T * G)
    y1 = single.forward(X, WG, W1, B1, W2, B2)
    g1 = single.backward(DY)
    torch.cuda.synchronize()

    hub = LoopbackHub(G)

    def rank_fn(r):
        torch.cuda.set_device(0)
        lay = MoELayer(N, k, d, f, replica_counts=cnt, num_gpus=G, rank=r, max_tokens=T)
        loc = lay.local_experts
        dl = DistributedMoELayer(lay, hub.endpoint(r), transport="p2p")
        xs = slice(r * T, (r + 1) * T)
        y = dl.forward(X[xs], WG, W1[loc].contiguous(), B1[loc].contiguous(), W2[loc].contiguous(),
                       B2[loc].contiguous())
        g = dl.backward(DY[xs])
        torch.cuda.synchronize()
        assert not dl.p2p_timed_out(), "a P2P arrival wait timed out"
        return dict(loc=loc, y=y.clone(), dx=g.dx.clone(), dw1=g.dw1.clone(), db1=g.db1.clone(),
                    dw2=g.dw2.clone(), db2=g.db2.clone(), dwg=g.dwg.clone())

    outs = run_ranks(G, rank_fn)
    for r, o in enumerate(outs):
        xs = slice(r * T, (r + 1) * T)
        assert torch.equal(o["y"], y1[xs]), f"y[rank {r}] differs from the single-GPU rows"
        assert torch.equal(o["dx"], g1.dx[xs]), f"dx[rank {r}] differs from the single-GPU rows"
        assert _rel(o["dwg"], g1.dwg) < 1e-2
        for i, e in enumerate(o["loc"]):
            tol = 1e-2 if e == hot else 1e-5
            for name in ("dw1", "db1", "dw2", "db2"):
                err = _rel(o[name][i], getattr(g1, name)[e])
                assert err < tol, f"{name}[expert {e} on rank {r}]: {err:.2e}"
    i0, i1 = outs[0]["loc"].index(hot), outs[1]["loc"].index(hot)
    for name in ("dw1", "db1", "dw2", "db2"):
        assert torch.equal(outs[0][name][i0], outs[1][name][i1]), f"replicas' {name} differ"
