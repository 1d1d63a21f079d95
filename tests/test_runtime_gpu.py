"""Dynamic placement in the loop, on one B200 with G virtual ranks (threads):
device gate -> all-gathered demand -> host scheduler (expand/shrink/migrate)
-> peer copies of expert weights + Adam state -> placement flip.

Checks: every rank sees the same placements and balance ratios; ops are
applied; replicas of every expert hold bit-identical state after migrations
and optimizer steps; the step output equals the fused single-GPU layer run
with the same weights (bf16 tolerance of test_layer_gpu.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2304_03946_b200 import scheduler as S  # noqa: E402
from paper_2304_03946_b200.distributed import LoopbackHub  # noqa: E402
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402
from paper_2304_03946_b200.runtime import FlexMoERuntime  # noqa: E402

from tests.test_layer_gpu import close_bf16  # noqa: E402
from tests.test_multigpu_gpu import run_ranks  # noqa: E402


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_runtime_dynamic_placement_loopback(transport):
    N, k, d, f, T, G, E, steps = 8, 2, 256, 256, 512, 4, 4, 10
    hub = LoopbackHub(G)
    gen = torch.Generator(device="cpu").manual_seed(0)
    wg = torch.randn(N, d, generator=gen) * d**-0.5
    wg[:, 0] = torch.tensor(np.log(1.0 / np.arange(1, N + 1) ** 1.5) * 2 + 3, dtype=torch.float32)
    xs = [torch.randn(T, d, generator=gen).to(torch.bfloat16) for _ in range(G)]
    for x in xs:
        x[:, 0] = 0.5
    dys = [(torch.randn(T, d, generator=gen) * 0.1).to(torch.bfloat16) for _ in range(G)]
    snap = {}

    def rank_fn(r):
        torch.cuda.set_device(0)
        rt = FlexMoERuntime(N, k, d, f, hub.endpoint(r), S.ClusterProfile.reference_default(G, E),
                            max_tokens=T, gate_weight=wg, lr=1e-3, transport=transport)
        x, dy = xs[r].cuda(), dys[r].cuda()
        hist = []
        for s in range(steps):
            if s == steps - 1:  # snapshot the weights the last step runs with
                hub.barrier.wait()
                for e in rt.layer.local_experts:
                    snap.setdefault(e, {kk: v.clone() for kk, v in rt.store.master[e].items()})
                hub.barrier.wait()
            out = rt.step(x, dy)
            hist.append((out.balance_ratio, out.replica_counts.tolist(), out.applied, out.accepted,
                         out.migration_bytes))
        torch.cuda.synchronize()
        states = {e: [t.clone() for t in rt.store.state(e)] for e in rt.layer.local_experts}
        return hist, out.y.float().cpu(), states, rt.slots.copy()

    outs = run_ranks(G, rank_fn)
    hists = [o[0] for o in outs]
    for h in hists[1:]:  # identical decisions everywhere
        assert [(a, b, c, d_) for a, b, c, d_, _ in h] == [(a, b, c, d_) for a, b, c, d_, _ in hists[0]]
    assert all((o[3] == outs[0][3]).all() for o in outs)
    applied = sum(len(s[2]) for s in hists[0])
    assert applied > 0, "the skewed gate should trigger placement changes"
    assert any(max(s[1]) > 1 for s in hists[0]), "some expert should be replicated"
    assert sum(s[4] for h in hists for s in h) > 0, "expert state must have moved between GPUs"
    assert hists[0][-1][0] < hists[0][0][0], "balance ratio should improve"

    # replicas hold bit-identical state
    by_expert = {}
    for _, _, states, _ in outs:
        for e, ts in states.items():
            by_expert.setdefault(e, []).append(ts)
    for e, copies in by_expert.items():
        for c in copies[1:]:
            assert all(torch.equal(a, b) for a, b in zip(copies[0], c)), f"expert {e} replicas diverged"

    # last step's output == fused single-GPU layer with the same weights
    fused = MoELayer(N, k, d, f, max_tokens=T)
    st = lambda kk: torch.stack([snap[e][kk] for e in range(N)])
    P = (wg.cuda().to(torch.bfloat16), st("w1").to(torch.bfloat16), st("b1"), st("w2").to(torch.bfloat16),
         st("b2"))
    for r in range(G):
        y_ref = fused.forward(xs[r].cuda(), *P).float().cpu()
        close_bf16(outs[r][1].numpy(), y_ref.numpy().astype(np.float64), f"y[rank {r}]")
