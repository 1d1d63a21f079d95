"""Dynamic placement in the loop, on one B200 with G virtual ranks (threads):
device gate -> all-gathered demand -> host scheduler (expand/shrink/migrate)
-> peer copies of expert weights + Adam state -> placement flip.

Checks: every rank sees the same placements and balance ratios; ops are
applied; replicas of every expert hold bit-identical state after migrations
and optimizer steps; the step output equals the fused single-GPU layer run
with the same weights (bf16 tolerance of test_layer_gpu.py). Both flip modes:
"modelled" (the reference's drain; the new replica computes in the step of its
copy) and "copy" (the new replica receives its state and the step's summed
gradient with zero rows routed to it, and takes tokens from the next step),
with the policy inline or on the scheduler's worker thread."""
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


@pytest.mark.parametrize("transport,flip,async_policy", [
    ("p2p", "modelled", False), ("nccl", "modelled", False),
    ("p2p", "copy", True), ("p2p", "copy", False), ("nccl", "copy", True)])
def test_runtime_dynamic_placement_loopback(transport, flip, async_policy):
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
                            max_tokens=T, gate_weight=wg, lr=1e-3, transport=transport, flip=flip,
                            async_policy=async_policy)
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
                         out.migration_bytes, out.issued))
        torch.cuda.synchronize()
        states = {e: [t.clone() for t in rt.store.state(e)] for e in rt.layer.local_experts}
        return hist, out.y.float().cpu(), states, rt.slots.copy()

    outs = run_ranks(G, rank_fn)
    hists = [o[0] for o in outs]
    for h in hists[1:]:  # identical decisions everywhere
        assert [(a, b, c, d_) for a, b, c, d_, _, _ in h] == [(a, b, c, d_) for a, b, c, d_, _, _ in hists[0]]
    assert all((o[3] == outs[0][3]).all() for o in outs)
    applied = sum(len(s[2]) for s in hists[0])
    assert applied > 0, "the skewed gate should trigger placement changes"
    assert any(max(s[1]) > 1 for s in hists[0]), "some expert should be replicated"
    assert sum(s[4] for h in hists for s in h) > 0, "expert state must have moved between GPUs"
    assert hists[0][-1][0] < hists[0][0][0], "balance ratio should improve"
    if flip == "copy":  # an op is issued one step before it becomes effective
        issued = [op for _, _, _, _, _, iss in hists[0] for op in iss]
        flipped = [op for _, _, ap, _, _, _ in hists[0] for op in ap]
        assert flipped == issued[: len(flipped)] and len(flipped) > 0

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


def test_placement_switch_is_async():
    """fm_layer_set_placement_async / fm_layer_set_operand_slots enqueue on
    the stream: they return while a long kernel still occupies it (no device
    or stream synchronisation, no allocation), and the next step routes on
    the new tables."""
    N, k, d, f, T, G = 8, 2, 256, 256, 256, 2
    counts = np.zeros((N, G), np.int32)
    counts[np.arange(N), np.arange(N) % G] = 1
    lay = MoELayer(N, k, d, f, replica_counts=counts, num_gpus=G, rank=0, max_tokens=T, slots_per_gpu=8)
    s = torch.cuda.current_stream()
    for i in range(6):  # 12 table uploads queued behind the sleeps
        torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU time on the stream
        new = counts.copy()
        new[i % N, 1 - (i % N) % G] = 1  # an extra replica of one expert
        hosted = np.zeros(N, bool)
        hosted[(i + 1) % N] = True  # a receiver whose copy is in flight
        lay.set_placement_async(new, hosted=hosted)
        slots = np.arange(N, dtype=np.int32)[::-1].copy()
        lay.set_operand_slots(slots, N)
        assert not s.query(), "the switch waited for the stream"
        expect = sorted(set(np.nonzero(new[:, 0] > 0)[0].tolist()) | {(i + 1) % N})
        assert lay.local_experts == expect
    torch.cuda.synchronize()


def test_runtime_switch_and_pull_do_not_block():
    """The runtime's placement boundary (flip "copy"): the table switch of the
    layer, the slot bookkeeping and the enqueue of the peer pulls return while
    the stream is still busy — no cudaFree, no device or stream sync."""
    N, k, d, f, T, G, E = 8, 2, 256, 256, 256, 2, 8
    hub = LoopbackHub(G)

    def rank_fn(r):
        torch.cuda.set_device(0)
        rt = FlexMoERuntime(N, k, d, f, hub.endpoint(r), S.ClusterProfile.reference_default(G, E),
                            max_tokens=T, flip="copy", async_policy=True)
        torch.cuda.synchronize()
        hub.barrier.wait()
        torch.cuda._sleep(400_000_000)
        expand = (S.EXPAND, 0, 1, -1, -1, -1, -1)  # expert 0 (on GPU 0) gains a replica on GPU 1
        nbytes, issue = rt._switch([], [expand])
        issue()
        busy = not torch.cuda.current_stream().query()
        local = rt.layer.local_experts
        torch.cuda.synchronize()
        hub.barrier.wait()
        return busy, nbytes, local, rt.hosted.copy()

    outs = run_ranks(G, rank_fn)
    for r, (busy, nbytes, local, hosted) in enumerate(outs):
        assert busy, f"rank {r}: the switch synchronised"
        assert hosted[0].tolist() == [True, True]
        assert (0 in local) and (nbytes > 0) == (r == 1)
