"""Comparison baselines on the device, G virtual ranks
on one B200 (loopback transport), demand replayed from reference traces
through the real gate (trace.replay_inputs):

* StaticEP: the device capacity drops (layer `kept`) equal the host
  baseline's kept demand, and the host StepReport equals the reference's
  run_baseline(StaticEP) on the same trace;
* FullReplicate: every step the hottest experts run as shadows on every GPU
  with the owner's weights (y == the fused single-GPU layer on the same
  weights), the replica-summed gradients of each owned expert equal the
  full-batch gradients, and the StepReport equals the reference's
  run_baseline(FullReplicate).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2304_03946_b200 import scheduler as S  # noqa: E402
from paper_2304_03946_b200 import trace as TR  # noqa: E402
from paper_2304_03946_b200.distributed import LoopbackHub  # noqa: E402
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402
from paper_2304_03946_b200.runtime import BaselineRuntime  # noqa: E402

from tests.test_layer_gpu import close_bf16, close_f32  # noqa: E402
from tests.test_multigpu_gpu import run_ranks  # noqa: E402

needs_ref = pytest.mark.skipif(not oracle.Reference.available(), reason="oracle/_ref not built")


def _setup(N, G, units, k, d, steps, zipf=1.25):
    tr = oracle.Reference().generate_trace(N, G, units, zipf=zipf, drift=0.02, seed=42, steps=steps)
    T = int(tr[0][:, 0].sum()) // k
    wg = TR.replay_inputs(tr[0][:, 0], k, d, device="cpu", dtype=torch.float32)[1]
    xs = [[TR.replay_inputs(tr[s][:, r], k, d, device="cpu")[0] for s in range(steps)] for r in range(G)]
    gen = torch.Generator().manual_seed(1)
    dys = [(torch.randn(T, d, generator=gen) * 0.1).to(torch.bfloat16) for _ in range(G)]
    return tr, T, wg, xs, dys


@needs_ref
def test_static_ep_on_device():
    N, G, E, k, d, f, steps, cf = 8, 4, 2, 2, 256, 256, 6, 1.0
    tr, T, wg, xs, dys = _setup(N, G, 8192, k, d, steps)
    hub = LoopbackHub(G)

    def rank_fn(r):
        torch.cuda.set_device(0)
        rt = BaselineRuntime(N, k, d, f, hub.endpoint(r), S.ClusterProfile.reference_default(G, E),
                             S.BaselineConfig.make("static-ep", capacity_factor=cf), max_tokens=T, gate_weight=wg)
        res = []
        for s in range(steps):
            o = rt.step(xs[r][s].cuda(), dys[r].cuda())
            torch.cuda.synchronize()
            kept = rt.layer.read("kept", N * G).reshape(N, G)
            h = o["host"]
            res.append((o["demand"], kept, h.demand, h.report.balance_ratio, h.report.makespan_s,
                        h.report.tokens_dropped))
        return res

    outs = run_ranks(G, rank_fn)
    ref = oracle.Reference().baseline_run(0, tr, E, cf=cf)
    for s in range(steps):
        D, kept, host_kept, ratio, mk, dropped = outs[0][s]
        np.testing.assert_array_equal(D, tr[s])  # the device gate reproduced the trace
        np.testing.assert_array_equal(kept, host_kept)  # device drops == reference rule
        assert ratio == ref["ratio"][s] and mk == ref["makespan"][s] and dropped == ref["dropped"][s]
        for o in outs[1:]:
            np.testing.assert_array_equal(o[s][1], kept)
    assert sum(o[5] for o in outs[0]) > 0, "skewed trace should drop tokens at cf 1.0"


@needs_ref
def test_full_replicate_on_device():
    N, G, E, k, d, f, steps, top = 8, 4, 2, 2, 256, 256, 4, 2
    tr, T, wg, xs, dys = _setup(N, G, 8192, k, d, steps)
    hub = LoopbackHub(G)
    snap = {}

    def rank_fn(r):
        torch.cuda.set_device(0)
        rt = BaselineRuntime(N, k, d, f, hub.endpoint(r), S.ClusterProfile.reference_default(G, E),
                             S.BaselineConfig.make("full-replicate", replicate_top=top), max_tokens=T,
                             gate_weight=wg, lr=1e-3)
        res = []
        for s in range(steps):
            if s == steps - 1:  # weights the last step runs with
                hub.barrier.wait()
                for e in rt.owned:
                    snap[e] = {kk: v.clone() for kk, v in rt.store.master[e].items()}
                hub.barrier.wait()
            o = rt.step(xs[r][s].cuda(), dys[r].cuda())
            h = o["host"]
            res.append((h.counts.copy(), h.report.balance_ratio, h.report.makespan_s, h.report.group_misses,
                        o["shadow_bytes"]))
        torch.cuda.synchronize()
        g = o["grads"]
        loc = o["local"]
        grads = {e: (g.dw1[i].cpu(), g.db1[i].cpu(), g.dw2[i].cpu(), g.db2[i].cpu()) for i, e in enumerate(loc)}
        return res, o["y"].float().cpu(), grads

    outs = run_ranks(G, rank_fn)
    ref = oracle.Reference().baseline_run(1, tr, E, replicate_top=top)
    for s in range(steps):
        counts, ratio, mk, misses, _ = outs[0][0][s]
        assert ratio == ref["ratio"][s] and mk == ref["makespan"][s] and misses == ref["misses"][s]
        np.testing.assert_array_equal(counts.sum(axis=1), ref["replicas"][s])
        hot = np.argsort(-tr[s].sum(axis=1), kind="stable")[:top]
        assert (counts[hot] > 0).all()
    assert sum(o[0][s][4] for o in outs for s in range(steps)) > 0, "shadows must be transferred"

    # last step: y per rank and the replica-summed grads == fused layer on all tokens
    fused = MoELayer(N, k, d, f, max_tokens=T * G)
    st = lambda kk: torch.stack([snap[e][kk] for e in range(N)])
    P = (wg.cuda().to(torch.bfloat16), st("w1").to(torch.bfloat16), st("b1"), st("w2").to(torch.bfloat16), st("b2"))
    X = torch.cat([xs[r][steps - 1] for r in range(G)]).cuda()
    y_ref = fused.forward(X, *P).float().cpu()
    g_ref = fused.backward(torch.cat(dys).cuda())
    for r in range(G):
        close_bf16(outs[r][1].numpy(), y_ref[r * T:(r + 1) * T].numpy().astype(np.float64), f"y[rank {r}]")
        for e, (dw1, db1, dw2, db2) in outs[r][2].items():
            close_f32(dw1.numpy(), g_ref.dw1[e].cpu().numpy(), f"dw1[e{e}@{r}]")
            close_f32(dw2.numpy(), g_ref.dw2[e].cpu().numpy(), f"dw2[e{e}@{r}]")
            close_f32(db1.numpy(), g_ref.db1[e].cpu().numpy(), f"db1[e{e}@{r}]")
            close_f32(db2.numpy(), g_ref.db2[e].cpu().numpy(), f"db2[e{e}@{r}]")
