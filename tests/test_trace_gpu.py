"""Trace replay through the real device path.

A reference trace (`generate_trace`, proj/src/workload.cpp:135-170) is
replayed with exact-arithmetic gate inputs (`trace.replay_inputs`): on every
virtual rank the REAL gate must reproduce that rank's TokenDemand column, so
the all-gathered device demand equals the trace step bit-exactly. Driving
FlexMoERuntime (device step + host scheduler + P2P state moves) with it, the
per-step modelled makespan, adjustment bytes and accepted ops must equal the
reference engine (`SimEngine::run`, sim_engine.cpp:329-449) on the same trace,
and the exported trace file must load back in the reference as the same trace.
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
from paper_2304_03946_b200._lib import call, ptr, stream_ptr  # noqa: E402
from paper_2304_03946_b200.runtime import FlexMoERuntime  # noqa: E402

from tests.test_multigpu_gpu import run_ranks  # noqa: E402


def _trace(N, G, units, zipf, steps, seed=42):
    if oracle.Reference.available():
        return oracle.Reference().generate_trace(N, G, units, zipf=zipf, drift=0.02, seed=seed, steps=steps)
    return oracle.Oracle().generate_trace(N, G, units, zipf=zipf, drift=0.02, seed=seed, steps=steps)


@pytest.mark.parametrize("N,k,units,zipf", [(16, 2, 131072, 1.25), (64, 1, 65536, 1.25),
                                             (32, 4, 65536, 0.8), (128, 8, 131072, 0.7)])
def test_gate_replays_trace_column(N, k, units, zipf):
    tr = _trace(N, 1, units, zipf, 1)
    col = tr[0][:, 0]
    x, wg = TR.replay_inputs(col, k, 1024)
    T = x.shape[0]
    lay = MoELayer(N, k, 1024, 256, max_tokens=T)
    hist = torch.empty(N, dtype=torch.int64, device="cuda")
    call("fm_layer_gate", lay._h, ptr(x), T, ptr(wg), ptr(hist), stream_ptr())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hist.cpu().numpy(), col)
    idx = lay.read("topk_idx", T * k).reshape(T, k)
    np.testing.assert_array_equal(idx, TR.replay_assignment(col, k))


def test_runtime_replays_reference_trace(tmp_path):
    # config-1 shape: N=8, G=4, k=2, 8192 units per step
    N, k, d, f, G, E, steps = 8, 2, 256, 256, 4, 4, 12
    tr = _trace(N, G, 8192, 1.25, steps)
    T = int(tr[0][:, 0].sum()) // k
    hub = LoopbackHub(G)
    wg = TR.replay_inputs(tr[0][:, 0], k, d, device="cpu", dtype=torch.float32)[1]
    xs = [[TR.replay_inputs(tr[s][:, r], k, d, device="cpu")[0] for s in range(steps)] for r in range(G)]
    dys = [(torch.randn(T, d, generator=torch.Generator().manual_seed(r)) * 0.1).to(torch.bfloat16)
           for r in range(G)]

    def rank_fn(r):
        torch.cuda.set_device(0)
        rec = TR.TraceRecorder()
        rt = FlexMoERuntime(N, k, d, f, hub.endpoint(r), S.ClusterProfile.reference_default(G, E),
                            max_tokens=T, gate_weight=wg, recorder=rec)
        hist = []
        for s in range(steps):
            out = rt.step(xs[r][s].cuda(), dys[r].cuda())
            hist.append((out.makespan_s, out.adjust_bytes, [tuple(o) for o in out.accepted]))
        torch.cuda.synchronize()
        return rec.trace(), hist

    outs = run_ranks(G, rank_fn)
    for rec_tr, _ in outs:
        np.testing.assert_array_equal(rec_tr, tr)  # device demand == the reference trace
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built: engine comparison needs the reference")
    ref = oracle.Reference()
    mk_r, ab_r, ops_r = ref.engine_detail(tr, E)
    n_ops = 0
    for s, (mk, ab, ops) in enumerate(outs[0][1]):
        assert mk == mk_r[s], s
        assert ab == ab_r[s], s
        assert ops == [tuple(o) for o in ops_r[s]], s
        n_ops += len(ops)
    assert n_ops > 0
    TR.save_trace(outs[0][0], tmp_path / "device.csv")
    np.testing.assert_array_equal(ref.load_trace(tmp_path / "device.csv"), tr)
