"""P2P transport across processes: two ranks (processes) map each other's
exchange arenas through CUDA IPC and run the layer's P2P phases — x rows
written into the peer's X_perm by the dispatch kernel, Y / dX rows read from
the peer by combine / un-permute, dY rows written by combine_bwd, device-side
arrival flags in between. Both processes share cuda:0 here (the 8-GPU box
path is the same code with NVLink under the IPC mapping); gloo carries only
the host control plane (IPC handles, the demand histogram).
Checked: y, dx and the non-replicated experts' weight gradients of every
rank against the full-batch oracle; no arrival wait timed out."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import layer as OL  # noqa: E402
from tests.test_layer_gpu import close_bf16, close_f32  # noqa: E402

N, K, D, F, T, G = 8, 2, 256, 256, 512, 2
PAIRS = [(e, e % 2) for e in range(N)] + [(0, 1)]  # expert 0 replicated on both GPUs


def _inputs():
    cnt = np.zeros((N, G), np.int32)
    for e, g in PAIRS:
        cnt[e, g] += 1
    rng = np.random.default_rng(3)
    p = 1.0 / np.arange(1, N + 1) ** 1.25
    skew = np.log(p / p.sum())[rng.permutation(N)] + 3
    X, wg, w1, b1, w2, b2 = OL.exact_inputs(rng, T * G, D, N, F, skew=skew)
    dY = OL.bf16(rng.standard_normal((T * G, D)) * 0.5)
    return cnt, X, wg, w1, b1, w2, b2, dY


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, q, cross=False):
    import torch.distributed as dist

    from paper_2304_03946_b200 import _lib as L
    from paper_2304_03946_b200.layer import MoELayer

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=G)
        torch.cuda.set_device(rank if cross else 0)
        cnt, X, wg, w1, b1, w2, b2, dY = _inputs()
        bf = torch.bfloat16
        dev = lambda a, dt=bf: torch.tensor(np.asarray(a), dtype=dt, device="cuda")
        lay = MoELayer(N, K, D, F, replica_counts=cnt, num_gpus=G, rank=rank, max_tokens=T)
        loc = lay.local_experts
        lay.enable_p2p()
        handles = [None] * G
        dist.all_gather_object(handles, lay.p2p_handle())
        lay.p2p_open_peer(1 - rank, handles[1 - rank])
        lib, h, s = L.lib(), lay._h, L.stream_ptr()
        xs = slice(rank * T, (rank + 1) * T)
        x, WG = dev(X[xs]), dev(wg)
        W1, B1, W2, B2 = dev(w1[loc]), dev(b1[loc], torch.float32), dev(w2[loc]), dev(b2[loc], torch.float32)
        hist = torch.empty(N, dtype=torch.int64, device="cuda")
        L.check(lib.fm_layer_gate(h, x.data_ptr(), T, WG.data_ptr(), hist.data_ptr(), s))
        parts = [torch.empty(N, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(parts, hist.cpu())
        gathered = torch.stack(parts).cuda()
        L.check(lib.fm_layer_route_p2p(h, gathered.data_ptr(), s))
        L.check(lib.fm_layer_dispatch_p2p(h, x.data_ptr(), s))
        L.check(lib.fm_layer_expert_forward_p2p(h, W1.data_ptr(), B1.data_ptr(), W2.data_ptr(), B2.data_ptr(), s))
        y = torch.empty(T, D, dtype=bf, device="cuda")
        L.check(lib.fm_layer_combine_p2p(h, y.data_ptr(), s))
        L.check(lib.fm_layer_combine_backward_p2p(h, dev(dY[xs]).data_ptr(), s))
        nl = len(loc)
        z = lambda *sh: torch.zeros(*sh, device="cuda")
        dw1, db1, dw2, db2, dwg = z(nl, F, D), z(nl, F), z(nl, D, F), z(nl, D), z(N, D)
        dx = torch.empty(T, D, dtype=bf, device="cuda")
        L.check(lib.fm_layer_expert_backward_p2p(h, W1.data_ptr(), W2.data_ptr(), dw1.data_ptr(), db1.data_ptr(),
                                                 dw2.data_ptr(), db2.data_ptr(), dwg.data_ptr(), s))
        L.check(lib.fm_layer_unpermute_backward_p2p(h, WG.data_ptr(), dx.data_ptr(), dwg.data_ptr(), s))
        torch.cuda.synchronize()
        status = lay.p2p_status()
        out = dict(loc=loc, y=y.float().cpu().numpy(), dx=dx.float().cpu().numpy(), dw1=dw1.cpu().numpy(),
                   dwg=dwg.cpu().numpy(), status=status)
        dist.barrier()  # the peer is done reading my arena
        q.put((rank, out))
        del lay
        dist.destroy_process_group()
    except BaseException as exc:
        q.put((rank, exc))


TWO_GPUS = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (cross-device P2P)")


@pytest.mark.timeout(300)
@pytest.mark.parametrize("cross", [False, pytest.param(True, marks=TWO_GPUS)], ids=["shared-gpu", "two-gpus"])
def test_p2p_transport_two_processes_ipc(cross):
    """cross=True: rank r on cuda:r — the release / acquire flags and the
    pushed / pulled rows cross a real NVLink between two devices."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, cross)) for r in range(G)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(G))
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        if isinstance(v, BaseException):
            raise v
    cnt, X, wg, w1, b1, w2, b2, dY = _inputs()
    st = OL.forward(X, wg, w1, b1, w2, b2, K)
    gr = OL.backward(st, dY)
    dwg_sum = sum(res[r]["dwg"] for r in range(G))  # each GPU holds its share
    close_f32(dwg_sum, gr["dwg"], "dwg (sum over GPUs)", tol=2e-2)
    for r in range(G):
        o = res[r]
        assert o["status"] == 0, f"rank {r}: a P2P arrival wait timed out"
        xs = slice(r * T, (r + 1) * T)
        close_bf16(o["y"], st["y"][xs], f"y[rank {r}]")
        close_bf16(o["dx"], gr["dx"][xs], f"dx[rank {r}]")
        for i, e in enumerate(o["loc"]):
            if (cnt[e] > 0).sum() == 1:  # replicated experts need the group sum
                close_f32(o["dw1"][i], gr["dw1"][e], f"dw1[e{e}@{r}]")
