"""The FlexMoE runtime across real processes (both token transports): two ranks (processes sharing
cuda:0), torch.distributed over gloo for the host control plane (histogram
all-gather, replica-group and gate all-reduces, handle exchange), CUDA IPC
for everything on the data plane: the P2P token transport between the
layers' arenas and the expert-state pulls between the ranks' pools when the
scheduler's expand / shrink / migrate ops become effective.

Checked: both ranks take identical decisions, expert state actually moved
between the processes, replicas of every expert hold bit-identical state
after the migrations and Adam steps, no P2P arrival wait timed out."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N, K, D, F, T, G, E, STEPS = 8, 2, 256, 256, 512, 2, 6, 10
TRANSPORTS = ["p2p", "nccl"]  # "nccl": the all-to-all path (gloo stands in for NCCL here)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, q, transport, cross=False):
    import torch.distributed as dist

    from paper_2304_03946_b200 import scheduler as S
    from paper_2304_03946_b200.distributed import TorchExchange
    from paper_2304_03946_b200.runtime import FlexMoERuntime

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=G)
        torch.cuda.set_device(rank if cross else 0)
        gen = torch.Generator(device="cpu").manual_seed(0)
        wg = torch.randn(N, D, generator=gen) * D**-0.5
        wg[:, 0] = torch.tensor(np.log(1.0 / np.arange(1, N + 1) ** 1.5) * 2 + 3, dtype=torch.float32)
        xs = [torch.randn(T, D, generator=gen).to(torch.bfloat16) for _ in range(G)]
        dys = [(torch.randn(T, D, generator=gen) * 0.1).to(torch.bfloat16) for _ in range(G)]
        x, dy = xs[rank].cuda(), dys[rank].cuda()
        x[:, 0] = 0.5
        rt = FlexMoERuntime(N, K, D, F, TorchExchange(), S.ClusterProfile.reference_default(G, E), max_tokens=T,
                            gate_weight=wg, lr=1e-3, transport=transport)
        hist = []
        for _ in range(STEPS):
            out = rt.step(x, dy)
            hist.append((round(out.balance_ratio, 12), out.replica_counts.tolist(), out.applied, out.accepted))
        torch.cuda.synchronize()
        states = {e: [t.cpu().numpy().copy() for t in rt.store.state(e)] for e in rt.layer.local_experts}  # by value
        res = dict(hist=hist, states=states, mig=rt.migration_stats(),
                   timed_out=rt.dl.p2p_timed_out() if transport == "p2p" else False)
        dist.barrier()  # peers are done reading my arena and pool
        q.put((rank, res))
        del rt
        dist.destroy_process_group()
    except BaseException as exc:
        q.put((rank, exc))


TWO_GPUS = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (cross-device P2P)")


@pytest.mark.timeout(400)
@pytest.mark.parametrize("cross", [False, pytest.param(True, marks=TWO_GPUS)], ids=["shared-gpu", "two-gpus"])
@pytest.mark.parametrize("transport", TRANSPORTS)
def test_runtime_two_processes(transport, cross):
    """cross=True: rank r on cuda:r (token rows and expert-state pulls over NVLink)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, transport, cross)) for r in range(G)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=360) for _ in range(G))
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        if isinstance(v, BaseException):
            raise v
    assert not res[0]["timed_out"] and not res[1]["timed_out"]
    assert res[0]["hist"] == res[1]["hist"], "ranks took different decisions"
    assert sum(len(h[2]) for h in res[0]["hist"]) > 0, "the skewed gate should trigger placement changes"
    assert res[0]["mig"]["bytes"] + res[1]["mig"]["bytes"] > 0, "expert state must move between processes"
    shared = set(res[0]["states"]) & set(res[1]["states"])
    for e in shared:
        for a, b in zip(res[0]["states"][e], res[1]["states"][e]):
            assert np.array_equal(a, b), f"expert {e} replicas diverged across processes"
