"""Expert state pool on the device (csrc/expert_pool.cu).

* pack: master -> bf16 weights / f32 biases, bit-exact vs torch's rounding;
* fused Adam: master/m/v updates vs an fp64 restatement of the same formula
  (rel. 1e-5), packed operands == bf16(master) bit-exact;
* migration: a pulled slot is a bit-exact copy of the source slot, in one
  process (linked pools) and across two processes through CUDA IPC (gloo for
  the handle exchange; both processes on cuda:0 — the NVLink path on an
  8-GPU box is the same cudaMemcpyAsync on an IPC-mapped peer range).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2304_03946_b200.pool import ExpertPool  # noqa: E402

d, f = 256, 512


def _fill(pool, slot, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    t = pool.slot_tensor(slot)
    t.copy_(torch.randn(3, pool.P, generator=g))
    t[2].abs_()  # v >= 0
    return t.clone()


def _packed(n):
    return (torch.zeros(n, f, d, dtype=torch.bfloat16, device="cuda"), torch.zeros(n, f, device="cuda"),
            torch.zeros(n, d, f, dtype=torch.bfloat16, device="cuda"), torch.zeros(n, d, device="cuda"))


def _split(master):
    o, out = 0, []
    for shape in ((f, d), (f,), (d, f), (d,)):
        n = int(np.prod(shape))
        out.append(master[o:o + n].view(shape))
        o += n
    return out


def test_pool_pack_and_adam():
    torch.cuda.set_device(0)
    pool = ExpertPool(4, d, f)
    assert pool.P == 2 * d * f + d + f and pool.slot_bytes >= 12 * pool.P
    ref = {s: _fill(pool, s, s) for s in range(4)}
    local = [3, 1]
    pk = _packed(2)
    pool.pack(local, pk)
    torch.cuda.synchronize()
    for i, s in enumerate(local):
        w1, b1, w2, b2 = _split(ref[s][0])
        assert torch.equal(pk[0][i], w1.to(torch.bfloat16)) and torch.equal(pk[1][i], b1)
        assert torch.equal(pk[2][i], w2.to(torch.bfloat16)) and torch.equal(pk[3][i], b2)

    g = torch.Generator(device="cpu").manual_seed(99)
    grads = [torch.randn(2, *shape, generator=g).cuda() for shape in ((f, d), (f,), (d, f), (d,))]
    lr, b1_, b2_, eps, step = 1e-3, 0.9, 0.999, 1e-8, 3
    pool.adam(local, grads, pk, lr, (b1_, b2_), eps, step)
    torch.cuda.synchronize()
    for i, s in enumerate(local):
        gcat = torch.cat([gg[i].reshape(-1) for gg in grads]).double()
        w, m, v = (ref[s][j].double() for j in range(3))
        m = b1_ * m + (1 - b1_) * gcat
        v = b2_ * v + (1 - b2_) * gcat * gcat
        w = w - lr * (m / (1 - b1_**step)) / ((v / (1 - b2_**step)).sqrt() + eps)
        got = pool.slot_tensor(s).double()
        for j, exp in enumerate((w, m, v)):
            err = ((got[j] - exp).norm() / exp.norm()).item()
            assert err < 1e-5, (s, j, err)
        w1, b1, w2, b2 = _split(pool.slot_tensor(s)[0])
        assert torch.equal(pk[0][i], w1.to(torch.bfloat16)) and torch.equal(pk[3][i], b2)
    # untouched slots unchanged
    for s in (0, 2):
        assert torch.equal(pool.slot_tensor(s), ref[s])


def test_pool_migrate_linked_in_process():
    torch.cuda.set_device(0)
    a, b = ExpertPool(3, d, f, world=2), ExpertPool(3, d, f, world=2)
    a.link_peer(1, b)
    b.link_peer(0, a)
    src = {s: _fill(b, s, 10 + s) for s in range(3)}
    _fill(a, 0, 5)
    keep = a.slot_tensor(0).clone()
    pk = _packed(3)
    a.migrate([(2, 1, 0), (1, 1, 2)], [0, 1, 2], pk)  # pull b:0 -> a:2, b:2 -> a:1
    a.wait_ready()
    torch.cuda.synchronize()
    assert torch.equal(a.slot_tensor(2), src[0]) and torch.equal(a.slot_tensor(1), src[2])
    assert torch.equal(a.slot_tensor(0), keep)
    assert torch.equal(pk[0][2], _split(src[0][0])[0].to(torch.bfloat16))
    ms, nbytes, copies = a.migration_stats()
    assert copies == 2 and nbytes == 2 * a.state_bytes and ms > 0
    with pytest.raises(Exception, match="not linked"):
        ExpertPool(1, d, f, world=2).migrate([(0, 1, 0)], [0], _packed(1))


# ------------------------------------------------------------- two processes, CUDA IPC
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, port, q):
    import torch.distributed as dist

    from paper_2304_03946_b200.distributed import TorchExchange

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        pool = ExpertPool(2, d, f, world=2)
        mine = _fill(pool, 0, 100 + rank)
        torch.cuda.synchronize()
        TorchExchange().share_pool(pool)  # IPC handles over gloo
        dist.barrier()  # both sources filled
        pk = _packed(2)
        pool.migrate([(1, 1 - rank, 0)], [0, 1], pk)  # pull the peer's slot 0 into slot 1
        pool.wait_ready()
        torch.cuda.synchronize()
        got = pool.slot_tensor(1).cpu()
        packed_ok = torch.equal(pk[2][1].cpu(), _split(got[0])[2].to(torch.bfloat16))
        dist.barrier()  # the peer finished reading my slot before I free it
        q.put((rank, (mine.cpu(), got, packed_ok, pool.migration_stats())))
        del pool
        dist.destroy_process_group()
    except BaseException as exc:
        q.put((rank, exc))


@pytest.mark.timeout(300)
def test_pool_migrate_ipc_two_processes():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        if isinstance(v, BaseException):
            raise v
    for r in range(2):
        mine, got, packed_ok, stats = res[r]
        assert torch.equal(got, res[1 - r][0]), f"rank {r}: pulled slot differs from the peer's"
        assert packed_ok
        assert stats[2] == 1 and stats[1] == 12 * (2 * d * f + d + f)
