"""Multi-GPU FlexMoE layer: one process per GPU, collectives between phases.

Per step (the exchanges the reference models in
cost_model.cpp:37-64):
  1. all-gather of each GPU's expert histogram -> full TokenDemand D[e][g],
     so every rank runs the identical deterministic route() (no broadcast);
  2. dispatch all-to-all (per-peer row counts from the flows);
  3. combine all-to-all back;
  4. the two backward mirrors;
  5. for every expert with >= 2 hosting GPUs, SUM all-reduce of its weight
     gradients within its replica group, issued in ascending expert id on
     every GPU (the deadlock-free order of proj/src/sim_engine.cpp:67-113),
     groups cached in an LRU (sim_engine.cpp:45-65, capacity 64);
     the data-parallel gate weight gradient is summed over all GPUs.
SUM (not mean) is the right reduction: tokens are partitioned across the
replicas, so the replica-group sum equals the single-replica gradient.

The compute phases run in libflexmoe_b200.so (`fm_layer_*` phase API);
torch.distributed (NCCL) is only the transport. `Exchange` abstracts the
transport so the same orchestration runs over NCCL, gloo, or an in-process
loopback (G virtual ranks on one GPU, used by the GPU tests).
"""
from __future__ import annotations

import ctypes as C
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


# ---------------------------------------------------------------- placement helpers
def replica_gpus(replica_counts, e) -> tuple[int, ...]:
    """Placement::replica_gpus (placement.cpp:109-117): ascending GPU ids hosting e."""
    row = np.asarray(replica_counts)[e]
    return tuple(int(g) for g in np.nonzero(row > 0)[0])


def collective_order(replica_counts) -> list[list[int]]:
    """Per GPU, the replicated experts it synchronises, ascending (sim_engine.cpp:67-79)."""
    cnt = np.asarray(replica_counts)
    G = cnt.shape[1]
    order = [[] for _ in range(G)]
    for e in range(cnt.shape[0]):
        grp = replica_gpus(cnt, e)
        if len(grp) >= 2:
            for g in grp:
                order[g].append(e)
    return order


def collective_order_deadlock_free(replica_counts) -> bool:
    """Simulates blocking collectives in the per-GPU order (sim_engine.cpp:81-113)."""
    cnt = np.asarray(replica_counts)
    order = collective_order(cnt)
    pos = [0] * cnt.shape[1]
    progress = True
    while progress:
        progress = False
        for e in range(cnt.shape[0]):
            grp = replica_gpus(cnt, e)
            if len(grp) < 2:
                continue
            if all(pos[g] < len(order[g]) and order[g][pos[g]] == e for g in grp):
                for g in grp:
                    pos[g] += 1
                progress = True
    return all(pos[g] == len(order[g]) for g in range(cnt.shape[1]))


class LruGroupCache:
    """LRU over replica-group keys (sorted GPU tuples); a miss creates the
    group. Mirrors LruGroupCache (sim_engine.hpp:70-86 / .cpp:45-65): touch()
    returns True on a hit; the least recently used group is evicted beyond
    `capacity`. `create` / `destroy` hook the real communicator lifetime."""

    def __init__(self, capacity=64, create=None, destroy=None):
        if capacity < 1:
            raise ValueError("LruGroupCache: capacity must be >= 1")
        self.capacity = capacity
        self._entries: OrderedDict[tuple, object] = OrderedDict()
        self.misses = 0
        self._create = create
        self._destroy = destroy

    def touch(self, group) -> bool:
        key = tuple(sorted(group))
        if key in self._entries:
            self._entries.move_to_end(key, last=False)
            return True
        self.misses += 1
        self._entries[key] = self._create(key) if self._create else key
        self._entries.move_to_end(key, last=False)
        if len(self._entries) > self.capacity:
            old_key, old = self._entries.popitem(last=True)
            if self._destroy:
                self._destroy(old)
        return False

    def get(self, group):
        self.touch(group)
        return self._entries[tuple(sorted(group))]

    def __len__(self):
        return len(self._entries)


# ---------------------------------------------------------------- transports
class Exchange:
    rank: int
    world: int

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:  # -> [world, *t.shape]
        raise NotImplementedError

    def all_to_all(self, out, inp, out_splits, in_splits) -> None:
        raise NotImplementedError

    def all_reduce(self, t: torch.Tensor | None, group: tuple[int, ...] | None) -> None:
        """SUM over `group` (None = all ranks). Every rank calls it for every
        group in the same order; ranks outside the group pass t=None."""
        raise NotImplementedError

    def all_reduce_many(self, ts, group: tuple[int, ...]) -> None:
        """SUM of several tensors over one replica group (ts = None on ranks
        outside it); the same call order rules as all_reduce."""
        for t in (ts if ts is not None else [None] * 4):
            self.all_reduce(t, group)

    def sync_group(self, group: tuple[int, ...]) -> None:
        """Called on EVERY rank, in ascending expert id, for every replica group
        (group creation is collective over the world in torch.distributed)."""

    def p2p(self, sends: list, recvs: list) -> None:
        """Point-to-point copies: sends [(dst, tensor)], recvs [(src, tensor)],
        matched per (src, dst) pair in list order. Called by every rank."""
        raise NotImplementedError

    def share_pool(self, pool) -> None:
        """Map every peer's ExpertPool into `pool` (collective): CUDA IPC handles
        across processes, plain pointers in one process."""
        raise NotImplementedError

    def share_layer(self, layer) -> None:
        """Map every peer's P2P exchange arena into `layer` (collective)."""
        raise NotImplementedError

    def fence(self) -> None:
        """Before a device-side arrival wait: every rank's preceding signals must
        be enqueued. Separate GPUs need nothing; ranks sharing one device
        stream (loopback) rendezvous on the host so no wait is queued ahead of
        the signal it waits for."""


class TorchExchange(Exchange):
    """torch.distributed transport (NCCL on B200 / NVLink; gloo on CPU)."""

    def __init__(self, max_live_groups=64):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.groups = LruGroupCache(max_live_groups, create=lambda key: dist.new_group(list(key)),
                                    destroy=lambda pg: dist.destroy_process_group(pg))

    def all_gather(self, t):
        flat = t.contiguous().reshape(-1)
        out = torch.empty(self.world * flat.numel(), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, flat)
        return out.view(self.world, *t.shape)

    def all_to_all(self, out, inp, out_splits, in_splits):
        self.dist.all_to_all_single(out, inp, output_split_sizes=list(out_splits),
                                    input_split_sizes=list(in_splits))

    def sync_group(self, group):
        self.groups.touch(group)

    def p2p(self, sends, recvs):
        ops = [self.dist.P2POp(self.dist.isend, t.contiguous(), dst) for dst, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, src) for src, t in recvs]
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def share_pool(self, pool):
        handles = [None] * self.world
        self.dist.all_gather_object(handles, pool.ipc_handle())
        for peer, h in enumerate(handles):
            if peer != self.rank:
                pool.open_peer(peer, h)

    def share_layer(self, layer):
        # the arenas are laid out from the layer shape: every rank must agree on it
        shape = (layer.N, layer.k, layer.d, layer.f, layer.G, layer.max_tokens)
        entries = [None] * self.world
        self.dist.all_gather_object(entries, (shape, layer.p2p_handle()))
        if any(sh != shape for sh, _ in entries):
            raise L.InvalidArgument(f"P2P transport: layer shapes differ across ranks: {[sh for sh, _ in entries]}")
        for peer, (_, h) in enumerate(entries):
            if peer != self.rank:
                layer.p2p_open_peer(peer, h)

    def all_reduce(self, t, group):
        if group is None:
            self.dist.all_reduce(t)
        elif t is not None and self.rank in group:
            self.dist.all_reduce(t, group=self.groups.get(group))

    def all_reduce_many(self, ts, group):
        """One NCCL group launch for an expert's four gradient slices (NCCL:
        coalesced; other backends: one call each)."""
        if ts is None or self.rank not in group:
            return
        pg = self.groups.get(group)
        if (ts[0].is_cuda and hasattr(self.dist, "_coalescing_manager")
                and self.dist.get_backend(pg) == "nccl"):
            with self.dist._coalescing_manager(group=pg, device=ts[0].device):
                for t in ts:
                    self.dist.all_reduce(t, group=pg)
        else:
            for t in ts:
                self.dist.all_reduce(t, group=pg)


class LoopbackHub:
    """In-process stand-in for G ranks (threads) sharing one device: used to
    run the real multi-GPU kernels and layouts on a single B200."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world, timeout=120)  # a failed rank breaks it, not a hang
        self.slots = [None] * world
        self.groups = LruGroupCache(64)

    def endpoint(self, rank):
        return LoopbackExchange(self, rank)


class LoopbackExchange(Exchange):
    def __init__(self, hub: LoopbackHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def _swap(self, obj):
        self.hub.barrier.wait()
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()
        got = list(self.hub.slots)
        self.hub.barrier.wait()
        return got

    def all_gather(self, t):
        return torch.stack(self._swap(t.clone()))

    def all_to_all(self, out, inp, out_splits, in_splits):
        offs = np.concatenate([[0], np.cumsum(in_splits)]).astype(int)
        chunks = [inp[offs[i]:offs[i + 1]] for i in range(self.world)]
        allc = self._swap(chunks)
        o = 0
        for src in range(self.world):
            c = allc[src][self.rank]
            out[o:o + c.shape[0]].copy_(c)
            o += c.shape[0]
        self._swap(None)  # keep sources alive until everyone copied

    def sync_group(self, group):
        if self.rank == 0:
            self.hub.groups.touch(group)

    def p2p(self, sends, recvs):
        allsends = self._swap(sends)
        inbox: dict[int, list] = {}
        for src in range(self.world):
            inbox[src] = [t for dst, t in allsends[src] if dst == self.rank]
        taken: dict[int, int] = {}
        for src, t in recvs:
            i = taken.get(src, 0)
            t.copy_(inbox[src][i])
            taken[src] = i + 1
        self._swap(None)  # senders keep their tensors alive until copied

    def share_pool(self, pool):
        for peer, other in enumerate(self._swap(pool)):
            if peer != self.rank:
                pool.link_peer(peer, other)

    def share_layer(self, layer):
        for peer, other in enumerate(self._swap(layer)):
            if peer != self.rank:
                layer.p2p_link_peer(peer, other)

    def fence(self):
        self.hub.barrier.wait()

    def all_reduce(self, t, group):
        members = range(self.world) if group is None else group
        allv = self._swap(t.clone() if (t is not None and self.rank in members) else None)
        if t is not None and self.rank in members:
            acc = torch.zeros_like(t)
            for g in members:
                acc += allv[g]
            t.copy_(acc)


# ---------------------------------------------------------------- the layer
@dataclass
class StepBuffers:
    send: torch.Tensor
    recv: torch.Tensor
    ret: torch.Tensor
    back: torch.Tensor
    send_rows: list[int]
    recv_rows: list[int]


class DistributedMoELayer:
    """FlexMoE layer on one GPU of G, driving fm_layer_* phases around `exchange`."""

    def __init__(self, layer, exchange: Exchange, transport: str = "nccl", reuse_grads: bool = False):
        """transport "nccl": dispatch / combine and their backward mirrors are
        all-to-alls of staging buffers (plus relayouts). "p2p": token rows
        cross NVLink inside the dispatch / combine / un-permute kernels,
        straight between the token's GPU and its expert GPU's permuted
        buffers (CUDA IPC-mapped arenas, device-side arrival flags).

        reuse_grads: backward() writes into the same gradient tensors every
        step (stream-ordered, like MoELayer.backward's `grads` argument) — the
        runtime consumes them within the step; a caller that keeps a step's
        gradients past the next backward must leave it off."""
        from .layer import MoELayer

        assert isinstance(layer, MoELayer)
        self.layer, self.ex = layer, exchange
        if layer.G != exchange.world or layer.rank != exchange.rank:
            raise L.InvalidArgument("DistributedMoELayer: layer and exchange disagree on rank/world")
        if transport not in ("nccl", "p2p"):
            raise L.InvalidArgument(f"DistributedMoELayer: unknown transport {transport!r}")
        self.transport = transport
        if transport == "p2p":
            layer.enable_p2p()
            exchange.share_layer(layer)
        self._st: StepBuffers | None = None
        self._saved = None
        self.reuse_grads = reuse_grads
        self._bufs: dict[str, torch.Tensor] = {}
        self._timing = False
        self._marks: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    # CUDA-event timing of the exchanges (a2a, all-gather, all-reduce)
    def set_timing(self, on: bool):
        self._timing = on
        self._marks = []

    def read_timing(self) -> dict[str, tuple[float, int]]:
        torch.cuda.synchronize()
        out: dict[str, list] = {}
        for name, a, b in self._marks:
            v = out.setdefault(name, [0.0, 0])
            v[0] += a.elapsed_time(b)
            v[1] += 1
        return {k: (v[0], v[1]) for k, v in out.items()}

    def _buf(self, name, shape, dtype, device):
        """A per-layer device buffer, reallocated only when its shape changes."""
        t = self._bufs.get(name)
        if t is None or t.shape != torch.Size(shape) or t.dtype != dtype or t.device != device:
            t = self._bufs[name] = torch.empty(shape, dtype=dtype, device=device)
        return t

    def _grads(self, T, nl, dev):
        from .layer import LayerGrads

        lay, f32 = self.layer, torch.float32
        d, f, N, m = lay.d, lay.f, lay.N, max(nl, 1)
        shapes = dict(dx=((T, d), torch.bfloat16), dwg=((N, d), f32), dw1=((m, f, d), f32), db1=((m, f), f32),
                      dw2=((m, d, f), f32), db2=((m, d), f32))
        if self.reuse_grads:
            return LayerGrads(**{n: self._buf("g_" + n, s, dt, dev) for n, (s, dt) in shapes.items()})
        return LayerGrads(**{n: torch.empty(s, dtype=dt, device=dev) for n, (s, dt) in shapes.items()})

    def _x(self, name, fn, *args):
        if not self._timing:
            return fn(*args)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn(*args)
        b.record()
        self._marks.append((name, a, b))
        return r

    @property
    def last_demand_host(self) -> np.ndarray:
        """This step's all-gathered TokenDemand D[e][g] on the host (waits for
        its copy if it is still in flight)."""
        if getattr(self, "_demand_event", None) is not None:
            self._demand_event.synchronize()
            self._demand_host = self._demand_pinned.numpy().T.copy()
            self._demand_event = None
        return self._demand_host

    @property
    def replica_counts(self):
        return self.layer.replica_counts

    def _call(self, name, *args):
        L.check(getattr(L.lib(), name)(self.layer._h, *args))

    def forward(self, x, wg, w1, b1, w2, b2, on_demand=None, before_experts=None, after_gather=None):
        """on_demand(D [N][G] host) -> None | (w1, b1, w2, b2): called once the
        step's TokenDemand is all-gathered and before routing; it may switch
        the layer's placement (a per-step placement such as FullReplicate's
        shadows, baselines.cpp:143-156) and return the operands of the new
        local experts. after_gather(): called right after the demand
        all-gather is enqueued — the first point of the step that every GPU
        passes only after finishing its previous step (optimizer update
        included); the runtime starts expert-state pulls there.
        before_experts(): called right before the expert FFN is enqueued (the
        runtime makes the stream wait for the pulls there, so the copies
        overlap routing and dispatch)."""
        lay, d, N, k = self.layer, self.layer.d, self.layer.N, self.layer.k
        T = x.shape[0]
        dev = x.device
        stream = L.stream_ptr()
        hist = self._buf("hist", (N,), torch.int64, dev)  # the all-gather copies it out
        self._call("fm_layer_gate", x.data_ptr(), T, wg.data_ptr(), hist.data_ptr(), stream)
        gathered = self._x("all_gather", self.ex.all_gather, hist)  # [G, N]
        if after_gather is not None:
            after_gather()
        if self.transport == "p2p":
            return self._forward_p2p(x, T, wg, w1, b1, w2, b2, gathered, on_demand, before_experts)
        if on_demand is not None:
            new = on_demand(gathered.cpu().numpy().T.copy())
            if new is not None:
                w1, b1, w2, b2 = new
        G = lay.G
        send_rows = np.zeros(G, np.int32)
        recv_rows = np.zeros(G, np.int32)
        self._call("fm_layer_route", gathered.data_ptr(), send_rows.ctypes.data, recv_rows.ctypes.data,
                   stream)
        send_rows, recv_rows = send_rows.tolist(), recv_rows.tolist()
        # fm_layer_route synchronised the stream: the demand is final, take the
        # host copy for the placement scheduler now (no extra sync later)
        self._demand_host = gathered.cpu().numpy().T.copy()  # TokenDemand [N][G]
        self._demand_event = None
        bf = torch.bfloat16
        send = torch.empty(max(T * k, 1), d, dtype=bf, device=dev)
        recv = torch.empty(max(sum(recv_rows), 1), d, dtype=bf, device=dev)
        ret = torch.empty_like(recv)
        back = torch.empty_like(send)
        self._call("fm_layer_dispatch", x.data_ptr(), send.data_ptr(), stream)
        self._x("a2a", self.ex.all_to_all, recv[: sum(recv_rows)], send[: T * k], recv_rows, send_rows)
        if before_experts is not None:
            before_experts()
        self._call("fm_layer_expert_forward", recv.data_ptr(), w1.data_ptr(), b1.data_ptr(),
                   w2.data_ptr(), b2.data_ptr(), ret.data_ptr(), stream)
        self._x("a2a", self.ex.all_to_all, back[: T * k], ret[: sum(recv_rows)], send_rows, recv_rows)
        y = torch.empty(T, d, dtype=bf, device=dev)
        self._call("fm_layer_combine", back.data_ptr(), y.data_ptr(), stream)
        self._st = StepBuffers(send, recv, ret, back, send_rows, recv_rows)
        self._saved = (T, wg, w1, w2, x)  # x: StaticEP backward re-reads dropped units
        self.last_demand = gathered
        return y

    def _forward_p2p(self, x, T, wg, w1, b1, w2, b2, gathered, on_demand, before_experts):
        stream = L.stream_ptr()
        if on_demand is not None:  # a per-step placement needs the demand before routing
            self._demand_host = gathered.cpu().numpy().T.copy()
            self._demand_event = None
            new = on_demand(self._demand_host.copy())
            if new is not None:
                w1, b1, w2, b2 = new
        else:  # no host sync in the step: the policy's copy lands asynchronously
            if getattr(self, "_demand_pinned", None) is None or self._demand_pinned.shape != gathered.shape:
                self._demand_pinned = torch.empty(gathered.shape, dtype=gathered.dtype, pin_memory=True)
            self._demand_pinned.copy_(gathered, non_blocking=True)
            self._demand_event = torch.cuda.Event()
            self._demand_event.record()
        self._call("fm_layer_route_p2p", gathered.data_ptr(), stream)
        self._call("fm_layer_dispatch_p2p", x.data_ptr(), stream)
        self.ex.fence()
        if before_experts is not None:
            before_experts()
        self._call("fm_layer_expert_forward_p2p", w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(),
                   stream)
        self.ex.fence()
        y = torch.empty(T, self.layer.d, dtype=torch.bfloat16, device=x.device)
        self._call("fm_layer_combine_p2p", y.data_ptr(), stream)
        self._st = None
        self._saved = (T, wg, w1, w2, x)
        self.last_demand = gathered
        return y

    def _backward_p2p(self, dy, sync, before_sync=None):
        T, wg, w1, w2, _x = self._saved
        lay, dev, stream = self.layer, dy.device, L.stream_ptr()
        nl = len(lay.local_experts)
        g = self._grads(T, nl, dev)
        self._call("fm_layer_combine_backward_p2p", dy.data_ptr(), stream)
        self.ex.fence()
        # the un-permute may ride beside this GPU's FFN1 weight gradients
        self._call("fm_layer_p2p_bind_dx", wg.data_ptr(), g.dx.data_ptr())
        self._call("fm_layer_expert_backward_p2p", w1.data_ptr(), w2.data_ptr(), g.dw1.data_ptr(),
                   g.db1.data_ptr(), g.dw2.data_ptr(), g.db2.data_ptr(), g.dwg.data_ptr(), stream)
        self.ex.fence()
        self._call("fm_layer_unpermute_backward_p2p", wg.data_ptr(), g.dx.data_ptr(), g.dwg.data_ptr(), stream)
        if nl == 0:
            g.dw1, g.db1, g.dw2, g.db2 = (t[:0] for t in (g.dw1, g.db1, g.dw2, g.db2))
        if sync:  # dwg holds this GPU's share: the all-GPU sum below completes it
            if before_sync is not None:
                before_sync()
            self._x("grad_sync", self.sync_grads, g)
        return g

    def p2p_timed_out(self) -> bool:
        """True if a device-side P2P arrival wait gave up (synchronises)."""
        return self.layer.p2p_status() != 0

    def backward(self, dy, sync=True, before_sync=None):
        """before_sync(): called right before the replica-group all-reduces
        are enqueued (the runtime makes the stream wait there for the state
        copies of replicas that join a group this step, flip_mode 1)."""
        if self.transport == "p2p":
            return self._backward_p2p(dy, sync, before_sync)
        T, wg, w1, w2, _x = self._saved
        st = self._st
        lay = self.layer
        dev = dy.device
        stream = L.stream_ptr()
        nl = len(lay.local_experts)
        k = lay.k
        dsend = torch.empty_like(st.send)
        drecv = torch.empty_like(st.recv)
        dret = torch.empty_like(st.recv)
        dback = torch.empty_like(st.send)
        g = self._grads(T, nl, dev)
        R = sum(st.recv_rows)
        self._call("fm_layer_combine_backward", dy.data_ptr(), st.back.data_ptr(), dsend.data_ptr(),
                   stream)
        self._x("a2a", self.ex.all_to_all, drecv[:R], dsend[: T * k], st.recv_rows, st.send_rows)
        self._call("fm_layer_expert_backward", drecv.data_ptr(), w1.data_ptr(), w2.data_ptr(),
                   g.dw1.data_ptr(), g.db1.data_ptr(), g.dw2.data_ptr(), g.db2.data_ptr(),
                   dret.data_ptr(), stream)
        self._x("a2a", self.ex.all_to_all, dback[: T * k], dret[:R], st.send_rows, st.recv_rows)
        self._call("fm_layer_unpermute_backward", dback.data_ptr(), st.send.data_ptr(),
                   wg.data_ptr(), g.dx.data_ptr(), g.dwg.data_ptr(), stream)
        if nl == 0:
            g.dw1, g.db1, g.dw2, g.db2 = (t[:0] for t in (g.dw1, g.db1, g.dw2, g.db2))
        if sync:
            if before_sync is not None:
                before_sync()
            self._x("grad_sync", self.sync_grads, g)
        return g

    def sync_grads(self, g):
        """Replica groups = the GPUs holding each expert's state: the routing
        replica counts, or `group_counts` when the runtime sets it (replicas
        whose state copy is in flight take part with zero gradients)."""
        cnt = self.group_counts if getattr(self, "group_counts", None) is not None else self.layer.replica_counts
        return sync_replica_grads(self.ex, cnt, self.layer.local_experts, g)


def sync_replica_grads(ex: Exchange, replica_counts, local_experts, g):
    """Replica-group SUM all-reduce of each replicated expert's (dw1, db1, dw2,
    db2), in ascending expert id on every rank, then the gate-weight gradient
    over all ranks. In place and copy-free: each expert's gradient is four
    contiguous slices of the layer's gradient arrays (dw1[i] is [f, d] etc.),
    reduced where they lie (NCCL runs them back to back on its stream)."""
    cnt = np.asarray(replica_counts)
    li = {e: i for i, e in enumerate(local_experts)}
    for e in range(cnt.shape[0]):
        grp = replica_gpus(cnt, e)
        if len(grp) < 2:
            continue
        ex.sync_group(grp)
        if ex.rank in grp:
            i = li[e]
            ex.all_reduce_many([g.dw1[i], g.db1[i], g.dw2[i], g.db2[i]], grp)
        else:  # non-members take part in the same calls (loopback rendezvous)
            ex.all_reduce_many(None, grp)
    ex.all_reduce(g.dwg, None)
    return g
