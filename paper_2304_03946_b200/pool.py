"""Expert state pool: f32 master weights + Adam moments of the hosted experts in
one device allocation per GPU (`fm_expert_pool`, csrc/expert_pool.cu), and
peer-to-peer migration of whole expert states on a side stream.

The reference turns a placement change into TransferDescriptor{src, dst,
bytes} (proj/include/moesim/placement.hpp:31-35, placement.cpp:143-232) and
models their drain (sim_engine.cpp:124-262). Here the receiving GPU pulls the
slot from the source GPU's pool (CUDA IPC mapping across processes, NVLink on
an NVSwitch box) with cudaMemcpyAsync on the pool's side stream; the compute
stream waits for it only before the expert FFN of the step.

Slot bookkeeping is deterministic and replicated: every rank keeps a
`SlotAllocator` for every rank and applies the same placement changes in the
same order, so a receiver knows the source's slot without asking.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L

_TENSORS = ("w1", "b1", "w2", "b2")


class _Cai:
    """A raw device range as a __cuda_array_interface__ object (zero-copy views)."""

    def __init__(self, ptr, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


class _AdamConfig(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("step", C.c_int)]


class ExpertPool:
    """ctypes handle of one `fm_expert_pool` on the current device."""

    def __init__(self, slots: int, d_model: int, d_ff: int, world: int = 1):
        if not torch.cuda.is_available():
            raise L.CudaError("ExpertPool needs a CUDA device (no CPU fallback)")
        h = C.c_void_p()
        L.check(L.lib().fm_pool_create(slots, d_model, d_ff, world, C.byref(h)))
        self._h = h
        self.slots, self.d, self.f, self.world = slots, d_model, d_ff, world
        P, sb = C.c_int64(), C.c_int64()
        L.check(L.lib().fm_pool_info(h, C.byref(P), C.byref(sb)))
        self.P, self.slot_bytes = P.value, sb.value
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._peers = []  # keep linked pools alive

    def __del__(self):
        try:
            L.release("fm_pool_destroy", getattr(self, "_h", None))
        except (TypeError, AttributeError):  # interpreter shutdown
            pass
        self._h = None

    @property
    def state_bytes(self) -> int:
        """Bytes pulled per migrated expert (master + m + v, f32)."""
        return 12 * self.P

    def slot_tensor(self, slot: int) -> torch.Tensor:
        """[3, P] f32 view of a slot: master, m, v."""
        p = C.c_void_p()
        L.check(L.lib().fm_pool_slot_ptr(self._h, slot, C.byref(p)))
        return torch.as_tensor(_Cai(p.value, (3, self.P)), device=self.device)

    def views(self, slot: int) -> list[dict[str, torch.Tensor]]:
        """[master, m, v] as {w1 [f,d], b1 [f], w2 [d,f], b2 [d]} views of the slot."""
        t = self.slot_tensor(slot)
        d, f = self.d, self.f
        out = []
        for i in range(3):
            row, o = t[i], 0
            dv = {}
            for k, shape in (("w1", (f, d)), ("b1", (f,)), ("w2", (d, f)), ("b2", (d,))):
                n = int(np.prod(shape))
                dv[k] = row[o:o + n].view(shape)
                o += n
            out.append(dv)
        return out

    # ------------------------------------------------------------ peers
    def ipc_handle(self) -> bytes:
        buf = (C.c_char * 64)()
        L.check(L.lib().fm_pool_ipc_handle(self._h, buf))
        return bytes(buf)

    def open_peer(self, peer: int, handle: bytes) -> None:
        buf = (C.c_char * 64).from_buffer_copy(handle)
        L.check(L.lib().fm_pool_open_peer(self._h, peer, buf))

    def link_peer(self, peer: int, other: "ExpertPool") -> None:
        L.check(L.lib().fm_pool_link_peer(self._h, peer, other._h))
        self._peers.append(other)

    # ------------------------------------------------------------ device work
    @staticmethod
    def _slots(local_slots):
        a = np.ascontiguousarray(local_slots, np.int32)
        return a, len(a)

    def migrate(self, moves, local_slots, packed, stream=None) -> None:
        """moves: [(dst_slot, peer, src_slot)]; then re-pack `local_slots` into
        `packed` (w1, b1, w2, b2 capacity buffers) on the side stream."""
        mv = np.ascontiguousarray(np.asarray(moves, np.int32).reshape(-1, 3))
        ls, n = self._slots(local_slots)
        w1, b1, w2, b2 = packed
        L.check(L.lib().fm_pool_migrate(self._h, mv.ctypes.data, len(mv), ls.ctypes.data, n, w1.data_ptr(),
                                        b1.data_ptr(), w2.data_ptr(), b2.data_ptr(), L.stream_ptr(stream)))

    def wait_ready(self, stream=None) -> None:
        L.check(L.lib().fm_pool_wait_ready(self._h, L.stream_ptr(stream)))

    def pack(self, local_slots, packed, stream=None) -> None:
        ls, n = self._slots(local_slots)
        w1, b1, w2, b2 = packed
        L.check(L.lib().fm_pool_pack(self._h, ls.ctypes.data, n, w1.data_ptr(), b1.data_ptr(), w2.data_ptr(),
                                     b2.data_ptr(), L.stream_ptr(stream)))

    def adam(self, local_slots, grads, packed, lr, betas, eps, step, stream=None) -> None:
        ls, n = self._slots(local_slots)
        dw1, db1, dw2, db2 = (g.contiguous() for g in grads)
        cfg = _AdamConfig(lr, betas[0], betas[1], eps, step)
        w1, b1, w2, b2 = packed
        L.check(L.lib().fm_pool_adam(self._h, ls.ctypes.data, n, dw1.data_ptr(), db1.data_ptr(),
                                     dw2.data_ptr(), db2.data_ptr(), C.byref(cfg), w1.data_ptr(),
                                     b1.data_ptr(), w2.data_ptr(), b2.data_ptr(), L.stream_ptr(stream)))

    def migration_stats(self) -> tuple[float, int, int]:
        """(side-stream copy ms, bytes pulled, slots pulled) so far (synchronises)."""
        ms, nb, nc = C.c_double(), C.c_int64(), C.c_int64()
        L.check(L.lib().fm_pool_migration_stats(self._h, C.byref(ms), C.byref(nb), C.byref(nc)))
        return ms.value, nb.value, nc.value


class SlotAllocator:
    """Slot table of one GPU's pool. A slot vacated in step s becomes free at
    the start of step s+1 (a peer may still be pulling it during step s)."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.slot_of: dict[int, int] = {}
        self._free = list(range(capacity))
        self._vacated: list[int] = []

    def begin_step(self) -> None:
        self._free = sorted(self._free + self._vacated)
        self._vacated = []

    def host(self, e: int) -> int:
        if e in self.slot_of:
            return self.slot_of[e]
        if not self._free:
            raise L.LogicError(f"expert pool: no free slot for expert {e} (capacity {self.capacity})")
        s = self._free.pop(0)
        self.slot_of[e] = s
        return s

    def vacate(self, e: int) -> None:
        s = self.slot_of.pop(e, None)
        if s is not None:
            self._vacated.append(s)


def state_moves(old_counts, new_counts) -> list[tuple[int, int, int]]:
    """(expert, src, dst) state copies of a placement change: every GPU that
    newly hosts an expert receives it from the lowest-id GPU that hosted it
    before (a holder of the up-to-date state; on one NVSwitch domain that is
    also the reference's nearest-by-bandwidth expand source, placement.cpp:
    160-169). Identical on every rank."""
    old_counts, new_counts = np.asarray(old_counts), np.asarray(new_counts)
    moves = []
    for e in range(old_counts.shape[0]):
        holders = np.nonzero(old_counts[e] > 0)[0]
        for g in np.nonzero((new_counts[e] > 0) & (old_counts[e] == 0))[0]:
            moves.append((e, int(holders[0]), int(g)))
    return moves


def apply_placement_change(slot_dir: list[SlotAllocator], old_counts, new_counts):
    """Updates every rank's slot table for one placement change and returns
    the pulls [(expert, src_gpu, src_slot, dst_gpu, dst_slot)]. Order: slots
    vacated last step become free; source slots are looked up before any
    vacate; GPUs that stop hosting an expert vacate its slot (readable until
    the next step); receivers take their lowest free slot."""
    old_counts, new_counts = np.asarray(old_counts), np.asarray(new_counts)
    for a in slot_dir:
        a.begin_step()
    moves = state_moves(old_counts, new_counts)
    src_slot = [slot_dir[src].slot_of[e] for e, src, _ in moves]
    for e in range(old_counts.shape[0]):
        for g in np.nonzero((old_counts[e] > 0) & (new_counts[e] == 0))[0]:
            slot_dir[g].vacate(e)
    return [(e, src, ss, dst, slot_dir[dst].host(e)) for (e, src, dst), ss in zip(moves, src_slot)]


class ExpertStore:
    """Parameters and Adam state of the experts hosted on this GPU, in an
    ExpertPool, plus the packed GEMM operands of the local experts
    (w1 [n,f,d] bf16, b1 [n,f] f32, w2 [n,d,f] bf16, b2 [n,d] f32; capacity
    buffers allocated once, so side-stream packing never races the allocator)."""

    def __init__(self, d, f, device, capacity, world=1, max_local=None, lr=1e-4, betas=(0.9, 0.999),
                 eps=1e-8, allocator: SlotAllocator | None = None, by_slot=False):
        """by_slot: the operands are indexed by pool slot (capacity rows; the
        layer addresses them through MoELayer.set_operand_slots), so placement
        changes move no weights and a migration re-packs only pulled slots.
        Otherwise they are packed in ascending local order (max_local rows)."""
        self.d, self.f, self.device = d, f, device
        self.lr, self.betas, self.eps = lr, betas, eps
        self.pool = ExpertPool(capacity, d, f, world)
        self.alloc = allocator or SlotAllocator(capacity)
        self.by_slot = by_slot
        if by_slot:
            L.check(L.lib().fm_pool_set_operand_layout(self.pool._h, 1))
        n = capacity if by_slot else max(1, max_local or capacity)
        bf = torch.bfloat16
        self._packed = (torch.zeros(n, f, d, dtype=bf, device=device), torch.zeros(n, f, device=device),
                        torch.zeros(n, d, f, dtype=bf, device=device), torch.zeros(n, d, device=device))
        self.t = 0

    @staticmethod
    def init_expert(e, d, f):
        g = torch.Generator(device="cpu").manual_seed(10_000 + e)  # identical on every rank
        return {"w1": torch.randn(f, d, generator=g) * d**-0.5, "b1": torch.randn(f, generator=g) * 0.02,
                "w2": torch.randn(d, f, generator=g) * f**-0.5, "b2": torch.randn(d, generator=g) * 0.02}

    def create(self, e):
        slot = self.alloc.host(e)
        master, m, v = self.pool.views(slot)
        for k, t in self.init_expert(e, self.d, self.f).items():
            master[k].copy_(t)
            m[k].zero_()
            v[k].zero_()

    def _views(self, which):
        return {e: self.pool.views(s)[which] for e, s in self.alloc.slot_of.items()}

    @property
    def master(self):
        return self._views(0)

    @property
    def m(self):
        return self._views(1)

    @property
    def v(self):
        return self._views(2)

    def state(self, e) -> list[torch.Tensor]:
        """The tensors that make up expert e's model state, in a fixed order."""
        master, m, v = self.pool.views(self.alloc.slot_of[e])
        return [master[k] for k in _TENSORS] + [m[k] for k in _TENSORS] + [v[k] for k in _TENSORS]

    def state_bytes(self, e=None) -> int:
        return self.pool.state_bytes

    def slots(self, local) -> list[int]:
        return [self.alloc.slot_of[e] for e in local]

    def packed(self, n=None):
        if self.by_slot:
            return self._packed
        return tuple(t[:n] for t in self._packed)

    def pack(self, local):
        """Layer operands for the local experts (ascending id; by_slot: at
        their slots), packed on the current stream."""
        if not local:
            return self.packed(1)
        self.pool.pack(self.slots(local), self._packed)
        return self.packed(len(local))

    def slot_table(self, num_experts) -> np.ndarray:
        """[N] operand row (= pool slot) of every hosted expert, -1 elsewhere."""
        t = -np.ones(num_experts, np.int32)
        for e, s in self.alloc.slot_of.items():
            t[e] = s
        return t

    def tick(self) -> int:
        """Advance the optimizer step count. Called on EVERY rank every step,
        hosting experts or not: Adam's bias correction depends on it, and an
        expert that later expands onto a GPU that hosted nothing must get the
        same update there as on its other replicas (bit-identical replicas)."""
        self.t += 1
        return self.t

    @torch.no_grad()
    def adam_step(self, local, grads):
        """One fused Adam step (step count `self.t`, see tick()) per local
        expert from the (replica-summed) gradients; refreshes the packed
        operands of `local` in the same pass."""
        if self.t < 1:
            raise L.LogicError("adam_step before the first tick()")
        self.pool.adam(self.slots(local), (grads.dw1, grads.db1, grads.dw2, grads.db2), self._packed,
                       self.lr, self.betas, self.eps, self.t)
