"""Host mirror of the FlexMoE MoE layer (one process per GPU).

`MoELayer` owns an `fm_layer` handle of libflexmoe_b200.so and the expert
parameters as torch tensors (PyTorch is used for device memory and streams
only). The placement is the reference's replica-count view
(Placement::replica_count_on, proj/include/moesim/placement.hpp:80-82);
weights are packed for the local experts in ascending expert id.

No CPU fallback: constructing a layer without the native library or without
a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

FIELDS = {
    "topk_idx": (0, np.int32), "topk_w": (1, np.float32), "unit_pos": (2, np.int32),
    "gate_grad": (3, np.float32), "hist": (4, np.int64), "demand": (5, np.int64),
    "flows": (6, np.int64), "seg_start": (7, np.int32), "seg_real": (8, np.int32),
    "seg_rows": (9, np.int32), "totals": (10, np.int32), "send_rows": (11, np.int32),
    "recv_rows": (12, np.int32), "x_perm": (13, np.uint16), "act": (14, np.uint16),
    "y_perm": (15, np.uint16), "dy_perm": (16, np.uint16), "dh": (17, np.uint16),
    "dx_perm": (18, np.uint16), "route_status": (19, np.int32), "kept": (20, np.int64),
    "dropped": (21, np.int64),
}


PHASES = ["gate", "scan", "route", "dispatch", "ffn1_fwd", "ffn2_fwd", "combine_fwd",
          "combine_bwd", "ffn2_dgrad", "ffn1_dgrad", "ffn2_wgrad", "ffn1_wgrad", "bias_grad",
          "unpermute", "gate_wgrad", "relayout"]  # FM_PHASE_* order


class _Config(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "num_experts", "top_k", "d_model", "d_ff", "num_gpus", "rank", "max_tokens", "slots_per_gpu")]


@dataclass
class LayerGrads:
    dx: torch.Tensor
    dwg: torch.Tensor
    dw1: torch.Tensor
    db1: torch.Tensor
    dw2: torch.Tensor
    db2: torch.Tensor


class MoELayer:
    def __init__(self, num_experts, top_k, d_model, d_ff, replica_counts=None, num_gpus=1, rank=0,
                 max_tokens=65536, slots_per_gpu=0, device=None):
        if not torch.cuda.is_available():
            raise L.CudaError("MoELayer needs a CUDA device (no CPU fallback)")
        self.N, self.k, self.d, self.f = num_experts, top_k, d_model, d_ff
        self.G, self.rank, self.max_tokens = num_gpus, rank, max_tokens
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        if replica_counts is None:
            replica_counts = np.zeros((num_experts, num_gpus), np.int32)
            replica_counts[np.arange(num_experts), np.arange(num_experts) % num_gpus] = 1
        self._cfg = _Config(num_experts, top_k, d_model, d_ff, num_gpus, rank, max_tokens, slots_per_gpu)
        cnt = np.ascontiguousarray(replica_counts, np.int32)
        h = C.c_void_p()
        lib = L.lib()
        L.check(lib.fm_layer_create(C.byref(self._cfg), cnt.ctypes.data, C.byref(h)))
        self._h = h
        self.replica_counts = cnt.copy()
        self._saved = None

    def __del__(self):
        try:
            L.release("fm_layer_destroy", getattr(self, "_h", None))
        except (TypeError, AttributeError):  # interpreter shutdown
            pass
        self._h = None

    # ---------------------------------------------------------------- placement
    @property
    def local_experts(self) -> list[int]:
        n = C.c_int(0)
        buf = np.zeros(self.N, np.int32)
        L.check(L.lib().fm_layer_local_experts(self._h, C.byref(n), buf.ctypes.data))
        return buf[: n.value].tolist()

    @property
    def side_jobs(self) -> int:
        """fm_layer_side_jobs: bit 0 = the tile column sums ran beside the FFN2
        weight-gradient GEMM, bit 1 = the un-permute beside the FFN1 one."""
        m = C.c_int(0)
        L.check(L.lib().fm_layer_side_jobs(self._h, C.byref(m)))
        return m.value

    def set_side_jobs(self, enable: bool) -> None:
        """fm_layer_set_side_jobs: False runs the column sums and the un-permute
        as their own kernels (same results, bit for bit)."""
        L.check(L.lib().fm_layer_set_side_jobs(self._h, 1 if enable else 0))

    def set_placement(self, replica_counts):
        cnt = np.ascontiguousarray(replica_counts, np.int32)
        L.check(L.lib().fm_layer_set_placement(self._h, cnt.ctypes.data))
        self.replica_counts = cnt.copy()

    def set_placement_async(self, replica_counts, hosted=None, stream=None):
        """The placement switch enqueued on the stream (no allocation, no host
        sync). hosted ([N] bool, optional): experts this rank keeps state for
        with replica count 0 (a replica whose state copy is in flight): local,
        with zero rows."""
        cnt = np.ascontiguousarray(replica_counts, np.int32)
        h = None if hosted is None else np.ascontiguousarray(np.asarray(hosted, bool).astype(np.int32))
        L.check(L.lib().fm_layer_set_placement_async(self._h, cnt.ctypes.data,
                                                     None if h is None else h.ctypes.data, L.stream_ptr(stream)))
        self.replica_counts = cnt.copy()

    def set_operand_slots(self, slot_of, capacity, stream=None):
        """slot_of [N]: operand row of every local expert (None: packed layout)."""
        if slot_of is None:
            L.check(L.lib().fm_layer_set_operand_slots(self._h, None, 0, L.stream_ptr(stream)))
            return
        t = np.ascontiguousarray(slot_of, np.int32)
        L.check(L.lib().fm_layer_set_operand_slots(self._h, t.ctypes.data, int(capacity), L.stream_ptr(stream)))

    def set_capacity_factor(self, capacity_factor: float) -> None:
        """StaticEP mode (baselines.cpp:81-131): > 0 drops units beyond capacity
        (bit-exact with fm_static_ep_kept); 0 / inf = no drops (FlexMoE)."""
        L.check(L.lib().fm_layer_set_capacity_factor(self._h, float(capacity_factor)))

    def init_params(self, seed=0, dtype=torch.bfloat16):
        """Random-init parameters of this layer's architecture (gate + local experts)."""
        g = torch.Generator(device="cpu").manual_seed(seed)
        nl, d, f = len(self.local_experts), self.d, self.f
        mk = lambda *s, scale: (torch.randn(*s, generator=g) * scale).to(self.device)
        return dict(
            wg=mk(self.N, d, scale=d**-0.5).to(dtype),
            w1=mk(nl, f, d, scale=d**-0.5).to(dtype),
            b1=mk(nl, f, scale=0.02).float(),
            w2=mk(nl, d, f, scale=f**-0.5).to(dtype),
            b2=mk(nl, d, scale=0.02).float(),
        )

    # ---------------------------------------------------------------- step
    def forward(self, x, wg, w1, b1, w2, b2, out=None, stream=None):
        T = x.shape[0]
        y = out if out is not None else torch.empty(T, self.d, device=x.device, dtype=torch.bfloat16)
        L.check(L.lib().fm_layer_forward(self._h, x.data_ptr(), T, wg.data_ptr(), w1.data_ptr(),
                                         b1.data_ptr(), w2.data_ptr(), b2.data_ptr(), y.data_ptr(),
                                         L.stream_ptr(stream)))
        self._saved = (T, x.device)
        # the native step keeps raw pointers to x (StaticEP backward re-reads the
        # gate input of dropped units) and to wg, w1, w2 (dgrad / gate backward):
        # hold the tensors until backward is enqueued, or the caching allocator
        # may hand their memory to the gradient buffers (fm_layer_forward contract)
        self._alive = (x, wg, w1, b1, w2, b2)
        return y

    def backward(self, dy, grads: LayerGrads | None = None, stream=None) -> LayerGrads:
        T, dev = self._saved
        nl = len(self.local_experts)
        if grads is None:
            z = lambda *s, dt=torch.float32: torch.empty(*s, device=dev, dtype=dt)
            grads = LayerGrads(dx=z(T, self.d, dt=torch.bfloat16), dwg=z(self.N, self.d),
                               dw1=z(nl, self.f, self.d), db1=z(nl, self.f),
                               dw2=z(nl, self.d, self.f), db2=z(nl, self.d))
        L.check(L.lib().fm_layer_backward(self._h, dy.data_ptr(), grads.dx.data_ptr(),
                                          grads.dwg.data_ptr(), grads.dw1.data_ptr(),
                                          grads.db1.data_ptr(), grads.dw2.data_ptr(),
                                          grads.db2.data_ptr(), L.stream_ptr(stream)))
        self._alive = None  # enqueued: later allocations are stream-ordered after it
        return grads

    # ---------------------------------------------------------------- P2P transport
    def enable_p2p(self) -> None:
        """Allocate the exchange arena for the peer-to-peer transport."""
        L.check(L.lib().fm_layer_enable_p2p(self._h))

    def p2p_handle(self) -> bytes:
        buf = (C.c_char * 64)()
        L.check(L.lib().fm_layer_p2p_handle(self._h, buf))
        return bytes(buf)

    def p2p_open_peer(self, peer: int, handle: bytes) -> None:
        buf = (C.c_char * 64).from_buffer_copy(handle)
        L.check(L.lib().fm_layer_p2p_open_peer(self._h, peer, buf))

    def p2p_link_peer(self, peer: int, other: "MoELayer") -> None:
        L.check(L.lib().fm_layer_p2p_link_peer(self._h, peer, other._h))
        self._p2p_peers = getattr(self, "_p2p_peers", []) + [other]  # keep the peer arena alive

    def p2p_status(self) -> int:
        st = C.c_int(0)
        L.check(L.lib().fm_layer_p2p_status(self._h, C.byref(st)))
        return st.value

    # ---------------------------------------------------------------- timing
    def set_timing(self, enable: bool) -> None:
        L.check(L.lib().fm_layer_set_timing(self._h, 1 if enable else 0))

    def read_timing(self) -> dict[str, tuple[float, int]]:
        """{phase: (total ms, launches)} since timing was enabled (synchronises)."""
        ms = np.zeros(len(PHASES), np.float64)
        n = np.zeros(len(PHASES), np.int32)
        L.check(L.lib().fm_layer_read_timing(self._h, ms.ctypes.data, n.ctypes.data))
        return {name: (float(ms[i]), int(n[i])) for i, name in enumerate(PHASES)}

    # ---------------------------------------------------------------- introspection
    def copy_out_async(self, field: str, host: torch.Tensor, stream=None) -> int:
        """Enqueue a copy of `field` into the page-locked tensor `host` on the
        stream (no device synchronisation); returns the bytes it will write."""
        code, _ = FIELDS[field]
        written = C.c_size_t(0)
        L.check(L.lib().fm_layer_copy_out_async(self._h, code, host.data_ptr(), host.numel() * host.element_size(),
                                                C.byref(written), L.stream_ptr(stream)))
        return written.value

    def read(self, field: str, count: int | None = None) -> np.ndarray:
        code, dt = FIELDS[field]
        itemsize = np.dtype(dt).itemsize
        nbytes = (count * itemsize) if count is not None else 1 << 34
        if count is None:
            raise ValueError("count required")
        out = np.zeros(count, dt)
        written = C.c_size_t(0)
        L.check(L.lib().fm_layer_copy_out(self._h, code, out.ctypes.data, nbytes, C.byref(written)))
        return out[: written.value // itemsize]
