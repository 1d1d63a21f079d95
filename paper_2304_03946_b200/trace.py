"""Trace export / replay.

The reference consumes the gate as a TokenDemand trace (file
format `step,expert,gpu,tokens`, proj/src/workload.cpp:175-341). This module
closes the loop in both directions:

* export: `TraceRecorder` collects the all-gathered device histogram of every
  step (the step's TokenDemand, bit-exact counts of the real gate) and
  `save_trace` writes it in the reference's format, so the reference
  engine/CLI can replay real gate traces;
* replay: `load_trace` reads a reference trace, and `replay_inputs` builds
  exact-arithmetic gate inputs (x, Wg) for one GPU's column, so the REAL
  device gate reproduces that column's demand exactly (no injected indices).

File I/O is the native library's (`fm_trace_save` / `fm_trace_load`, same
acceptance rules and "<path>:<line>: <what>" errors as the reference loader).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib as L


def save_trace(trace, path, step_ids=None) -> None:
    """save_trace (workload.hpp:79): trace [steps][N][G] int64."""
    tr = np.ascontiguousarray(trace, np.int64)
    if tr.ndim != 3:
        raise L.InvalidArgument("trace must be [steps][experts][gpus]")
    ids = None if step_ids is None else np.ascontiguousarray(step_ids, np.int32)
    L.call("fm_trace_save", os.fsencode(path), tr.ctypes.data, None if ids is None else ids.ctypes.data,
           tr.shape[0], tr.shape[1], tr.shape[2])


def load_trace(path, num_experts: int = 0, num_gpus: int = 0) -> np.ndarray:
    """load_trace (workload.hpp:82-86): [steps][N][G] int64; dimensions
    inferred from the largest ids when not given."""
    s, n, g = C.c_int(), C.c_int(), C.c_int()
    p = os.fsencode(path)
    L.call("fm_trace_load", p, num_experts, num_gpus, None, 0, C.addressof(s), C.addressof(n), C.addressof(g))
    out = np.zeros((s.value, n.value, g.value), np.int64)
    L.call("fm_trace_load", p, num_experts, num_gpus, out.ctypes.data, out.size,
           C.addressof(s), C.addressof(n), C.addressof(g))
    return out


class TraceRecorder:
    """Per-step TokenDemand of a running layer/runtime (host copies of the
    all-gathered device histogram)."""

    def __init__(self):
        self.steps: list[np.ndarray] = []

    def record(self, demand_NG) -> None:
        self.steps.append(np.array(demand_NG, np.int64, copy=True))

    def trace(self) -> np.ndarray:
        return np.stack(self.steps) if self.steps else np.zeros((0, 0, 0), np.int64)

    def save(self, path) -> None:
        save_trace(self.trace(), path)


def replay_assignment(column, top_k: int) -> np.ndarray:
    """Expert choices [T][k] (distinct per token) whose per-expert unit counts
    equal `column` (one GPU's TokenDemand column, Σ = T·k).

    Units sorted by expert are dealt column-major: token t takes units
    t, t+T, ..., t+(k-1)T. A run of one expert is at most T long, so it never
    holds two units T apart: the k choices of a token are distinct."""
    col = np.asarray(column, np.int64)
    total = int(col.sum())
    if top_k < 1 or total % top_k:
        raise L.InvalidArgument(f"replay: demand total {total} is not a multiple of top_k {top_k}")
    T = total // top_k
    if (col < 0).any() or (col > T).any():
        raise L.InvalidArgument("replay: an expert's demand exceeds the token count (k choices are distinct)")
    units = np.repeat(np.arange(col.size, dtype=np.int32), col)
    return units.reshape(top_k, T).T.copy()


def replay_inputs(column, top_k: int, d_model: int, device=None, dtype=torch.bfloat16):
    """(x [T,d], Wg [N,d]) on `device` such that the gate (Eq. 3,
    logits = x·Wgᵀ, top-k, ties to the lower id) picks exactly
    `replay_assignment(column, top_k)`: Wg is the identity on the first N
    features, token t carries (k-j)/8 at the feature of its j-th expert.
    Every logit is exact in bf16/f32, the k picks are strictly ordered."""
    col = np.asarray(column, np.int64)
    N = col.size
    if d_model < N:
        raise L.InvalidArgument(f"replay: d_model {d_model} < num_experts {N}")
    choice = replay_assignment(col, top_k)
    T = choice.shape[0]
    x = np.zeros((T, d_model), np.float32)
    for j in range(top_k):
        x[np.arange(T), choice[:, j]] = (top_k - j) / 8.0
    wg = np.zeros((N, d_model), np.float32)
    wg[np.arange(N), np.arange(N)] = 1.0
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(x).to(dev).to(dtype), torch.from_numpy(wg).to(dev).to(dtype)
