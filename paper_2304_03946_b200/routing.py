"""Count-level FlexMoE routing through the C ABI (host side).

Mirrors the reference's router / metrics API (proj/include/moesim/router.hpp,
policy.hpp:38, workload.hpp:90, baselines.cpp:89-122) on numpy arrays:
``demand[e][g]`` int64, ``replica_counts[e][g]`` int32, ``flows[e][src][dst]``
int64. Every call goes to libflexmoe_b200.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def route(demand, replica_counts) -> np.ndarray:
    """`route(TokenDemand, Placement)` (router.hpp:62): flows[e][src][dst]."""
    D, cnt = _i64(demand), _i32(replica_counts)
    if D.shape != cnt.shape:
        raise L.InvalidArgument("route: demand and placement disagree on shape")
    N, G = D.shape
    flows = np.zeros((N, G, G), np.int64)
    L.call("fm_route_counts", L.ptr(D), L.ptr(cnt), N, G, L.ptr(flows))
    return flows


def received_matrix(flows) -> np.ndarray:
    f = _i64(flows)
    N, G, _ = f.shape
    out = np.zeros((N, G), np.int64)
    L.call("fm_received_matrix", L.ptr(f), N, G, L.ptr(out))
    return out


def per_gpu_received(flows) -> np.ndarray:
    f = _i64(flows)
    N, G, _ = f.shape
    out = np.zeros(G, np.int64)
    L.call("fm_per_gpu_received", L.ptr(f), N, G, L.ptr(out))
    return out


def balance_ratio(flows) -> float:
    """Eq. 7 (policy.cpp:32-46)."""
    f = _i64(flows)
    N, G, _ = f.shape
    r = C.c_double(0.0)
    L.check(L.lib().fm_balance_ratio(L.ptr(f), N, G, C.byref(r)))
    return r.value


def largest_remainder_round(exact, total) -> np.ndarray:
    x = np.ascontiguousarray(exact, dtype=np.float64)
    out = np.zeros(x.shape[0], np.int64)
    L.call("fm_largest_remainder_round", L.ptr(x), x.shape[0], int(total), L.ptr(out))
    return out


def static_ep_kept(demand, capacity_factor=1.0):
    """StaticEP capacity drops (baselines.cpp:89-122): (kept[e][g], dropped)."""
    D = _i64(demand)
    N, G = D.shape
    kept = np.zeros_like(D)
    dropped = C.c_int64(0)
    L.check(L.lib().fm_static_ep_kept(L.ptr(D), N, G, float(capacity_factor), L.ptr(kept), C.byref(dropped)))
    return kept, dropped.value
