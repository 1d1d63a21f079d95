"""TEST INFRASTRUCTURE ONLY — the parity checker for the FlexMoE hot path.

Two independent CPU implementations the product is checked against:

* ``Oracle``    — ctypes over ``oracle/liboracle.so``, the plain-C restatement
                  of the reference's count-level algorithms (flexmoe_oracle.c).
* ``Reference`` — ctypes over ``oracle/_ref/libmoesim_ref.so``, the UNMODIFIED
                  reference sources (/root/reference/proj/src) compiled by
                  oracle/Makefile, behind our extern "C" shim (ref_shim.cpp).
                  Optional: absent on boxes where it was never built.

plus ``oracle.layer`` (numpy restatement of the layer math that has no
reference implementation: gate/top-k/softmax, permutation, FFN, combine).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline and
``--impl reference`` legs may import this package. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libmoesim_ref.so"

_P = C.c_void_p


def build(reference: bool = True) -> None:
    """Builds liboracle.so (always) and the reference shim (when sources exist)."""
    targets = ["oracle"] + (["ref"] if reference else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(_P)


class _Base:
    _lib_path: Path
    _err_fn: str
    _sigs: dict

    def __init__(self):
        if not self._lib_path.exists():
            raise FileNotFoundError(f"{self._lib_path} not built (make -C oracle)")
        self.lib = C.CDLL(str(self._lib_path))
        getattr(self.lib, self._err_fn).restype = C.c_char_p
        for name, (args, res) in self._sigs.items():
            f = getattr(self.lib, name)
            f.argtypes = args
            f.restype = res

    def _check(self, status):
        if status != 0:
            msg = getattr(self.lib, self._err_fn)().decode()
            exc = {1: ValueError, 2: RuntimeError, 4: IndexError}.get(status, RuntimeError)
            raise exc(msg)


class Oracle(_Base):
    """Plain-C restatement (flexmoe_oracle.c)."""

    _lib_path = ORACLE_SO
    _err_fn = "orc_last_error"
    _sigs = {
        "orc_route": ([_P, _P, C.c_int, C.c_int, _P], C.c_int),
        "orc_largest_remainder_round": ([_P, C.c_int, C.c_int64, _P], C.c_int),
        "orc_static_ep_kept": ([_P, C.c_int, C.c_int, C.c_double, C.c_int64, _P, _P], C.c_int),
        "orc_balance_ratio": ([_P, C.c_int, C.c_int, _P], C.c_int),
        "orc_generate_trace": (
            [C.c_int, C.c_int, C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int, _P],
            C.c_int,
        ),
        "orc_mt64_first": ([C.c_uint64, C.c_int], C.c_uint64),
        "orc_bf16_round_f32": ([_P, C.c_int64], None),
    }

    def bf16_round_f32(self, a):
        """In place (contiguous float32), OpenMP."""
        self.lib.orc_bf16_round_f32(_p(a), a.size)
        return a

    def route(self, D, cnt):
        D, cnt = _i64(D), _i32(cnt)
        N, G = D.shape
        flows = np.zeros((N, G, G), np.int64)
        self._check(self.lib.orc_route(_p(D), _p(cnt), N, G, _p(flows)))
        return flows

    def largest_remainder_round(self, exact, total):
        exact = _f64(exact)
        out = np.zeros(exact.shape[0], np.int64)
        self._check(self.lib.orc_largest_remainder_round(_p(exact), exact.shape[0], int(total), _p(out)))
        return out

    def static_ep_kept(self, D, cf, tokens_per_step=0):
        D = _i64(D)
        N, G = D.shape
        kept = np.zeros_like(D)
        dropped = np.zeros(1, np.int64)
        self._check(self.lib.orc_static_ep_kept(_p(D), N, G, float(cf), int(tokens_per_step), _p(kept), _p(dropped)))
        return kept, int(dropped[0])

    def balance_ratio(self, flows):
        flows = _i64(flows)
        N, G, _ = flows.shape
        r = np.zeros(1, np.float64)
        self._check(self.lib.orc_balance_ratio(_p(flows), N, G, _p(r)))
        return float(r[0])

    def generate_trace(self, N, G, tokens_per_step, zipf=1.25, drift=0.02, seed=42, steps=1):
        out = np.zeros((steps, N, G), np.int64)
        self._check(self.lib.orc_generate_trace(N, G, int(tokens_per_step), float(zipf), float(drift), int(seed), steps, _p(out)))
        return out


class Reference(_Base):
    """The unmodified reference library behind ref_shim.cpp."""

    _lib_path = REF_SO
    _err_fn = "ref_last_error"
    _sigs = {
        "ref_route": ([_P, _P, C.c_int, C.c_int, C.c_int, _P], C.c_int),
        "ref_balance_ratio": ([_P, _P, C.c_int, C.c_int, C.c_int, _P], C.c_int),
        "ref_largest_remainder_round": ([_P, C.c_int, C.c_int64, _P], C.c_int),
        "ref_generate_trace": (
            [C.c_int, C.c_int, C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int, _P],
            C.c_int,
        ),
        "ref_static_ep": ([_P, C.c_int, C.c_int, C.c_int, C.c_double, _P, _P], C.c_int),
        "ref_baseline_run": ([C.c_int, _P] + [C.c_int] * 4 + [C.c_double, C.c_int, C.c_int] + [_P] * 8, C.c_int),
        "ref_topology_load": ([C.c_char_p, _P, _P, _P, _P], C.c_int),
        "ref_save_trace": ([C.c_char_p, _P, C.c_int, C.c_int, C.c_int], C.c_int),
        "ref_load_trace": ([C.c_char_p, C.c_int, C.c_int, _P, C.c_int64, _P], C.c_int),
        "ref_engine_run": (
            [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P],
            C.c_int,
        ),
        "ref_make_scheduling_plan": (
            [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int],
            C.c_int,
        ),
        "ref_time_route": ([_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P], C.c_int),
        "ref_time_count_path": ([_P] + [C.c_int] * 6 + [C.c_double, _P], C.c_int),
        "ref_step_cost": ([_P, _P, C.c_int, C.c_int, C.c_int, _P, _P], C.c_int),
        "ref_plan_migrations": ([_P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P], C.c_int),
        "ref_engine_detail": (
            [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, C.c_int],
            C.c_int,
        ),
    }

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    @staticmethod
    def _slots(cnt, slots):
        return int(slots) if slots else int(max(1, np.asarray(cnt).sum(axis=0).max()))

    def route(self, D, cnt, slots=None):
        D, cnt = _i64(D), _i32(cnt)
        N, G = D.shape
        flows = np.zeros((N, G, G), np.int64)
        self._check(self.lib.ref_route(_p(D), _p(cnt), N, G, self._slots(cnt, slots), _p(flows)))
        return flows

    def balance_ratio(self, D, cnt, slots=None):
        D, cnt = _i64(D), _i32(cnt)
        N, G = D.shape
        r = np.zeros(1)
        self._check(self.lib.ref_balance_ratio(_p(D), _p(cnt), N, G, self._slots(cnt, slots), _p(r)))
        return float(r[0])

    def largest_remainder_round(self, exact, total):
        exact = _f64(exact)
        out = np.zeros(exact.shape[0], np.int64)
        self._check(self.lib.ref_largest_remainder_round(_p(exact), exact.shape[0], int(total), _p(out)))
        return out

    def generate_trace(self, N, G, tokens_per_step, zipf=1.25, drift=0.02, seed=42, steps=1):
        out = np.zeros((steps, N, G), np.int64)
        self._check(self.lib.ref_generate_trace(N, G, int(tokens_per_step), float(zipf), float(drift), int(seed), steps, _p(out)))
        return out

    def topology_load(self, path):
        ints, dbl = np.zeros(3, np.int32), np.zeros(6)
        intra, inter = np.zeros(65), np.zeros(65)
        self._check(self.lib.ref_topology_load(str(path).encode(), _p(ints), _p(dbl), _p(intra), _p(inter)))
        return ints, dbl, intra, inter

    def save_trace(self, trace, path):
        trace = _i64(trace)
        S, N, G = trace.shape
        self._check(self.lib.ref_save_trace(str(path).encode(), _p(trace), S, N, G))

    def load_trace(self, path, N=0, G=0):
        dims = np.zeros(3, np.int32)
        self._check(self.lib.ref_load_trace(str(path).encode(), N, G, None, 0, _p(dims)))
        out = np.zeros(tuple(int(v) for v in dims), np.int64)
        self._check(self.lib.ref_load_trace(str(path).encode(), N, G, _p(out), out.size, _p(dims)))
        return out

    def baseline_run(self, kind, trace, slots, cf=1.0, replicate_top=1, metric=0):
        trace = _i64(trace)
        S, N, G = trace.shape
        out = dict(ratio=np.zeros(S), metric=np.zeros(S), makespan=np.zeros(S),
                   misses=np.zeros(S, np.int32), dropped=np.zeros(S, np.int64),
                   reassigned=np.zeros(S, np.int64), util=np.zeros(S), replicas=np.zeros((S, N), np.int32))
        self._check(self.lib.ref_baseline_run(int(kind), _p(trace), S, N, G, int(slots), float(cf),
                                              int(replicate_top), int(metric),
                                              *[_p(out[k]) for k in ("ratio", "metric", "makespan", "misses",
                                                                     "dropped", "reassigned", "util",
                                                                     "replicas")]))
        return out

    def static_ep(self, trace, cf=1.0):
        trace = _i64(trace)
        S, N, G = trace.shape
        dropped = np.zeros(S, np.int64)
        ratio = np.zeros(S)
        self._check(self.lib.ref_static_ep(_p(trace), S, N, G, float(cf), _p(dropped), _p(ratio)))
        return dropped, ratio

    def engine_run(self, trace, slots, policy_mode=0, interval=10):
        """policy_mode: 0 Dynamic, 1 FixedInterval, 2 Static (sim_engine.hpp:33)."""
        trace = _i64(trace)
        S, N, G = trace.shape
        ratio = np.zeros(S)
        replicas = np.zeros((S, N), np.int32)
        ops = np.zeros(3, np.int64)
        self._check(self.lib.ref_engine_run(_p(trace), S, N, G, slots, policy_mode, interval, _p(ratio), _p(replicas), _p(ops)))
        return ratio, replicas, ops

    def make_scheduling_plan(self, D, cnt, slots, horizon=50):
        D, cnt = _i64(D), _i32(cnt)
        N, G = D.shape
        ops = np.zeros((16, 7), np.int32)
        n = np.zeros(1, np.int32)
        self._check(self.lib.ref_make_scheduling_plan(_p(D), _p(cnt), N, G, slots, horizon, _p(ops), _p(n), 16))
        return ops[: n[0]]

    def step_cost(self, D, cnt, slots):
        D, cnt = _i64(D), _i32(cnt)
        N, G = D.shape
        mk = np.zeros(1)
        per = np.zeros((G, 3))
        self._check(self.lib.ref_step_cost(_p(D), _p(cnt), N, G, slots, _p(mk), _p(per)))
        return float(mk[0]), per

    def plan_migrations(self, cnt, slots, horizon=50):
        cnt = _i32(cnt)
        N, G = cnt.shape
        ops = np.zeros((4, 7), np.int32)
        n = np.zeros(1, np.int32)
        self._check(self.lib.ref_plan_migrations(_p(cnt), N, G, slots, horizon, _p(ops), _p(n)))
        return ops[: n[0]]

    def engine_detail(self, trace, slots, policy_mode=0, interval=10, metric=0, max_ops=64):
        trace = _i64(trace)
        S, N, G = trace.shape
        mk = np.zeros(S)
        ab = np.zeros(S)
        n = np.zeros(S, np.int32)
        ops = np.zeros((S, max_ops, 7), np.int32)
        self._check(self.lib.ref_engine_detail(_p(trace), S, N, G, slots, policy_mode, interval, metric,
                                               _p(mk), _p(ab), _p(n), _p(ops), max_ops))
        return mk, ab, [ops[s, : n[s]] for s in range(S)]

    COUNT_PATH = ("route", "step_cost", "make_scheduling_plan", "plan_migrations", "engine_step")

    def time_count_path(self, trace, slots, policy_mode=0, interval=10, min_seconds=0.2) -> dict:
        """Seconds per call on one host thread of the reference's count-level
        per-step path: route (+balance_ratio), step_cost,
        make_scheduling_plan, plan_migrations on trace step 0 and
        Placement::initial, and one SimEngine step over the trace."""
        trace = _i64(trace)
        S, N, G = trace.shape
        out = np.zeros(6)
        self._check(self.lib.ref_time_count_path(_p(trace), S, N, G, int(slots), policy_mode, interval,
                                                 float(min_seconds), _p(out)))
        return dict(zip(self.COUNT_PATH, out[:5].tolist()))

    def time_route(self, D, cnt, slots=None, iters=1000):
        D, cnt = _i64(D), _i32(cnt)
        N, G = D.shape
        s = np.zeros(1)
        self._check(self.lib.ref_time_route(_p(D), _p(cnt), N, G, self._slots(cnt, slots), iters, _p(s)))
        return float(s[0])
