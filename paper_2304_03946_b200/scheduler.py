"""Host placement scheduler (C ABI in libflexmoe_b200.so).

Mirrors the reference's policy layer on numpy arrays: the cluster profile
(ClusterTopology), the vExpert slot table (Placement), step_cost,
make_scheduling_plan, plan_migrations, Placement::apply, and the Alg. 1 step
driver with its adjustment queue (SimEngine::run_step). It consumes the
TokenDemand the device gate produces each step.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

MAX_GROUP = 64
EXPAND, SHRINK, MIGRATE = 0, 1, 2


class ClusterProfile(C.Structure):
    _fields_ = [("num_gpus", C.c_int), ("gpus_per_node", C.c_int), ("slots_per_gpu", C.c_int),
                ("intra_node_bandwidth_bps", C.c_double), ("inter_node_bandwidth_bps", C.c_double),
                ("tps", C.c_double), ("expert_param_bytes", C.c_double),
                ("expert_state_bytes", C.c_double), ("token_bytes", C.c_double),
                ("allreduce_bps_intra", C.c_double * (MAX_GROUP + 1)),
                ("allreduce_bps_inter", C.c_double * (MAX_GROUP + 1))]

    @classmethod
    def reference_default(cls, num_gpus, slots_per_gpu):
        """ClusterTopology::default_profile (topology.cpp:140-184), A100-like."""
        p = cls()
        L.check(L.lib().fm_profile_reference_default(num_gpus, slots_per_gpu, C.byref(p)))
        return p

    @classmethod
    def from_json(cls, cfg):
        """ClusterTopology::from_json / from_file (topology.cpp:64-138): a dict,
        a JSON string or a path."""
        import json
        import os
        if isinstance(cfg, (str, bytes, os.PathLike)) and not str(cfg).lstrip().startswith("{"):
            try:
                with open(cfg) as fh:
                    cfg = json.load(fh)
            except OSError:
                raise L.FlexMoEError(f"cannot open topology config: {os.fspath(cfg)}") from None
        elif isinstance(cfg, (str, bytes)):
            cfg = json.loads(cfg)
        return _profile_from_json(cls, cfg)

    def to_json(self) -> dict:
        """ClusterTopology::to_json (topology.cpp:222-255)."""
        G, gpn = self.num_gpus, self.gpus_per_node
        cfg = {"num_gpus": G, "gpus_per_node": gpn, "vexperts_per_gpu": self.slots_per_gpu,
               "intra_node_bandwidth_bps": self.intra_node_bandwidth_bps, "tps": self.tps,
               "expert_param_bytes": self.expert_param_bytes, "expert_state_bytes": self.expert_state_bytes,
               "token_bytes": self.token_bytes}
        if self.inter_node_bandwidth_bps > 0:
            cfg["inter_node_bandwidth_bps"] = self.inter_node_bandwidth_bps
        bps = {}
        max_intra = min(gpn, G)
        if max_intra >= 2:
            bps["intra"] = {str(n): self.allreduce_bps_intra[n] for n in range(2, max_intra + 1)}
        if G > gpn:
            bps["inter"] = {str(n): self.allreduce_bps_inter[n] for n in range(2, G + 1)}
        if bps:
            cfg["allreduce_bps"] = bps
        return cfg

    @classmethod
    def b200(cls, num_gpus, slots_per_gpu, tps, expert_param_bytes, expert_state_bytes, token_bytes,
             link_bps=770e9, allreduce_bus_bps=725e9):
        """One NVSwitch node of B200s: uniform peers (NVLink 5, measured 770 GB/s
        per direction), all-reduce throughput from the measured bus bandwidth."""
        p = cls()
        p.num_gpus, p.gpus_per_node, p.slots_per_gpu = num_gpus, num_gpus, slots_per_gpu
        p.intra_node_bandwidth_bps = link_bps
        p.inter_node_bandwidth_bps = link_bps
        p.tps, p.expert_param_bytes = tps, expert_param_bytes
        p.expert_state_bytes, p.token_bytes = expert_state_bytes, token_bytes
        for n in range(2, num_gpus + 1):  # algorithm bandwidth = bus bandwidth * n / (2(n-1))
            p.allreduce_bps_intra[n] = allreduce_bus_bps * n / (2.0 * (n - 1))
        return p


def _topology_error(msg):
    return L.InvalidArgument("topology config: " + msg)


def _positive(cfg, key):
    if key not in cfg:
        raise _topology_error(f"missing field '{key}'")
    v = float(cfg[key])
    if not v > 0:
        raise _topology_error(f"non-positive {key}")
    return v


def _bps_table(table, max_size, span):
    out = [0.0] * (max_size + 1)
    for n in range(2, max_size + 1):
        key = str(n)
        if key not in table:
            raise _topology_error(f"allreduce_bps.{span} missing entry for group size {key}")
        v = float(table[key])
        if not v > 0:
            raise _topology_error(f"non-positive allreduce_bps.{span}[{key}]")
        if n > 2 and v > out[n - 1]:
            raise _topology_error(f"allreduce_bps.{span} must be non-increasing in group size")
        out[n] = v
    return out


def _profile_from_json(cls, cfg):
    """ClusterTopology::from_json (topology.cpp:64-128): same fields, checks
    and messages."""
    for key in ("num_gpus", "gpus_per_node", "vexperts_per_gpu"):
        if key not in cfg:
            raise _topology_error(f"missing field '{key}'")
    G, gpn, E = int(cfg["num_gpus"]), int(cfg["gpus_per_node"]), int(cfg["vexperts_per_gpu"])
    if G < 1:
        raise _topology_error("num_gpus must be >= 1")
    if gpn < 1 or G % gpn != 0:
        raise _topology_error("num_gpus must be a positive multiple of gpus_per_node")
    if E < 1:
        raise _topology_error("vexperts_per_gpu must be >= 1")
    if G > MAX_GROUP:
        raise L.InvalidArgument(f"profile: at most {MAX_GROUP} GPUs")
    p = cls()
    p.num_gpus, p.gpus_per_node, p.slots_per_gpu = G, gpn, E
    p.intra_node_bandwidth_bps = _positive(cfg, "intra_node_bandwidth_bps")
    p.tps = _positive(cfg, "tps")
    p.expert_param_bytes = _positive(cfg, "expert_param_bytes")
    p.expert_state_bytes = _positive(cfg, "expert_state_bytes")
    p.token_bytes = _positive(cfg, "token_bytes")
    multi = G > gpn
    if multi or "inter_node_bandwidth_bps" in cfg:
        p.inter_node_bandwidth_bps = _positive(cfg, "inter_node_bandwidth_bps")
    if G >= 2:
        if "allreduce_bps" not in cfg:
            raise _topology_error("missing field 'allreduce_bps'")
        tables = cfg["allreduce_bps"]
        max_intra = min(gpn, G)
        intra = inter = None
        if max_intra >= 2:
            if "intra" not in tables:
                raise _topology_error("missing allreduce_bps.intra")
            intra = _bps_table(tables["intra"], max_intra, "intra")
            for n, v in enumerate(intra):
                p.allreduce_bps_intra[n] = v
        if multi:
            if "inter" not in tables:
                raise _topology_error("missing allreduce_bps.inter")
            inter = _bps_table(tables["inter"], G, "inter")
            for n in range(2, max_intra + 1):
                if inter[n] > intra[n]:
                    raise _topology_error(f"inter-node bps exceeds intra-node bps for group size {n}")
            for n, v in enumerate(inter):
                p.allreduce_bps_inter[n] = v
    return p


class PlacementOp(C.Structure):
    _fields_ = [("kind", C.c_int), ("expert", C.c_int), ("gpu", C.c_int), ("a_gpu", C.c_int),
                ("a_slot", C.c_int), ("b_gpu", C.c_int), ("b_slot", C.c_int)]

    def as_tuple(self):
        return (self.kind, self.expert, self.gpu, self.a_gpu, self.a_slot, self.b_gpu, self.b_slot)


class SchedulerConfig(C.Structure):
    _fields_ = [("threshold", C.c_double), ("metric", C.c_int), ("policy_mode", C.c_int),
                ("interval_steps", C.c_int), ("amortization_horizon", C.c_int),
                ("adjust_bandwidth_fraction", C.c_double), ("max_live_groups", C.c_int),
                ("group_creation_latency_s", C.c_double), ("flip_mode", C.c_int), ("async_policy", C.c_int)]

    @classmethod
    def defaults(cls, **kw):
        """SimConfig defaults (sim_engine.hpp:35-49); flip_mode / async_policy
        0 = the reference's modelled drain and inline policy
        (include/flexmoe_b200.h documents the device modes)."""
        c = cls(1.1, 0, 0, 10, 50, 0.5, 64, 0.005, 0, 0)
        for k, v in kw.items():
            setattr(c, k, v)
        return c


class StepReport(C.Structure):
    _fields_ = [("balance_ratio", C.c_double), ("metric_value", C.c_double), ("makespan_s", C.c_double),
                ("adjust_s", C.c_double), ("adjust_bytes", C.c_double), ("group_misses", C.c_int),
                ("n_accepted", C.c_int), ("n_applied", C.c_int), ("pending_ops", C.c_int),
                ("n_issued", C.c_int)]


def slots_from_counts(counts, slots_per_gpu):
    """Placement::from_counts slot fill (placement.cpp:74-107): per GPU, experts
    ascending, each taking its count of consecutive slots."""
    cnt = np.asarray(counts, np.int32)
    N, G = cnt.shape
    slots = -np.ones((G, slots_per_gpu), np.int32)
    for g in range(G):
        s = 0
        for e in range(N):
            for _ in range(cnt[e, g]):
                slots[g, s] = e
                s += 1
    return slots


def counts_from_slots(slots, num_experts):
    slots = np.asarray(slots)
    G = slots.shape[0]
    cnt = np.zeros((num_experts, G), np.int32)
    for g in range(G):
        for e in slots[g]:
            if e >= 0:
                cnt[e, g] += 1
    return cnt


def _ops(buf, n):
    return [buf[i].as_tuple() for i in range(n.value)]


def step_cost(D, slots, prof: ClusterProfile):
    D = np.ascontiguousarray(D, np.int64)
    slots = np.ascontiguousarray(slots, np.int32)
    mk = C.c_double()
    per = np.zeros((prof.num_gpus, 3))
    L.check(L.lib().fm_step_cost(D.ctypes.data, slots.ctypes.data, D.shape[0], C.byref(prof),
                                 C.byref(mk), per.ctypes.data))
    return mk.value, per


def make_scheduling_plan(D, slots, prof: ClusterProfile, horizon=50):
    D = np.ascontiguousarray(D, np.int64)
    slots = np.ascontiguousarray(slots, np.int32)
    buf = (PlacementOp * 16)()
    n = C.c_int()
    L.check(L.lib().fm_make_scheduling_plan(D.ctypes.data, slots.ctypes.data, D.shape[0], C.byref(prof),
                                            horizon, buf, 16, C.byref(n)))
    return _ops(buf, n)


def plan_migrations(slots, num_experts, prof: ClusterProfile, horizon=50):
    slots = np.ascontiguousarray(slots, np.int32)
    buf = (PlacementOp * 4)()
    n = C.c_int()
    L.check(L.lib().fm_plan_migrations(slots.ctypes.data, num_experts, C.byref(prof), horizon, buf, 4,
                                       C.byref(n)))
    return _ops(buf, n)


def apply_op(slots, num_experts, prof: ClusterProfile, op):
    """Returns (new slot table, transfers [(src, dst, bytes)])."""
    s = np.ascontiguousarray(slots, np.int32).copy()
    o = PlacementOp(*op)
    t = np.zeros((2, 3))
    n = C.c_int()
    L.check(L.lib().fm_placement_apply(s.ctypes.data, num_experts, C.byref(prof), C.byref(o),
                                       t.ctypes.data, C.byref(n)))
    return s, [(int(a), int(b), float(c)) for a, b, c in t[: n.value]]


@dataclass
class StepResult:
    report: StepReport
    accepted: list
    applied: list


class Scheduler:
    """SimEngine::run_step driver over device-produced demand."""

    def __init__(self, prof: ClusterProfile, num_experts: int, cfg: SchedulerConfig | None = None):
        self.prof, self.N = prof, num_experts
        self.cfg = cfg or SchedulerConfig.defaults()
        h = C.c_void_p()
        L.check(L.lib().fm_scheduler_create(C.byref(prof), C.byref(self.cfg), num_experts, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            L.release("fm_scheduler_destroy", getattr(self, "_h", None))
        except (TypeError, AttributeError):  # interpreter shutdown
            pass
        self._h = None

    def step(self, D) -> StepResult:
        D = np.ascontiguousarray(D, np.int64)
        rep = StepReport()
        L.check(L.lib().fm_scheduler_step(self._h, D.ctypes.data, C.byref(rep)))
        return StepResult(rep, self._ops(0, rep.n_accepted), self._ops(1, rep.n_applied))

    def begin_step(self) -> list:
        """Drain half: returns the ops that became effective at this boundary
        (flip_mode 1: `self.issued` holds the ops whose copies start now)."""
        rep = StepReport()
        L.check(L.lib().fm_scheduler_begin_step(self._h, C.byref(rep)))
        self._begin = rep
        self.issued = self._ops(2, rep.n_issued)
        return self._ops(1, rep.n_applied)

    def join_policy(self) -> list:
        """async_policy: wait for the worker, enqueue its ops, return them."""
        n = C.c_int()
        L.check(L.lib().fm_scheduler_join_policy(self._h, C.byref(n)))
        if n.value == 0:
            return []
        buf = (PlacementOp * 4096)()
        got = C.c_int()
        L.check(L.lib().fm_scheduler_ops(self._h, 0, buf, 4096, C.byref(got)))
        return _ops(buf, got)[-n.value:]

    def finish_step(self, D) -> StepResult:
        D = np.ascontiguousarray(D, np.int64)
        rep = StepReport()
        L.check(L.lib().fm_scheduler_finish_step(self._h, D.ctypes.data, C.byref(rep)))
        return StepResult(rep, self._ops(0, rep.n_accepted), self._ops(1, rep.n_applied))

    def _ops(self, which, n):
        buf = (PlacementOp * max(n, 1))()
        got = C.c_int()
        L.check(L.lib().fm_scheduler_ops(self._h, which, buf, max(n, 1), C.byref(got)))
        return _ops(buf, got)

    def placement(self, which="effective"):
        G, E = self.prof.num_gpus, self.prof.slots_per_gpu
        slots = np.zeros((G, E), np.int32)
        counts = np.zeros((self.N, G), np.int32)
        L.check(L.lib().fm_scheduler_placement(self._h, 0 if which == "effective" else 1,
                                               slots.ctypes.data, counts.ctypes.data))
        return slots, counts

    def reset(self, slots):
        s = np.ascontiguousarray(slots, np.int32)
        L.check(L.lib().fm_scheduler_reset(self._h, s.ctypes.data))


# ---------------------------------------------------------------- baselines
STATIC_EP, FULL_REPLICATE, STRICT_REBALANCE = 0, 1, 2
BASELINES = {"static-ep": STATIC_EP, "full-replicate": FULL_REPLICATE, "strict-rebalance": STRICT_REBALANCE}


class BaselineConfig(C.Structure):
    """BaselineConfig (proj/include/moesim/baselines.hpp) + the SimConfig
    fields a baseline step uses."""

    _fields_ = [("kind", C.c_int), ("capacity_factor", C.c_double), ("replicate_top", C.c_int),
                ("metric", C.c_int), ("max_live_groups", C.c_int), ("group_creation_latency_s", C.c_double)]

    @classmethod
    def make(cls, kind, capacity_factor=1.0, replicate_top=1, metric=0, max_live_groups=64,
             group_creation_latency_s=0.005):
        kind = BASELINES[kind] if isinstance(kind, str) else int(kind)
        return cls(kind, float(capacity_factor), int(replicate_top), int(metric), int(max_live_groups),
                   float(group_creation_latency_s))


class BaselineReport(C.Structure):
    _fields_ = [("balance_ratio", C.c_double), ("metric_value", C.c_double), ("makespan_s", C.c_double),
                ("slot_utilization", C.c_double), ("group_misses", C.c_int), ("tokens_total", C.c_int64),
                ("tokens_dropped", C.c_int64), ("tokens_reassigned", C.c_int64)]


@dataclass
class BaselineStep:
    report: BaselineReport
    counts: np.ndarray   # [N][G] placement the step ran on
    demand: np.ndarray   # [N][G] routed demand (post-drop / rebalanced)
    flows: np.ndarray    # [N][G][G]


class Baseline:
    """run_baseline (baselines.cpp:81-276), one step at a time over
    device-produced demand: StaticEP, FullReplicate, StrictRebalance."""

    def __init__(self, prof: ClusterProfile, num_experts: int, cfg: BaselineConfig):
        self.prof, self.N, self.cfg = prof, num_experts, cfg
        h = C.c_void_p()
        L.check(L.lib().fm_baseline_create(C.byref(prof), C.byref(cfg), num_experts, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            L.release("fm_baseline_destroy", getattr(self, "_h", None))
        except (TypeError, AttributeError):  # interpreter shutdown
            pass
        self._h = None

    def step(self, D) -> BaselineStep:
        D = np.ascontiguousarray(D, np.int64)
        G = self.prof.num_gpus
        rep = BaselineReport()
        counts = np.zeros((self.N, G), np.int32)
        demand = np.zeros((self.N, G), np.int64)
        flows = np.zeros((self.N, G, G), np.int64)
        L.check(L.lib().fm_baseline_step(self._h, D.ctypes.data, C.byref(rep), counts.ctypes.data,
                                         demand.ctypes.data, flows.ctypes.data))
        return BaselineStep(rep, counts, demand, flows)

    def placement(self):
        e = C.c_int()
        L.check(L.lib().fm_baseline_placement(self._h, None, None, C.byref(e)))
        slots = np.zeros((self.prof.num_gpus, e.value), np.int32)
        counts = np.zeros((self.N, self.prof.num_gpus), np.int32)
        L.check(L.lib().fm_baseline_placement(self._h, slots.ctypes.data, counts.ctypes.data, C.byref(e)))
        return slots, counts
