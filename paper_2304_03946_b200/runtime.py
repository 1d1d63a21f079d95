"""FlexMoE runtime: the device step in the loop with the host scheduler.

Per training step on every rank (one process per GPU):
  1. scheduler.begin_step(): adjustments whose (modelled) transfers drained
     become effective (SimEngine::run_step order, sim_engine.cpp:331-336);
     their expert states move peer-to-peer (weights + optimizer state), the
     layer switches placement and re-packs its local experts;
  2. the layer step on the device (DistributedMoELayer): the gate's
     all-gathered histogram is the step's TokenDemand;
  3. optimizer step on the local experts (replicas receive identical summed
     gradients, so they stay bit-identical);
  4. scheduler.finish_step(D): trigger, expand/shrink policy on the target
     placement, migration pass — ops enter the adjustment queue.
Every rank runs the same deterministic scheduler on the same all-gathered
demand, so placements agree without any broadcast.

Expert state moved per transfer = bf16 weights + f32 master weights + Adam
m/v (14 bytes per parameter); the peer copies use the
exchange's P2P path (NCCL send/recv over NVLink with torch.distributed).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import scheduler as S
from .distributed import DistributedMoELayer, Exchange
from .layer import MoELayer

_TENSORS = ("w1", "b1", "w2", "b2")


class ExpertStore:
    """Parameters and Adam state of the experts hosted on this GPU."""

    def __init__(self, d, f, device, lr=1e-4, betas=(0.9, 0.999), eps=1e-8):
        self.d, self.f, self.device = d, f, device
        self.lr, self.betas, self.eps = lr, betas, eps
        self.master: dict[int, dict[str, torch.Tensor]] = {}  # f32
        self.m: dict[int, dict[str, torch.Tensor]] = {}
        self.v: dict[int, dict[str, torch.Tensor]] = {}
        self.t = 0

    @staticmethod
    def init_expert(e, d, f):
        g = torch.Generator(device="cpu").manual_seed(10_000 + e)  # identical on every rank
        return {"w1": torch.randn(f, d, generator=g) * d**-0.5, "b1": torch.randn(f, generator=g) * 0.02,
                "w2": torch.randn(d, f, generator=g) * f**-0.5, "b2": torch.randn(d, generator=g) * 0.02}

    def create(self, e):
        p = self.init_expert(e, self.d, self.f)
        self.master[e] = {k: v.to(self.device) for k, v in p.items()}
        self.m[e] = {k: torch.zeros_like(v) for k, v in self.master[e].items()}
        self.v[e] = {k: torch.zeros_like(v) for k, v in self.master[e].items()}

    def state(self, e) -> list[torch.Tensor]:
        """The tensors that make up expert e's model state, in a fixed order."""
        return [self.master[e][k] for k in _TENSORS] + [self.m[e][k] for k in _TENSORS] + \
               [self.v[e][k] for k in _TENSORS]

    def empty_state(self, e):
        shapes = {"w1": (self.f, self.d), "b1": (self.f,), "w2": (self.d, self.f), "b2": (self.d,)}
        self.master[e] = {k: torch.empty(s, device=self.device) for k, s in shapes.items()}
        self.m[e] = {k: torch.empty(s, device=self.device) for k, s in shapes.items()}
        self.v[e] = {k: torch.empty(s, device=self.device) for k, s in shapes.items()}
        return self.state(e)

    def drop(self, e):
        for d_ in (self.master, self.m, self.v):
            d_.pop(e, None)

    def state_bytes(self, e) -> int:
        return sum(t.numel() * t.element_size() for t in self.state(e)) + \
            sum(self.master[e][k].numel() * 2 for k in ("w1", "w2"))  # + the bf16 working copy

    def pack(self, local):
        """Layer operands for the local experts (ascending id): bf16 weights, f32 biases."""
        if not local:
            z = torch.zeros(1, device=self.device)
            return z.to(torch.bfloat16), z, z.to(torch.bfloat16), z
        st = lambda k: torch.stack([self.master[e][k] for e in local])
        return st("w1").to(torch.bfloat16), st("b1"), st("w2").to(torch.bfloat16), st("b2")

    @torch.no_grad()
    def adam_step(self, local, grads):
        """One Adam step per local expert from the (replica-summed) gradients."""
        self.t += 1
        b1, b2 = self.betas
        c1, c2 = 1 - b1**self.t, 1 - b2**self.t
        for i, e in enumerate(local):
            for k, gk in zip(_TENSORS, (grads.dw1[i], grads.db1[i], grads.dw2[i], grads.db2[i])):
                m, v, w = self.m[e][k], self.v[e][k], self.master[e][k]
                m.mul_(b1).add_(gk, alpha=1 - b1)
                v.mul_(b2).addcmul_(gk, gk, value=1 - b2)
                w.addcdiv_(m / c1, (v / c2).sqrt_().add_(self.eps), value=-self.lr)


@dataclass
class RuntimeStep:
    y: torch.Tensor
    balance_ratio: float
    applied: list
    accepted: list
    migration_bytes: int = 0
    migration_ms: float = 0.0
    replica_counts: np.ndarray = field(default_factory=lambda: np.zeros(0))
    makespan_s: float = 0.0  # modelled step time on the effective placement (Eq. 5)
    adjust_bytes: float = 0.0


class FlexMoERuntime:
    def __init__(self, num_experts, top_k, d_model, d_ff, exchange: Exchange, profile: S.ClusterProfile,
                 sched_cfg: S.SchedulerConfig | None = None, max_tokens=65536, gate_weight=None,
                 lr=1e-4, optimizer=True, recorder=None):
        self.N, self.k, self.d, self.f = num_experts, top_k, d_model, d_ff
        self.recorder = recorder  # trace.TraceRecorder: per-step device TokenDemand export
        self.ex = exchange
        self.rank, self.G = exchange.rank, exchange.world
        self.prof = profile
        self.sched = S.Scheduler(profile, num_experts, sched_cfg)
        self.slots, counts = self.sched.placement("effective")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.layer = MoELayer(num_experts, top_k, d_model, d_ff, replica_counts=counts, num_gpus=self.G,
                              rank=self.rank, max_tokens=max_tokens, slots_per_gpu=profile.slots_per_gpu)
        self.dl = DistributedMoELayer(self.layer, exchange)
        self.store = ExpertStore(d_model, d_ff, dev, lr=lr)
        for e in self.layer.local_experts:
            self.store.create(e)
        if gate_weight is None:
            g = torch.Generator(device="cpu").manual_seed(7)
            gate_weight = torch.randn(num_experts, d_model, generator=g) * d_model**-0.5
        self.wg = gate_weight.to(dev).to(torch.bfloat16)
        self.optimizer = optimizer
        self.packed = self.store.pack(self.layer.local_experts)
        self.history: list[RuntimeStep] = []

    # ------------------------------------------------------------ migrations
    def _moves(self, old_counts, new_counts):
        """(expert, src, dst) state copies: every GPU that newly hosts an expert
        receives it from the lowest-id GPU that hosted it before (a holder of
        the up-to-date state). Identical on every rank, so sends and receives
        pair up without negotiation."""
        moves = []
        for e in range(self.N):
            holders = np.nonzero(old_counts[e] > 0)[0]
            for g in np.nonzero((new_counts[e] > 0) & (old_counts[e] == 0))[0]:
                moves.append((e, int(holders[0]), int(g)))
        return moves

    def _apply(self, ops):
        """Make `ops` effective on this rank: move expert states, re-pack."""
        old_counts = S.counts_from_slots(self.slots, self.N)
        for op in ops:  # Placement::apply in queue order (sim_engine.cpp:256-260)
            self.slots, _ = S.apply_op(self.slots, self.N, self.prof, op)
        counts = S.counts_from_slots(self.slots, self.N)
        new_local = [e for e in range(self.N) if counts[e, self.rank] > 0]
        t0 = time.perf_counter()
        sends, recvs, nbytes = [], [], 0
        for e, src, dst in self._moves(old_counts, counts):
            if src == self.rank:
                sends += [(dst, t) for t in self.store.state(e)]
                nbytes += sum(t.numel() * t.element_size() for t in self.store.state(e))
            if dst == self.rank:
                recvs += [(src, t) for t in self.store.empty_state(e)]
        self.ex.p2p(sends, recvs)
        old_local = set(np.nonzero(old_counts[:, self.rank] > 0)[0].tolist())
        for e in old_local - set(new_local):
            self.store.drop(e)
        self.layer.set_placement(counts)
        self.packed = self.store.pack(new_local)
        torch.cuda.synchronize()
        return nbytes, (time.perf_counter() - t0) * 1e3

    # ------------------------------------------------------------ one step
    def step(self, x, dy) -> RuntimeStep:
        applied = self.sched.begin_step()
        mig_bytes, mig_ms = self._apply(applied) if applied else (0, 0.0)
        w1, b1, w2, b2 = self.packed
        y = self.dl.forward(x, self.wg, w1, b1, w2, b2)
        D = self.dl.last_demand_host  # TokenDemand [N][G], copied when routing synchronised
        if self.recorder is not None:
            self.recorder.record(D)
        grads = self.dl.backward(dy)
        if self.optimizer and self.layer.local_experts:
            self.store.adam_step(self.layer.local_experts, grads)
            self.packed = self.store.pack(self.layer.local_experts)
        res = self.sched.finish_step(D)
        out = RuntimeStep(y=y, balance_ratio=res.report.balance_ratio, applied=applied,
                          accepted=res.accepted, migration_bytes=mig_bytes, migration_ms=mig_ms,
                          replica_counts=S.counts_from_slots(self.slots, self.N).sum(axis=1),
                          makespan_s=res.report.makespan_s, adjust_bytes=res.report.adjust_bytes)
        self.history.append(out)
        return out


class BaselineRuntime:
    """The paper's comparison systems on the device,
    driven by the same gate histogram as FlexMoERuntime
    (proj/src/baselines.cpp:81-161):

    * StaticEP (DeepSpeed-like): round-robin placement, the layer in capacity
      mode drops over-capacity units on the device (the device port of the
      reference's drop rule) — `host.demand` is the reference's kept demand;
    * FullReplicate (FasterMoE-like shadowing): each step, after the demand
      is all-gathered, the hottest `replicate_top` experts are shadowed on
      every GPU: the owner (round-robin home, e % G) sends the bf16 weights +
      f32 biases peer-to-peer, the shadows' gradients are SUM-reduced within
      the replica group, and only the owner keeps optimizer state and steps.

    Every rank runs the same host baseline on the same demand: placements
    agree without a broadcast. `step()` returns the reference's StepReport
    fields (`host`) next to the device outputs."""

    def __init__(self, num_experts, top_k, d_model, d_ff, exchange: Exchange, profile: S.ClusterProfile,
                 cfg: S.BaselineConfig, max_tokens=65536, gate_weight=None, lr=1e-4, optimizer=True):
        if cfg.kind not in (S.STATIC_EP, S.FULL_REPLICATE):
            raise ValueError("BaselineRuntime runs StaticEP or FullReplicate (StrictRebalance rewrites "
                             "the gate's demand: count level only, scheduler.Baseline)")
        self.N, self.k, self.d, self.f = num_experts, top_k, d_model, d_ff
        self.ex, self.rank, self.G = exchange, exchange.rank, exchange.world
        self.cfg = cfg
        self.base = S.Baseline(profile, num_experts, cfg)
        _, counts = self.base.placement()
        self.home = np.arange(num_experts) % self.G  # round-robin owner (placement.cpp:52-68)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        slots = int(np.asarray(counts).sum(axis=0).max()) + (cfg.replicate_top if cfg.kind == S.FULL_REPLICATE else 0)
        self.layer = MoELayer(num_experts, top_k, d_model, d_ff, replica_counts=counts, num_gpus=self.G,
                              rank=self.rank, max_tokens=max_tokens, slots_per_gpu=slots)
        if cfg.kind == S.STATIC_EP:
            self.layer.set_capacity_factor(cfg.capacity_factor)
        self.dl = DistributedMoELayer(self.layer, exchange)
        self.store = ExpertStore(d_model, d_ff, dev, lr=lr)
        self.owned = [e for e in range(num_experts) if self.home[e] == self.rank]
        for e in self.owned:
            self.store.create(e)
        if gate_weight is None:
            g = torch.Generator(device="cpu").manual_seed(7)
            gate_weight = torch.randn(num_experts, d_model, generator=g) * d_model**-0.5
        self.wg = gate_weight.to(dev).to(torch.bfloat16)
        self.optimizer = optimizer
        self.history: list = []

    def _params(self, e):
        m = self.store.master[e]
        return [m["w1"].to(torch.bfloat16), m["b1"], m["w2"].to(torch.bfloat16), m["b2"]]

    def _shadow(self, counts):
        """Switch to this step's placement; owners send the shadows' weights."""
        self.layer.set_placement(counts)
        local = self.layer.local_experts
        sends, recvs, got, nbytes = [], [], {}, 0
        for e in range(self.N):  # ascending expert id on every rank: P2P pairs match in order
            h = int(self.home[e])
            for g in np.nonzero(counts[e] > 0)[0].tolist():
                if g == h:
                    continue
                if h == self.rank:
                    ts = self._params(e)
                    sends += [(g, t) for t in ts]
                    nbytes += sum(t.numel() * t.element_size() for t in ts)
                if g == self.rank:
                    got[e] = [torch.empty(self.f, self.d, dtype=torch.bfloat16, device=self.device),
                              torch.empty(self.f, device=self.device),
                              torch.empty(self.d, self.f, dtype=torch.bfloat16, device=self.device),
                              torch.empty(self.d, device=self.device)]
                    recvs += [(h, t) for t in got[e]]
        self.ex.p2p(sends, recvs)
        if not local:
            z = torch.zeros(1, device=self.device)
            return (z.to(torch.bfloat16), z, z.to(torch.bfloat16), z), nbytes
        ps = [got[e] if e in got else self._params(e) for e in local]
        return tuple(torch.stack([p[i] for p in ps]) for i in range(4)), nbytes

    def step(self, x, dy):
        info = {}

        def on_demand(D):
            res = self.base.step(D)
            info["host"], info["D"] = res, D
            if self.cfg.kind == S.FULL_REPLICATE:
                ops, info["shadow_bytes"] = self._shadow(res.counts)
                return ops
            return None

        packed = self.store.pack(self.owned) if self.cfg.kind == S.STATIC_EP else (None,) * 4
        y = self.dl.forward(x, self.wg, *packed, on_demand=on_demand)
        grads = self.dl.backward(dy)  # SUM over each replica group (shadows included)
        local = self.layer.local_experts
        if self.optimizer and self.owned:
            idx = torch.tensor([local.index(e) for e in self.owned], device=self.device)
            from .layer import LayerGrads
            sub = LayerGrads(dx=grads.dx, dwg=grads.dwg, dw1=grads.dw1[idx], db1=grads.db1[idx],
                             dw2=grads.dw2[idx], db2=grads.db2[idx])
            self.store.adam_step(self.owned, sub)
        out = dict(y=y, grads=grads, host=info["host"], demand=info["D"],
                   shadow_bytes=info.get("shadow_bytes", 0), local=list(local))
        self.history.append(out)
        return out
