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

Expert state lives in a per-GPU ExpertPool (pool.py, csrc/expert_pool.cu):
f32 master weights + Adam m/v, 12 bytes per parameter (the bf16 working copy
is re-derived on arrival, so the 14 B/param of SURVEY.md §8d shrink to 12).
A transfer is a peer-to-peer cudaMemcpyAsync of one slot, pulled by the
receiving GPU on the pool's side stream (CUDA IPC mapping of the source's
pool), issued once the step's demand all-gather is enqueued; the compute
stream waits for it only before the expert FFN, so the copy overlaps routing
and the dispatch all-to-all.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import scheduler as S
from .distributed import DistributedMoELayer, Exchange
from .layer import MoELayer
from .pool import ExpertStore, SlotAllocator, apply_placement_change

@dataclass
class RuntimeStep:
    y: torch.Tensor | None  # None in `history` (entries keep no device tensors)
    balance_ratio: float
    applied: list
    accepted: list
    migration_bytes: int = 0  # expert state pulled by this GPU this step (copies run async)
    replica_counts: np.ndarray = field(default_factory=lambda: np.zeros(0))
    makespan_s: float = 0.0  # modelled step time on the effective placement (Eq. 5)
    adjust_bytes: float = 0.0


class FlexMoERuntime:
    def __init__(self, num_experts, top_k, d_model, d_ff, exchange: Exchange, profile: S.ClusterProfile,
                 sched_cfg: S.SchedulerConfig | None = None, max_tokens=65536, gate_weight=None,
                 lr=1e-4, optimizer=True, recorder=None, transport="p2p"):
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
        self.dl = DistributedMoELayer(self.layer, exchange, transport=transport, reuse_grads=True)
        # every rank tracks every rank's slot table (same ops, same order): a
        # receiver knows the source's slot without a round trip. A GPU hosts at
        # most E experts; vacated slots stay readable for one step -> 2E slots.
        E = profile.slots_per_gpu
        self.slot_dir = [SlotAllocator(2 * E) for _ in range(self.G)]
        self.store = ExpertStore(d_model, d_ff, dev, capacity=2 * E, world=self.G, max_local=E, lr=lr,
                                 allocator=self.slot_dir[self.rank])
        for g in range(self.G):
            for e in range(num_experts):
                if counts[e, g] > 0:
                    self.slot_dir[g].host(e)
        for e in self.layer.local_experts:
            self.store.create(e)
        exchange.share_pool(self.store.pool)
        if gate_weight is None:
            g = torch.Generator(device="cpu").manual_seed(7)
            gate_weight = torch.randn(num_experts, d_model, generator=g) * d_model**-0.5
        self.wg = gate_weight.to(dev).to(torch.bfloat16)
        self.optimizer = optimizer
        self.packed = self.store.pack(self.layer.local_experts)
        self.history: list[RuntimeStep] = []

    # ------------------------------------------------------------ migrations
    def _apply(self, ops):
        """Make `ops` effective on this rank: update every rank's slot table and
        the layer's placement. Returns (bytes this GPU pulls, a callable that
        enqueues the pulls of the states it newly hosts and the operand
        re-pack on the pool's side stream).

        The pulls are issued after the step's demand all-gather: a source GPU
        joins that collective only after its previous step's optimizer update,
        so the pulled state is the one the source starts this step with. The
        source's next update comes after this step's gradient all-reduces,
        which the receiver joins only after its expert FFN waited for the pull."""
        old_counts = S.counts_from_slots(self.slots, self.N)
        for op in ops:  # Placement::apply in queue order (sim_engine.cpp:256-260)
            self.slots, _ = S.apply_op(self.slots, self.N, self.prof, op)
        counts = S.counts_from_slots(self.slots, self.N)
        pulls = [(ds, src, ss) for _, src, ss, dst, ds in apply_placement_change(self.slot_dir, old_counts, counts)
                 if dst == self.rank]
        new_local = [e for e in range(self.N) if counts[e, self.rank] > 0]
        self.layer.set_placement(counts)
        self.packed = self.store.packed(max(1, len(new_local)))
        local_slots = self.store.slots(new_local)

        def issue():
            self.store.pool.migrate(pulls, local_slots, self.store.packed(max(1, len(new_local))))

        return len(pulls) * self.store.pool.state_bytes, issue

    def migration_stats(self) -> dict:
        """Side-stream copy time, bytes and slots pulled by this GPU so far."""
        ms, nbytes, copies = self.store.pool.migration_stats()
        return {"copy_ms": ms, "bytes": nbytes, "copies": copies}

    # ------------------------------------------------------------ one step
    def step(self, x, dy) -> RuntimeStep:
        applied = self.sched.begin_step()
        mig_bytes, issue = self._apply(applied) if applied else (0, None)
        w1, b1, w2, b2 = self.packed
        y = self.dl.forward(x, self.wg, w1, b1, w2, b2, after_gather=issue,
                            before_experts=lambda: self.store.pool.wait_ready())
        grads = self.dl.backward(dy)
        D = self.dl.last_demand_host  # TokenDemand [N][G] (its host copy overlapped the step)
        if self.recorder is not None:
            self.recorder.record(D)
        if self.optimizer:
            self.store.tick()  # every rank, with or without local experts (same Adam step count everywhere)
            if self.layer.local_experts:
                self.store.adam_step(self.layer.local_experts, grads)  # refreshes self.packed in place
        res = self.sched.finish_step(D)
        out = RuntimeStep(y=y, balance_ratio=res.report.balance_ratio, applied=applied,
                          accepted=res.accepted, migration_bytes=mig_bytes,
                          replica_counts=S.counts_from_slots(self.slots, self.N).sum(axis=1),
                          makespan_s=res.report.makespan_s, adjust_bytes=res.report.adjust_bytes)
        self.history.append(replace(out, y=None))  # no device tensors kept past the step
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
                 cfg: S.BaselineConfig, max_tokens=65536, gate_weight=None, lr=1e-4, optimizer=True,
                 transport="p2p"):
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
        self.dl = DistributedMoELayer(self.layer, exchange, transport=transport, reuse_grads=True)
        self.owned = [e for e in range(num_experts) if self.home[e] == self.rank]
        self.store = ExpertStore(d_model, d_ff, dev, capacity=max(1, len(self.owned)), lr=lr)
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
        if self.optimizer:
            self.store.tick()
        if self.optimizer and self.owned:
            idx = torch.tensor([local.index(e) for e in self.owned], device=self.device)
            from .layer import LayerGrads
            sub = LayerGrads(dx=grads.dx, dwg=grads.dwg, dw1=grads.dw1[idx], db1=grads.db1[idx],
                             dw2=grads.dw2[idx], db2=grads.db2[idx])
            self.store.adam_step(self.owned, sub)
        out = dict(y=y, grads=grads, host=info["host"], demand=info["D"],
                   shadow_bytes=info.get("shadow_bytes", 0), local=list(local))
        self.history.append({kk: v for kk, v in out.items() if kk not in ("y", "grads")})
        return out
