"""FlexMoE runtime: the device step in the loop with the host scheduler.

Per training step on every rank (one process per GPU):
  1. scheduler.begin_step(): the placement boundary. Two flip modes
     (fm_scheduler_config.flip_mode, include/flexmoe_b200.h):
     * "modelled" (the reference, SimEngine::run_step, sim_engine.cpp:331-336):
       ops whose MODELLED bytes drained become effective; their expert states
       are pulled peer-to-peer during this step and the expert FFN waits for
       them (they compute this step);
     * "copy" (the device mode): the ops issued at the previous boundary
       become effective — their state copies ran during that step — and the
       next queue prefix is issued: receivers pull the state now, join the
       expert's replica group with zero rows routed to them (zero gradients),
       wait for the copy only before the group all-reduce and apply the same
       Adam update as the other replicas, so the new replica is up to date when
       it takes tokens at the next boundary. Nothing waits on the copy before
       the all-reduce, and nothing synchronises the host;
     the layer switches placement with one async table upload (no allocation,
     no weight movement: the operands stay in their pool slots);
  2. the layer step on the device (DistributedMoELayer): the gate's
     all-gathered histogram is the step's TokenDemand;
  3. optimizer step on the hosted experts (replicas receive identical summed
     gradients, so they stay bit-identical);
  4. scheduler.finish_step(D): trigger, expand/shrink policy on the target
     placement, migration pass — inline, or (async_policy) on the scheduler's
     worker thread while the host enqueues the next step; those ops then enter
     the queue at the next finish_step.
Every rank runs the same deterministic scheduler on the same all-gathered
demand, so placements agree without any broadcast.

Expert state lives in a per-GPU ExpertPool (pool.py, csrc/expert_pool.cu):
f32 master weights + Adam m/v, 12 bytes per parameter (the bf16 working copy
is re-derived from the master, so the 14 B/param of SURVEY.md §8d shrink to
12), and the GEMM operands sit at the expert's pool slot. A transfer is a
peer-to-peer cudaMemcpyAsync of one slot, pulled by the receiving GPU on the
pool's side stream (CUDA IPC mapping of the source's pool), issued once the
step's demand all-gather is enqueued.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import scheduler as S
from .distributed import DistributedMoELayer, Exchange
from .layer import MoELayer
from .pool import ExpertStore, SlotAllocator, apply_placement_change

FLIP_MODES = {"modelled": 0, "copy": 1}


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
    issued: list = field(default_factory=list)  # flip "copy": ops whose copies started this step


class FlexMoERuntime:
    def __init__(self, num_experts, top_k, d_model, d_ff, exchange: Exchange, profile: S.ClusterProfile,
                 sched_cfg: S.SchedulerConfig | None = None, max_tokens=65536, gate_weight=None,
                 lr=1e-4, optimizer=True, recorder=None, transport="p2p", flip="modelled", async_policy=False):
        self.N, self.k, self.d, self.f = num_experts, top_k, d_model, d_ff
        self.recorder = recorder  # trace.TraceRecorder: per-step device TokenDemand export
        self.ex = exchange
        self.rank, self.G = exchange.rank, exchange.world
        self.prof = profile
        if flip not in FLIP_MODES:
            raise ValueError(f"flip must be one of {sorted(FLIP_MODES)}")
        self.flip = flip
        cfg = S.SchedulerConfig.defaults() if sched_cfg is None else S.SchedulerConfig.from_buffer_copy(sched_cfg)
        cfg.flip_mode = FLIP_MODES[flip]
        cfg.async_policy = 1 if async_policy else 0
        self.sched = S.Scheduler(profile, num_experts, cfg)
        self.slots, counts = self.sched.placement("effective")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.layer = MoELayer(num_experts, top_k, d_model, d_ff, replica_counts=counts, num_gpus=self.G,
                              rank=self.rank, max_tokens=max_tokens, slots_per_gpu=profile.slots_per_gpu)
        self.dl = DistributedMoELayer(self.layer, exchange, transport=transport, reuse_grads=True)
        # every rank tracks every rank's slot table (same ops, same order): a
        # receiver knows the source's slot without a round trip. A GPU hosts at
        # most E experts plus, in flight, the receivers of one issued batch;
        # vacated slots stay readable for one step -> 3E slots.
        E = profile.slots_per_gpu
        cap = 3 * E
        self.slot_dir = [SlotAllocator(cap) for _ in range(self.G)]
        self.store = ExpertStore(d_model, d_ff, dev, capacity=cap, world=self.G, lr=lr,
                                 allocator=self.slot_dir[self.rank], by_slot=True)
        self.hosted = counts > 0  # [N][G] GPUs holding each expert's state
        for g in range(self.G):
            for e in range(num_experts):
                if self.hosted[e, g]:
                    self.slot_dir[g].host(e)
        for e in self.layer.local_experts:
            self.store.create(e)
        exchange.share_pool(self.store.pool)
        if gate_weight is None:
            g = torch.Generator(device="cpu").manual_seed(7)
            gate_weight = torch.randn(num_experts, d_model, generator=g) * d_model**-0.5
        self.wg = gate_weight.to(dev).to(torch.bfloat16)
        self.optimizer = optimizer
        self.packed = self.store.pack(self.layer.local_experts)  # operands at their pool slots
        self.layer.set_operand_slots(self.store.slot_table(num_experts), cap)
        self.dl.group_counts = self.hosted.astype(np.int32)
        self.history: list[RuntimeStep] = []

    # ------------------------------------------------------------ migrations
    def _switch(self, applied, issued):
        """The placement boundary on this rank: `applied` ops become effective
        (routing placement), the receivers of `issued` ops start hosting
        state. Updates every rank's slot table and the layer's tables (async,
        on the current stream). Returns (bytes this GPU pulls, a callable that
        enqueues the pulls on the pool's side stream).

        The pulls are issued after the step's demand all-gather: a source GPU
        joins that collective only after its previous step's optimizer update,
        so the pulled state is the one the source starts this step with. The
        source's next update comes after this step's replica-group
        all-reduce, which the receiver joins only after waiting for the pull
        (modelled: before its expert FFN; copy: before the all-reduce)."""
        for op in applied:  # Placement::apply in queue order (sim_engine.cpp:256-260)
            self.slots, _ = S.apply_op(self.slots, self.N, self.prof, op)
        counts = S.counts_from_slots(self.slots, self.N)
        hosted = counts > 0
        if issued:
            pend = self.slots
            for op in issued:
                pend, _ = S.apply_op(pend, self.N, self.prof, op)
            hosted = hosted | (S.counts_from_slots(pend, self.N) > 0)
        changes = apply_placement_change(self.slot_dir, self.hosted, hosted)
        self.hosted = hosted
        pulls = [(ds, src, ss) for _, src, ss, dst, ds in changes if dst == self.rank]
        self.layer.set_placement_async(counts, hosted=hosted[:, self.rank])
        self.layer.set_operand_slots(self.store.slot_table(self.N), self.store.pool.slots)
        self.dl.group_counts = hosted.astype(np.int32)
        pulled = [ds for ds, _, _ in pulls]

        def issue():
            self.store.pool.migrate(pulls, pulled, self.packed)  # re-packs only the pulled slots

        return len(pulls) * self.store.pool.state_bytes, issue

    def migration_stats(self) -> dict:
        """Side-stream copy time, bytes and slots pulled by this GPU so far."""
        ms, nbytes, copies = self.store.pool.migration_stats()
        return {"copy_ms": ms, "bytes": nbytes, "copies": copies}

    # ------------------------------------------------------------ one step
    def step(self, x, dy) -> RuntimeStep:
        t0 = time.perf_counter()
        applied = self.sched.begin_step()
        issued = self.sched.issued if self.flip == "copy" else []
        mig_bytes, issue = self._switch(applied, issued) if (applied or issued) else (0, None)
        self.last_switch_us = (time.perf_counter() - t0) * 1e6  # host time of the placement boundary
        wait = lambda: self.store.pool.wait_ready()  # noqa: E731
        copy = self.flip == "copy"
        y = self.dl.forward(x, self.wg, *self.packed, after_gather=issue,
                            before_experts=None if copy else wait)
        grads = self.dl.backward(dy, before_sync=wait if copy else None)
        D = self.dl.last_demand_host  # TokenDemand [N][G] (its host copy overlapped the step)
        if self.recorder is not None:
            self.recorder.record(D)
        local = self.layer.local_experts
        if self.optimizer:
            self.store.tick()  # every rank, with or without local experts (same Adam step count everywhere)
            if local:
                self.store.adam_step(local, grads)  # refreshes the operands at their slots
        t0 = time.perf_counter()
        res = self.sched.finish_step(D)
        self.last_finish_us = (time.perf_counter() - t0) * 1e6  # host time of the policy half (inline or join)
        out = RuntimeStep(y=y, balance_ratio=res.report.balance_ratio, applied=applied,
                          accepted=res.accepted, migration_bytes=mig_bytes,
                          replica_counts=S.counts_from_slots(self.slots, self.N).sum(axis=1),
                          makespan_s=res.report.makespan_s, adjust_bytes=res.report.adjust_bytes,
                          issued=list(issued))
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
