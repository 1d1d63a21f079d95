"""FlexMoE's dynamic placement measured on the device (one B200, G virtual ranks).

    python profiles/dynamic_loopback.py [--steps S] [--out profiles/r01_dynamic_loopback.json]

G ranks run as threads sharing one B200 with the in-process loopback exchange
(distributed.LoopbackHub): every rank's REAL gate produces its TokenDemand
column from drifting Zipf traffic (workload.cpp:164-170 walk, applied
through the gate's skew column), the all-gathered demand feeds the C++ host
scheduler (expand / shrink / migrate, B200 cluster profile), accepted ops
drain through the adjustment queue, and when they become effective the
expert state (f32 master + Adam m/v) is pulled peer to peer from the source
rank's pool (side-stream cudaMemcpyAsync; linked pools in one process).
The same traffic also runs with the placement frozen (policy "static") for
comparison. Recorded per step: the balance ratio of the routed load (Eq. 7,
from the device flows), applied ops, bytes pulled, replica counts.

Token-exchange and step TIMES are not meaningful here (all ranks share one
GPU and the host loopback copies); the load balance, the decisions and the
migration traffic are.
"""
from __future__ import annotations

import argparse
import json
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2304_03946_b200 import scheduler as S  # noqa: E402
from paper_2304_03946_b200.distributed import LoopbackHub  # noqa: E402
from paper_2304_03946_b200.profile import b200_profile  # noqa: E402
from paper_2304_03946_b200.runtime import BaselineRuntime, FlexMoERuntime  # noqa: E402


def zipf_logp(N, s, seed):
    rng = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, N + 1) ** s
    return np.log(p / p.sum())[rng.permutation(N)]


def run(mode, N, k, d, f, T, G, steps, zipf, transport):
    """mode: "static" / "dynamic" (FlexMoERuntime; policy frozen or FlexMoE's),
    "static-ep" (DeepSpeed-like capacity 1.0, drops), "full-replicate"
    (FasterMoE-like shadowing of the hottest expert) — BaselineRuntime."""
    hub = LoopbackHub(G)
    E = 2 * -(-N // G)
    prof = b200_profile(G, E, tps=2.0e7, d=d, f=f)
    baseline = mode in ("static-ep", "full-replicate")
    cfg = S.SchedulerConfig.defaults(policy_mode={"dynamic": 0, "dynamic-copy": 0, "static": 2}.get(mode, 2))
    g = torch.Generator(device="cpu").manual_seed(1234)
    wg0 = torch.randn(N, d, generator=g) * d**-0.5
    logp0 = zipf_logp(N, zipf, 42)
    xs = [torch.randn(T, d, generator=g).to(torch.bfloat16) for _ in range(G)]
    for x in xs:
        x[:, 0] = 0.5
    dys = [(torch.randn(T, d, generator=g) * 0.1).to(torch.bfloat16) for _ in range(G)]
    rec = [None] * G
    errs = [None] * G

    def rank_fn(r):
        try:
            torch.cuda.set_device(0)
            if baseline:
                rt = BaselineRuntime(N, k, d, f, hub.endpoint(r), prof,
                                     S.BaselineConfig.make(mode, capacity_factor=1.0, replicate_top=1),
                                     max_tokens=T, gate_weight=wg0.clone(), lr=1e-4, transport=transport)
            else:
                copy = mode == "dynamic-copy"  # flips on completed copies, policy on the worker thread
                rt = FlexMoERuntime(N, k, d, f, hub.endpoint(r), prof, sched_cfg=cfg, max_tokens=T,
                                    gate_weight=wg0.clone(), lr=1e-4, transport=transport,
                                    flip="copy" if copy else "modelled", async_policy=copy)
            x, dy = xs[r].cuda(), dys[r].cuda()
            walk = np.random.default_rng(42)  # the same drift on every rank
            logp = logp0.copy()
            out = []
            for s in range(steps):
                logp = logp + walk.uniform(-0.02, 0.02, N)
                logp -= np.log(np.exp(logp).sum())
                rt.wg[:, 0] = torch.tensor(logp * 2, dtype=torch.float32).to(rt.wg)
                st = rt.step(x, dy)
                flows = rt.layer.read("flows", N * G * G).reshape(N, G, G)
                recv = flows.sum(axis=1).sum(axis=0)  # per-GPU received units
                if baseline:
                    rep = st["host"].report
                    out.append({"step": s, "balance_ratio": float(recv.max() / recv.mean()),
                                "tokens_dropped": int(rep.tokens_dropped), "tokens_total": int(rep.tokens_total),
                                "applied": [], "shadow_bytes": int(st["shadow_bytes"])})
                    continue
                out.append({"step": s, "balance_ratio": float(recv.max() / recv.mean()),
                            "scheduler_ratio": st.balance_ratio, "applied": [list(o) for o in st.applied],
                            "pulled_bytes": int(st.migration_bytes), "issued": [list(o) for o in st.issued],
                            "switch_host_us": rt.last_switch_us, "finish_host_us": rt.last_finish_us,
                            "replicas": [int(c) for c in st.replica_counts]})
            torch.cuda.synchronize()
            mig = {"bytes": 0, "copy_ms": 0.0, "copies": 0} if baseline else rt.migration_stats()
            rec[r] = {"steps": out, "migration": mig}
        except BaseException as exc:
            errs[r] = exc

    th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(G)]
    t0 = time.time()
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    steps0 = rec[0]["steps"]
    ratios = [s["balance_ratio"] for s in steps0]
    tail = ratios[len(ratios) // 2:]
    return {
        "mode": mode,
        "wall_s": round(time.time() - t0, 1),
        "balance_ratio_first": ratios[0],
        "balance_ratio_tail_mean": float(np.mean(tail)),
        "balance_ratio_tail_max": float(np.max(tail)),
        "ops_applied": sum(len(s["applied"]) for s in steps0),
        "switch_host_us_max": max((s.get("switch_host_us", 0.0) for s in steps0), default=0.0),
        "finish_host_us_mean": float(np.mean([s.get("finish_host_us", 0.0) for s in steps0])),
        "expert_state_pulled_bytes": sum(rec[r]["migration"]["bytes"] for r in range(G)),
        "expert_state_copy_ms": sum(rec[r]["migration"]["copy_ms"] for r in range(G)),
        "slots_pulled": sum(rec[r]["migration"]["copies"] for r in range(G)),
        "tokens_dropped_fraction": (sum(s.get("tokens_dropped", 0) for s in steps0) /
                                    max(1, sum(s.get("tokens_total", 0) for s in steps0))) if baseline else 0.0,
        "shadow_bytes_per_step_per_rank": (float(np.mean([np.mean([s.get("shadow_bytes", 0) for s in rec[r]["steps"]])
                                                          for r in range(G)])) if baseline else 0.0),
        "decisions_identical_on_all_ranks": all(
            [s["applied"] for s in rec[r]["steps"]] == [s["applied"] for s in steps0] for r in range(G)),
        "per_step": steps0,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=120)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_dynamic_loopback.json"))
    ap.add_argument("--modes", default="static,static-ep,full-replicate,dynamic,dynamic-copy")
    ap.add_argument("--shape", default="32,2,768,3072,8192,4,1.25", help="N,k,d,f,T,G,zipf")
    a = ap.parse_args()
    # default: BERT-MoE-like layer (configs[3] dims) at 4 virtual GPUs, 8K tokens per GPU
    N, k, d, f, T, G, zipf = (t(v) for t, v in zip((int,) * 6 + (float,), a.shape.split(",")))
    res = {"what": __doc__.strip().splitlines()[0],
           "workload": {"experts": N, "top_k": k, "d_model": d, "d_ff": f, "tokens_per_gpu": T, "gpus_virtual": G,
                        "zipf": zipf, "drift": "p *= exp(U[-0.02, 0.02]) per step (workload.cpp:164-170)",
                        "transport": "p2p", "steps": a.steps},
           "runs": [run(m, N, k, d, f, T, G, a.steps, zipf, "p2p")
                    for m in a.modes.split(",")]}
    Path(a.out).write_text(json.dumps(res, indent=1))
    for r in res["runs"]:
        print(json.dumps({kk: v for kk, v in r.items() if kk != "per_step"}))


if __name__ == "__main__":
    main()
