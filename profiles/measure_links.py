"""Measures the two cluster-profile numbers the cost model borrows on a
single-GPU box (paper_2304_03946_b200/profile.py LINK_BPS / ALLREDUCE_BUS_BPS;
ClusterTopology's intra_node_bandwidth_bps and allreduce_bps table,
proj/src/topology.cpp:64-128):

* p2p_bps: peer-to-peer copy bandwidth between two GPUs (one direction,
  cudaMemcpyPeerAsync of 256 MiB through torch, CUDA events, best of 10) —
  what an expert-state pull moves at (fm_pool_migrate);
* allreduce_bus_bps_by_group: NCCL all-reduce bus bandwidth (algorithm
  bandwidth x 2(n-1)/n) of a 256 MiB f32 buffer for every group size 2..G —
  what a replica-group gradient sum moves at.

    python profiles/measure_links.py --out profiles/links_b200.json
    python -m paper_2304_03946_b200.profile --config cfg3 --links profiles/links_b200.json ...

With fewer than 2 GPUs it writes {"skipped": ...} and exits 0.
"""
from __future__ import annotations

import argparse
import json
import os

import torch

MIB = 1 << 20


def p2p_bps(a=0, b=1, nbytes=256 * MIB, reps=10):
    src = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a}")
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{b}")
    best = 0.0
    with torch.cuda.device(a):
        for _ in range(reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize(a)
            torch.cuda.synchronize(b)
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3))
    return best


def _allreduce_worker(rank, world, nbytes, reps, out):
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29631")
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    res = {}
    t = torch.ones(nbytes // 4, device="cuda")
    for n in range(2, world + 1):
        grp = dist.new_group(list(range(n)))
        if rank < n:
            for _ in range(3):
                dist.all_reduce(t, group=grp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                dist.all_reduce(t, group=grp)
            e1.record()
            torch.cuda.synchronize()
            sec = e0.elapsed_time(e1) * 1e-3 / reps
            res[str(n)] = nbytes / sec * 2 * (n - 1) / n
        dist.barrier()
    if rank == 0:
        out.update(res)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/links_b200.json")
    ap.add_argument("--mib", type=int, default=256)
    a = ap.parse_args()
    G = torch.cuda.device_count()
    if G < 2:
        res = {"skipped": f"{G} GPU visible: peer-to-peer and all-reduce bandwidth need >= 2 GPUs"}
    else:
        import torch.multiprocessing as mp

        pairs = {f"{i}->{j}": p2p_bps(i, j, a.mib * MIB) for i in range(min(G, 2)) for j in range(G) if i != j}
        mgr = mp.Manager()
        out = mgr.dict()
        mp.spawn(_allreduce_worker, args=(G, a.mib * MIB, 10, out), nprocs=G, join=True)
        res = {"gpus": G, "p2p_bps_pairs": pairs, "p2p_bps": min(pairs.values()),
               "allreduce_bus_bps_by_group": dict(out),
               "how": "p2p: dst.copy_(src) 256 MiB across devices, best of 10; all-reduce: NCCL SUM of a 256 MiB "
                      "f32 buffer, 10 back to back, bus bandwidth = bytes/s x 2(n-1)/n"}
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
