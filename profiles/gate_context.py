"""What the gate pays for its predecessor: the configs[1] gate kernel timed
with adjacent CUDA events (the bench's in-step method) after different
predecessors on the stream:

  read     a 256 MiB read (L2 left clean)
  write    a 256 MiB memset (L2 left full of dirty lines)
  bwd      the layer's own backward (the bench's real predecessor)
  bwd+read the backward, then a 256 MiB read (its dirty lines written back
           before the gate starts)

Usage: python profiles/gate_context.py [N]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_03946_b200 import _lib as L  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = dict(bench.CFG2, N=N)
dev = torch.device("cuda", 0)
arm = bench.FusedArm(cfg, dev, 0)
_, x_h, dy_h, _ = bench.bench_inputs(cfg)
x, dy = x_h.to(dev), dy_h.to(dev)
lay = arm.layer
flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
acc = torch.empty((), device=dev)
hist = torch.empty(N, dtype=torch.int64, device=dev)
wg = arm.P[0]
for _ in range(3):
    arm.step(x, dy)
torch.cuda.synchronize()


def gate():
    L.call("fm_layer_gate", lay._h, L.ptr(x), x.shape[0], L.ptr(wg), L.ptr(hist), L.stream_ptr())


def run(pred, reps=20):
    gs = []
    for _ in range(reps):
        arm.step(x, dy) if "bwd" in pred else None  # leaves the backward as the last work
        if pred in ("read", "bwd+read"):
            torch.sum(flush, dim=0, out=acc)
        elif pred == "write":
            flush.fill_(1.0)
        torch.cuda._sleep(200_000)
        lay.set_timing(True)
        gate()
        ph = lay.read_timing()
        lay.set_timing(False)
        gs.append(ph["gate"][0] * 1e3)
    return statistics.median(gs)


for pred in ("read", "write", "bwd", "bwd+read"):
    us = run(pred)
    mb = (x.numel() * 2 + N * 1024 * 2 + x.shape[0] * cfg["k"] * 12) / 1e6
    print(f"N={N} gate after {pred:9s}: {us:6.1f} us  ({mb / us * 1e3:5.0f} GB/s, "
          f"{mb / us * 1e3 / bench.measured_peaks()['hbm']:.3f} of HBM)")
