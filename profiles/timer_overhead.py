"""Cost of the per-phase CUDA-event timer on the configs[1] step: the same
fused step timed with the layer's phase events on and off, interleaved."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
arm = bench.FusedArm(bench.CFG2, dev, 0)
_, x_h, dy_h, _ = bench.bench_inputs(bench.CFG2)
x, dy = x_h.to(dev), dy_h.to(dev)
for _ in range(5):
    arm.step(x, dy)
torch.cuda.synchronize()
res = {True: [], False: []}
for rep in range(6):
    for on in (True, False):
        arm.set_timing(on)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(30):
            arm.step(x, dy)
        e1.record()
        torch.cuda.synchronize()
        res[on].append(e0.elapsed_time(e1) / 30)
        arm.timing() if on else None
        arm.set_timing(False)
for on in (True, False):
    print(f"timer {'on ' if on else 'off'}: ms/step median {statistics.median(res[on]):.4f}  all {[round(v, 3) for v in res[on]]}")
