"""Weight-gradient GEMM (FM_GEMM_WGRAD) alone on three row distributions, to
locate its DRAM re-reads (run under ncu with dram__bytes_read.sum):

  cfg1      the configs[1] expert loads of the bench (Zipf 1.25, 16 experts, 131,072 units)
  balanced  16 x 8,192 rows
  one       1 x 131,072 rows

For each: both wgrad shapes of the step (dW2: M_w = d = 1024, N = f = 4096;
dW1: M_w = f = 4096, N = d = 1024), median of 10 event-timed launches, and the
algorithmic operand bytes (rows x (M_w + N) x 2). Usage: python profiles/wgrad_traffic.py [dist ...]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2304_03946_b200 import _lib as L  # noqa: E402

d, f = 1024, 4096


def cfg1_rows():
    import bench

    arm = bench.FusedArm(bench.CFG2, torch.device("cuda", 0), 0)
    _, x_h, dy_h, _ = bench.bench_inputs(bench.CFG2)
    arm.step(x_h.cuda(), dy_h.cuda())
    torch.cuda.synchronize()
    rows = [int(v) for v in arm.hist()]
    del arm
    return rows


DISTS = {"balanced": lambda: [8192] * 16, "one": lambda: [131072], "cfg1": cfg1_rows,
         "two": lambda: [65536] * 2, "four": lambda: [32768] * 4, "eight": lambda: [16384] * 8}
names = sys.argv[1:] or ["cfg1", "balanced", "one"]
shapes = [(d, f), (f, d)]
if names and names[0] in ("dW2", "dW1"):
    shapes = [(d, f)] if names[0] == "dW2" else [(f, d)]
    names = names[1:]
for name in names:
    rows = DISTS[name]()
    pad = [((r + 127) // 128) * 128 for r in rows]
    start = [0]
    for p in pad[:-1]:
        start.append(start[-1] + p)
    total = sum(pad)
    st = torch.tensor(start, dtype=torch.int32, device="cuda")
    pr = torch.tensor(pad, dtype=torch.int32, device="cuda")
    G = len(rows)
    for Mw, N in shapes:
        A = torch.randn(total, Mw, device="cuda").to(torch.bfloat16)
        B = torch.randn(total, N, device="cuda").to(torch.bfloat16)
        C = torch.empty(G, Mw, N, device="cuda", dtype=torch.float32)
        run = lambda: L.call("fm_grouped_gemm", L.FM_GEMM_WGRAD, L.ptr(A), L.ptr(B), L.ptr(C), None, None,
                             L.ptr(st), L.ptr(pr), None, G, total, Mw, N, 0, L.stream_ptr())
        for _ in range(2):
            run()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ops = total * (Mw + N) * 2 / 1e6
        flop = 2.0 * total * Mw * N
        us = statistics.median(ts)
        print(f"{name:8s} groups={G:3d} max_rows={max(rows):6d} M_w={Mw} N={N}: {us:7.1f} us "
              f"{flop / us / 1e6:6.0f} TFLOP/s, operands {ops:6.0f} MB, out {G * Mw * N * 4 / 1e6:5.0f} MB")
        del A, B, C
