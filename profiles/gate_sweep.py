"""Gate kernel alone over a token sweep: fixed cost vs streaming rate.

argv: N [tokens ...]. For each T: the gate kernel (fm_layer_gate = gate +
expert scan) after an L2-cleaning read of a 256 MiB buffer, median of 30,
plus a reference streaming read of the same x bytes (torch sum over dim 1)
— the achievable read bandwidth for this size. A linear fit t(T) = a + b*T
separates the per-launch fixed cost (a) from the streaming rate (1/b)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2304_03946_b200 import _lib as L  # noqa: E402
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
Ts = [int(t) for t in sys.argv[2:]] or [8192, 16384, 32768, 65536, 131072, 262144]
k, d = (2 if N <= 32 else 1), 1024
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
acc = torch.empty((), device="cuda")


def timed(fn, reps=30):
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=acc)
        torch.cuda._sleep(300_000)  # the host enqueues the timed launch while the GPU is still busy
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


rows = []
for T in Ts:
    lay = MoELayer(N, k, d, 256, max_tokens=T)
    x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    wg = (torch.randn(N, d, device="cuda") * d**-0.5).to(torch.bfloat16)
    hist = torch.empty(N, dtype=torch.int64, device="cuda")
    out = torch.empty(T, device="cuda", dtype=torch.bfloat16)
    g = lambda: L.call("fm_layer_gate", lay._h, L.ptr(x), T, L.ptr(wg), L.ptr(hist), L.stream_ptr())
    r = lambda: torch.sum(x, dim=1, out=out)
    for _ in range(3):
        g(), r()
    tg, tr = timed(g), timed(r)
    lay.set_timing(True)  # the bench's in-step method: events adjacent to each kernel
    timed(g)
    ph = lay.read_timing()
    lay.set_timing(False)
    t_gate = ph["gate"][0] / ph["gate"][1] * 1e3
    t_scan = ph["scan"][0] / ph["scan"][1] * 1e3
    mb = T * d * 2 / 1e6
    rows.append((T, tg, tr, t_gate))
    print(f"N={N} T={T:7d} x={mb:7.1f} MB  gate+scan {tg:7.1f} us ({mb / tg * 1e3:6.0f} GB/s)  "
          f"[gate {t_gate:6.1f} us = {mb / t_gate * 1e3:5.0f} GB/s, scan {t_scan:5.1f} us]  "
          f"torch row-sum {tr:7.1f} us ({mb / tr * 1e3:6.0f} GB/s)")
    del lay
if len(rows) >= 2:
    import numpy as np

    T = np.array([r[0] for r in rows], float)
    for name, col in (("gate+scan", 1), ("torch read", 2), ("gate alone", 3)):
        y = np.array([r[col] for r in rows])
        b, a = np.polyfit(T, y, 1)
        print(f"{name}: fixed {a:.1f} us + {b * 1e3:.3f} ns/token -> streaming {d * 2 / b / 1e3:.0f} GB/s")
