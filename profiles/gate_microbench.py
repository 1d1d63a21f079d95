"""Gate phase microbenchmark: fm_layer_gate (gate kernel + expert scan) alone.

argv: [N] [flush] — flush "write" (memset a 256 MiB buffer: L2 left full of
dirty lines, as after the step's f32 wgrad) or "read" (sum it: L2 left clean).
The difference is the write-back the gate pays for its predecessor."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2304_03946_b200 import _lib as L
from paper_2304_03946_b200.layer import MoELayer

N, k, d, T = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 2, 1024, 65536
lay = MoELayer(N, k, d, 4096, max_tokens=T)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
wg = (torch.randn(N, d, device="cuda") * d**-0.5).to(torch.bfloat16)
hist = torch.empty(N, dtype=torch.int64, device="cuda")
mode = sys.argv[2] if len(sys.argv) > 2 else "write"
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
acc = torch.empty((), device="cuda")
f = lambda: L.call("fm_layer_gate", lay._h, L.ptr(x), T, L.ptr(wg), L.ptr(hist), L.stream_ptr())
for _ in range(5):
    f()
ts = []
for _ in range(50):
    if mode == "write":
        flush.fill_(1.0)
    else:
        torch.sum(flush, dim=0, out=acc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f(); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
us = ts[len(ts) // 2] * 1e3
print(f"N={N} flush={mode} gate+scan median {us:.1f} us  min {ts[0]*1e3:.1f}  -> {T*d*2/us/1e3:.0f} GB/s (x read only)")
