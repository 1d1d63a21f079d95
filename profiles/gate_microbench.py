"""Gate phase microbenchmark: fm_layer_gate (gate kernel + expert scan) alone."""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
f = lambda: L.call("fm_layer_gate", lay._h, L.ptr(x), T, L.ptr(wg), L.ptr(hist), L.stream_ptr())
for _ in range(5):
    f()
ts = []
for _ in range(50):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f(); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
us = ts[len(ts) // 2] * 1e3
print(f"N={N} gate+scan median {us:.1f} us  min {ts[0]*1e3:.1f}  -> {T*d*2/us/1e3:.0f} GB/s (x read only)")
