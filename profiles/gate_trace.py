"""Gate pipeline timeline of block 0 (diagnostic build: NVCC_EXTRA=-DFM_GATE_TRACE).

argv: N T [T ...]. For each T: runs the gate a few times after an L2-cleaning
read, then prints block 0's globaltimer stamps relative to its start:
prologue done, per k-block TMA issue (producer) and full-barrier wake (MMA
warp), per tile the epilogue's accumulator wake and finish, and exit."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2304_03946_b200 import _lib as L  # noqa: E402
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402

N = int(sys.argv[1])
Ts = [int(t) for t in sys.argv[2:]] or [128, 37888, 65536]
k, d = (2 if N <= 32 else 1), 1024
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
acc = torch.empty((), device="cuda")
fn = L.lib().fm_debug_gate_trace
buf = (C.c_ulonglong * 256)()
for T in Ts:
    lay = MoELayer(N, k, d, 256, max_tokens=T)
    x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    wg = (torch.randn(N, d, device="cuda") * d**-0.5).to(torch.bfloat16)
    hist = torch.empty(N, dtype=torch.int64, device="cuda")
    for rep in range(4):
        torch.sum(flush, dim=0, out=acc)
        L.call("fm_layer_gate", lay._h, L.ptr(x), T, L.ptr(wg), L.ptr(hist), L.stream_ptr())
        torch.cuda.synchronize()
    assert fn(buf) == 0
    t0 = buf[0]
    rel = lambda i: (buf[i] - t0) / 1e3 if buf[i] >= t0 and buf[i] - t0 < 10**7 else None
    print(f"N={N} T={T}: prologue {rel(1)} us, exit {rel(150)} us")
    for it in range(4):
        iss = [rel(2 + it * 16 + kb) for kb in range(16)]
        full = [rel(66 + it * 16 + kb) for kb in range(16)]
        if iss[0] is None:
            break
        f = lambda v: "  -  " if v is None else f"{v:5.2f}"
        print(f"  tile{it} issue: " + " ".join(f(v) for v in iss))
        print(f"  tile{it} full : " + " ".join(f(v) for v in full))
        print(f"  tile{it} epilogue wake {rel(130 + 2 * it)}  done {rel(131 + 2 * it)}")
        if it == 0:
            print("  tile0 epilogue: top-k %s  masks %s  barrier %s  outputs %s  counts %s  barrier %s" %
                  tuple(rel(i) for i in range(140, 146)))
    blk = (C.c_ulonglong * 1024)()
    assert L.lib().fm_debug_gate_blocks(blk) == 0
    nb = min(512, 2 * 148, (T + 127) // 128)
    st = [blk[2 * b] for b in range(nb)]
    en = [blk[2 * b + 1] for b in range(nb)]
    m = min(st)
    ss = sorted((x - m) / 1e3 for x in st)
    ee = sorted((x - m) / 1e3 for x in en)
    q = lambda a: " ".join(f"{a[int(p * (len(a) - 1))]:.2f}" for p in (0, 0.1, 0.5, 0.9, 1.0))
    print(f"  blocks ({nb}): start min/p10/p50/p90/max {q(ss)} us; exit {q(ee)} us")
    for i in range(len(buf)):
        buf[i] = 0
    torch.cuda.synchronize()
    del lay
