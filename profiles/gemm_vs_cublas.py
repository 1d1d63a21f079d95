"""Sustained-throughput comparison, same process, same data: our grouped GEMM
vs cuBLAS (torch.mm) on dense random bf16 inputs. Each measurement runs
back-to-back launches for ~2 s (power-capped steady state)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2304_03946_b200 import _lib as L  # noqa: E402

dev = "cuda"
G, R = 8, 16384
i32 = lambda v: torch.tensor(v, device=dev, dtype=torch.int32)


def timed(fn, secs=2.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n, t0 = 0, time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def case(K, N, relu_a=False):
    total = G * R
    A = torch.randn(total, K, device=dev).to(torch.bfloat16)
    if relu_a:
        A = A.clamp_min(0)
    W = (torch.randn(G, N, K, device=dev) * K**-0.5).to(torch.bfloat16)
    b = torch.randn(G, N, device=dev)
    C = torch.empty(total, N, device=dev, dtype=torch.bfloat16)
    mask = torch.empty(total, N // 32, device=dev, dtype=torch.int32)
    st, pr = i32([g * R for g in range(G)]), i32([R] * G)
    tp = i32([g * (R // 128) for g in range(G + 1)])
    flops = 2.0 * total * K * N

    def ours(variant):
        def f():
            L.call("fm_grouped_gemm", variant, L.ptr(A), L.ptr(W), L.ptr(C), L.ptr(b),
                   L.ptr(mask) if variant == L.FM_GEMM_FWD_BIAS_RELU else None,
                   L.ptr(st), L.ptr(pr), L.ptr(tp), G, total, 0, N, K, L.stream_ptr())
        return f

    def cublas():
        for g in range(G):
            torch.mm(A[g * R:(g + 1) * R], W[g].T, out=C[g * R:(g + 1) * R])

    res = {}
    for name, fn in [("ours_relu", ours(L.FM_GEMM_FWD_BIAS_RELU)), ("cublas", cublas),
                     ("ours_none", ours(L.FM_GEMM_FWD_BIAS)), ("cublas2", cublas),
                     ("ours_relu2", ours(L.FM_GEMM_FWD_BIAS_RELU))]:
        ms = timed(fn)
        res[name] = round(flops / ms / 1e9, 1)
    print(f"K={K} N={N} relu_a={relu_a} TFLOP/s", res, flush=True)


for cg in (2,):
    L.call("fm_set_gemm_cta_group", cg)
    case(1024, 4096)
    case(4096, 1024)
    case(1024, 4096, relu_a=True)
