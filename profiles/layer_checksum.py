"""Checksums of every output of one fused layer step (y, dx and the six
gradients) for an A/B of two library builds that must agree bit for bit.

    FLEXMOE_B200_LIB=abtest/libA.so python profiles/layer_checksum.py
    FLEXMOE_B200_LIB=abtest/libB.so python profiles/layer_checksum.py

Real-valued seeded inputs; shapes: configs[1] (k 2, d 1024), configs[3]'s
d 768 with k 2, and a top-1 case (k 1) — the combine backward's three paths.
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402

CASES = [(16, 2, 1024, 4096, 65536), (32, 2, 768, 3072, 16384), (64, 1, 1024, 4096, 16384)]


def digest(t: torch.Tensor) -> str:
    return hashlib.sha256(t.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:16]


def main():
    torch.cuda.set_device(0)
    for N, k, d, f, T in CASES:
        layer = MoELayer(N, k, d, f, max_tokens=T)
        p = layer.init_params(seed=1)
        g = torch.Generator(device="cpu").manual_seed(2)
        x = torch.randn(T, d, generator=g).to("cuda", torch.bfloat16)
        dy = (torch.randn(T, d, generator=g) * 0.5).to("cuda", torch.bfloat16)
        y = layer.forward(x, p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
        gr = layer.backward(dy)
        torch.cuda.synchronize()
        out = {"y": y, "dx": gr.dx, "dwg": gr.dwg, "dw1": gr.dw1, "db1": gr.db1, "dw2": gr.dw2, "db2": gr.db2}
        print(f"N{N} k{k} d{d} f{f} T{T}", " ".join(f"{n}={digest(v)}" for n, v in out.items()))


if __name__ == "__main__":
    main()
