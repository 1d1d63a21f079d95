"""Second sanitizer case: top-1, 64 experts, d 768 / f 3072, 8,192 tokens —
single-CTA (cta_group::1) GEMM tiles (few rows per expert), gate_kernel<1>,
the standalone column sums and un-permute (36 tiles per expert: no side jobs)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2304_03946_b200.layer import MoELayer  # noqa: E402

N, k, d, f, T = 64, 1, 768, 3072, 8192
lay = MoELayer(N, k, d, f, max_tokens=T)
p = lay.init_params(seed=2)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
dy = torch.randn(T, d, device="cuda").to(torch.bfloat16)
y = lay.forward(x, p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
g = lay.backward(dy)
torch.cuda.synchronize()
print("side", lay.side_jobs, float(g.dx.float().abs().sum()))
