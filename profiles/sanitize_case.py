import sys, torch
sys.path.insert(0, ".")
from paper_2304_03946_b200.layer import MoELayer
# configs[1]-shaped layer at 8K tokens: 64 tiles per expert -> both side jobs run
N, k, d, f, T = 16, 2, 1024, 4096, 8192
lay = MoELayer(N, k, d, f, max_tokens=T)
p = lay.init_params(seed=1)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
dy = torch.randn(T, d, device="cuda").to(torch.bfloat16)
for side in (True, False):
    lay.set_side_jobs(side)
    y = lay.forward(x, p["wg"], p["w1"], p["b1"], p["w2"], p["b2"])
    g = lay.backward(dy)
    torch.cuda.synchronize()
    print("side", side, "mask", lay.side_jobs, float(g.dx.float().abs().sum()))
