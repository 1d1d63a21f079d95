"""Parity of the tcgen05 grouped GEMM against a torch fp32 reference.

Tolerances: bf16 outputs are compared with |d| <= 2^-7 |ref| + 1e-2 * rms(ref)
(one bf16 rounding of the f32 accumulator plus accumulation-order noise);
f32 weight-gradient outputs within 1e-4 relative Frobenius error.
"""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2304_03946_b200 import _lib as L  # noqa: E402


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"], autouse=True)
def cta_group(request):
    """Every GEMM test runs with single-CTA 128x256 tiles and CTA-pair 256x256 tiles."""
    L.call("fm_set_gemm_cta_group", request.param)
    yield request.param
    L.call("fm_set_gemm_cta_group", 0)


def _segments(rows_per_group, device):
    pad = [((r + 127) // 128) * 128 for r in rows_per_group]
    start = [0]
    for p in pad[:-1]:
        start.append(start[-1] + p)
    tiles = lambda n_tiles: [0] + list(torch.tensor([p // 128 * n_tiles for p in pad]).cumsum(0).tolist())
    return pad, start, tiles


def _unpack_bits(words, N):
    w = words.to(torch.int64) & 0xFFFFFFFF
    sh = torch.arange(32, device=words.device)
    return ((w.unsqueeze(-1) >> sh) & 1).reshape(words.shape[0], N).bool()


def _pack_bits(b):
    rows, N = b.shape
    sh = torch.arange(32, device=b.device)
    w = (b.reshape(rows, N // 32, 32).to(torch.int64) << sh).sum(-1)
    return torch.where(w >= 2**31, w - 2**32, w).to(torch.int32).contiguous()


def _close_bf16(out, ref):
    out = out.float()
    rms = ref.pow(2).mean().sqrt().item()
    bad = (out - ref).abs() > (ref.abs() * 2**-7 + 1e-2 * rms)
    assert bad.float().mean().item() < 1e-4, f"{bad.sum().item()} mismatches"
    rel = ((out - ref).norm() / ref.norm()).item()
    assert rel < 4e-3, rel


def _setup(rows, d_in, d_out, seed=0):
    torch.manual_seed(seed)
    dev = "cuda"
    pad, start, tiles = _segments(rows, dev)
    total = sum(pad)
    A = torch.zeros(total, d_in, device=dev, dtype=torch.bfloat16)
    for g, r in enumerate(rows):
        A[start[g] : start[g] + r] = torch.randn(r, d_in, device=dev).to(torch.bfloat16)
    i32 = lambda v: torch.tensor(v, device=dev, dtype=torch.int32)
    return pad, start, tiles, total, A, i32


@pytest.mark.parametrize("rows", [[200, 0, 77, 512], [1000], [128, 384, 130, 0, 900]])
@pytest.mark.parametrize("relu", [True, False])
def test_fwd(rows, relu):
    K, N = 512, 768
    pad, start, tiles, total, A, i32 = _setup(rows, K, N)
    G = len(rows)
    W = (torch.randn(G, N, K, device="cuda") * K**-0.5).to(torch.bfloat16)
    b = torch.randn(G, N, device="cuda")
    C = torch.full((total, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    mask = torch.zeros(total, N // 32, device="cuda", dtype=torch.int32)
    st, pr, tp = i32(start), i32(pad), i32(tiles(1))
    variant = L.FM_GEMM_FWD_BIAS_RELU if relu else L.FM_GEMM_FWD_BIAS
    L.call("fm_grouped_gemm", variant, L.ptr(A), L.ptr(W), L.ptr(C), L.ptr(b),
           L.ptr(mask) if relu else None, L.ptr(st), L.ptr(pr), L.ptr(tp), G, total, 0, N, K,
           L.stream_ptr())
    torch.cuda.synchronize()
    for g in range(G):
        seg = slice(start[g], start[g] + pad[g])
        pre = A[seg].float() @ W[g].float().T + b[g]
        ref = pre.clamp_min(0) if relu else pre
        if pad[g]:
            _close_bf16(C[seg], ref)
            if relu:  # ReLU bits agree with the kernel's own output wherever it is not ~0
                bits = _unpack_bits(mask[seg], N)
                assert torch.equal(bits, C[seg].float() > 0) or \
                    ((bits != (C[seg].float() > 0)) & (pre.abs() > 1e-3)).sum() == 0


@pytest.mark.parametrize("mask", [True, False])
def test_dgrad(mask):
    rows = [300, 128, 0, 640]
    K, N = 768, 512  # A [rows, K] . W_g [K, N]
    pad, start, tiles, total, A, i32 = _setup(rows, K, N, seed=1)
    G = len(rows)
    W = (torch.randn(G, K, N, device="cuda") * K**-0.5).to(torch.bfloat16)
    aux = torch.randn(total, N, device="cuda").clamp_min(0).to(torch.bfloat16)
    bits = _pack_bits(aux.float() > 0)
    C = torch.full((total, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    st, pr, tp = i32(start), i32(pad), i32(tiles(1))
    variant = L.FM_GEMM_DGRAD_RELU_MASK if mask else L.FM_GEMM_DGRAD
    colsum = torch.full((total // 128, N), float("nan"), device="cuda") if mask else None
    L.call("fm_grouped_gemm", variant, L.ptr(A), L.ptr(W), L.ptr(C), L.ptr(colsum), L.ptr(bits),
           L.ptr(st), L.ptr(pr), L.ptr(tp), G, total, 0, N, K, L.stream_ptr())
    torch.cuda.synchronize()
    if mask:  # per-128-row-tile column sums of the stored bf16 output (bias-grad partials)
        ref_cs = C.float().reshape(total // 128, 128, N).sum(1)
        assert torch.allclose(colsum, ref_cs, rtol=1e-5, atol=1e-4)
    for g in range(G):
        seg = slice(start[g], start[g] + pad[g])
        ref = A[seg].float() @ W[g].float()
        if mask:
            ref = ref * (aux[seg].float() > 0)
        if pad[g]:
            _close_bf16(C[seg], ref)


def test_wgrad():
    rows = [333, 0, 1024, 64]
    Mw, N = 256, 768
    pad, start, tiles, total, A, i32 = _setup(rows, Mw, N, seed=2)
    B = torch.zeros(total, N, device="cuda", dtype=torch.bfloat16)
    for g, r in enumerate(rows):
        B[start[g] : start[g] + r] = torch.randn(r, N, device="cuda").to(torch.bfloat16)
    G = len(rows)
    C = torch.full((G, Mw, N), float("nan"), device="cuda", dtype=torch.float32)
    st, pr = i32(start), i32(pad)
    L.call("fm_grouped_gemm", L.FM_GEMM_WGRAD, L.ptr(A), L.ptr(B), L.ptr(C), None, None, L.ptr(st),
           L.ptr(pr), None, G, total, Mw, N, 0, L.stream_ptr())
    torch.cuda.synchronize()
    for g in range(G):
        seg = slice(start[g], start[g] + pad[g])
        ref = A[seg].float().T @ B[seg].float()
        if pad[g] == 0:
            assert torch.all(C[g] == 0)
        else:
            rel = ((C[g] - ref).norm() / ref.norm()).item()
            assert rel < 1e-4, rel
