"""The float32 layer restatement (the CPU baseline bench.py times) against the
float64 one (the parity oracle) on exact-arithmetic inputs: identical routing
(indices, positions, histogram), forward and all gradients within the bf16
storage tolerance of DESIGN.md §6; and the C oracle's OpenMP bf16 rounding
bit-equal to the numpy restatement."""
import numpy as np

from oracle import layer as OL


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def test_float32_layer_matches_float64():
    rng = np.random.default_rng(3)
    T, d, N, f, k = 512, 256, 8, 512, 2
    skew = np.log(1.0 / np.arange(1, N + 1) ** 1.25)
    x, wg, w1, b1, w2, b2 = OL.exact_inputs(rng, T, d, N, f, skew=skew)
    dy = OL.bf16(rng.standard_normal((T, d)) * 0.1)
    s64 = OL.forward(x, wg, w1, b1, w2, b2, k)
    g64 = OL.backward(s64, dy)
    f32 = np.float32
    s32 = OL.forward(x.astype(f32), wg.astype(f32), w1.astype(f32), b1.astype(f32), w2.astype(f32),
                     b2.astype(f32), k, dtype=f32)
    g32 = OL.backward(s32, dy.astype(f32))
    assert np.array_equal(s32["idx"], s64["idx"]) and np.array_equal(s32["pos"], s64["pos"])
    assert np.array_equal(s32["hist"], s64["hist"])
    assert _rel(s32["y"], s64["y"]) < 1e-2
    for name in ("dx", "dw1", "dw2", "db1", "db2", "dwg"):
        assert _rel(g32[name], g64[name]) < 1e-2, name


def test_openmp_bf16_rounding_equals_numpy():
    a = np.random.default_rng(0).standard_normal(3 << 20).astype(np.float32) * 17
    ref = a.copy().view(np.uint32)
    ref += np.uint32(0x7FFF) + ((ref >> np.uint32(16)) & np.uint32(1))
    ref &= np.uint32(0xFFFF0000)
    out = OL.bf16_f32(a.copy())  # >= 1 Mi elements: the C oracle's OpenMP loop
    assert np.array_equal(out.view(np.uint32), ref)
