"""CPU checks of numeric constants baked into the CUDA kernels (no GPU).

The representative pass 1 (rep1_kernel, fp_rep.cu) evaluates a quarter of its
exponentials 2^x (x <= 0) on the FMA pipe: x = j + f with j = rint(x) from the
1.5 * 2^23 magic add, 2^f by a degree-5 polynomial, 2^j added into the exponent
field. This test re-evaluates exactly that recipe in float32 (numpy) with the
coefficients parsed from the kernel source and checks it against 2^x in
float64: the row sums it feeds (the softmax normaliser of the
representative attention) must stay at ex2.approx accuracy.
"""
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2502_20766_b200", "csrc", "fp_rep.cu")


def _coeffs():
    src = open(SRC).read()
    body = src[src.index("FP_DEV void exp2_emu2("):]
    body = body[: body.index("\n}\n")]
    nums = [float(v) for v in re.findall(r"(-?\d+\.\d+(?:e-?\d+)?)f", body)]
    # magic, clamp (x0, x1), then c5, c5 (the two lanes), c4, c3, c2, c1, c0
    magic, clamp, clamp_b = nums[0], nums[1], nums[2]
    c5, c5b, c4, c3, c2, c1, c0 = nums[3:10]
    assert clamp == clamp_b and c5 == c5b
    return magic, clamp, [c5, c4, c3, c2, c1, c0]


def _emu(x, magic, clamp, c):
    f32 = np.float32
    x = np.maximum(x.astype(f32), f32(clamp))
    M = f32(magic)
    t = (x + M).astype(f32)
    j = (t - M).astype(f32)
    fr = (x - j).astype(f32)
    p = (f32(c[0]) * fr + f32(c[1])).astype(f32)
    for k in c[2:]:
        p = (p * fr + f32(k)).astype(f32)
    bits = (t.view(np.uint32).astype(np.uint64) * 8388608 + p.view(np.uint32).astype(np.uint64)) % 2**32
    return bits.astype(np.uint32).view(np.float32)


def test_fma_exp2_polynomial_accuracy():
    magic, clamp, c = _coeffs()
    assert magic == 12582912.0 and clamp == -125.0
    x = np.linspace(-125.0, 0.0, 1_000_001, dtype=np.float32)
    y = _emu(x, magic, clamp, c).astype(np.float64)
    ref = np.exp2(x.astype(np.float64))
    rel = np.abs(y - ref) / ref
    assert rel.max() < 3e-7, rel.max()
    # exact at the integers (f = 0: the polynomial's constant term ~ 1)
    xi = np.arange(-125, 1, dtype=np.float32)
    yi = _emu(xi, magic, clamp, c).astype(np.float64)
    assert np.all(np.abs(yi / np.exp2(xi.astype(np.float64)) - 1) < 2e-7)


def test_fma_exp2_masked_keys_vanish_against_a_row_sum():
    magic, clamp, c = _coeffs()
    y = _emu(np.array([-np.inf, -1e30, -200.0], dtype=np.float32), magic, clamp, c)
    # clamped to 2^-125: below an ulp of any row sum (>= 1, the row max contributes 2^0)
    assert np.all(y > 0) and np.all(y < 1e-37)
    assert np.all(np.float32(1.0) + y == np.float32(1.0))
