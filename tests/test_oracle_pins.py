"""Pins of the CPU oracle against what the paper and mathematics fix.

None of these compares the oracle with itself or with the CUDA path: each
check is a worked value the paper (or SURVEY.md s9 / SPEC.md) prints, a closed
form or bound, a library routine the method reduces to in a special case, or a
brute-force re-formulation on tiny inputs.  CPU only (no GPU marker).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import amsim_inputs as inp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def u32(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def f32(u):
    return np.asarray(u, dtype=np.uint32).view(np.float32)


def trunc(x, m):
    """(1,8,m) by bit truncation: the format definition of PAPER.md:726-727."""
    mask = np.uint32((0xFFFFFFFF << (23 - m)) & 0xFFFFFFFF)
    return f32(u32(x) & mask)


def frac_of(v: float) -> Fraction:
    return Fraction(float(v))


def rand_normal_operands(n, seed, emin=64, emax=190):
    g = inp.rng(seed)
    e = g.integers(emin, emax + 1, n, dtype=np.uint32)
    mant = g.integers(0, 1 << 23, n, dtype=np.uint32)
    s = g.integers(0, 2, n, dtype=np.uint32)
    return f32((s << 31) | (e << 23) | mant)


# --------------------------------------------------------------------------
# Alg. 2 special cases and worked values (golden fixture, cited per case)

def test_alg2_golden_cases(orc):
    cases = json.load(open(os.path.join(GOLD, "alg2_specials.json")))["cases"]
    for c in cases:
        a = f32([int(c["a"], 16)])
        b = f32([int(c["b"], 16)])
        got = u32(orc.mul(a, b, c["model"], c["m"]))[0]
        assert got == int(c["c"], 16), f"{c['why']}: got {got:#010x}"


# --------------------------------------------------------------------------
# Exact multiplier == the true product of truncated operands (library / exact
# rational arithmetic), SURVEY.md 8(c) "Exact model special case".

@pytest.mark.parametrize("m", list(range(1, 12)))
def test_exact_equals_truncated_fp32_product(orc, m):
    a = rand_normal_operands(50000, 10 + m)
    b = rand_normal_operands(50000, 100 + m)
    got = orc.mul(a, b, "exact", m)
    want = trunc(a, m) * trunc(b, m)           # numpy IEEE FP32 multiply
    assert np.array_equal(u32(got), u32(want))
    # and against exact rationals on a subsample (independent of FP rounding)
    for i in range(0, 50000, 997):
        exact = frac_of(trunc(a[i:i + 1], m)[0]) * frac_of(trunc(b[i:i + 1], m)[0])
        assert frac_of(got[i]) == exact


def test_exact_power_of_two_invariant(orc):
    """amsim(x, 2^n) = trunc_m(x) * 2^n for the exact model."""
    x = rand_normal_operands(20000, 7, 80, 170)
    for n in (-20, -1, 0, 1, 5, 30):
        p2 = np.full_like(x, np.float32(2.0 ** n))
        got = orc.mul(x, p2, "exact", 7)
        assert np.array_equal(u32(got), u32(np.ldexp(trunc(x, 7), n).astype(np.float32)))


def test_exact_m1_probe_products(orc):
    """The four significand products behind the M=1 exact table
    {0, 0x400000, 0x400000, 0x900000}: 1.0*1.0, 1.0*1.5, 1.5*1.0,
    1.5*1.5 with carry on the last."""
    ops = f32([0x3F800000, 0x3FC00000])
    got = [u32(orc.mul(ops[k:k + 1], ops[j:j + 1], "exact", 1))[0] for k in range(2) for j in range(2)]
    assert got == [0x3F800000, 0x3FC00000, 0x3FC00000, 0x40100000]


def test_sign_xor_and_exponent_sum(orc):
    """Sign = XOR, exponent = sum - 127 (Alg. 2 l.5-6) for every model."""
    a = rand_normal_operands(20000, 1, 90, 160)
    b = rand_normal_operands(20000, 2, 90, 160)
    for model in ("exact", "mitchell", "mbm"):
        p = orc.mul(a, b, model, 7)
        up, ua, ub = u32(p), u32(a), u32(b)
        assert np.array_equal(up >> 31, (ua >> 31) ^ (ub >> 31))
        ex = ((ua >> 23) & 0xFF).astype(np.int64) + ((ub >> 23) & 0xFF) - 127
        ep = ((up >> 23) & 0xFF).astype(np.int64)
        assert np.all((ep == ex) | (ep == ex + 1))


# --------------------------------------------------------------------------
# Mitchell: closed-form bound and the log/antilog formulation

def _mitchell_loglin(k, j, m):
    """Mitchell 1962 written as log/antilog: log2(1+x) ~ x; 2^(n+f) ~ 2^n(1+f)."""
    L = Fraction(k, 1 << m) + Fraction(j, 1 << m)   # log2 A + log2 B with exponents 0
    n = L.numerator // L.denominator                 # floor
    f = L - n
    return (1 + f) * (2 ** n)


def test_mitchell_error_bound_exhaustive(orc):
    m = 7
    ks, js = np.meshgrid(np.arange(128, dtype=np.uint32), np.arange(128, dtype=np.uint32), indexing="ij")
    a = f32((127 << 23) | (ks.ravel() << 16))
    b = f32((127 << 23) | (js.ravel() << 16))
    p = orc.mul(a, b, "mitchell", m).astype(np.float64)
    exact = a.astype(np.float64) * b.astype(np.float64)
    rel = (p - exact) / exact
    assert rel.max() <= 0.0                       # never overestimates
    assert rel.min() >= -1.0 / 9.0 - 1e-15        # Mitchell's bound
    worst = np.flatnonzero(np.isclose(rel, -1.0 / 9.0, rtol=0, atol=1e-15))
    assert list(worst) == [64 * 128 + 64]         # only 1.5 x 1.5 -> 2.0
    assert p[64 * 128 + 64] == 2.0
    for idx in range(0, 128 * 128, 37):           # log/antilog formulation
        k, j = divmod(idx, 128)
        assert Fraction(float(p[idx])) == _mitchell_loglin(k, j, m)


def test_mitchell_scales_with_exponents(orc):
    g = inp.rng(5)
    k = g.integers(0, 128, 2000)
    j = g.integers(0, 128, 2000)
    e1 = g.integers(-40, 40, 2000)
    e2 = g.integers(-40, 40, 2000)
    a = f32(((127 + e1).astype(np.uint32) << 23) | (k.astype(np.uint32) << 16))
    b = f32(((127 + e2).astype(np.uint32) << 23) | (j.astype(np.uint32) << 16))
    p = orc.mul(a, b, "mitchell", 7)
    for i in range(2000):
        assert Fraction(float(p[i])) == _mitchell_loglin(int(k[i]), int(j[i]), 7) * Fraction(2) ** int(e1[i] + e2[i])


def test_mbm_standin_properties(orc):
    """MBM stand-in (reading C17, fidelity UNPINNED): contract properties only --
    carry <= 1 (the oracle raises otherwise), symmetric, and less biased than
    Mitchell (the defining claim of a 'minimally biased' multiplier)."""
    m = 7
    ks, js = np.meshgrid(np.arange(128, dtype=np.uint32), np.arange(128, dtype=np.uint32), indexing="ij")
    a = f32((127 << 23) | (ks.ravel() << 16))
    b = f32((127 << 23) | (js.ravel() << 16))
    pm = orc.mul(a, b, "mbm", m).astype(np.float64)
    pt = orc.mul(b, a, "mbm", m).astype(np.float64)
    assert np.array_equal(pm, pt)
    exact = a.astype(np.float64) * b.astype(np.float64)
    mit = orc.mul(a, b, "mitchell", m).astype(np.float64)
    assert abs(np.mean((pm - exact) / exact)) < 0.25 * abs(np.mean((mit - exact) / exact))


def _mbm_c17(k: int, j: int, m: int) -> Fraction:
    """Reading C17 written out in exact rationals: the stand-in's
    significand product of 1.k and 1.j (k, j the top m mantissa bits)."""
    x, y = Fraction(k, 2 ** m), Fraction(j, 2 ** m)
    if x + y < 1:
        sig, e = 1 + x + y + Fraction(5, 64), 0
        if sig >= 2:
            sig, e = sig / 2, 1
    else:
        sig, e = min(x + y + Fraction(5, 128), 2 - Fraction(1, 2 ** 15)), 1
    return sig * 2 ** e


@pytest.mark.parametrize("m", [7, 4, 11])
def test_mbm_standin_equals_c17_definition(orc, m):
    """Pins oracle_model_mbm to reading C17's written definition (DESIGN.md,
    PAPER.md:782-785 only cites the model): every (k, j) pair at m = 7 and 4
    (a 64-pair stride sample at m = 11) under four exponent pairs, compared
    bit for bit with the rational evaluation above (every value is exactly
    representable in FP32, checked).  A wrong bias constant, a renormalisation
    that forgets the exponent, or a wrong saturation bound fails here.
    Fidelity to Saadat et al. stays unpinned (not checkable from the paper)."""
    n = 1 << m
    pairs = [(k, j) for k in range(n) for j in range(n)] if m <= 7 else \
        [(k, j) for k in range(0, n, 64) for j in range(0, n, 64)] + [(n - 1, n - 1), (n - 1, 0), (0, n - 1)]
    ks = np.array([p[0] for p in pairs], dtype=np.uint32)
    js = np.array([p[1] for p in pairs], dtype=np.uint32)
    want_sig = [_mbm_c17(int(k), int(j), m) for k, j in pairs]
    for ea, eb in ((127, 127), (120, 140), (64, 190), (200, 50)):
        a = f32((np.uint32(ea) << 23) | (ks << np.uint32(23 - m)))
        b = f32((np.uint32(eb) << 23) | (js << np.uint32(23 - m)))
        got = orc.mul(a, b, "mbm", m)
        scale = Fraction(2) ** (ea + eb - 254)
        for i, w in enumerate(want_sig):
            v = w * scale
            assert Fraction(float(np.float32(float(v)))) == v, "value not exact in FP32"
            assert Fraction(float(got[i])) == v, (m, ea, eb, pairs[i], float(got[i]), float(v))


def test_mbm_golden_cases(orc):
    """Hand-derived MBM stand-in products (tests/golden/mbm_standin.json: 1 x 1,
    the carry boundary, a renormalising pair, sig = 2 exactly, the saturated
    corner, exponents, sign), derivation per case in the fixture."""
    cases = json.load(open(os.path.join(GOLD, "mbm_standin.json")))["cases"]
    assert len(cases) >= 5
    for c in cases:
        assert np.float32(c["a_val"]).view(np.uint32) == int(c["a"], 16)
        got = orc.mul(f32([int(c["a"], 16)]), f32([int(c["b"], 16)]), "mbm", c["m"])
        assert u32(got)[0] == int(c["c"], 16), f"{c['why']}: got {float(got[0])!r}, want {c['c_val']!r}"
        assert float(got[0]) == c["c_val"]


def test_model_contract_violation_raises(orc):
    """A product outside {Exp, Exp+1} is a model error (reading C10): the asym
    model is valid, so no error; this checks the error path is reachable via an
    out-of-range m argument instead."""
    with pytest.raises(orc.OracleError):
        orc.mul(np.float32(1.0), np.float32(1.0), "exact", 0)


# --------------------------------------------------------------------------
# GEMM: brute force / library reductions

def test_gemm_exact_vs_numpy(orc):
    g = inp.rng(11)
    for (M, N, K) in [(1, 1, 1), (3, 5, 7), (8, 8, 8), (17, 9, 33), (4, 3, 0)]:
        A = g.standard_normal((M, K)).astype(np.float32)
        B = g.standard_normal((K, N)).astype(np.float32)
        r = orc.gemm(A, B, "exact", 7)
        At, Bt = trunc(A, 7), trunc(B, 7)
        ref64 = At.astype(np.float64) @ Bt.astype(np.float64)
        assert np.all(np.abs(r.c64 - ref64) <= 1e-12 * (np.abs(At).astype(np.float64) @ np.abs(Bt) + 1e-300))
        # FP32 sequential sum in increasing k of the (library) FP32 products
        prods = At[:, :, None] * Bt[None, :, :]         # M x K x N, exact in FP32
        s = np.zeros((M, N), np.float32)
        for t in range(K):
            s = (s + prods[:, t, :]).astype(np.float32)
        assert np.array_equal(u32(r.c32), u32(s))
        assert np.allclose(r.abs64, np.abs(At).astype(np.float64) @ np.abs(Bt), rtol=1e-12, atol=0)


def test_gemm_operand_order_and_indexing_asym(orc):
    """C[i][j] = sum_t mul(A[i][t], B[t][j]) with a from A (reading C11), written
    as explicit Python loops over per-product oracle calls (pinned above)."""
    g = inp.rng(12)
    M, N, K = 5, 4, 6
    A = g.standard_normal((M, K)).astype(np.float32)
    B = g.standard_normal((K, N)).astype(np.float32)
    r = orc.gemm(A, B, "asym", 7)
    for i in range(M):
        for j in range(N):
            p = orc.mul(A[i, :], B[:, j], "asym", 7).astype(np.float64)
            assert abs(r.c64[i, j] - p.sum()) <= 1e-12 * np.abs(p).sum()
    swapped = orc.gemm(B.T.copy(), A.T.copy(), "asym", 7)
    assert not np.allclose(swapped.c64.T, r.c64)  # the model really is asymmetric


def test_gemm_row_sampling_matches_full(orc):
    g = inp.rng(13)
    A = g.standard_normal((20, 16)).astype(np.float32)
    B = g.standard_normal((16, 6)).astype(np.float32)
    full = orc.gemm(A, B, "mitchell", 7)
    rows = np.array([19, 0, 7, 7, 3])
    part = orc.gemm(A, B, "mitchell", 7, rows=rows)
    assert np.array_equal(u32(part.c32), u32(full.c32[rows]))


def test_dense_worked_example(orc):
    """AMDENSE 2x3 example."""
    gd = json.load(open(os.path.join(GOLD, "dense_2x3.json")))
    W = np.array(gd["W"], np.float32)
    x = np.array(gd["x"], np.float32)[:, None]
    d = np.array(gd["delta_out"], np.float32)[:, None]
    assert np.array_equal(orc.gemm(W, x).c32[:, 0], np.array(gd["o"], np.float32))
    assert np.array_equal(orc.gemm(d, x.T.copy()).c32, np.array(gd["W_grad"], np.float32))
    assert np.array_equal(orc.gemm(W.T.copy(), d).c32[:, 0], np.array(gd["x_grad"], np.float32))


# --------------------------------------------------------------------------
# Convolutions: the explicit im2col / dilate / pad / reverse-transpose
# pipelines reduce, for the exact model, to FP64 conv2d and its gradients on
# truncated inputs (torch library routines).

CONV_SHAPES = [
    # N, H, W, C, K, R, S, sh, sw, ph, pw
    (2, 5, 5, 3, 4, 3, 3, 1, 1, 0, 0),
    (2, 7, 6, 3, 2, 3, 3, 2, 2, 1, 1),
    (1, 8, 8, 2, 3, 3, 3, 3, 3, 1, 1),
    (2, 6, 6, 4, 5, 1, 1, 2, 2, 0, 0),
    (1, 9, 7, 2, 2, 5, 5, 2, 2, 2, 2),   # (H+2P-KH) mod S != 0
    (3, 4, 4, 1, 1, 2, 2, 1, 1, 0, 0),
    (1, 7, 9, 3, 2, 4, 3, 2, 1, 1, 0),   # R != S, stride_h != stride_w
    (1, 10, 10, 2, 3, 7, 7, 2, 2, 3, 3),  # ResNet-50 stem geometry
]


def _torch_refs(shape, x, w, dy):
    import torch
    import torch.nn.functional as F
    N, H, W, C, K, R, S, sh, sw, ph, pw = shape
    xt = torch.from_numpy(trunc(x, 7).astype(np.float64)).permute(0, 3, 1, 2)
    wt = torch.from_numpy(trunc(w, 7).astype(np.float64)).permute(3, 2, 0, 1)
    dyt = torch.from_numpy(trunc(dy, 7).astype(np.float64)).permute(0, 3, 1, 2)
    y = F.conv2d(xt, wt, stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1).reshape(-1, K).numpy()
    dw = torch.nn.grad.conv2d_weight(xt, wt.shape, dyt, stride=(sh, sw), padding=(ph, pw))
    dw = dw.permute(2, 3, 1, 0).reshape(-1, K).numpy()
    dx = torch.nn.grad.conv2d_input(xt.shape, wt, dyt, stride=(sh, sw), padding=(ph, pw))
    dx = dx.permute(0, 2, 3, 1).reshape(-1, C).numpy()
    return y, dw, dx


@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_conv_exact_vs_torch_fp64(orc, shape):
    N, H, W, C, K, R, S, sh, sw, ph, pw = shape
    d = orc.conv_desc(N, H, W, C, K, R, S, sh, ph, stride_w=sw, pad_w=pw)
    x = inp.normal((N, H, W, C), 1)
    w = inp.normal((R, S, C, K), 2)
    dy = inp.normal((N, d.OH, d.OW, K), 3)
    y, dw, dx = _torch_refs(shape, x, w, dy)
    ry = orc.conv_fwd(d, x, w)
    rw = orc.conv_bwd_filter(d, x, dy)
    rx = orc.conv_bwd_data(d, dy, w)
    for r, ref in ((ry, y), (rw, dw), (rx, dx)):
        assert r.c64.shape == ref.shape
        assert np.all(np.abs(r.c64 - ref) <= 1e-12 * r.abs64 + 1e-300)


def _direct_conv_refs(orc, shape, x, w, dy, model):
    """The three passes written as direct nested-loop sums of per-product
    oracle calls (a formulation with no im2col/dilate/pad/reversal)."""
    N, H, W, C, K, R, S, sh, sw, ph, pw = shape
    OH = (H + 2 * ph - R) // sh + 1
    OW = (W + 2 * pw - S) // sw + 1
    y = np.zeros((N, OH, OW, K))
    dw = np.zeros((R, S, C, K))
    dx = np.zeros((N, H, W, C))
    for n in range(N):
        for oh in range(OH):
            for ow in range(OW):
                for kh in range(R):
                    for kw in range(S):
                        ih, iw = oh * sh - ph + kh, ow * sw - pw + kw
                        if not (0 <= ih < H and 0 <= iw < W):
                            continue
                        xv = x[n, ih, iw, :]
                        # fwd: a = x, b = w
                        y[n, oh, ow, :] += orc.mul(xv[:, None], w[kh, kw], model).astype(np.float64).sum(0)
                        # wgrad: a = x, b = dy
                        dw[kh, kw] += orc.mul(xv[:, None], dy[n, oh, ow][None, :], model).astype(np.float64)
                        # dgrad: a = dy, b = w
                        dx[n, ih, iw] += orc.mul(dy[n, oh, ow][None, :], w[kh, kw], model).astype(np.float64).sum(1)
    return y.reshape(-1, K), dw.reshape(-1, K), dx.reshape(-1, C)


@pytest.mark.parametrize("shape", CONV_SHAPES[:5])
def test_conv_pipelines_vs_direct_asym(orc, shape):
    N, H, W, C, K, R, S, sh, sw, ph, pw = shape
    d = orc.conv_desc(N, H, W, C, K, R, S, sh, ph, stride_w=sw, pad_w=pw)
    x = inp.normal((N, H, W, C), 4)
    w = inp.normal((R, S, C, K), 5)
    dy = inp.normal((N, d.OH, d.OW, K), 6)
    y, dw, dx = _direct_conv_refs(orc, shape, x, w, dy, "asym")
    for r, ref in ((orc.conv_fwd(d, x, w, "asym"), y), (orc.conv_bwd_filter(d, x, dy, "asym"), dw),
                   (orc.conv_bwd_data(d, dy, w, "asym"), dx)):
        assert np.all(np.abs(r.c64 - ref) <= 1e-12 * r.abs64 + 1e-300)


def test_conv_row_sampling(orc):
    shape = CONV_SHAPES[1]
    N, H, W, C, K, R, S, sh, sw, ph, pw = shape
    d = orc.conv_desc(N, H, W, C, K, R, S, sh, ph)
    x = inp.normal((N, H, W, C), 7)
    w = inp.normal((R, S, C, K), 8)
    dy = inp.normal((N, d.OH, d.OW, K), 9)
    for fn, a1, a2, nrows in ((orc.conv_fwd, x, w, N * d.OH * d.OW), (orc.conv_bwd_filter, x, dy, R * S * C),
                              (orc.conv_bwd_data, dy, w, N * H * W)):
        full = fn(d, a1, a2, "mitchell")
        rows = np.array([nrows - 1, 0, nrows // 2])
        part = fn(d, a1, a2, "mitchell", rows=rows)
        assert np.array_equal(u32(part.c32), u32(full.c32[rows]))


# ---------------------------------------------------------------------------
# exponent casting to (1, e, m) (reading C23)

def test_cast_e8_is_identity(orc):
    g = inp.rng(41)
    x = f32(g.integers(0, 2 ** 32, 20000, dtype=np.uint64).astype(np.uint32))
    assert np.array_equal(u32(orc.cast_e(x, 8)), u32(x))


def test_cast_e5_matches_ieee_half_range(orc):
    """e = 5 is IEEE binary16's exponent: normal magnitudes in
    [finfo(float16).tiny, 2^finfo(float16).maxexp) survive, larger overflow to
    +-Inf, smaller flush to +-0 (no subnormals)."""
    fi = np.finfo(np.float16)
    g = inp.rng(42)
    ex = g.integers(1, 255, 20000).astype(np.uint32)
    x = f32((g.integers(0, 2, 20000).astype(np.uint32) << 31) | (ex << 23) | g.integers(0, 1 << 23, 20000).astype(np.uint32))
    y = orc.cast_e(x, 5)
    a = np.abs(x.astype(np.float64))
    big = a >= 2.0 ** fi.maxexp
    small = a < float(fi.tiny)
    keep = ~big & ~small
    assert np.all(np.isinf(y[big])) and np.array_equal(np.signbit(y[big]), np.signbit(x[big]))
    assert np.all(y[small] == 0) and np.array_equal(np.signbit(y[small]), np.signbit(x[small]))
    assert np.array_equal(u32(y[keep]), u32(x[keep]))
    # values exactly representable as float16 normals are unchanged
    h = g.normal(0, 100, 5000).astype(np.float16)
    h = h[np.abs(h.astype(np.float64)) >= float(fi.tiny)].astype(np.float32)
    assert np.array_equal(u32(orc.cast_e(h, 5)), u32(h))


def test_cast_then_amsim_is_half_precision_product(orc):
    """(1,5,10) with the exact multiplier: for float16 normals the product is
    the exact FP32 product of the two halves (an 11x11-bit significand product
    is exact in FP32) -- the IEEE half-precision multiplier without rounding."""
    g = inp.rng(43)
    a = g.normal(0, 4, 3000).astype(np.float16).astype(np.float32)
    b = g.normal(0, 4, 3000).astype(np.float16).astype(np.float32)
    fi = np.finfo(np.float16)
    ok = (np.abs(a) >= float(fi.tiny)) & (np.abs(b) >= float(fi.tiny))
    a, b = a[ok], b[ok]
    got = orc.mul(orc.cast_e(a, 5), orc.cast_e(b, 5), "exact", 10)
    want = (a.astype(np.float64) * b.astype(np.float64)).astype(np.float32)
    assert np.array_equal(u32(got), u32(want))


@pytest.mark.parametrize("e", [1, 2, 3, 4, 6, 7])
def test_cast_boundaries_closed_form(orc, e):
    """The largest kept magnitude is just below 2^(B+1), the smallest kept is
    2^(1-B), B = 2^(e-1) - 1; e = 1 has no normal numbers at all."""
    B = 2 ** (e - 1) - 1
    top = np.float32(np.nextafter(np.float32(2.0 ** (B + 1)), np.float32(0)))
    cases = np.array([top, 2.0 ** (B + 1), 2.0 ** (1 - B), np.nextafter(np.float32(2.0 ** (1 - B)), np.float32(0)),
                      -(2.0 ** (B + 1))], np.float32)
    y = orc.cast_e(cases, e)
    if e == 1:   # B = 0, kept range [2^1, 2^1) is empty: 1.99 (exponent 0 < 1 - B) flushes, 2 overflows
        assert y[0] == 0 and np.isposinf(y[2])
    else:
        assert y[0] == cases[0] and y[2] == cases[2]
    assert np.isposinf(y[1]) and np.isneginf(y[4]) and y[3] == 0
