"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (north_star):
  * per product: bit-exact (K = 1 outer products, C = +0 + p),
  * GEMM / conv outputs: |gpu - c64| <= 1e-5 * sum|p| + FLT_MIN per element,
  * non-split kernels accumulate each output in increasing k from +0 exactly
    as the oracle's c32, so they are also checked bit-for-bit against c32.
"""
import numpy as np
import pytest

import amsim_inputs as inp

pytestmark = pytest.mark.gpu

FLT_MIN = np.finfo(np.float32).tiny


@pytest.fixture(scope="module")
def am():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    from paper_2209_04161_b200 import build
    build.build()
    import paper_2209_04161_b200 as am
    am.amsim_set_path_policy(0)
    return am


@pytest.fixture(scope="module")
def luts(am):
    cache = {}

    def get(model, m=7):
        if (model, m) not in cache:
            cache[(model, m)] = am.Lut.build(model, m)
        return cache[(model, m)]
    return get


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def assert_bits(got, want, what=""):
    """Bit equality; two NaNs match whatever their payloads (IEEE 754 leaves
    the payload of e.g. Inf - Inf to the implementation: GPU 0x7FFFFFFF, x86
    0xFFC00000)."""
    g = np.ascontiguousarray(got, np.float32).view(np.uint32)
    w = np.ascontiguousarray(want, np.float32).view(np.uint32)
    both_nan = np.isnan(g.view(np.float32)) & np.isnan(w.view(np.float32))
    bad = np.flatnonzero((g.ravel() != w.ravel()) & ~both_nan.ravel())
    assert bad.size == 0, (f"{what}: {bad.size} of {g.size} differ; first at {bad[:5]}: "
                           f"got {g.ravel()[bad[:5]]} want {w.ravel()[bad[:5]]}")


def assert_tol(got, res, what=""):
    err = np.abs(got.astype(np.float64) - res.c64)
    tol = 1e-5 * res.abs64 + FLT_MIN
    bad = np.flatnonzero((err > tol).ravel())
    assert bad.size == 0, f"{what}: {bad.size} outside tolerance, worst ratio {np.max(err / tol):.3g}"


class exact_order:
    """Policy bit 1: no split-K, so every output is the FP32 sum from +0 in
    increasing k -- the oracle's c32 order (bit-exact comparisons)."""

    def __init__(self, am, careful=False):
        self.am = am
        self.policy = 2 | (1 if careful else 0)

    def __enter__(self):
        self.am.amsim_set_path_policy(self.policy)

    def __exit__(self, *a):
        self.am.amsim_set_path_policy(0)


def run_gemm(am, lut, A, B, trans_a=False, trans_b=False, C0=None, accumulate=False):
    import torch
    M = A.shape[1] if trans_a else A.shape[0]
    N = B.shape[0] if trans_b else B.shape[1]
    C = dev(C0) if C0 is not None else torch.full((M, N), float("nan"), device="cuda")
    am.amsim_gemm(lut, dev(A), dev(B), C, trans_a, trans_b, accumulate)
    return host(C)


# ---------------------------------------------------------------------------
# per-product bit-exactness

@pytest.mark.parametrize("model,m", [("exact", 7), ("mitchell", 7), ("mbm", 7), ("exact", 1), ("exact", 4),
                                     ("exact", 5), ("exact", 6), ("mitchell", 8), ("mitchell", 3)])
@pytest.mark.parametrize("policy", [0, 1])
def test_k1_outer_product_exhaustive(am, luts, orc, model, m, policy):
    """All m-bit mantissas x exponents {1,2,63,64,65,126,127,128,190,253,254}
    x signs, plus zero/subnormal/Inf/NaN, as a K = 1 outer product
    (SURVEY.md 8(d) config 1), under automatic and forced-careful dispatch."""
    v = inp.operand_grid(m)
    am.amsim_set_path_policy(policy)
    try:
        got = run_gemm(am, luts(model, m), v[:, None], v[None, :])  # K = 1: never split
    finally:
        am.amsim_set_path_policy(0)
    want = orc.mul(v[:, None], v[None, :], model, m)
    assert_bits(got, want, f"{model} m={m} policy={policy}")


def _sampled_grid(m, n_mant=96, seed=5):
    """operand_grid restricted to a sample of the 2^m mantissas (the first and
    last four always included) -- the exhaustive grid is too large for m >= 9."""
    v = inp.operand_grid(m).view(np.uint32)
    mant = (v >> np.uint32(23 - m)) & np.uint32((1 << m) - 1)
    keep = np.unique(np.concatenate([np.arange(4), (1 << m) - 1 - np.arange(4),
                                     inp.rng(seed).integers(0, 1 << m, n_mant)]))
    normal = ((v >> 23) & 0xFF) != 0
    normal &= ((v >> 23) & 0xFF) != 0xFF
    sel = ~normal | np.isin(mant, keep)
    return v[sel].view(np.float32)


@pytest.mark.parametrize("model,m,width", [("exact", 8, 32), ("exact", 11, 32), ("mitchell", 9, 16),
                                           ("mitchell", 11, 16), ("mbm", 10, 16)])
@pytest.mark.parametrize("policy", [0, 1])
def test_k1_outer_product_global_table(am, luts, orc, model, m, width, policy):
    """Tables too large for shared memory (m >= 8 with 32-bit entries, m >= 9)
    are read from global memory / L2; per-product bits are unchanged."""
    lut = luts(model, m)
    assert lut.info() == (m, width)
    v = _sampled_grid(m)
    am.amsim_set_path_policy(policy)
    try:
        got = run_gemm(am, lut, v[:, None], v[None, :])
    finally:
        am.amsim_set_path_policy(0)
    assert_bits(got, orc.mul(v[:, None], v[None, :], model, m), f"{model} m={m} policy={policy}")


@pytest.mark.parametrize("model,m", [("mitchell", 9), ("exact", 8)])
def test_global_table_gemm_and_conv(am, luts, orc, model, m):
    lut = luts(model, m)
    A = inp.normal((130, 77), 81)
    B = inp.normal((77, 200), 82)
    shape = (2, 14, 14, 16, 72, 3, 3, 2, 1)
    x, w, dy, OH, OW = _conv_tensors(shape, 83)
    d = am.conv_desc(*shape)
    od = orc.conv_desc(*shape)
    with exact_order(am):
        assert_bits(run_gemm(am, lut, A, B), orc.gemm(A, B, model, m).c32, "gemm")
        assert_bits(_run_conv(am, lut, d, x, w, dy, "fwd"), orc.conv_fwd(od, x, w, model, m).c32, "fwd")
        assert_bits(_run_conv(am, lut, d, x, w, dy, "dgrad"), orc.conv_bwd_data(od, dy, w, model, m).c32, "dgrad")
        assert_bits(_run_conv(am, lut, d, x, w, dy, "wgrad"), orc.conv_bwd_filter(od, x, dy, model, m).c32, "wgrad")
    assert_tol(_run_conv(am, lut, d, x, w, dy, "wgrad"), orc.conv_bwd_filter(od, x, dy, model, m), "wgrad split")


@pytest.mark.parametrize("model", ["exact", "mitchell", "mbm"])
def test_fast_path_full_exponent_range(am, luts, orc, model):
    """Operands whose exponent ranges keep every Exp in [1, 253] take the FTZ
    fast path; it must equal Alg. 2 bit-for-bit, including Exp = 1 and 253."""
    g = inp.rng(21)
    n = 512
    ea = g.integers(64, 191, n).astype(np.uint32)
    ea[:2] = (64, 190)
    a = ((g.integers(0, 2, n).astype(np.uint32) << 31) | (ea << 23) |
         g.integers(0, 1 << 23, n).astype(np.uint32)).view(np.float32)
    b = np.roll(a, 3)
    got = run_gemm(am, luts(model), a[:, None], b[None, :])
    assert_bits(got, orc.mul(a[:, None], b[None, :], model, 7), model)


# ---------------------------------------------------------------------------
# GEMM

GEMM_SHAPES = [(1, 1, 1), (3, 5, 7), (64, 128, 16), (130, 200, 77), (257, 33, 300), (100, 64, 1000),
               (65, 129, 17), (5, 300, 31)]


@pytest.mark.parametrize("shape", GEMM_SHAPES)
@pytest.mark.parametrize("trans", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_vs_oracle(am, luts, orc, shape, trans):
    M, N, K = shape
    ta, tb = trans
    A = inp.normal((M, K), 31)
    B = inp.normal((K, N), 32)
    res = orc.gemm(A, B, "mitchell", 7)
    args = (A.T.copy() if ta else A, B.T.copy() if tb else B, ta, tb)
    got = run_gemm(am, luts("mitchell"), *args)
    assert_tol(got, res, f"{shape} {trans}")
    with exact_order(am):
        got = run_gemm(am, luts("mitchell"), *args)
    assert_bits(got, res.c32, f"{shape} {trans} vs c32")


def test_gemm_config1_256(am, luts, orc):
    """BASELINE config 1: 256^3, Mitchell m = 7."""
    A = inp.normal((256, 256), 1)
    B = inp.normal((256, 256), 2)
    res = orc.gemm(A, B, "mitchell", 7)
    assert_tol(run_gemm(am, luts("mitchell"), A, B), res)
    with exact_order(am):
        assert_bits(run_gemm(am, luts("mitchell"), A, B), res.c32)


def test_gemm_leading_dims_and_accumulate(am, luts, orc):
    import torch
    M, N, K = 70, 90, 40
    Abig = inp.normal((M, K + 9), 41)
    Bbig = inp.normal((K, N + 5), 42)
    A = dev(Abig)[:, :K]
    B = dev(Bbig)[:, :N]
    C0 = inp.normal((M, N + 3), 43)
    C = dev(C0)
    lut = luts("exact")
    with exact_order(am):
        am.amsim_gemm(lut, A, B, C[:, :N], accumulate=True)
    res = orc.gemm(Abig[:, :K], Bbig[:, :N], "exact", 7)
    got = host(C)
    want = (C0[:, :N] + res.c32).astype(np.float32)      # C + S, S formed from +0 (header semantics)
    assert_bits(got[:, :N], want)
    assert_bits(got[:, N:], C0[:, N:], "columns beyond N untouched")


def test_gemm_degenerate(am, luts):
    import torch
    lut = luts("exact")
    C = torch.full((3, 4), 7.0, device="cuda")
    am.amsim_gemm(lut, torch.empty((3, 0), device="cuda"), torch.empty((0, 4), device="cuda"), C)
    assert np.all(host(C) == 0.0) and not np.signbit(host(C)).any()
    C.fill_(7.0)
    am.amsim_gemm(lut, torch.empty((3, 0), device="cuda"), torch.empty((0, 4), device="cuda"), C, accumulate=True)
    assert np.all(host(C) == 7.0)
    am.amsim_gemm(lut, torch.empty((0, 5), device="cuda"), torch.ones((5, 4), device="cuda"),
                  torch.empty((0, 4), device="cuda"))
    assert am.lib().amsim_gemm(lut.handle, 0, 0, -1, 2, 2, None, 2, None, 2, None, 2, 0, None) == 1


def test_policy_careful_equals_fast(am, luts):
    A = inp.normal((200, 150), 51)
    B = inp.normal((150, 170), 52)
    lut = luts("mitchell")
    with exact_order(am):
        fast = run_gemm(am, lut, A, B)
    with exact_order(am, careful=True):
        careful = run_gemm(am, lut, A, B)
    assert_bits(fast, careful)


def test_determinism(am, luts):
    A = inp.normal((300, 257), 61)
    B = inp.normal((257, 190), 62)
    lut = luts("mbm")
    assert_bits(run_gemm(am, lut, A, B), run_gemm(am, lut, A, B))


def test_dense_layer_passes(am, luts, orc):
    """AMDENSE as GEMMs with the conv operand order
    (reading C11): fwd Y = X W (a = x), wgrad dW = X^T dY (a = x),
    dgrad dX = dY W^T (a = dy).  Asymmetric-order check with the MBM table."""
    B_, IN, OUT = 64, 400, 120
    X = inp.relu_normal((B_, IN), 71)
    W = inp.he_uniform((IN, OUT), IN, 72)
    dY = inp.normal((B_, OUT), 73, 2 ** -4)
    lut = luts("mbm")
    with exact_order(am):
        y = run_gemm(am, lut, X, W)
        dW = run_gemm(am, lut, X, dY, trans_a=True)
        dX = run_gemm(am, lut, dY, W, trans_b=True)
    assert_bits(y, orc.gemm(X, W, "mbm").c32)
    assert_bits(dW, orc.gemm(X.T.copy(), dY, "mbm").c32)
    assert_bits(dX, orc.gemm(dY, W.T.copy(), "mbm").c32)
    assert_tol(run_gemm(am, lut, X, dY, trans_a=True), orc.gemm(X.T.copy(), dY, "mbm"))


# ---------------------------------------------------------------------------
# convolutions

CONV = [
    # N, H, W, C, K, R, S, stride, pad
    (2, 5, 5, 3, 4, 3, 3, 1, 0),
    (2, 7, 6, 3, 2, 3, 3, 2, 1),
    (1, 8, 8, 2, 3, 3, 3, 3, 1),
    (2, 6, 6, 4, 5, 1, 1, 2, 0),
    (1, 9, 7, 2, 2, 5, 5, 2, 2),
    (3, 4, 4, 1, 1, 2, 2, 1, 0),
    (2, 12, 12, 8, 36, 3, 3, 1, 1),      # vectorised loads, several N tiles
    (2, 14, 14, 16, 72, 3, 3, 2, 1),     # stride-2 3x3, C % 4 == 0
    (3, 9, 9, 12, 130, 1, 1, 2, 0),      # 1x1 stride-2 downsample
    (2, 20, 20, 3, 16, 7, 7, 2, 3),      # stem geometry
    (4, 28, 28, 1, 6, 5, 5, 1, 2),       # LeNet c1
    (2, 7, 7, 16, 40, 1, 1, 1, 0),       # 1x1 stride 1: TMA-staged x (fwd, wgrad) and dy (dgrad)
    (1, 5, 9, 20, 32, 1, 1, 1, 0),       # 1x1 stride 1, K % 16 == 0: TMA weight taps in dgrad too
    (2, 9, 9, 8, 48, 3, 3, 1, 1),        # 3x3, K % 16 == 0: 3-D TMA weight taps in dgrad
    (2, 6, 6, 6, 32, 1, 1, 1, 0),        # 1x1 stride 1 with C % 4 != 0: cp.async fallback
    (2, 9, 9, 16, 32, 3, 3, 1, 1),       # C, K % 16 == 0: im2col-mode TMA for fwd x and stride-1 dgrad dy
    (3, 12, 10, 16, 16, 5, 5, 1, 2),     # 5x5 pad 2 im2col, ragged pixel tiles across images
    (2, 20, 20, 32, 16, 7, 7, 2, 3),     # 7x7 stride 2 im2col (traversal stride 2)
    (2, 9, 11, 16, 32, 3, 1, 1, 0),      # R != S im2col
    (2, 11, 11, 32, 48, 3, 3, 2, 0),     # stride 2 unpadded, (H - R) % S != 0
    (2, 9, 9, 64, 32, 3, 3, 1, 1),       # C % 64 == 0: im2col TMA for the wgrad activations too
    (1, 10, 10, 128, 64, 3, 3, 2, 1),    # C % 128 == 0, stride 2
]


def _conv_tensors(shape, seed):
    N, H, W, C, K, R, S, st, pd = shape
    OH = (H + 2 * pd - R) // st + 1
    OW = (W + 2 * pd - S) // st + 1
    x = inp.relu_normal((N, H, W, C), seed)
    w = inp.he_normal((R, S, C, K), R * S * C, seed + 1)
    dy = inp.normal((N, OH, OW, K), seed + 2, 0.5)
    return x, w, dy, OH, OW


def _run_conv(am, lut, d, x, w, dy, which):
    import torch
    N, H, W, C, K = d.N, d.H, d.W, d.C, d.K
    if which == "fwd":
        y = torch.full((N, d.OH, d.OW, K), float("nan"), device="cuda")
        am.amsim_conv2d_fwd(lut, d, dev(x), dev(w), y)
        return host(y).reshape(-1, K)
    if which == "dgrad":
        dx = torch.full((N, H, W, C), float("nan"), device="cuda")
        am.amsim_conv2d_bwd_data(lut, d, dev(dy), dev(w), dx)
        return host(dx).reshape(-1, C)
    dw = torch.full((d.R, d.S, C, K), float("nan"), device="cuda")
    nbytes = am.amsim_conv2d_bwd_filter_workspace(lut, d)
    ws = torch.empty(max(nbytes // 4, 1), device="cuda")
    am.amsim_conv2d_bwd_filter(lut, d, dev(x), dev(dy), dw, ws)
    return host(dw).reshape(-1, K)


@pytest.mark.parametrize("shape", CONV)
@pytest.mark.parametrize("which", ["fwd", "dgrad", "wgrad"])
@pytest.mark.parametrize("model", ["mitchell", "exact"])
def test_conv_vs_oracle(am, luts, orc, shape, which, model):
    N, H, W, C, K, R, S, st, pd = shape
    x, w, dy, OH, OW = _conv_tensors(shape, 100)
    d = am.conv_desc(N, H, W, C, K, R, S, st, pd)
    od = orc.conv_desc(N, H, W, C, K, R, S, st, pd)
    omodel = model
    lut = luts(omodel)
    got = _run_conv(am, lut, d, x, w, dy, which)
    if which == "fwd":
        res = orc.conv_fwd(od, x, w, omodel)
    elif which == "dgrad":
        res = orc.conv_bwd_data(od, dy, w, omodel)
    else:
        res = orc.conv_bwd_filter(od, x, dy, omodel)
    assert_tol(got, res, f"{which} {shape}")
    with exact_order(am):
        got = _run_conv(am, lut, d, x, w, dy, which)
    assert_bits(got, res.c32, f"{which} {shape} vs c32")


@pytest.mark.parametrize("model,m,width", [("mitchell", 7, 8), ("exact", 3, 8), ("mbm", 7, 16), ("exact", 6, 16),
                                             ("mitchell", 8, 16), ("mitchell", 5, 8), ("exact", 4, 16)])
def test_entry_layout_never_changes_bits(am, luts, orc, model, m, width):
    """The narrow device layouts (8-bit: carry | 7 mantissa bits; 16-bit) give
    the same bits as the 32-bit Alg. 1 layout (policy bit 2), for GEMM and all
    three conv passes; and the narrow layout matches the oracle's c32."""
    lut = luts(model, m)
    assert lut.info() == (m, width)
    A = inp.normal((150, 90), 71)
    B = inp.normal((90, 140), 72)
    shape = (2, 14, 14, 16, 72, 3, 3, 2, 1)
    x, w, dy, OH, OW = _conv_tensors(shape, 73)
    d = am.conv_desc(*shape)
    outs = {}
    for pol in (0, 4, 2, 6):
        am.amsim_set_path_policy(pol)
        try:
            outs[pol] = [run_gemm(am, lut, A, B)] + [_run_conv(am, lut, d, x, w, dy, k)
                                                      for k in ("fwd", "dgrad", "wgrad")]
        finally:
            am.amsim_set_path_policy(0)
    for i in range(4):
        # default plans compare bit for bit while both layouts keep the table in
        # shared memory (same tile configuration, hence the same stream-K
        # pieces); the 32-bit m = 8 table (256 KB) moves to global memory with
        # its own tile set, so there only the exact order is layout-independent
        if m <= 7:
            assert_bits(outs[0][i], outs[4][i], f"{model} m={m} part {i} split")
        assert_bits(outs[2][i], outs[6][i], f"{model} m={m} part {i} exact order")
    assert_tol(outs[0][3], orc.conv_bwd_filter(orc.conv_desc(*shape), x, dy, model, m), "wgrad default plan")
    assert_tol(outs[4][3], orc.conv_bwd_filter(orc.conv_desc(*shape), x, dy, model, m), "wgrad default plan, 32-bit")
    assert_bits(outs[2][0], orc.gemm(A, B, model, m).c32, "gemm vs c32")
    assert_bits(outs[2][1], orc.conv_fwd(orc.conv_desc(*shape), x, w, model, m).c32, "fwd vs c32")


def test_conv_operand_order_asymmetric(am, orc):
    """An asymmetric table must give a = x for fwd/wgrad and a = dy for dgrad
    (reading C11).  The user model is a Python callback passed through the
    function-pointer ABI: exact product of a with b's significand cut to 3
    fraction bits (the oracle implements the same model independently in C)."""
    import struct
    from paper_2209_04161_b200 import _lib

    @_lib.MUL_FN
    def asym(a, b):
        ub = struct.unpack("<I", struct.pack("<f", b))[0] & 0xFFF00000
        return a * struct.unpack("<f", struct.pack("<I", ub))[0]

    lut = am.Lut.build(asym, 7)
    shape = (2, 9, 9, 4, 8, 3, 3, 2, 1)
    N, H, W, C, K, R, S, st, pd = shape
    x, w, dy, OH, OW = _conv_tensors(shape, 200)
    d = am.conv_desc(N, H, W, C, K, R, S, st, pd)
    od = orc.conv_desc(N, H, W, C, K, R, S, st, pd)
    for which, res in (("fwd", orc.conv_fwd(od, x, w, "asym")), ("dgrad", orc.conv_bwd_data(od, dy, w, "asym")),
                       ("wgrad", orc.conv_bwd_filter(od, x, dy, "asym"))):
        with exact_order(am):
            got = _run_conv(am, lut, d, x, w, dy, which)
        assert_bits(got, res.c32, which)


def test_plan_cache_separates_symmetric_and_asymmetric_tables(am, luts, orc):
    """the transposed orientation reads LUT^T, so a plan made for a
    symmetric table (MBM, 16-bit entries) must not be reused for an asymmetric
    table of the same m and entry width on the same shape.  The MBM call comes
    first (it plans the transposed orientation for this 64-channel layer),
    then the asymmetric table, checked against the oracle in both plans."""
    import struct
    from paper_2209_04161_b200 import _lib

    @_lib.MUL_FN
    def asym(a, b):
        ub = struct.unpack("<I", struct.pack("<f", b))[0] & 0xFFF00000
        return a * struct.unpack("<f", struct.pack("<I", ub))[0]

    lut_a = am.Lut.build(asym, 7)
    assert lut_a.info() == luts("mbm").info() == (7, 16)
    shape = (4, 16, 16, 64, 64, 3, 3, 1, 1)
    x, w, dy, OH, OW = _conv_tensors(shape, 500)
    d, od = am.conv_desc(*shape), orc.conv_desc(*shape)
    for which in ("fwd", "dgrad", "wgrad"):
        for pol in (0, 2):
            am.amsim_set_path_policy(pol)
            try:
                _run_conv(am, luts("mbm"), d, x, w, dy, which)          # plans (and caches) for the symmetric table
                got = _run_conv(am, lut_a, d, x, w, dy, which)
            finally:
                am.amsim_set_path_policy(0)
            ref = {"fwd": lambda: orc.conv_fwd(od, x, w, "asym"), "dgrad": lambda: orc.conv_bwd_data(od, dy, w, "asym"),
                   "wgrad": lambda: orc.conv_bwd_filter(od, x, dy, "asym")}[which]()
            if pol:
                assert_bits(got, ref.c32, f"asym {which} after symmetric plan (exact order)")
            else:
                assert_tol(got, ref, f"asym {which} after symmetric plan")


@pytest.mark.parametrize("model", ["mbm", "exact"])
def test_lenet5_step_layers(am, luts, orc, model):
    """BASELINE config 2 shapes (LeNet-5, batch 64) with MNIST-like inputs."""
    lut = luts(model)
    am.amsim_set_path_policy(2)  # exact c32 order; the tolerance path is covered elsewhere
    try:
        _lenet(am, lut, orc, model)
    finally:
        am.amsim_set_path_policy(0)


def _lenet(am, lut, orc, model):
    for i, L in enumerate(inp.lenet5_layers(64)):
        if isinstance(L, inp.ConvLayer):
            shape = (L.N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)
            x = inp.mnist_like((L.N, L.H, L.W, L.C), 3 + i) if L.first else inp.relu_normal((L.N, L.H, L.W, L.C), 3 + i)
            w = inp.he_uniform((L.R, L.S, L.C, L.K), L.R * L.S * L.C, 4 + i)
            dy = inp.normal((L.N, L.OH, L.OW, L.K), 5 + i, 2 ** -8)
            d = am.conv_desc(*shape)
            od = orc.conv_desc(*shape)
            assert_bits(_run_conv(am, lut, d, x, w, dy, "fwd"), orc.conv_fwd(od, x, w, model).c32, L.name)
            r = orc.conv_bwd_filter(od, x, dy, model)
            assert_tol(_run_conv(am, lut, d, x, w, dy, "wgrad"), r, L.name)
            if not L.first:
                assert_bits(_run_conv(am, lut, d, x, w, dy, "dgrad"), orc.conv_bwd_data(od, dy, w, model).c32, L.name)
        else:
            X = inp.relu_normal((L.N, L.IN), 3 + i)
            W = inp.he_uniform((L.IN, L.OUT), L.IN, 4 + i)
            dY = inp.normal((L.N, L.OUT), 5 + i, 2 ** -8)
            assert_bits(run_gemm(am, lut, X, W), orc.gemm(X, W, model).c32, L.name)
            assert_bits(run_gemm(am, lut, X, dY, trans_a=True), orc.gemm(X.T.copy(), dY, model).c32, L.name)
            assert_bits(run_gemm(am, lut, dY, W, trans_b=True), orc.gemm(dY, W.T.copy(), model).c32, L.name)


# ---------------------------------------------------------------------------
# full BASELINE sizes, sampled outputs

FULL_LAYERS = ["stem", "l1.0.conv2", "l2.0.conv2", "l2.0.down", "l4.0.conv2", "l4.2.conv3"]


@pytest.mark.parametrize("name,model", [(n, "mbm") for n in FULL_LAYERS] +
                         [(n, "exact") for n in FULL_LAYERS[:3]] + [("l3.1.conv2", "mitchell")])
def test_resnet50_full_size_sampled(am, luts, orc, name, model):
    """ResNet-50 b256 layers at full size in the bench's launch configuration
    (the bench's MBM table: 16-bit packed path, TMA weight / error tiles, the
    planner's tile shapes and split-K); the oracle recomputes sampled output
    rows one by one."""
    import torch
    L = {l.name: l for l in inp.resnet50_layers(256)}[name]
    shape = (L.N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)
    d = am.conv_desc(*shape)
    od = orc.conv_desc(*shape)
    g = inp.rng(7)
    x = inp.relu_normal((L.N, L.H, L.W, L.C), 1000)
    w = inp.he_normal((L.R, L.S, L.C, L.K), L.R * L.S * L.C, 1001)
    dy = inp.normal((L.N, L.OH, L.OW, L.K), 1002, 2 ** -10)
    lut = luts(model)
    y = _run_conv(am, lut, d, x, w, dy, "fwd")
    rows = np.unique(np.concatenate([[0, y.shape[0] - 1], g.integers(0, y.shape[0], 14)]))
    res = orc.conv_fwd(od, x, w, model, rows=rows)
    assert_tol(y[rows], res, f"{name} fwd")
    with exact_order(am):
        y = _run_conv(am, lut, d, x, w, dy, "fwd")
    assert_bits(y[rows], res.c32, f"{name} fwd (exact order)")
    if not L.first:
        dx = _run_conv(am, lut, d, x, w, dy, "dgrad")
        rows = np.unique(np.concatenate([[0, dx.shape[0] - 1], g.integers(0, dx.shape[0], 14)]))
        res = orc.conv_bwd_data(od, dy, w, model, rows=rows)
        assert_tol(dx[rows], res, f"{name} dgrad")
    dw = _run_conv(am, lut, d, x, w, dy, "wgrad")
    rows = np.unique(np.concatenate([[0, dw.shape[0] - 1], g.integers(0, dw.shape[0], 6)]))
    res = orc.conv_bwd_filter(od, x, dy, model, rows=rows)
    assert_tol(dw[rows], res, f"{name} wgrad")
    torch.cuda.empty_cache()


@pytest.mark.parametrize("width", [8, 16, 32])
def test_lut_lookup_microbench(am, width):
    idx = inp.rng(3).integers(0, 128, 1 << 16).astype(np.uint32)
    r = am.amsim_bench_lut_lookup(7, width, idx, iters=256)
    assert r > 1e11


def test_dp_shard_sum_equals_full_batch(am, luts, orc):
    """The data-parallel identity on one device: wgrad of two batch shards,
    summed (what the NCCL all-reduce does), equals the full-batch wgrad within
    the reading-C12 tolerance."""
    import torch
    from paper_2209_04161_b200.dp import shard_batch
    N, H, W, C, K, R, S, st, pd = 6, 14, 14, 16, 32, 3, 3, 2, 1
    x, w, dy, OH, OW = _conv_tensors((N, H, W, C, K, R, S, st, pd), 300)
    lut = luts("mbm")
    full = _run_conv(am, lut, am.conv_desc(N, H, W, C, K, R, S, st, pd), x, w, dy, "wgrad")
    acc = np.zeros_like(full, dtype=np.float64)
    for r in range(2):
        s0, c = shard_batch(N, 2, r)
        acc += _run_conv(am, lut, am.conv_desc(c, H, W, C, K, R, S, st, pd), x[s0:s0 + c], w, dy[s0:s0 + c], "wgrad")
    res = orc.conv_bwd_filter(orc.conv_desc(N, H, W, C, K, R, S, st, pd), x, dy, "mbm")
    assert_tol(full, res, "full")
    assert np.all(np.abs(acc - res.c64) <= 1e-5 * res.abs64 + FLT_MIN)


def test_train_step_lenet(am, luts, orc):
    """The bench's TrainStep on LeNet-5 shapes (default plan, as the bench
    runs it): every pass through the C ABI; each weight gradient, read from
    the flat all-reduce buffer at its planned offset, and the outputs of one
    conv and one dense pass taken from inside the step, against the oracle."""
    import torch
    from paper_2209_04161_b200.train_step import TrainStep
    lut = luts("mbm")
    step = TrainStep(inp.lenet5_layers(64), lut, device="cuda", seed=5, first_input="mnist")
    n0 = am.amsim_launch_count()
    step.step()
    torch.cuda.synchronize()
    assert am.amsim_launch_count() - n0 >= 14          # 5 fwd + 5 wgrad + 4 dgrad passes
    flat = step.flat_grad.cpu().numpy()
    for ly in step.layers:
        l = ly.spec
        x, dy = ly.x.cpu().numpy(), ly.dy.cpu().numpy()
        off = ly.dw.storage_offset()
        got = flat[off:off + ly.dw.numel()]
        if ly.kind == "conv":
            ref = orc.conv_bwd_filter(orc.conv_desc(l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad), x, dy, "mbm")
        else:
            ref = orc.gemm(np.ascontiguousarray(x.T), dy, "mbm")
        assert_tol(got.reshape(ref.c64.shape), ref, f"{l.name} wgrad in the flat buffer")
    # the last forward output of each kind stays in the step's y scratch: re-run
    # one conv (c2) and one dense (f3) forward pass exactly as forward() does
    for ly in (step.layers[1], step.layers[2]):
        l = ly.spec
        step.timers = None
        if ly.kind == "conv":
            y = step.y_scratch[: l.N * l.OH * l.OW * l.K]
            am.amsim_conv2d_fwd(lut, ly.desc, ly.x, ly.w, y)
            ref = orc.conv_fwd(orc.conv_desc(l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad),
                               ly.x.cpu().numpy(), ly.w.cpu().numpy(), "mbm")
            assert_tol(host(y).reshape(ref.c64.shape), ref, f"{l.name} fwd")
        else:
            y = step.y_scratch[: l.N * l.OUT].view(l.N, l.OUT)
            am.amsim_gemm(lut, ly.x, ly.w, y)
            ref = orc.gemm(ly.x.cpu().numpy(), ly.w.cpu().numpy(), "mbm")
            assert_tol(host(y), ref, f"{l.name} fwd")
        # dgrad into the dx scratch
        if ly.kind == "conv":
            dx = step.dx_scratch[: l.N * l.H * l.W * l.C]
            am.amsim_conv2d_bwd_data(lut, ly.desc, ly.dy, ly.w, dx)
            ref = orc.conv_bwd_data(orc.conv_desc(l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad),
                                    ly.dy.cpu().numpy(), ly.w.cpu().numpy(), "mbm")
        else:
            dx = step.dx_scratch[: l.N * l.IN].view(l.N, l.IN)
            am.amsim_gemm(lut, ly.dy, ly.w, dx, trans_b=True)
            ref = orc.gemm(ly.dy.cpu().numpy(), np.ascontiguousarray(ly.w.cpu().numpy().T), "mbm")
        assert_tol(host(dx).reshape(ref.c64.shape), ref, f"{l.name} dgrad")


@pytest.mark.parametrize("model", ["mbm", "exact"])
def test_lenet5_default_plan(am, luts, orc, model):
    """BASELINE config 2 (LeNet-5 b64) in the DEFAULT launch plan the bench
    runs (split-K, transposed orientation, TMA where eligible): tolerance
    against the oracle for every pass (reading C12)."""
    lut = luts(model)
    for i, L in enumerate(inp.lenet5_layers(64)):
        if isinstance(L, inp.ConvLayer):
            shape = (L.N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)
            x = inp.mnist_like((L.N, L.H, L.W, L.C), 3 + i) if L.first else inp.relu_normal((L.N, L.H, L.W, L.C), 3 + i)
            w = inp.he_uniform((L.R, L.S, L.C, L.K), L.R * L.S * L.C, 4 + i)
            dy = inp.normal((L.N, L.OH, L.OW, L.K), 5 + i, 2 ** -8)
            d, od = am.conv_desc(*shape), orc.conv_desc(*shape)
            assert_tol(_run_conv(am, lut, d, x, w, dy, "fwd"), orc.conv_fwd(od, x, w, model), L.name + " fwd")
            assert_tol(_run_conv(am, lut, d, x, w, dy, "wgrad"), orc.conv_bwd_filter(od, x, dy, model), L.name + " wgrad")
            if not L.first:
                assert_tol(_run_conv(am, lut, d, x, w, dy, "dgrad"), orc.conv_bwd_data(od, dy, w, model),
                           L.name + " dgrad")
        else:
            X = inp.relu_normal((L.N, L.IN), 3 + i)
            W = inp.he_uniform((L.IN, L.OUT), L.IN, 4 + i)
            dY = inp.normal((L.N, L.OUT), 5 + i, 2 ** -8)
            assert_tol(run_gemm(am, lut, X, W), orc.gemm(X, W, model), L.name + " fwd")
            assert_tol(run_gemm(am, lut, X, dY, trans_a=True), orc.gemm(X.T.copy(), dY, model), L.name + " wgrad")
            assert_tol(run_gemm(am, lut, dY, W, trans_b=True), orc.gemm(dY, W.T.copy(), model), L.name + " dgrad")


def _distinct(layers):
    seen, out = set(), []
    for L in layers:
        key = (L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, L.first) if isinstance(L, inp.ConvLayer) else \
            ("dense", L.IN, L.OUT)
        if key not in seen:
            seen.add(key)
            out.append(L)
    return out


R18 = _distinct(inp.resnet18_cifar_layers(128))


@pytest.mark.parametrize("name", [L.name for L in R18])
def test_resnet18_cifar_full_size_sampled(am, luts, orc, name):
    """BASELINE config 3 (ResNet-18 CIFAR b128): every
    distinct pass shape at full size with the MBM table.  Default plan:
    sampled output rows within the reading-C12 tolerance; exact order (no
    split): the same rows bit-identical to the oracle's c32."""
    import torch
    L = {l.name: l for l in R18}[name]
    g = inp.rng(11)
    lut = luts("mbm")
    if isinstance(L, inp.DenseLayer):
        X = inp.relu_normal((L.N, L.IN), 2000)
        W = inp.he_normal((L.IN, L.OUT), L.IN, 2001)
        dY = inp.normal((L.N, L.OUT), 2002, 2 ** -10)
        for what, A, B, ta, tb in (("fwd", X, W, False, False), ("wgrad", X, dY, True, False),
                                   ("dgrad", dY, W, False, True)):
            ref = orc.gemm(A.T.copy() if ta else A, B.T.copy() if tb else B, "mbm")
            assert_tol(run_gemm(am, lut, A, B, trans_a=ta, trans_b=tb), ref, f"fc {what}")
            with exact_order(am):
                assert_bits(run_gemm(am, lut, A, B, trans_a=ta, trans_b=tb), ref.c32, f"fc {what} (exact order)")
        return
    shape = (L.N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)
    d, od = am.conv_desc(*shape), orc.conv_desc(*shape)
    x = inp.relu_normal((L.N, L.H, L.W, L.C), 2000)
    w = inp.he_normal((L.R, L.S, L.C, L.K), L.R * L.S * L.C, 2001)
    dy = inp.normal((L.N, L.OH, L.OW, L.K), 2002, 2 ** -10)
    passes = [("fwd", lambda rows: orc.conv_fwd(od, x, w, "mbm", rows=rows), 24),
              ("wgrad", lambda rows: orc.conv_bwd_filter(od, x, dy, "mbm", rows=rows), 6)]
    if not L.first:
        passes.append(("dgrad", lambda rows: orc.conv_bwd_data(od, dy, w, "mbm", rows=rows), 24))
    for which, oracle_rows, nsamp in passes:
        out = _run_conv(am, lut, d, x, w, dy, which)
        rows = np.unique(np.concatenate([[0, out.shape[0] - 1], g.integers(0, out.shape[0], nsamp)]))
        res = oracle_rows(rows)
        assert_tol(out[rows], res, f"{name} {which}")
        with exact_order(am):
            out = _run_conv(am, lut, d, x, w, dy, which)
        assert_bits(out[rows], res.c32, f"{name} {which} (exact order)")
    torch.cuda.empty_cache()


def test_resnet50_fc_full_size(am, luts, orc):
    """The ResNet-50 fc layer at size (256 x 2048 x 1000):
    fwd Y = X W, wgrad dW = X^T dY, dgrad dX = dY W^T through amsim_gemm in the
    bench's plan; sampled output rows against the oracle (tolerance), and bit
    equality with c32 in exact order."""
    L = [l for l in inp.resnet50_layers(256) if l.name == "fc"][0]
    g = inp.rng(12)
    X = inp.relu_normal((L.N, L.IN), 3000)
    W = inp.he_normal((L.IN, L.OUT), L.IN, 3001)
    dY = inp.normal((L.N, L.OUT), 3002, 2 ** -10)
    lut = luts("mbm")
    for what, A, B, ta, tb in (("fwd", X, W, False, False), ("wgrad", X, dY, True, False),
                               ("dgrad", dY, W, False, True)):
        Ao = np.ascontiguousarray(A.T) if ta else A
        Bo = np.ascontiguousarray(B.T) if tb else B
        out = run_gemm(am, lut, A, B, trans_a=ta, trans_b=tb)
        rows = np.unique(np.concatenate([[0, out.shape[0] - 1], g.integers(0, out.shape[0], 30)]))
        res = orc.gemm(Ao, Bo, "mbm", rows=rows)
        assert_tol(out[rows], res, f"fc {what}")
        with exact_order(am):
            out = run_gemm(am, lut, A, B, trans_a=ta, trans_b=tb)
        assert_bits(out[rows], res.c32, f"fc {what} (exact order)")


# ---------------------------------------------------------------------------
# measurement instruments: direct model evaluation (no table) and native multiply

@pytest.mark.parametrize("model,m", [("exact", 7), ("mitchell", 7), ("mbm", 7), ("exact", 11), ("mitchell", 4),
                                     ("mbm", 10), ("exact", 1)])
def test_direct_mode_equals_table(am, luts, orc, model, m):
    """AMSIM_MUL_DIRECT evaluates the built-in model per product on the device
    (the paper's "direct simulation") -- same bits as the
    table and the oracle, on the special-value grid (fast and careful paths)."""
    lut = luts(model, m)
    v = _sampled_grid(m) if m > 7 else inp.operand_grid(m)
    want = orc.mul(v[:, None], v[None, :], model, m)
    for policy in (0, 1):
        am.amsim_set_path_policy(policy)
        try:
            with am.multiply_mode(am.AMSIM_MUL_DIRECT):
                got = run_gemm(am, lut, v[:, None], v[None, :])
        finally:
            am.amsim_set_path_policy(0)
        assert_bits(got, want, f"direct {model} m={m} policy={policy}")


@pytest.mark.parametrize("model", ["exact", "mitchell", "mbm"])
def test_direct_mode_conv_equals_table(am, luts, model):
    lut = luts(model)
    shape = (2, 14, 14, 16, 72, 3, 3, 2, 1)
    x, w, dy, OH, OW = _conv_tensors(shape, 91)
    d = am.conv_desc(*shape)
    # exact order: the direct mode plans its own tile shapes (no table in shared
    # memory), so only the fixed k order makes the two plans comparable bit for bit
    for which in ("fwd", "dgrad", "wgrad"):
        with exact_order(am):
            ref = _run_conv(am, lut, d, x, w, dy, which)
            with am.multiply_mode(am.AMSIM_MUL_DIRECT):
                got = _run_conv(am, lut, d, x, w, dy, which)
        assert_bits(got, ref, f"{model} {which}")


def test_direct_mode_needs_builtin_model(am, luts):
    import torch
    lut = am.Lut.from_entries(luts("exact", 4).entries(), 4)
    C = torch.empty((2, 2), device="cuda")
    with am.multiply_mode(am.AMSIM_MUL_DIRECT):
        with pytest.raises(am.AmsimError):
            am.amsim_gemm(lut, torch.ones((2, 3), device="cuda"), torch.ones((3, 2), device="cuda"), C)


def test_native_mode_is_fp32_gemm(am, luts):
    """AMSIM_MUL_NATIVE (the ATnG analog): IEEE FP32 products of the
    UNtruncated operands, fma-accumulated from +0 in increasing k."""
    A = inp.normal((130, 300), 95)
    B = inp.normal((300, 70), 96)
    with exact_order(am), am.multiply_mode(am.AMSIM_MUL_NATIVE):
        got = run_gemm(am, luts("mbm"), A, B)
    want = np.zeros((130, 70), np.float32)
    for k in range(300):                       # sequential fp32 fma order
        want = (want.astype(np.float64) + A[:, k:k + 1].astype(np.float64) * B[k:k + 1, :]).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    absum = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    assert np.all(np.abs(got - ref) <= 1e-5 * absum)
    assert np.max(np.abs(got.astype(np.float64) - want)) <= 1e-6 * absum.max()


# ---------------------------------------------------------------------------
# (1, e, m) exponent casting (reading C23)

@pytest.mark.parametrize("model,m,e", [("exact", 10, 5), ("exact", 7, 5), ("mitchell", 7, 4), ("mbm", 7, 2),
                                       ("exact", 3, 1), ("mitchell", 7, 8)])
@pytest.mark.parametrize("policy", [0, 1])
def test_exponent_cast_per_product(am, luts, orc, model, m, e, policy):
    lut = luts(model, m).with_exponent_bits(e)
    assert lut.exponent_bits() == e
    v = _sampled_grid(m) if m > 7 else inp.operand_grid(m, exponents=(1, 60, 100, 110, 113, 120, 126, 127, 128, 134,
                                                                      141, 142, 150, 200, 254))
    am.amsim_set_path_policy(policy)
    try:
        got = run_gemm(am, lut, v[:, None], v[None, :])
    finally:
        am.amsim_set_path_policy(0)
    c = orc.cast_e(v, e)
    assert_bits(got, orc.mul(c[:, None], c[None, :], model, m), f"e={e} {model} m={m}")


@pytest.mark.parametrize("e", [5, 4])
def test_exponent_cast_gemm_and_conv(am, luts, orc, e):
    lut = luts("mitchell").with_exponent_bits(e)
    A = inp.normal((70, 90), 101) * np.float32(300.0)        # spans the e-bit range and beyond
    B = inp.normal((90, 50), 102) * np.float32(1e-3)
    shape = (2, 10, 10, 8, 36, 3, 3, 2, 1)
    x, w, dy, OH, OW = _conv_tensors(shape, 103)
    x = x * np.float32(1e3)
    d = am.conv_desc(*shape)
    od = orc.conv_desc(*shape)
    cx, cw, cdy = orc.cast_e(x, e), orc.cast_e(w, e), orc.cast_e(dy, e)
    with exact_order(am):
        assert_bits(run_gemm(am, lut, A, B), orc.gemm(orc.cast_e(A, e), orc.cast_e(B, e), "mitchell", 7).c32)
        assert_bits(_run_conv(am, lut, d, x, w, dy, "fwd"), orc.conv_fwd(od, cx, cw, "mitchell").c32, "fwd")
        assert_bits(_run_conv(am, lut, d, x, w, dy, "dgrad"), orc.conv_bwd_data(od, cdy, cw, "mitchell").c32, "dgrad")
        assert_bits(_run_conv(am, lut, d, x, w, dy, "wgrad"), orc.conv_bwd_filter(od, cx, cdy, "mitchell").c32, "wgrad")


# ---------------------------------------------------------------------------
# TMA-staged operand tiles (policy bit 3 forces cp.async everywhere)

def test_tma_staging_equals_cp_async(am, luts, orc):
    """Box-shaped operand tiles (GEMM A / B, conv fwd weights, wgrad errors,
    dgrad weight taps via 3-D maps, 1x1 / stride-1 activations and errors,
    1x1 strided errors (dgrad phase (0, 0)), 64-byte swizzled where k is
    contiguous) are loaded by TMA by default; the
    bits equal the all-cp.async path and the oracle, including ragged
    M / N / K edges (TMA zero fill)."""
    lut = luts("mbm")
    A = inp.normal((133, 77), 111)
    B = inp.normal((77, 204), 112)            # ldb = 204: 16-byte row pitch -> TMA eligible
    At = np.ascontiguousarray(inp.normal((77, 132), 113))   # trans_a, lda = 132 -> TMA eligible A
    shapes = [(3, 13, 11, 12, 40, 3, 3, 2, 1), (2, 9, 7, 16, 48, 1, 1, 1, 0), (2, 8, 8, 12, 32, 3, 3, 1, 1),
              (2, 10, 10, 8, 64, 3, 3, 2, 1), (3, 9, 9, 32, 48, 3, 3, 1, 1), (2, 15, 15, 16, 32, 3, 3, 2, 1),
              (2, 9, 9, 128, 64, 3, 3, 1, 1), (2, 12, 12, 64, 128, 3, 3, 2, 1), (2, 9, 7, 32, 48, 1, 1, 2, 0),
              (3, 10, 12, 16, 64, 1, 1, 2, 0)]
    outs = {}
    for pol in (2, 10):
        am.amsim_set_path_policy(pol)
        try:
            outs[pol] = [run_gemm(am, lut, A, B), run_gemm(am, lut, At, B, trans_a=True)]
            for k, shape in enumerate(shapes):
                x, w, dy, OH, OW = _conv_tensors(shape, 114 + k)
                d = am.conv_desc(*shape)
                outs[pol] += [_run_conv(am, lut, d, x, w, dy, which) for which in ("fwd", "wgrad", "dgrad")]
        finally:
            am.amsim_set_path_policy(0)
    for i in range(len(outs[2])):
        assert_bits(outs[2][i], outs[10][i], f"part {i}")
    assert_bits(outs[2][0], orc.gemm(A, B, "mbm", 7).c32, "gemm vs c32")
    assert_bits(outs[2][1], orc.gemm(np.ascontiguousarray(At.T), B, "mbm", 7).c32, "gemm trans_a vs c32")
    for k in (8, 9):   # 1x1 strided dgrad (TMA box of dy for phase (0, 0), zeros elsewhere) vs the oracle
        x, w, dy, OH, OW = _conv_tensors(shapes[k], 114 + k)
        want = orc.conv_bwd_data(orc.conv_desc(*shapes[k]), dy, w, "mbm").c32
        assert_bits(outs[2][2 + 3 * k + 2], want, f"{shapes[k]} dgrad vs c32")


# ---------------------------------------------------------------------------
# transposed orientation for skinny N (policy bit 4 disables it)

@pytest.mark.parametrize("model", ["mbm", "mitchell"])
def test_transposed_orientation_equals_normal(am, luts, orc, model):
    """For N <= 128 << M and a symmetric table the planner may make the output
    channels the warp-shared rows (the kernel computes C^T, the epilogue and
    split-K reduction write C transposed).  Same bits as the normal
    orientation and as the oracle's sequential order."""
    lut = luts(model)
    A = inp.normal((1000, 300), 121)
    B = inp.normal((300, 40), 122)
    shapes = [(4, 16, 16, 16, 32, 3, 3, 1, 1), (2, 20, 20, 64, 64, 1, 1, 1, 0), (3, 14, 14, 32, 48, 3, 3, 2, 1),
              (2, 12, 12, 128, 64, 3, 3, 1, 1)]
    outs = {}
    for pol in (2, 18, 0, 16):
        am.amsim_set_path_policy(pol)
        try:
            outs[pol] = [run_gemm(am, lut, A, B), run_gemm(am, lut, np.ascontiguousarray(A.T), B, trans_a=True)]
            for k, shape in enumerate(shapes):
                x, w, dy, OH, OW = _conv_tensors(shape, 123 + k)
                d = am.conv_desc(*shape)
                outs[pol] += [_run_conv(am, lut, d, x, w, dy, which) for which in ("fwd", "wgrad", "dgrad")]
        finally:
            am.amsim_set_path_policy(0)
    for i in range(len(outs[2])):
        assert_bits(outs[2][i], outs[18][i], f"exact order, part {i}")
    assert_bits(outs[2][0], orc.gemm(A, B, model, 7).c32, "gemm vs c32")
    res = orc.gemm(A, B, model, 7)
    assert_tol(outs[0][0], res, "gemm split")
    assert_tol(outs[16][0], res, "gemm split, normal orientation")


@pytest.mark.parametrize("force", ["14", "12", "15", "16", "18", "19", "6", "20"])
def test_transposed_orientation_forced(am, luts, orc, force, monkeypatch):
    """Every pass in the transposed orientation (AMSIM_FORCE_CFG >= 10 forces
    it wherever it is allowed), cp.async operand gathers (C % BN != 0) and TMA
    alike, against the oracle's sequential order."""
    lut = luts("mbm")
    monkeypatch.setenv("AMSIM_FORCE_CFG", force)
    for k, shape in enumerate([(2, 20, 20, 16, 16, 3, 3, 1, 1), (1, 18, 18, 32, 24, 1, 1, 1, 0),
                               (2, 16, 16, 64, 32, 3, 3, 1, 1)]):
        x, w, dy, OH, OW = _conv_tensors(shape, 140 + k)
        d = am.conv_desc(*shape)
        od = orc.conv_desc(*shape)
        with exact_order(am):
            assert_bits(_run_conv(am, lut, d, x, w, dy, "fwd"), orc.conv_fwd(od, x, w, "mbm").c32, f"{shape} fwd")
            assert_bits(_run_conv(am, lut, d, x, w, dy, "wgrad"), orc.conv_bwd_filter(od, x, dy, "mbm").c32,
                        f"{shape} wgrad")
            assert_bits(_run_conv(am, lut, d, x, w, dy, "dgrad"), orc.conv_bwd_data(od, dy, w, "mbm").c32,
                        f"{shape} dgrad")
        assert_tol(_run_conv(am, lut, d, x, w, dy, "wgrad"), orc.conv_bwd_filter(od, x, dy, "mbm"), f"{shape} wgrad split")
    A = inp.normal((700, 90), 150)
    B = inp.normal((90, 30), 151)
    with exact_order(am):
        assert_bits(run_gemm(am, lut, A, B), orc.gemm(A, B, "mbm", 7).c32, "gemm")


@pytest.mark.parametrize("force", [None, "1", "2", "12", "14", "15", "16", "18"])
def test_wgrad_multi_tap_tma(am, luts, orc, force, monkeypatch):
    """wgrad activation tiles whose rows span several taps (rows a multiple of a
    power-of-two C >= 32: one TMA im2col box per tap, smem tap-blocked; the
    tap blocks past R*S*C are zero-filled) give the same bits as the cp.async
    gather (policy bit 5) and the oracle's sequential order, in both
    orientations, with ragged tap counts, strides, 5x5 taps and ragged pixels."""
    lut = luts("mbm")
    if force:
        monkeypatch.setenv("AMSIM_FORCE_CFG", force)
    shapes = [(2, 12, 12, 32, 48, 3, 3, 1, 1), (2, 11, 11, 64, 32, 3, 3, 2, 1), (2, 9, 9, 32, 40, 5, 5, 1, 2),
              (1, 10, 10, 128, 24, 3, 3, 1, 1), (3, 7, 9, 64, 16, 3, 3, 1, 1)]
    for k, shape in enumerate(shapes):
        x, w, dy, OH, OW = _conv_tensors(shape, 170 + k)
        d = am.conv_desc(*shape)
        od = orc.conv_desc(*shape)
        got = {}
        for pol in (2, 2 | 32):
            am.amsim_set_path_policy(pol)
            try:
                got[pol] = _run_conv(am, lut, d, x, w, dy, "wgrad")
            finally:
                am.amsim_set_path_policy(0)
        want = orc.conv_bwd_filter(od, x, dy, "mbm")
        assert_bits(got[2], want.c32, f"{shape} multi-tap TMA vs c32")
        assert_bits(got[2 | 32], want.c32, f"{shape} cp.async vs c32")
        assert_tol(_run_conv(am, lut, d, x, w, dy, "wgrad"), want, f"{shape} split")


@pytest.mark.parametrize("force", [None, "2", "5", "16", "15", "20"])
def test_strided_dgrad_phase_tma(am, luts, orc, force, monkeypatch):
    """Stride-2 dgrad reads dy through one im2col TMA descriptor per stride
    phase (lower corner from the phase's first tap, upper from its extent):
    the oracle's bits in exact order and the cp.async gather's (policy bit 5),
    odd and even sizes, pads 0..2, 3x3 / 5x5 / 2x2 / 1x3 kernels, both
    orientations."""
    if force:
        monkeypatch.setenv("AMSIM_FORCE_CFG", force)
    lut = luts("mbm")
    shapes = [(2, 14, 14, 16, 32, 3, 3, 2, 1), (2, 13, 11, 8, 48, 3, 3, 2, 1), (2, 15, 15, 16, 16, 5, 5, 2, 2),
              (3, 10, 12, 12, 32, 2, 2, 2, 0), (2, 9, 9, 24, 16, 1, 3, 2, 0), (2, 11, 11, 32, 64, 3, 3, 2, 0)]
    for k, shape in enumerate(shapes):
        x, w, dy, OH, OW = _conv_tensors(shape, 210 + k)
        d = am.conv_desc(*shape)
        want = orc.conv_bwd_data(orc.conv_desc(*shape), dy, w, "mbm")
        got = {}
        for pol in (2, 2 | 32):
            am.amsim_set_path_policy(pol)
            try:
                got[pol] = _run_conv(am, lut, d, x, w, dy, "dgrad")
            finally:
                am.amsim_set_path_policy(0)
            assert_bits(got[pol], want.c32, f"{shape} dgrad policy {pol}")
        assert_tol(_run_conv(am, lut, d, x, w, dy, "dgrad"), want, f"{shape} dgrad split")


@pytest.mark.parametrize("policy", [2 | 16, 2 | 16 | 4])
def test_zero_row_skipping_bits(am, luts, orc, policy):
    """Normal orientation (policy bit 4), 16- and 32-bit table layouts: warp-
    shared A elements that are +0, -0 or subnormal (zero exponent field) have
    their lookups predicated off; rows that start with zeros (no entry loaded
    yet), alternate, or are all zero give the oracle's c32 bits, as do the
    conv fwd / wgrad passes on ReLU activations."""
    lut = luts("mbm")
    g = inp.rng(190)
    M, N, K = 300, 200, 150
    A = inp.normal((M, K), 191)
    z = g.random((M, K)) < 0.6
    A[z] = 0.0
    A[g.random((M, K)) < 0.05] = -0.0
    sub = g.random((M, K)) < 0.03
    A[sub] = (g.integers(1, 1 << 23, int(sub.sum())).astype(np.uint32)).view(np.float32)
    A[:7, :] = 0.0           # all-zero rows
    A[7:20, :40] = 0.0       # rows whose first k-tiles are all zero
    A[:, ::5] = -0.0
    B = inp.normal((K, N), 192)
    shape = (2, 12, 12, 32, 64, 3, 3, 1, 1)
    x, w, dy, OH, OW = _conv_tensors(shape, 193)
    d = am.conv_desc(*shape)
    od = orc.conv_desc(*shape)
    am.amsim_set_path_policy(policy)
    try:
        got = run_gemm(am, lut, A, B)
        fwd = _run_conv(am, lut, d, x, w, dy, "fwd")
        wgr = _run_conv(am, lut, d, x, w, dy, "wgrad")
    finally:
        am.amsim_set_path_policy(0)
    assert_bits(got, orc.gemm(A, B, "mbm", 7).c32, "gemm with zero / subnormal rows")
    assert_bits(fwd, orc.conv_fwd(od, x, w, "mbm").c32, "fwd")
    assert_bits(wgr, orc.conv_bwd_filter(od, x, dy, "mbm").c32, "wgrad")


@pytest.mark.parametrize("model", ["mbm", "mitchell"])
@pytest.mark.parametrize("policy", [2, 0])
def test_zero_row_branch_skipping_16x8(am, luts, orc, model, policy, monkeypatch):
    """Conv fwd / wgrad on the normal-orientation 16 x 8 tile (AMSIM_FORCE_CFG=5),
    where a zero warp-shared layer-input element skips its whole row (lookups,
    IMAD, FFMA) by a uniform branch: inputs with +0, -0 and subnormal elements,
    all-zero pixels and channels, for the 16-bit (MBM) and 8-bit (Mitchell)
    layouts -- the oracle's c32 bits in exact order (policy bit 1), the C12
    tolerance in the default (stream-K) plan."""
    monkeypatch.setenv("AMSIM_FORCE_CFG", "5")
    lut = luts(model)
    g = inp.rng(260)
    for k, shape in enumerate([(2, 13, 13, 32, 256, 3, 3, 1, 1), (3, 9, 9, 64, 300, 1, 1, 1, 0)]):
        x, w, dy, OH, OW = _conv_tensors(shape, 261 + k)
        x[g.random(x.shape) < 0.1] = -0.0
        sub = g.random(x.shape) < 0.03
        x[sub] = (g.integers(1, 1 << 23, int(sub.sum())).astype(np.uint32)).view(np.float32)
        x[0, :3] = 0.0            # all-zero pixels (rows of the fwd A operand)
        x[..., :5] = 0.0          # all-zero channels (rows of the wgrad A operand)
        d, od = am.conv_desc(*shape), orc.conv_desc(*shape)
        refs = {"fwd": orc.conv_fwd(od, x, w, model), "wgrad": orc.conv_bwd_filter(od, x, dy, model)}
        am.amsim_set_path_policy(policy)
        try:
            outs = {which: _run_conv(am, lut, d, x, w, dy, which) for which in refs}
        finally:
            am.amsim_set_path_policy(0)
        for which, ref in refs.items():
            if policy & 2:
                assert_bits(outs[which], ref.c32, f"{model} {shape} {which} (exact order)")
            else:
                assert_tol(outs[which], ref, f"{model} {shape} {which}")


@pytest.mark.parametrize("model", ["mbm", "mitchell"])
def test_tall_tiles_129_to_160_rows(am, luts, orc, model, monkeypatch):
    """Problems of 129..160 rows (the stem's wgrad: M = 7*7*3 = 147) may use
    the 160 x 64 Tall tiles (20 x 2 register tiles); forced (AMSIM_FORCE_CFG=7)
    and automatic plans give the oracle's bits in exact order and meet the
    tolerance with split-K, including ragged rows / columns and the C = 3
    activation gather."""
    lut = luts(model)
    shape = (2, 20, 20, 3, 24, 7, 7, 2, 3)
    x, w, dy, OH, OW = _conv_tensors(shape, 180)
    d = am.conv_desc(*shape)
    od = orc.conv_desc(*shape)
    A = inp.normal((150, 333), 181)
    B = inp.normal((333, 70), 182)
    for force in ("7", "19", None):
        if force:
            monkeypatch.setenv("AMSIM_FORCE_CFG", force)
        else:
            monkeypatch.delenv("AMSIM_FORCE_CFG", raising=False)
        want = orc.conv_bwd_filter(od, x, dy, model)
        with exact_order(am):
            assert_bits(_run_conv(am, lut, d, x, w, dy, "wgrad"), want.c32, f"force={force} wgrad")
            assert_bits(run_gemm(am, lut, A, B), orc.gemm(A, B, model, 7).c32, f"force={force} gemm")
        assert_tol(_run_conv(am, lut, d, x, w, dy, "wgrad"), want, f"force={force} wgrad split")
        assert_tol(run_gemm(am, lut, A, B), orc.gemm(A, B, model, 7), f"force={force} gemm split")


@pytest.mark.parametrize("force", [None, "14", "16", "6"])
def test_gemm_accumulate_and_leading_dims_transposed(am, luts, orc, force, monkeypatch):
    """C += A B with padded leading dimensions in both orientations (the
    transposed epilogue's read-modify-write path and its split-K reduction)."""
    if force:
        monkeypatch.setenv("AMSIM_FORCE_CFG", force)
    M, N, K = 900, 24, 700
    Abig = inp.normal((M, K + 3), 161)
    Bbig = inp.normal((K, N + 5), 162)
    C0 = inp.normal((M, N + 7), 163)
    A = dev(Abig)[:, :K]
    B = dev(Bbig)[:, :N]
    lut = luts("mbm")
    res = orc.gemm(Abig[:, :K], Bbig[:, :N], "mbm", 7)
    for exact in (True, False):
        C = dev(C0)
        if exact:
            with exact_order(am):
                am.amsim_gemm(lut, A, B, C[:, :N], accumulate=True)
        else:
            am.amsim_gemm(lut, A, B, C[:, :N], accumulate=True)
        got = host(C)
        if exact:
            assert_bits(got[:, :N], (C0[:, :N] + res.c32).astype(np.float32), "C + S exact order")
        else:
            err = np.abs(got[:, :N].astype(np.float64) - (C0[:, :N].astype(np.float64) + res.c64))
            assert np.all(err <= 1e-5 * res.abs64 + np.abs(C0[:, :N]) * 2 ** -23 + FLT_MIN)
        assert_bits(got[:, N:], C0[:, N:], "columns beyond N untouched")


# ---------------------------------------------------------------------------
# M-sharded GEMM (SURVEY.md §8(e), config 5 at N GPUs)

@pytest.mark.parametrize("world", [2, 3, 8])
def test_gemm_row_shards_bit_identical(am, luts, orc, world):
    """Each rank's row block (dp.sharded_gemm: amsim_gemm on A[r0:r0+n], C[r0:r0+n])
    in exact order is bit-identical to the single-GPU GEMM and the oracle's c32;
    in the default launch configuration (the planner may pick other tiles /
    split-K for the smaller M) it meets the GEMM tolerance against the oracle."""
    import torch
    from paper_2209_04161_b200.dp import sharded_gemm
    M, N, K = 1000, 384, 1040
    Ah, Bh = inp.normal((M, K), 41), inp.normal((K, N), 42)
    A, B = dev(Ah), dev(Bh)
    res = orc.gemm(Ah, Bh, "mitchell", 7)
    lut = luts("mitchell")
    for policy in (0, 2):
        am.amsim_set_path_policy(policy)
        try:
            C = torch.full((M, N), float("nan"), device="cuda")
            cover = np.zeros(M, int)
            for r in range(world):
                r0, n = sharded_gemm(am, lut, A, B, C, world, r)
                cover[r0:r0 + n] += 1
            assert (cover == 1).all()
            if policy == 2:
                full = torch.empty((M, N), device="cuda")
                am.amsim_gemm(lut, A, B, full)
                assert_bits(host(C), host(full), f"world {world}: shards vs one GEMM")
                assert_bits(host(C), res.c32, f"world {world}: shards vs oracle c32")
            else:
                assert_tol(host(C), res, f"world {world}")
        finally:
            am.amsim_set_path_policy(0)


def test_gemm_16384_rank_block_sampled(am, luts, orc):
    """Config 5 at full size in the bench's launch configuration
    (bench.py --workload gemm): the last rank's block of 16384^3 at 8 GPUs
    (2048 x 16384 x 16384, Mitchell m = 7), sampled rows against the oracle."""
    import torch
    from amsim_inputs import device as gen
    from paper_2209_04161_b200.dp import sharded_gemm
    n = 16384
    A = gen.normal((n, n), 1, device="cuda")
    B = gen.normal((n, n), 2, device="cuda")
    C = torch.full((n, n), float("nan"), device="cuda")
    r0, rows = sharded_gemm(am, luts("mitchell"), A, B, C, 8, 7)
    assert (r0, rows) == (14336, 2048)
    sample = np.array([r0, r0 + 1, r0 + 977, n - 1])
    Ah = A[torch.from_numpy(sample).cuda()].cpu().numpy()
    res = orc.gemm(Ah, B.cpu().numpy(), "mitchell", 7)
    assert_tol(host(C)[sample], res, "16384^3 rank 7 of 8")
    assert torch.isnan(C[:r0]).all()
    del A, B, C
    torch.cuda.empty_cache()


def test_first_call_inside_graph_capture(am, orc):
    """A table's first use on a device may happen inside CUDA graph capture:
    the upload runs on a private stream in relaxed capture mode, the graph
    holds only the compute launch, and its replays give the oracle's bits."""
    import torch
    lut = am.Lut.build("mitchell", 6)          # fresh handle: not yet uploaded
    A = inp.normal((70, 48), 81)
    B = inp.normal((48, 90), 82)
    Ad, Bd = dev(A), dev(B)
    C = torch.full((70, 90), float("nan"), device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    am.amsim_set_path_policy(2)
    try:
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                am.amsim_gemm(lut, Ad, Bd, C)
    finally:
        am.amsim_set_path_policy(0)
    g.replay()
    assert_bits(host(C), orc.gemm(A, B, "mitchell", 6).c32, "captured first call")
    C.fill_(float("nan"))
    g.replay()
    assert_bits(host(C), orc.gemm(A, B, "mitchell", 6).c32, "second replay")


def test_path_policy_is_per_thread(am, luts, orc):
    """amsim_set_path_policy affects only the calling thread: a worker thread
    forcing exact order (policy bit 1) gets the oracle's c32 bits, and the main
    thread's default-plan result is unchanged before and after."""
    import threading
    A = inp.normal((64, 65536), 83)
    B = inp.normal((65536, 64), 84)
    lut = luts("mbm")
    before = run_gemm(am, lut, A, B)
    out = {}

    def worker():
        am.amsim_set_path_policy(2)
        out["exact"] = run_gemm(am, lut, A, B)

    t = threading.Thread(target=worker)
    t.start()
    t.join()
    after = run_gemm(am, lut, A, B)
    assert_bits(after, before, "main thread default plan")
    ref = orc.gemm(A, B, "mbm")
    assert_bits(out["exact"], ref.c32, "worker thread exact order")
    assert_tol(before, ref, "main thread")


# ---------------------------------------------------------------------------
# stream-K schedule (SubP in csrc/amsim_device.cuh): the pieces of a tile are
# summed by a binary tree over their k order that depends only on the plan
# (each node added by the second of its two subtrees to finish)

SK_CASES = [
    # (kind, args): GEMM (M, N, K) or conv shape; chosen so tiles are cut into
    # 1, 2 and many pieces, with fewer stream-K CTAs than SMs, ragged edges,
    # several sub-problems with K = 0 tiles (strided 1x1 / stride-3 dgrad)
    ("gemm", (64, 64, 200000)),        # one tile, cut into ~G pieces
    ("gemm", (130, 70, 3000)),         # few tiles, W / 4 < G: fewer CTAs
    ("gemm", (1000, 300, 777)),        # ragged, pieces straddle tile ends
    ("gemm", (2048, 1000, 256)),       # the ResNet-50 fc shape (tile count not a multiple of G)
    ("conv", (3, 17, 17, 16, 24, 1, 1, 2, 0)),    # 1x1 stride 2: 3 of 4 dgrad phases have K = 0
    ("conv", (2, 19, 19, 16, 32, 3, 3, 3, 1)),    # stride 3: 9 phases, uneven K
    ("conv", (4, 16, 16, 64, 64, 3, 3, 1, 1)),    # 64-channel layer (transposed orientation)
]


@pytest.mark.parametrize("case", range(len(SK_CASES)))
@pytest.mark.parametrize("sched", ["sk", "dp"])
def test_stream_k_schedule(am, luts, orc, case, sched, monkeypatch):
    """Forced stream-K (AMSIM_SCHED=sk) and forced data-parallel tiles give
    results within the reading-C12 tolerance of the oracle, and a repeated
    call is bit-identical (the pieces and their order depend only on the
    plan, not on which CTA finishes last)."""
    monkeypatch.setenv("AMSIM_SCHED", sched)
    kind, args = SK_CASES[case]
    lut = luts("mbm")
    if kind == "gemm":
        M, N, K = args
        A = inp.normal((M, K), 90 + case)
        B = inp.normal((K, N), 91 + case)
        outs = [run_gemm(am, lut, A, B) for _ in range(2)]
        assert_bits(outs[1], outs[0], "repeat")
        rows = np.unique(np.concatenate([[0, M - 1], inp.rng(case).integers(0, M, 20)]))
        assert_tol(outs[0][rows], orc.gemm(A, B, "mbm", rows=rows), f"gemm {args}")
        C0 = inp.normal((M, N), 92 + case)
        got = run_gemm(am, lut, A, B, C0=C0, accumulate=True)
        ref = orc.gemm(A, B, "mbm", rows=rows)
        err = np.abs(got[rows].astype(np.float64) - (ref.c64 + C0[rows]))
        assert np.all(err <= 1e-5 * (ref.abs64 + np.abs(C0[rows])) + FLT_MIN), "accumulate"
        return
    x, w, dy, OH, OW = _conv_tensors(args, 95 + case)
    d, od = am.conv_desc(*args), orc.conv_desc(*args)
    for which, ref in (("fwd", lambda: orc.conv_fwd(od, x, w, "mbm")), ("dgrad", lambda: orc.conv_bwd_data(od, dy, w, "mbm")),
                       ("wgrad", lambda: orc.conv_bwd_filter(od, x, dy, "mbm"))):
        outs = [_run_conv(am, lut, d, x, w, dy, which) for _ in range(2)]
        assert_bits(outs[1], outs[0], f"{which} repeat")
        assert_tol(outs[0], ref(), f"{args} {which}")


def test_stream_k_transposed_and_forced_configs(am, luts, orc, monkeypatch):
    """Stream-K pieces in the transposed orientation (the epilogue writes
    C^T) and with several forced tile configurations."""
    monkeypatch.setenv("AMSIM_SCHED", "sk")
    shape = (2, 20, 20, 64, 48, 3, 3, 1, 1)
    x, w, dy, OH, OW = _conv_tensors(shape, 120)
    d, od = am.conv_desc(*shape), orc.conv_desc(*shape)
    lut = luts("mbm")
    refs = {"fwd": orc.conv_fwd(od, x, w, "mbm"), "dgrad": orc.conv_bwd_data(od, dy, w, "mbm"),
            "wgrad": orc.conv_bwd_filter(od, x, dy, "mbm")}
    for force in ("14", "12", "16", "2", "5", "0"):
        monkeypatch.setenv("AMSIM_FORCE_CFG", force)
        for which, ref in refs.items():
            assert_tol(_run_conv(am, lut, d, x, w, dy, which), ref, f"force={force} {which}")


@pytest.mark.parametrize("policy", [0, 8, 32])
def test_flat8_narrow_tile(am, luts, orc, policy, monkeypatch):
    """The 64 x 512 transposed tile (AMSIM_FORCE_CFG=20, narrow shared-memory
    layout, lane tiles loaded as two 256-row TMA boxes): conv fwd and dgrad of
    64-channel layers -- 3x3 stride 1 (im2col boxes), stride 2 (per-phase
    boxes), 1x1 (2-D boxes) -- with pixel counts that leave ragged 512-lane
    tiles; bits in exact order, tolerance in the default plan.  Policy bits 3 /
    5 (cp.async gathers) make the planner fall back to a padded tile."""
    monkeypatch.setenv("AMSIM_FORCE_CFG", "20")
    lut = luts("mbm")
    for k, shape in enumerate([(3, 15, 15, 64, 64, 3, 3, 1, 1), (2, 23, 23, 64, 64, 3, 3, 2, 1),
                               (3, 14, 13, 256, 64, 1, 1, 1, 0), (2, 17, 17, 64, 48, 1, 1, 2, 0)]):
        x, w, dy, OH, OW = _conv_tensors(shape, 230 + k)
        d, od = am.conv_desc(*shape), orc.conv_desc(*shape)
        refs = {"fwd": orc.conv_fwd(od, x, w, "mbm"), "dgrad": orc.conv_bwd_data(od, dy, w, "mbm")}
        for which, ref in refs.items():
            am.amsim_set_path_policy(policy | 2)
            try:
                got = _run_conv(am, lut, d, x, w, dy, which)
            finally:
                am.amsim_set_path_policy(0)
            assert_bits(got, ref.c32, f"{shape} {which} policy {policy} (exact order)")
            am.amsim_set_path_policy(policy)
            try:
                got = _run_conv(am, lut, d, x, w, dy, which)
            finally:
                am.amsim_set_path_policy(0)
            assert_tol(got, ref, f"{shape} {which} policy {policy}")
