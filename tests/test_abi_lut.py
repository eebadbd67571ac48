"""CPU tests of libamsim's C ABI: the library loads, exports every symbol
include/amsim.h declares, and its host-side Alg. 1 table build / file I/O /
error paths behave.  The table is checked exhaustively against the ORACLE's
direct functional-model products (independent implementations).  No GPU.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2209_04161_b200 as am
from paper_2209_04161_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def built():
    from paper_2209_04161_b200 import build
    build.build()
    return am.lib()


def test_exports_every_declared_symbol(built):
    hdr = open(os.path.join(ROOT, "include", "amsim.h")).read()
    declared = set(re.findall(r"\b(amsim_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS)
    nn = set(re.findall(r"\b(amsim_[a-z0-9_]+)\s*\(", open(os.path.join(ROOT, "include", "amsim_nn.h")).read()))
    assert nn == set(_lib.NN_EXPORTS)
    declared |= nn
    for name in declared:
        assert hasattr(built, name), name
    assert built.amsim_abi_version() == 1


def _oracle_table(orc, model, m):
    """Alg. 1 entries derived from the oracle's direct model products on the
    probe operands 1.k, 1.j (exponent field 127)."""
    n = 1 << m
    k, j = np.meshgrid(np.arange(n, dtype=np.uint32), np.arange(n, dtype=np.uint32), indexing="ij")
    a = ((127 << 23) | (k.ravel() << (23 - m))).astype(np.uint32).view(np.float32)
    b = ((127 << 23) | (j.ravel() << (23 - m))).astype(np.uint32).view(np.float32)
    c = orc.mul(a, b, model, m).view(np.uint32)
    ec = (c >> 23) & 0xFF
    assert np.all((ec == 127) | (ec == 128)) and np.all(c >> 31 == 0)
    return ((ec - 127).astype(np.uint32) << 23) | (c & 0x7FFFFF)


@pytest.mark.parametrize("model", ["exact", "mitchell", "mbm"])
@pytest.mark.parametrize("m", list(range(1, 12)))
def test_lut_exhaustive_vs_oracle_models(built, orc, model, m):
    lut = am.Lut.build(model, m)
    e = lut.entries()
    assert e.size == 1 << (2 * m) and e.nbytes == 4 << (2 * m)   # 2^(2M) x 4 B
    assert np.all(e >> 24 == 0)
    assert np.array_equal(e, _oracle_table(orc, model, m))
    if model in ("exact", "mitchell"):                            # symmetric tables
        n = 1 << m
        t = e.reshape(n, n)
        assert np.array_equal(t, t.T)


def test_lut_sizes_match_paper(built):
    assert am.Lut.build("exact", 1).entries().nbytes == 16         # PAPER.md:392 "1 (16 Bytes)"
    assert am.Lut.build("exact", 7).entries().nbytes == 65536      # PAPER.md:342 "65.53 kB"
    assert am.Lut.build("exact", 11).entries().nbytes == 16777216  # PAPER.md:392 "11 (16.8MB"


def test_m1_exact_table(built):
    assert list(am.Lut.build("exact", 1).entries()) == [0x0, 0x400000, 0x400000, 0x900000]


def test_device_entry_width(built):
    # exact at m=7: products of 8-bit significands need 15 fraction bits -> 16-bit entries
    assert am.Lut.build("exact", 7).info() == (7, 16)
    assert am.Lut.build("mbm", 7).info() == (7, 16)
    # Mitchell: carry + the m-bit sum of the operand mantissas -> 8-bit entries up to m = 7
    assert am.Lut.build("mitchell", 7).info() == (7, 8)
    assert am.Lut.build("mitchell", 8).info() == (8, 16)
    # every table whose entries fit 8 bits gets the 8-bit layout (round 2: with the
    # 16 x 8 tiles it is 19 % faster than 16-bit rows also where those fit one
    # wavefront, m <= 6): Mitchell m <= 7, exact m <= 3
    assert am.Lut.build("mitchell", 6).info() == (6, 8)
    assert am.Lut.build("mitchell", 1).info() == (1, 8)
    assert am.Lut.build("exact", 3).info() == (3, 8)
    assert am.Lut.build("exact", 4).info() == (4, 16)
    assert am.Lut.build("exact", 11).info() == (11, 32)


@pytest.mark.parametrize("model", ["exact", "mitchell", "mbm"])
def test_builtin_models_match_oracle_models(built, orc, model):
    """The library's integer-arithmetic models agree with the oracle's
    independent double-arithmetic models on random normal operands."""
    g = np.random.default_rng(3)
    e = g.integers(64, 190, 4000).astype(np.uint32)  # product exponent in range (Alg. 2 calls models only there)
    mant = g.integers(0, 1 << 23, 4000).astype(np.uint32)
    s = g.integers(0, 2, 4000).astype(np.uint32)
    a = ((s << 31) | (e << 23) | mant).view(np.float32)
    b = np.roll(a, 7)
    for m in (7, 11):
        mask = np.uint32((0xFFFFFFFF << (23 - m)) & 0xFFFFFFFF)
        at = (a.view(np.uint32) & mask).view(np.float32)
        bt = (b.view(np.uint32) & mask).view(np.float32)
        for i in range(0, 4000, 3):
            got = np.float32(am.model_call(model, float(at[i]), float(bt[i])))
            want = np.float32(orc.model_call(model, float(at[i]), float(bt[i])))
            assert got.view(np.uint32) == want.view(np.uint32)


def test_lut_file_roundtrip_and_errors(built, tmp_path):
    lut = am.Lut.build("mitchell", 7)
    p = str(tmp_path / "mit7.amlt")
    lut.save(p)
    raw = open(p, "rb").read()
    assert raw[:4] == b"AMLT" and raw[4] == 1 and raw[5] == 7 and len(raw) == 8 + 65536
    back = am.Lut.load(p)
    assert np.array_equal(back.entries(), lut.entries())
    bad = {
        "magic": b"XMLT" + raw[4:],
        "version": raw[:4] + b"\x02" + raw[5:],
        "m12": raw[:5] + b"\x0c" + raw[6:],
        "truncated": raw[:-3],
        "trailing": raw + b"\x00",
    }
    for name, blob in bad.items():
        q = str(tmp_path / f"bad_{name}.amlt")
        open(q, "wb").write(blob)
        with pytest.raises(am.AmsimError) as ei:
            am.Lut.load(q)
        assert ei.value.status == 6, name  # AMSIM_ERR_IO
    with pytest.raises(am.AmsimError) as ei:
        am.Lut.load(str(tmp_path / "missing.amlt"))
    assert ei.value.status == 6


def test_lut_build_errors(built):
    for m in (0, 12, -1):
        with pytest.raises(am.AmsimError) as ei:
            am.Lut.build("exact", m)
        assert ei.value.status == 2  # AMSIM_ERR_UNSUPPORTED

    @_lib.MUL_FN
    def doubling(a, b):  # carry of 2 at large mantissas -> breaks Alg. 1's contract
        return a * b * 2.0

    with pytest.raises(am.AmsimError) as ei:
        am.Lut.build(doubling, 4)
    assert ei.value.status == 3 and "k=" in str(ei.value)

    @_lib.MUL_FN
    def negating(a, b):
        return -(a * b)

    with pytest.raises(am.AmsimError) as ei:
        am.Lut.build(negating, 3)
    assert ei.value.status == 3

    @_lib.MUL_FN
    def user_exact(a, b):  # a user model passed through the function-pointer ABI
        return a * b

    assert np.array_equal(am.Lut.build(user_exact, 5).entries(), am.Lut.build("exact", 5).entries())


def test_from_entries_validation(built):
    e = am.Lut.build("exact", 3).entries()
    assert np.array_equal(am.Lut.from_entries(e, 3).entries(), e)
    e2 = e.copy()
    e2[5] |= 0x01000000
    with pytest.raises(am.AmsimError) as ei:
        am.Lut.from_entries(e2, 3)
    assert ei.value.status == 1


def test_compute_without_gpu_fails_loudly(built):
    """No CPU fallback: without an sm_100 device compute calls return an error
    (argument validation still runs first)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = built
    lut = am.Lut.build("exact", 7)
    st = L.amsim_gemm(lut.handle, 0, 0, -1, 4, 4, None, 4, None, 4, None, 4, 0, None)
    assert st == 1  # INVALID_ARG before any device access
    buf = (ctypes.c_float * 64)()
    st = L.amsim_gemm(lut.handle, 0, 0, 4, 4, 4, ctypes.cast(buf, ctypes.c_void_p), 4,
                      ctypes.cast(buf, ctypes.c_void_p), 4, ctypes.cast(buf, ctypes.c_void_p), 4, 0, None)
    assert st == 2, L.amsim_last_error()  # AMSIM_ERR_UNSUPPORTED: no device


def test_exponent_bits_handle(built):
    lut = am.Lut.build("exact", 7)
    assert lut.exponent_bits() == 8
    l5 = lut.with_exponent_bits(5)
    assert l5.exponent_bits() == 5 and l5.info() == lut.info()
    assert np.array_equal(l5.entries(), lut.entries())
    for bad in (0, 9, -1):
        with pytest.raises(am.AmsimError):
            lut.with_exponent_bits(bad)


def _build_example(tmp_path):
    import subprocess
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    pkg = os.path.join(ROOT, "paper_2209_04161_b200")
    exe = str(tmp_path / "amsim_example")
    subprocess.run(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
                    os.path.join(ROOT, "examples", "amsim_example.c"), "-L", pkg, "-lamsim",
                    "-L", os.path.join(cuda, "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{pkg}", "-o", exe],
                   check=True, capture_output=True, text=True)
    return exe


def test_c_example_builds_against_the_abi(built, tmp_path):
    """The ABI is usable from plain C (no Python / PyTorch): examples/amsim_example.c
    compiles and links against libamsim.so + cudart."""
    assert os.path.exists(_build_example(tmp_path))


@pytest.mark.gpu
def test_c_example_runs(built, tmp_path):
    import subprocess
    r = subprocess.run([_build_example(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "amsim_example: ok" in r.stdout, r.stdout + r.stderr


def test_binding_rejects_inconsistent_gemm_shapes(built):
    """The binding checks what the C ABI cannot see from pointers: op(A)'s K
    must match op(B)'s and C must be M x N (host-side, before any call)."""
    import torch
    lut = am.Lut.build("mitchell", 7)
    with pytest.raises(ValueError, match="op\\(A\\)"):
        am.amsim_gemm(lut, torch.zeros(2, 3), torch.zeros(4, 5), torch.zeros(2, 5))
    with pytest.raises(ValueError, match="op\\(A\\)"):
        am.amsim_gemm(lut, torch.zeros(2, 3), torch.zeros(3, 5), torch.zeros(2, 4))
    with pytest.raises(ValueError, match="op\\(A\\)"):
        am.amsim_gemm(lut, torch.zeros(3, 2), torch.zeros(3, 5), torch.zeros(3, 5), trans_a=True)
