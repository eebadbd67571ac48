"""CPU oracle for the AMSim hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2209_04161_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``amsim_oracle.c`` (plain C, OpenMP
over output rows, IEEE FP32 without FTZ).  See that file's header for the
passages of /root/reference/PAPER.md each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "amsim_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MODELS = {"exact": 0, "mitchell": 1, "mbm": 2, "asym": 3}


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off", "-std=c11",
             "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.oracle_mul.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_int, ctypes.c_int, f32p]
        L.oracle_mul.restype = ctypes.c_int
        L.oracle_mul_vec.argtypes = [f32p, f32p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, f32p]
        L.oracle_mul_vec.restype = ctypes.c_int
        L.oracle_cast_e_vec.argtypes = [f32p, ctypes.c_int64, ctypes.c_int, f32p]
        L.oracle_cast_e_vec.restype = None
        L.oracle_model_call.argtypes = [ctypes.c_int, ctypes.c_float, ctypes.c_float]
        L.oracle_model_call.restype = ctypes.c_float
        L.oracle_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                  f32p, f32p, i64p, ctypes.c_int64, f32p, f64p, f64p]
        L.oracle_gemm.restype = ctypes.c_int
        for name in ("oracle_conv_fwd", "oracle_conv_bwd_filter", "oracle_conv_bwd_data"):
            fn = getattr(L, name)
            fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, f32p, f32p, i64p, ctypes.c_int64,
                           f32p, f64p, f64p]
            fn.restype = ctypes.c_int
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _check(code: int, what: str):
    if code == 1:
        raise OracleError(f"{what}: multiplier model broke the Alg. 1 contract (exponent/sign)")
    if code != 0:
        raise OracleError(f"{what}: invalid argument (code {code})")


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def num_threads() -> int:
    return lib().oracle_num_threads()


def model_call(model: str, a: float, b: float) -> float:
    return float(lib().oracle_model_call(MODELS[model], a, b))


def cast_e(x, e: int) -> np.ndarray:
    """Exponent cast of every element to the (1, e, m) range (reading C23,
    amsim_oracle.c oracle_cast_e); applied to both operands before AMSim."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(a)
    f32p = ctypes.POINTER(ctypes.c_float)
    lib().oracle_cast_e_vec(a.ctypes.data_as(f32p), a.size, int(e), out.ctypes.data_as(f32p))
    return out


def mul(a, b, model: str = "exact", m: int = 7) -> np.ndarray:
    """Elementwise approximate product (Alg. 2 via direct model calls)."""
    a, b = np.broadcast_arrays(_f32(a), _f32(b))
    shape = a.shape
    a = _f32(a).ravel()
    b = _f32(b).ravel()
    out = np.empty_like(a)
    _check(lib().oracle_mul_vec(_ptr(a, ctypes.c_float), _ptr(b, ctypes.c_float), a.size,
                                MODELS[model], m, _ptr(out, ctypes.c_float)), "oracle_mul")
    return out.reshape(shape)


@dataclass
class Result:
    c32: np.ndarray   # FP32 sequential sum in the paper's order (increasing k)
    c64: np.ndarray   # double sum of the same bit-exact products
    abs64: np.ndarray  # sum |p|

    def tol(self, rel: float = 1e-5) -> np.ndarray:
        """Per-element acceptance bound |gpu - c64| <= rel*sum|p| + FLT_MIN (reading C12)."""
        return rel * self.abs64 + np.finfo(np.float32).tiny


def _rows(rows):
    if rows is None:
        return None, 0
    r = np.ascontiguousarray(rows, dtype=np.int64)
    return r, r.size


def gemm(A, B, model: str = "exact", m: int = 7, rows=None) -> Result:
    """C = A @ B with every product approximated; A is M x K, B is K x N."""
    A = _f32(A)
    B = _f32(B)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    r, nr = _rows(rows)
    nout = nr if r is not None else M
    c32 = np.empty((nout, N), np.float32)
    c64 = np.empty((nout, N), np.float64)
    a64 = np.empty((nout, N), np.float64)
    _check(lib().oracle_gemm(MODELS[model], m, M, N, K, _ptr(A, ctypes.c_float), _ptr(B, ctypes.c_float),
                             None if r is None else _ptr(r, ctypes.c_int64), nr,
                             _ptr(c32, ctypes.c_float), _ptr(c64, ctypes.c_double), _ptr(a64, ctypes.c_double)),
           "oracle_gemm")
    return Result(c32, c64, a64)


class ConvDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("N", "H", "W", "C", "K", "R", "S", "stride_h", "stride_w", "pad_h", "pad_w")]

    @property
    def OH(self):
        return (self.H + 2 * self.pad_h - self.R) // self.stride_h + 1

    @property
    def OW(self):
        return (self.W + 2 * self.pad_w - self.S) // self.stride_w + 1


def conv_desc(N, H, W, C, K, R, S, stride=1, pad=0, stride_w=None, pad_w=None) -> ConvDesc:
    return ConvDesc(N, H, W, C, K, R, S, stride, stride if stride_w is None else stride_w,
                    pad, pad if pad_w is None else pad_w)


def _conv(fn, d: ConvDesc, first, second, model, m, rows, nrows_all, ncols) -> Result:
    first = _f32(first)
    second = _f32(second)
    r, nr = _rows(rows)
    nout = nr if r is not None else nrows_all
    c32 = np.empty((nout, ncols), np.float32)
    c64 = np.empty((nout, ncols), np.float64)
    a64 = np.empty((nout, ncols), np.float64)
    _check(fn(MODELS[model], m, ctypes.byref(d), _ptr(first, ctypes.c_float), _ptr(second, ctypes.c_float),
              None if r is None else _ptr(r, ctypes.c_int64), nr,
              _ptr(c32, ctypes.c_float), _ptr(c64, ctypes.c_double), _ptr(a64, ctypes.c_double)), fn.__name__)
    return Result(c32, c64, a64)


def conv_fwd(d: ConvDesc, x, w, model="exact", m=7, rows=None) -> Result:
    """Alg. 3: y rows (n,oh,ow) x K.  x NHWC, w HWIO."""
    return _conv(lib().oracle_conv_fwd, d, x, w, model, m, rows, d.N * d.OH * d.OW, d.K)


def conv_bwd_filter(d: ConvDesc, x, dy, model="exact", m=7, rows=None) -> Result:
    """Alg. 4 l.4-5: dW rows (kh,kw,ci) x K.  x NHWC, dy NHWC (N,OH,OW,K)."""
    return _conv(lib().oracle_conv_bwd_filter, d, x, dy, model, m, rows, d.R * d.S * d.C, d.K)


def conv_bwd_data(d: ConvDesc, dy, w, model="exact", m=7, rows=None) -> Result:
    """Alg. 4 l.6-8: dX rows (n,h,w) x C.  dy NHWC, w HWIO."""
    return _conv(lib().oracle_conv_bwd_data, d, dy, w, model, m, rows, d.N * d.H * d.W, d.C)
