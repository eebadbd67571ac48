"""ctypes binding of libamsim (include/amsim.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
CPU fallback -- if libamsim.so is missing or the device is not sm_100 the
calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AMSIM_LIB") or os.path.join(PKG, "libamsim.so")

AMSIM_OK = 0
_STATUS = {0: "AMSIM_OK", 1: "AMSIM_ERR_INVALID_ARG", 2: "AMSIM_ERR_UNSUPPORTED", 3: "AMSIM_ERR_MODEL",
           4: "AMSIM_ERR_NOMEM", 5: "AMSIM_ERR_CUDA", 6: "AMSIM_ERR_IO"}

MUL_FN = ctypes.CFUNCTYPE(ctypes.c_float, ctypes.c_float, ctypes.c_float)


class AmsimError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


class ConvDesc(ctypes.Structure):
    """amsim_conv2d_desc: x NHWC [N][H][W][C], w HWIO [R][S][C][K]."""
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


# every symbol include/amsim.h declares
EXPORTS = [
    "amsim_lut_build", "amsim_lut_from_entries", "amsim_lut_entries", "amsim_lut_info", "amsim_lut_save",
    "amsim_lut_load", "amsim_lut_destroy", "amsim_last_error", "amsim_model_exact", "amsim_model_mitchell",
    "amsim_model_mbm", "amsim_gemm", "amsim_conv2d_fwd", "amsim_conv2d_bwd_data",
    "amsim_conv2d_bwd_filter_workspace", "amsim_conv2d_bwd_filter", "amsim_set_path_policy",
    "amsim_launch_count", "amsim_bench_lut_lookup", "amsim_abi_version", "amsim_set_multiply_mode",
    "amsim_lut_with_exponent_bits", "amsim_lut_exponent_bits",
]

# every symbol include/amsim_nn.h declares (the non-approximated layers)
NN_EXPORTS = [
    "amsim_nn_workspace_bytes", "amsim_bn_fwd_train", "amsim_bn_fwd_infer", "amsim_bn_bwd", "amsim_bias_act_fwd",
    "amsim_bias_act_bwd", "amsim_maxpool_fwd", "amsim_maxpool_bwd", "amsim_avgpool_fwd", "amsim_avgpool_bwd",
    "amsim_softmax_xent", "amsim_add", "amsim_sgd_momentum",
]

# amsim_set_multiply_mode values (include/amsim.h)
AMSIM_MUL_LUT, AMSIM_MUL_NATIVE, AMSIM_MUL_DIRECT = 0, 1, 2

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2209_04161_b200.build` "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, u32p = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32)
    L.amsim_lut_build.argtypes = [vp, i32, ctypes.POINTER(vp)]
    L.amsim_lut_from_entries.argtypes = [u32p, i32, ctypes.POINTER(vp)]
    L.amsim_lut_entries.argtypes = [vp, ctypes.POINTER(u32p), ctypes.POINTER(ctypes.c_size_t)]
    L.amsim_lut_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.amsim_lut_save.argtypes = [vp, ctypes.c_char_p]
    L.amsim_lut_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.amsim_lut_with_exponent_bits.argtypes = [vp, i32, ctypes.POINTER(vp)]
    L.amsim_lut_exponent_bits.argtypes = [vp, ctypes.POINTER(i32)]
    L.amsim_lut_destroy.argtypes = [vp]
    L.amsim_lut_destroy.restype = None
    L.amsim_last_error.restype = ctypes.c_char_p
    for name in ("amsim_model_exact", "amsim_model_mitchell", "amsim_model_mbm"):
        getattr(L, name).argtypes = [ctypes.c_float, ctypes.c_float]
        getattr(L, name).restype = ctypes.c_float
    L.amsim_gemm.argtypes = [vp, i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, vp]
    L.amsim_conv2d_fwd.argtypes = [vp, ctypes.POINTER(ConvDesc), vp, vp, vp, vp]
    L.amsim_conv2d_bwd_data.argtypes = [vp, ctypes.POINTER(ConvDesc), vp, vp, vp, vp]
    L.amsim_conv2d_bwd_filter_workspace.argtypes = [vp, ctypes.POINTER(ConvDesc), ctypes.POINTER(ctypes.c_size_t)]
    L.amsim_conv2d_bwd_filter.argtypes = [vp, ctypes.POINTER(ConvDesc), vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.amsim_set_path_policy.argtypes = [i32]
    L.amsim_set_multiply_mode.argtypes = [i32]
    L.amsim_launch_count.restype = ctypes.c_uint64
    L.amsim_bench_lut_lookup.argtypes = [i32, i32, i32, u32p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_double), vp]
    L.amsim_abi_version.restype = i32
    f32, sz = ctypes.c_float, ctypes.c_size_t
    L.amsim_nn_workspace_bytes.argtypes = [i64, i32]
    L.amsim_nn_workspace_bytes.restype = sz
    L.amsim_bn_fwd_train.argtypes = [vp, i64, i32, vp, vp, f32, vp, i32, vp, vp, vp, vp, vp, f32, vp, sz, vp]
    L.amsim_bn_fwd_infer.argtypes = [vp, i64, i32, vp, vp, vp, vp, f32, vp, i32, vp, vp]
    L.amsim_bn_bwd.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp, sz, vp]
    L.amsim_bias_act_fwd.argtypes = [vp, i64, i32, vp, i32, vp, vp]
    L.amsim_bias_act_bwd.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, sz, vp]
    L.amsim_maxpool_fwd.argtypes = [vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp, vp]
    L.amsim_maxpool_bwd.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp]
    L.amsim_avgpool_fwd.argtypes = [vp, i32, i32, i32, vp, vp]
    L.amsim_avgpool_bwd.argtypes = [vp, i32, i32, i32, vp, vp]
    L.amsim_softmax_xent.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp, sz, vp]
    L.amsim_add.argtypes = [vp, vp, vp, i64, vp]
    L.amsim_sgd_momentum.argtypes = [vp, vp, vp, i64, f32, f32, f32, vp]
    _lib = L
    return L


def _check(status: int, fn: str):
    if status != AMSIM_OK:
        msg = lib().amsim_last_error()
        raise AmsimError(status, fn, msg.decode() if msg else "")


MODEL_FNS = ("exact", "mitchell", "mbm")


def model_fn_ptr(name: str) -> int:
    """Address of a built-in functional model (amsim_model_<name>)."""
    return ctypes.cast(getattr(lib(), f"amsim_model_{name}"), ctypes.c_void_p).value


def model_call(name: str, a: float, b: float) -> float:
    return float(getattr(lib(), f"amsim_model_{name}")(a, b))


class Lut:
    """Owner of an amsim_lut handle (Alg. 1 table)."""

    def __init__(self, handle: int, keep=None):
        self.handle = ctypes.c_void_p(handle)
        self._keep = keep

    @classmethod
    def build(cls, model, m: int) -> "Lut":
        """amsim_lut_build.  `model` is a built-in name ('exact', 'mitchell',
        'mbm'), a ctypes MUL_FN, or an integer function address."""
        keep = None
        if isinstance(model, str):
            fp = model_fn_ptr(model)
        elif isinstance(model, MUL_FN):
            keep = model
            fp = ctypes.cast(model, ctypes.c_void_p).value
        else:
            fp = int(model)
        out = ctypes.c_void_p()
        _check(lib().amsim_lut_build(fp, m, ctypes.byref(out)), "amsim_lut_build")
        return cls(out.value, keep)

    @classmethod
    def from_entries(cls, entries, m: int) -> "Lut":
        e = np.ascontiguousarray(entries, dtype=np.uint32)
        out = ctypes.c_void_p()
        _check(lib().amsim_lut_from_entries(e.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), m, ctypes.byref(out)),
               "amsim_lut_from_entries")
        return cls(out.value)

    def with_exponent_bits(self, e: int) -> "Lut":
        """amsim_lut_with_exponent_bits: a (1, e, m) copy (operands cast to e exponent bits)."""
        out = ctypes.c_void_p()
        _check(lib().amsim_lut_with_exponent_bits(self.handle, int(e), ctypes.byref(out)),
               "amsim_lut_with_exponent_bits")
        return Lut(out.value)

    def exponent_bits(self) -> int:
        e = ctypes.c_int()
        _check(lib().amsim_lut_exponent_bits(self.handle, ctypes.byref(e)), "amsim_lut_exponent_bits")
        return e.value

    @classmethod
    def load(cls, path: str) -> "Lut":
        out = ctypes.c_void_p()
        _check(lib().amsim_lut_load(path.encode(), ctypes.byref(out)), "amsim_lut_load")
        return cls(out.value)

    def save(self, path: str):
        _check(lib().amsim_lut_save(self.handle, path.encode()), "amsim_lut_save")

    def entries(self) -> np.ndarray:
        p = ctypes.POINTER(ctypes.c_uint32)()
        n = ctypes.c_size_t()
        _check(lib().amsim_lut_entries(self.handle, ctypes.byref(p), ctypes.byref(n)), "amsim_lut_entries")
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy()

    def info(self):
        m = ctypes.c_int()
        eb = ctypes.c_int()
        _check(lib().amsim_lut_info(self.handle, ctypes.byref(m), ctypes.byref(eb)), "amsim_lut_info")
        return m.value, eb.value

    @property
    def m(self):
        return self.info()[0]

    def __del__(self):
        if getattr(self, "handle", None) is not None and self.handle.value and _lib is not None:
            _lib.amsim_lut_destroy(self.handle)
            self.handle = ctypes.c_void_p(0)


def amsim_lut_build(model, m: int) -> Lut:
    return Lut.build(model, m)


# ---------------------------------------------------------------------------
# compute entry points over torch CUDA tensors (device memory, current stream)

_torch = None


def _T():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


def _stream(stream):
    """cudaStream_t of `stream` (default: PyTorch's current stream on the current device)."""
    if stream is None:
        torch = _T()
        return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dptr(t, name):
    if t is None:
        return None
    if not t.is_cuda or t.dtype is not _T().float32:
        raise TypeError(f"{name} must be a float32 CUDA tensor")
    return t.data_ptr()


def amsim_gemm(lut: Lut, A, B, C, trans_a: bool = False, trans_b: bool = False, accumulate: bool = False,
               stream=None):
    """C (M x N) = [C +] op(A) op(B) with AMSim products; 2-D row-major tensors
    (leading dimension = stride(0))."""
    M = A.shape[1] if trans_a else A.shape[0]
    K = A.shape[0] if trans_a else A.shape[1]
    N = B.shape[0] if trans_b else B.shape[1]
    KB = B.shape[1] if trans_b else B.shape[0]
    if KB != K or tuple(C.shape) != (M, N):
        raise ValueError(f"amsim_gemm: op(A) is {M}x{K}, op(B) {KB}x{N}, C {tuple(C.shape)}")
    dev = _T().cuda.current_device()
    for t, nm in ((A, "A"), (B, "B"), (C, "C")):
        if t.is_cuda and t.device.index != dev:
            raise ValueError(f"{nm} is on {t.device}, not the current device cuda:{dev}")
    lds = []
    for t, nm in ((A, "A"), (B, "B"), (C, "C")):
        if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
            raise ValueError(f"{nm} must be 2-D with unit column stride")
        lds.append(t.stride(0) if t.shape[0] > 1 else t.shape[1])  # a size-1 dim's stride is arbitrary
    _check(lib().amsim_gemm(lut.handle, int(trans_a), int(trans_b), M, N, K, _dptr(A, "A"), lds[0],
                            _dptr(B, "B"), lds[1], _dptr(C, "C"), lds[2], int(accumulate),
                            _stream(stream)), "amsim_gemm")
    return C


def _conv_ptr(t, name, numel):
    """Device pointer of a conv operand after the checks the C ABI cannot make
    (it sees only a pointer): float32, on the current CUDA device, contiguous,
    and exactly the element count the descriptor implies."""
    p = _dptr(t, name)
    torch = _T()
    if t.device.index != torch.cuda.current_device():
        raise ValueError(f"{name} is on {t.device}, not the current device cuda:{torch.cuda.current_device()}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (NHWC / HWIO)")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements; the descriptor needs {numel}")
    return p


def _conv_sizes(d: ConvDesc):
    """Element counts of x, w, y for descriptor d."""
    return d.N * d.H * d.W * d.C, d.R * d.S * d.C * d.K, d.N * d.OH * d.OW * d.K


def amsim_conv2d_fwd(lut: Lut, d: ConvDesc, x, w, y, stream=None):
    nx, nw, ny = _conv_sizes(d)
    _check(lib().amsim_conv2d_fwd(lut.handle, ctypes.byref(d), _conv_ptr(x, "x", nx), _conv_ptr(w, "w", nw),
                                  _conv_ptr(y, "y", ny), _stream(stream)), "amsim_conv2d_fwd")
    return y


def amsim_conv2d_bwd_data(lut: Lut, d: ConvDesc, dy, w, dx, stream=None):
    nx, nw, ny = _conv_sizes(d)
    _check(lib().amsim_conv2d_bwd_data(lut.handle, ctypes.byref(d), _conv_ptr(dy, "dy", ny), _conv_ptr(w, "w", nw),
                                       _conv_ptr(dx, "dx", nx), _stream(stream)), "amsim_conv2d_bwd_data")
    return dx


def amsim_conv2d_bwd_filter_workspace(lut: Lut, d: ConvDesc) -> int:
    n = ctypes.c_size_t()
    _check(lib().amsim_conv2d_bwd_filter_workspace(lut.handle, ctypes.byref(d), ctypes.byref(n)),
           "amsim_conv2d_bwd_filter_workspace")
    return n.value


def amsim_conv2d_bwd_filter(lut: Lut, d: ConvDesc, x, dy, dw, workspace=None, stream=None):
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    if workspace is not None and (not workspace.is_cuda or not workspace.is_contiguous()):
        raise ValueError("workspace must be a contiguous CUDA tensor")
    nx, nw, ny = _conv_sizes(d)
    _check(lib().amsim_conv2d_bwd_filter(lut.handle, ctypes.byref(d), _conv_ptr(x, "x", nx), _conv_ptr(dy, "dy", ny),
                                         _conv_ptr(dw, "dw", nw),
                                         None if workspace is None else ctypes.c_void_p(workspace.data_ptr()),
                                         ws_bytes, _stream(stream)), "amsim_conv2d_bwd_filter")
    return dw


def amsim_set_path_policy(policy: int):
    _check(lib().amsim_set_path_policy(policy), "amsim_set_path_policy")


def amsim_set_multiply_mode(mode: int):
    _check(lib().amsim_set_multiply_mode(mode), "amsim_set_multiply_mode")


class multiply_mode:
    """Context manager: run the enclosed calls in AMSIM_MUL_NATIVE / _DIRECT
    (measurement instruments), restoring AMSIM_MUL_LUT afterwards."""

    def __init__(self, mode: int):
        self.mode = mode

    def __enter__(self):
        amsim_set_multiply_mode(self.mode)

    def __exit__(self, *a):
        amsim_set_multiply_mode(AMSIM_MUL_LUT)


def amsim_launch_count() -> int:
    return int(lib().amsim_launch_count())


def amsim_bench_lut_lookup(m: int, entry_bits: int, b_idx, iters: int = 4096, stream=None) -> float:
    idx = np.ascontiguousarray(b_idx, dtype=np.uint32)
    out = ctypes.c_double()
    _check(lib().amsim_bench_lut_lookup(m, entry_bits, iters, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                        idx.size, ctypes.byref(out), _stream(stream)), "amsim_bench_lut_lookup")
    return out.value


# ---------------------------------------------------------------------------
# non-approximated layers (include/amsim_nn.h): argument marshalling only

def _p(t):
    """Device pointer of an optional tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _ws(ws):
    return (None, 0) if ws is None else (ctypes.c_void_p(ws.data_ptr()), ws.numel() * ws.element_size())


def amsim_nn_workspace_bytes(P: int, C: int) -> int:
    return int(lib().amsim_nn_workspace_bytes(P, C))


def amsim_bn_fwd_train(x, P, C, gamma, beta, eps, res, relu, y, save_mean, save_invstd, running_mean, running_var,
                       momentum, ws, stream=None):
    w, wb = _ws(ws)
    _check(lib().amsim_bn_fwd_train(_p(x), P, C, _p(gamma), _p(beta), eps, _p(res), int(relu), _p(y), _p(save_mean),
                                    _p(save_invstd), _p(running_mean), _p(running_var), momentum, w, wb,
                                    _stream(stream)), "amsim_bn_fwd_train")


def amsim_bn_fwd_infer(x, P, C, gamma, beta, running_mean, running_var, eps, res, relu, y, stream=None):
    _check(lib().amsim_bn_fwd_infer(_p(x), P, C, _p(gamma), _p(beta), _p(running_mean), _p(running_var), eps, _p(res),
                                    int(relu), _p(y), _stream(stream)), "amsim_bn_fwd_infer")


def amsim_bn_bwd(dy, y, x, P, C, gamma, save_mean, save_invstd, relu, dx, dres, dgamma, dbeta, ws, stream=None):
    w, wb = _ws(ws)
    _check(lib().amsim_bn_bwd(_p(dy), _p(y), _p(x), P, C, _p(gamma), _p(save_mean), _p(save_invstd), int(relu),
                              _p(dx), _p(dres), _p(dgamma), _p(dbeta), w, wb, _stream(stream)), "amsim_bn_bwd")


def amsim_bias_act_fwd(x, P, C, bias, relu, y, stream=None):
    _check(lib().amsim_bias_act_fwd(_p(x), P, C, _p(bias), int(relu), _p(y), _stream(stream)), "amsim_bias_act_fwd")


def amsim_bias_act_bwd(dy, y, P, C, relu, dx, dbias, ws, stream=None):
    w, wb = _ws(ws)
    _check(lib().amsim_bias_act_bwd(_p(dy), _p(y), P, C, int(relu), _p(dx), _p(dbias), w, wb, _stream(stream)),
           "amsim_bias_act_bwd")


def amsim_maxpool_fwd(x, N, H, W, C, R, S, stride, pad, y, argmax, stream=None):
    _check(lib().amsim_maxpool_fwd(_p(x), N, H, W, C, R, S, stride, pad, _p(y), _p(argmax), _stream(stream)),
           "amsim_maxpool_fwd")


def amsim_maxpool_bwd(dy, argmax, N, H, W, C, R, S, stride, pad, dx, stream=None):
    _check(lib().amsim_maxpool_bwd(_p(dy), _p(argmax), N, H, W, C, R, S, stride, pad, _p(dx), _stream(stream)),
           "amsim_maxpool_bwd")


def amsim_avgpool_fwd(x, N, HW, C, y, stream=None):
    _check(lib().amsim_avgpool_fwd(_p(x), N, HW, C, _p(y), _stream(stream)), "amsim_avgpool_fwd")


def amsim_avgpool_bwd(dy, N, HW, C, dx, stream=None):
    _check(lib().amsim_avgpool_bwd(_p(dy), N, HW, C, _p(dx), _stream(stream)), "amsim_avgpool_bwd")


def amsim_softmax_xent(logits, labels, N, K, loss, dlogits, ws, grad_denominator=0, stream=None):
    w, wb = _ws(ws)
    _check(lib().amsim_softmax_xent(_p(logits), _p(labels), N, K, int(grad_denominator), _p(loss), _p(dlogits), w, wb,
                                    _stream(stream)),
           "amsim_softmax_xent")


def amsim_add(a, b, out, n, stream=None):
    _check(lib().amsim_add(_p(a), _p(b), _p(out), n, _stream(stream)), "amsim_add")


def amsim_sgd_momentum(w, g, v, n, lr, momentum, weight_decay, stream=None):
    _check(lib().amsim_sgd_momentum(_p(w), _p(g), _p(v), n, lr, momentum, weight_decay, _stream(stream)),
           "amsim_sgd_momentum")
