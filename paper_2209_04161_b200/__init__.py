"""AMSim approximate-multiply GEMM / convolution hot path of ApproxTrain
(arXiv 2209.04161) on B200 (sm_100a).

The compute lives in libamsim.so (include/amsim.h); this package is its thin
ctypes binding plus the data-parallel training-step driver.  Import is cheap;
the shared library is loaded on first use and raises if missing.
"""
from ._lib import (ConvDesc, Lut, AmsimError, conv_desc, amsim_lut_build, amsim_gemm,  # noqa: F401
                   amsim_conv2d_fwd, amsim_conv2d_bwd_data, amsim_conv2d_bwd_filter,
                   amsim_conv2d_bwd_filter_workspace, amsim_set_path_policy, amsim_launch_count,
                   amsim_bench_lut_lookup, model_call, lib, LIB_PATH, EXPORTS, amsim_set_multiply_mode,
                   multiply_mode, AMSIM_MUL_LUT, AMSIM_MUL_NATIVE, AMSIM_MUL_DIRECT)
