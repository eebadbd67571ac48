"""Build libamsim.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2209_04161_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libamsim.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = [
    ("amsim_host.cpp", "g++"),
    ("amsim_gemm.cu", "nvcc"),
    ("amsim_conv_fwd.cu", "nvcc"),
    ("amsim_conv_dgrad.cu", "nvcc"),
    ("amsim_conv_wgrad.cu", "nvcc"),
    ("amsim_bench.cu", "nvcc"),
    ("amsim_nn.cu", "nvcc"),
]
HEADERS = [os.path.join(CSRC, "amsim_internal.h"), os.path.join(CSRC, "amsim_device.cuh"),
           os.path.join(CSRC, "amsim_dispatch.cuh"), os.path.join(ROOT, "include", "amsim.h"), os.path.join(ROOT, "include", "amsim_nn.h")]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    procs = []
    for src, tool in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if not force and not _newer(o, [s] + HEADERS):
            continue
        if tool == "nvcc":
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-I", os.path.join(CUDA, "include"),
                   "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{out}")
        if verbose:
            print(out)
    if force or _newer(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


def build_variant(tag: str, defines, only=None) -> str:
    """Experimental build with extra -D flags (tuning sweeps): build/variants/libamsim_<tag>.so.
    Load it by setting AMSIM_LIB to the returned path.  `only`: the translation
    units to rebuild with the flags (the others are linked from the main build)."""
    vdir = os.path.join(BUILD, "variants")
    os.makedirs(vdir, exist_ok=True)
    host_o = os.path.join(BUILD, "amsim_host.cpp.o")
    build()  # host object
    so = os.path.join(vdir, f"libamsim_{tag}.so")
    objs, procs = [host_o], []
    for src, tool in SOURCES:
        if tool != "nvcc":
            continue
        if only and src not in only:
            objs.append(os.path.join(BUILD, src + ".o"))
            continue
        ko = os.path.join(vdir, f"{src}_{tag}.o")
        objs.append(ko)
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
               "-c", os.path.join(CSRC, src), "-o", ko]
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"variant build failed: {p.args}")
    subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", so, *objs, "-lpthread", "-ldl", "-lrt"],
                   check=True)
    return so


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        # --variant TAG [-DFLAG ...] [+unit.cu ...]
        args = sys.argv[3:]
        print(build_variant(sys.argv[2], [a for a in args if not a.startswith("+")],
                            [a[1:] for a in args if a.startswith("+")] or None))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
