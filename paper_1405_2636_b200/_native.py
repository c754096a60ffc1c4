"""Loading and building of the package's native libraries.

* `libps_host.so`   - C++ symbolic analysis (csrc/ps_host.cpp)
* `libps_b200.so`   - the sm_100a CUDA engine and its C ABI (csrc/ps_b200.cu,
                      declared in include/ps_b200.h)

Both are built in-tree (into paper_1405_2636_b200/lib/) so they travel with
the repository snapshot to the GPU box.  There is no fallback: a missing
engine library raises, it never degrades to a CPU path.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")

HOST_LIB = os.path.join(LIBDIR, "libps_host.so")
ENGINE_LIB = os.path.join(LIBDIR, "libps_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

_ENGINE_SOURCES = ["ps_b200.cu"]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_host(force=False):
    os.makedirs(LIBDIR, exist_ok=True)
    src = os.path.join(CSRC, "ps_host.cpp")
    if force or _stale(HOST_LIB, [src]):
        tmp = HOST_LIB + ".tmp"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC",
                               "-o", tmp, src])
        os.replace(tmp, HOST_LIB)
    return HOST_LIB


def engine_sources():
    srcs = [os.path.join(CSRC, s) for s in _ENGINE_SOURCES]
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    return srcs, hdrs + [os.path.join(INCLUDE, "ps_b200.h")]


def build_engine(force=False, verbose=False):
    os.makedirs(LIBDIR, exist_ok=True)
    srcs, deps = engine_sources()
    if force or _stale(ENGINE_LIB, srcs + deps):
        tmp = ENGINE_LIB + ".tmp"
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
               "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
               *os.environ.get("PS_NVCC_EXTRA", "").split(),  # tuning experiments (-D...)
               "-o", tmp, *srcs]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(tmp, ENGINE_LIB)
    return ENGINE_LIB


_host = None
_engine = None


def host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB) or _stale(HOST_LIB, [os.path.join(CSRC, "ps_host.cpp")]):
            build_host()
        lib = ctypes.CDLL(HOST_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.psh_nested_dissection.argtypes = [I, P, P, I, P, P, I, P]
        lib.psh_nested_dissection.restype = ctypes.c_int
        lib.psh_etree.argtypes = [I, P, P, P]
        lib.psh_etree.restype = None
        lib.psh_postorder.argtypes = [I, P, P]
        lib.psh_postorder.restype = None
        lib.psh_symbolic.argtypes = [I, P, P, P]
        lib.psh_symbolic.restype = P
        lib.psh_symbolic_sizes.argtypes = [P, P, P, P]
        lib.psh_symbolic_sizes.restype = None
        lib.psh_symbolic_fetch.argtypes = [P, P, P, P]
        lib.psh_symbolic_fetch.restype = None
        lib.psh_symbolic_free.argtypes = [P]
        lib.psh_symbolic_free.restype = None
        _host = lib
    return _host


def engine_lib():
    """The CUDA engine.  Raises if it was not built (no CPU fallback)."""
    global _engine
    if _engine is None:
        alt = os.environ.get("PS_ENGINE_LIB")  # dev: a tuning variant built elsewhere
        if alt:
            from . import _abi
            _engine = _abi.bind(ctypes.CDLL(alt))
            return _engine
        if not os.path.exists(ENGINE_LIB):
            raise RuntimeError(
                f"CUDA engine library missing: {ENGINE_LIB}. Run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a).")
        from . import _abi
        _engine = _abi.bind(ctypes.CDLL(ENGINE_LIB))
    return _engine


def ptr(a):
    """Raw data pointer of a numpy array (ctypes void*)."""
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)
