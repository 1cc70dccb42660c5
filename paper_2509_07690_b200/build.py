"""In-tree native builds (the .so files travel to the GPU box with the repo snapshot).

* ``lib/libhylu_b200.so`` — the sm_100a CUDA kernels behind the C ABI in
  ``include/hylu_b200.h`` (nvcc, ``-gencode arch=compute_100a,code=sm_100a``).
* ``lib/libhymetis.so``  — C shim over METIS_NodeND (CUDA toolkit static lib).
"""

from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
INCLUDE = os.path.join(REPO, "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n%s\n%s%s" % (" ".join(cmd), r.stdout, r.stderr))
    return r.stdout + r.stderr


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build_metis(force=False):
    os.makedirs(LIBDIR, exist_ok=True)
    out = os.path.join(LIBDIR, "libhymetis.so")
    src = os.path.join(CSRC, "metis_shim.c")
    if force or _stale(out, [src]):
        lib = os.path.join(CUDA, "targets", "x86_64-linux", "lib", "libmetis_static.a")
        _run(["gcc", "-shared", "-fPIC", "-O2", src, "-o", out, lib, "-lm"])
    return out


def build_cuda(force=False, verbose=False, out=None, extra=None):
    """extra: additional nvcc flags (default $HYLU_NVCC_EXTRA); out: variant path."""
    os.makedirs(LIBDIR, exist_ok=True)
    out = out or os.path.join(LIBDIR, "libhylu_b200.so")
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    if force or _stale(out, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
               "-I", INCLUDE, *(extra if extra is not None else os.environ.get("HYLU_NVCC_EXTRA", "")).split(), "-o", out, *srcs]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        log = _run(cmd)
        if verbose:
            print(log)
    return out


def build_all(force=False):
    return build_metis(force), build_cuda(force)


if __name__ == "__main__":
    import sys
    print(build_all(force="--force" in sys.argv))
