"""Builds the in-tree native artefacts (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

* paper_1711_00289_b200/libconvgpu.so  -- the product: sm_100a kernels + C ABI
* oracle/liboracle.so, oracle/_ref/libconvref.so  -- test-only parity checkers
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = [os.path.join(PKG, "csrc", "convgpu.cu")]
DEPS = SOURCES + [os.path.join(PKG, "csrc", f) for f in ("colmath.cuh", "convgpu_kernels.cuh", "bulkcopy.cuh", "exp_gl_table.h")] + [
    os.path.join(ROOT, "include", "convgpu.h")]


def _run(cmd, **kw):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, **kw)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_cuda(force=False, verbose=False):
    out = os.path.join(PKG, "libconvgpu.so")
    if not force and not _stale(out, DEPS):
        return out
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-o", out, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    _run(cmd)
    return out


def build_oracle(force=False):
    od = os.path.join(ROOT, "oracle")
    args = ["make", "-C", od, "oracle"]
    ref_src = os.environ.get("CONVPROXY_REF", "/root/reference/proj/src/core")
    if os.path.isdir(ref_src):
        args.append("ref")
        args.append(f"REF={ref_src}")
    if force:
        args.insert(1, "-B")
    _run(args)


def build_cpp_tests(force=False):
    """tests/cpp/test_dropin: the C++ drop-in vs the reference's own types and
    CPU implementation (needs the reference headers: build container only)."""
    ref_src = os.environ.get("CONVPROXY_REF", "/root/reference/proj/src/core")
    if not os.path.isdir(ref_src):
        return
    args = ["make", "-C", os.path.join(ROOT, "tests", "cpp"), f"REF={ref_src}"]
    if force:
        args.insert(1, "-B")
    _run(args)


def build_all(force=False):
    build_cuda(force)
    build_oracle(force)
    build_cpp_tests(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
