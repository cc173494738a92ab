"""Compile the sm_100a CUDA sources into in-tree shared libraries (nvcc, no JIT cache)."""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "--expt-extended-lambda", "-I", os.path.join(ROOT, "include")]

# library name -> sources
LIBS = {
    "libhistospec.so": ["hs_index.cu", "hs_draft.cu", "hs_accept.cu"],
    "libhsmodel.so": ["hm_ops.cu", "hm_gemm.cu", "hm_attn.cu", "hm_attn_tc.cu"],
}


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps += [os.path.join(ROOT, "include", h) for h in os.listdir(os.path.join(ROOT, "include"))]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> list[str]:
    built = []
    for lib, srcs in LIBS.items():
        out = os.path.join(PKG, lib)
        paths = [os.path.join(CSRC, s) for s in srcs]
        if not force and not _stale(out, paths):
            continue
        objs = []
        for src in paths:
            obj = os.path.join(CSRC, os.path.basename(src).replace(".cu", ".o"))
            cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
            objs.append(obj)
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs]
        subprocess.run(cmd, check=True)
        built.append(out)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
