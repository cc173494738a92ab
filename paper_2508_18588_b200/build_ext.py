"""Compile the sm_100a CUDA sources into in-tree shared libraries (nvcc, no JIT cache).

A library is rebuilt when the sha256 over its sources, every header they may
include, the nvcc flags and the nvcc version differs from the digest recorded
next to it (`<lib>.sha256`) -- content, not mtimes, so a library copied from
another tree or restored by a checkout is never trusted by accident.
Objects compile in parallel.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "--expt-extended-lambda", "-I", os.path.join(ROOT, "include")]

# library name -> sources
LIBS = {
    "libhistospec.so": ["hs_index.cu", "hs_draft.cu", "hs_accept.cu", "hs_route.cu"],
    "libhsmodel.so": ["hm_ops.cu", "hm_gemm.cu", "hm_attn.cu", "hm_attn_tc.cu", "hm_fp32.cu"],
}


def _nvcc_version() -> str:
    try:
        return subprocess.run([NVCC, "--version"], capture_output=True, text=True, check=True).stdout
    except (OSError, subprocess.CalledProcessError):
        return "unknown"


def digest(srcs) -> str:
    h = hashlib.sha256()
    headers = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
    headers += sorted(os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include")))
    for path in list(srcs) + headers:
        h.update(os.path.basename(path).encode())
        with open(path, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    h.update(_nvcc_version().encode())
    return h.hexdigest()


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(CSRC, os.path.basename(src).replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, verbose: bool = False) -> list[str]:
    built = []
    for lib, srcs in LIBS.items():
        out = os.path.join(PKG, lib)
        paths = [os.path.join(CSRC, s) for s in srcs]
        want = digest(paths)
        stamp = out + ".sha256"
        have = open(stamp).read().strip() if os.path.exists(stamp) and os.path.exists(out) else None
        if not force and have == want:
            continue
        with ThreadPoolExecutor(max_workers=min(len(paths), os.cpu_count() or 1)) as ex:
            objs = list(ex.map(lambda p: _compile(p, verbose), paths))
        subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *objs], check=True)
        with open(stamp, "w") as fh:
            fh.write(want + "\n")
        built.append(out)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
