"""CPU checks of the C-ABI boundary: every symbol declared in include/*.h is exported."""

import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT

HEADERS = sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))
# header -> shared library that implements it
LIB_OF = {"histospec.h": "paper_2508_18588_b200/libhistospec.so",
          "hsmodel.h": "paper_2508_18588_b200/libhsmodel.so"}


def declared(header):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b((?:hs|hm)_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2508_18588_b200 import build_ext
    build_ext.build()


@pytest.mark.parametrize("header", [os.path.basename(h) for h in HEADERS])
def test_header_symbols_exported(header):
    names = declared(os.path.join(ROOT, "include", header))
    assert names, header
    lib = ctypes.CDLL(os.path.join(ROOT, LIB_OF[header]))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2508_18588_b200 import _lib
    names = declared(os.path.join(ROOT, "include", "histospec.h"))
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)
    lib = _lib.load()
    assert lib.hs_version() >= 1


def test_gpu_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2508_18588_b200.history import build_tree, Response
    with pytest.raises(RuntimeError):
        build_tree("p", 1, [Response("p", 1, [1, 2, 3], 1.0)])
