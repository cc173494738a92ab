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


def test_attention_work_size_host_only():
    """hm_attention_work_size is host arithmetic (no GPU): tile prefix (n_seq + 1) plus one entry per
    128-row tcgen05 tile of every sequence; invalid shapes return 0."""
    from paper_2508_18588_b200 import model as Mo
    L = Mo.lib()
    assert L.hm_attention_work_size(1024, 33, 12, 2) == 1025 + 1024 * 2    # 33 queries x 6 heads = 198 rows
    assert L.hm_attention_work_size(1024, 21, 12, 2) == 1025 + 1024        # 126 rows fit one tile
    assert L.hm_attention_work_size(5, 1, 4, 4) == 6 + 5
    assert L.hm_attention_work_size(0, 1, 12, 2) == 0
    assert L.hm_attention_work_size(8, 4, 12, 5) == 0                      # H % KVH != 0
