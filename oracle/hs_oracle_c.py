"""ctypes front-end of oracle/hs_oracle.c (TEST INFRASTRUCTURE ONLY)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhs_oracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
                os.path.join(HERE, "hs_oracle.c")):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.hso_draft.restype = ctypes.c_int32
        _lib.hso_replay.restype = ctypes.c_int32
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def layout(prompts):
    """prompts: list (per prompt) of [(tokens, reward)] -> flat text with -1 terminals."""
    text, rid, rew, poff = [], [], [], [0]
    r = 0
    for corpus in prompts:
        for toks, reward in corpus:
            toks = np.asarray(toks, dtype=np.int32)
            text.append(toks)
            text.append(np.array([-1], dtype=np.int32))
            rid.append(np.full(len(toks) + 1, r, dtype=np.int32))
            rew.append(float(reward))
            r += 1
        poff.append(poff[-1] + sum(len(t) + 1 for t, _ in corpus))
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
    return (cat(text, np.int32), cat(rid, np.int32), np.asarray(rew, dtype=np.float64),
            np.asarray(poff, dtype=np.int64))


def draft(corpus, prefix, window):
    """(tokens, found, mass) by brute-force scan (history.py:302-333 semantics)."""
    text, rid, rew, _ = layout([corpus])
    pre = np.asarray(prefix, dtype=np.int32)
    out = np.zeros(max(window, 1), dtype=np.int32)
    n = ctypes.c_int32(0)
    mass = ctypes.c_double(0.0)
    found = lib().hso_draft(_p(text), _p(rid), _p(rew), ctypes.c_int64(len(text)), _p(pre),
                            ctypes.c_int32(len(pre)), ctypes.c_int32(window), _p(out),
                            ctypes.byref(n), ctypes.byref(mass))
    if found < 0:
        raise ValueError("invalid prefix/window")
    return out[:n.value].tolist(), bool(found), mass.value


def replay_batch(histories, truths, truth_prompt, cfg=(1, 2, 2, 32, 7, 3), speculate=True,
                 has_tree=None, threads=1):
    """Replay each truth against histories[truth_prompt[i]].

    Returns (tokens_per_iter list per truth, stats [n,5] int64)."""
    text, rid, rew, poff = layout(histories)
    if has_tree is None:
        has_tree = np.ones(len(histories), dtype=np.uint8)
    has_tree = np.asarray(has_tree, dtype=np.uint8)
    toff = np.zeros(len(truths) + 1, dtype=np.int64)
    toff[1:] = np.cumsum([len(t) for t in truths])
    tcat = (np.concatenate([np.asarray(t, dtype=np.int32) for t in truths]) if truths
            else np.zeros(0, np.int32))
    tp = np.asarray(truth_prompt, dtype=np.int32)
    c6 = np.asarray(cfg, dtype=np.int32)
    tpi = np.zeros(max(int(toff[-1]), 1), dtype=np.int32)
    niter = np.zeros(max(len(truths), 1), dtype=np.int64)
    stats = np.zeros((max(len(truths), 1), 5), dtype=np.int64)
    rc = lib().hso_replay(_p(text), _p(rid), _p(rew), _p(poff), _p(has_tree),
                          ctypes.c_int32(len(histories)), _p(tcat), _p(toff), _p(tp),
                          ctypes.c_int32(len(truths)), _p(c6), ctypes.c_int32(int(speculate)),
                          _p(tpi), _p(niter), _p(stats), ctypes.c_int32(threads))
    if rc != 0:
        raise ValueError("invalid config")
    per = [tpi[toff[i]:toff[i] + niter[i]].tolist() for i in range(len(truths))]
    return per, stats[:len(truths)]


def replay_arrays(text, rid, rew, poff, has_tree, tcat, toff, tprompt, cfg, speculate, threads):
    """Array-level entry used by bench.py's CPU baseline (no Python per-token work)."""
    n = len(toff) - 1
    tpi = np.zeros(max(int(toff[-1]), 1), dtype=np.int32)
    niter = np.zeros(max(n, 1), dtype=np.int64)
    stats = np.zeros((max(n, 1), 5), dtype=np.int64)
    rc = lib().hso_replay(_p(text), _p(rid), _p(rew), _p(poff), _p(has_tree),
                          ctypes.c_int32(len(poff) - 1), _p(tcat), _p(toff), _p(tprompt),
                          ctypes.c_int32(n), _p(np.asarray(cfg, dtype=np.int32)),
                          ctypes.c_int32(int(speculate)), _p(tpi), _p(niter), _p(stats),
                          ctypes.c_int32(threads))
    if rc != 0:
        raise ValueError("invalid config")
    return tpi, niter[:n], stats[:n]
