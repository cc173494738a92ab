"""token_similarity_replay (tracegen.py:306-353): oracle vs the reference's golden vectors (CPU)
and the GPU kernel (hs_similarity_replay) vs golden, oracle and size-independent properties.

Golden vectors: tests/golden/similarity.json.gz, made by make_similarity_golden.py from the
reference itself.
"""

import random

import numpy as np
import pytest

from conftest import load_golden
from oracle import hs_oracle


def _epochs(case):
    return {int(e): {pid: rs for pid, rs in d.items()} for e, d in case["trace"].items()}


def test_oracle_matches_reference_golden():
    for case in load_golden("similarity.json.gz"):
        tr = _epochs(case)
        for r in case["results"]:
            a, b = r["pair"]
            want = (r["accepted"], r["total"], r["warmup"])
            got = hs_oracle.token_similarity_replay(tr.get(a, {}), tr.get(b, {}), r["prefix_len"])
            assert got == want, (r, got)
            got = hs_oracle.token_similarity_replay_indexed(tr.get(a, {}), tr.get(b, {}), r["prefix_len"])
            assert got == want, (r, got)


def test_oracle_rejects_bad_prefix():
    with pytest.raises(ValueError):
        hs_oracle.token_similarity_replay({}, {}, 0)


def test_result_properties_cpu():
    from paper_2508_18588_b200.similarity import ReplayResult
    r = ReplayResult(accepted=6, total=10, warmup=2)
    assert r.acceptance == 0.6 and r.acceptance_after_warmup == 0.75
    assert ReplayResult(0, 0, 0).acceptance == 0.0
    assert ReplayResult(0, 3, 3).acceptance_after_warmup == 0.0


def _to_trace(tr):
    return {e: {pid: [(t, 0.0) for t in rs] for pid, rs in d.items()} for e, d in tr.items()}


@pytest.fixture(params=["isa", "plain"])
def variant(request, monkeypatch):
    """Both search kernels: ISA-seeded (default) and plain binary search (HS_SIM_SEARCH)."""
    monkeypatch.setenv("HS_SIM_SEARCH", request.param)
    return request.param


def test_unknown_search_mode_is_an_error(monkeypatch):
    """A typo in HS_SIM_SEARCH raises instead of silently selecting the slower kernel."""
    from paper_2508_18588_b200 import similarity
    monkeypatch.setenv("HS_SIM_SEARCH", "ISA")
    with pytest.raises(ValueError):
        similarity._search_mode()


@pytest.mark.gpu
def test_gpu_matches_reference_golden(variant):
    from paper_2508_18588_b200.similarity import token_similarity_replay
    for case in load_golden("similarity.json.gz"):
        trace = _to_trace(_epochs(case))
        for r in case["results"]:
            got = token_similarity_replay(trace, tuple(r["pair"]), r["prefix_len"])
            assert (got.accepted, got.total, got.warmup) == (r["accepted"], r["total"], r["warmup"]), r


@pytest.mark.gpu
def test_gpu_errors_like_reference():
    from paper_2508_18588_b200.similarity import token_similarity_replay
    trace = {1: {"a": [([1, 2, 3], 1.0)]}, 2: {"a": [([1, 2, 3], 1.0)]}}
    with pytest.raises(ValueError):
        token_similarity_replay(trace, (1, 2), 0)
    with pytest.raises(KeyError):
        token_similarity_replay(trace, (1, 3), 2)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gpu_matches_oracle_random(seed, variant):
    """Random small-vocabulary epochs (many collisions, ragged and tiny lengths)."""
    from paper_2508_18588_b200.similarity import token_similarity_replay
    rng = random.Random(seed)
    prev, cur = {}, {}
    for p in range(6):
        vocab = rng.choice([2, 3, 7, 50])
        base = [rng.randrange(vocab) for _ in range(rng.randint(1, 120))]
        def child():
            t = [x if rng.random() < 0.7 else rng.randrange(vocab) for x in base]
            return t[:rng.randint(1, len(t))] if rng.random() < 0.3 else t
        if p != 5:
            prev[f"p{p}"] = [child() for _ in range(rng.randint(1, 4))]
        if p != 4:
            cur[f"p{p}"] = [child() for _ in range(rng.randint(1, 4))]
    trace = _to_trace({1: prev, 2: cur})
    for plen in (1, 2, 3, 4, 7):
        want = hs_oracle.token_similarity_replay(prev, cur, plen)
        got = token_similarity_replay(trace, (1, 2), plen)
        assert (got.accepted, got.total, got.warmup) == want, plen


@pytest.mark.gpu
def test_gpu_full_size_properties(variant):
    """configs[1]-sized epoch (64 prompts x 8 x 4096): identical epochs accept everything after
    the warm-up; a disjoint vocabulary accepts nothing; a shifted copy accepts all but warm-up."""
    import torch
    from paper_2508_18588_b200.similarity import token_similarity_replay
    rng = np.random.default_rng(7)
    prev = {f"p{i}": [rng.integers(0, 151_936, 4096) for _ in range(8)] for i in range(64)}
    trace = {1: {k: [(t, 1.0) for t in v] for k, v in prev.items()}}
    trace[2] = trace[1]
    for plen in (3, 7):
        r = token_similarity_replay(trace, (1, 2), plen)
        assert r.total == 64 * 8 * 4096 and r.warmup == 64 * 8 * plen
        assert r.accepted == r.total - r.warmup
    trace[3] = {k: [(t + 200_000, 0.0) for t in v] for k, v in prev.items()}
    assert token_similarity_replay(trace, (1, 3), 3).accepted == 0
    torch.cuda.synchronize()
