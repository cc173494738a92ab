"""Pin the CPU oracle (Python + C restatements) to the reference's golden outputs.

Fixtures come from running the reference package (tests/golden/make_golden.py).
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import load_golden
from oracle import hs_oracle as O
from oracle import hs_oracle_c as C
from paper_2508_18588_b200.synth import TraceSpec, generate_trace


def test_python_oracle_kats():
    k = load_golden("kats.json")
    for d in k["drafts"]:
        corpus = [(t, r) for t, r in d["corpus"]]
        toks, matched, prio = O.extract_draft(corpus, d["prefix"], d["window"])
        assert toks == d["tokens"] and matched == d["matched"] and prio == d["priority"]
    for v in k["verify"]:
        assert O.lcp(v["draft"], v["truth"]) == v["accepted"]
    for g in k["gate"]:
        assert O.gate_check(g["table"], g["batch"], g["acc"]) == g["speculate"]


def test_python_oracle_drafts_golden():
    cases = load_golden("drafts.json.gz")
    n = 0
    for case in cases[:120]:
        corpus = [(t, r) for t, r in case["corpus"]]
        for q in case["queries"]:
            toks, matched, prio = O.extract_draft(corpus, q["prefix"], q["window"])
            assert toks == q["tokens"]
            assert (matched > 0) == q["found"] and matched == q["matched"]
            assert prio == q["priority"]
            n += 1
    assert n == 960


def test_c_oracle_drafts_golden():
    cases = load_golden("drafts.json.gz")
    for case in cases:
        corpus = [(t, r) for t, r in case["corpus"]]
        for q in case["queries"]:
            toks, found, mass = C.draft(corpus, q["prefix"], q["window"])
            assert toks == q["tokens"] and found == q["found"]
            assert mass == q["priority"]


def test_python_oracle_replays_golden():
    for case in load_golden("replays.json.gz")[:40]:
        wi, wa, wm, pi, pm = case["config"]
        cfg = O.Config(True, wi, wa, wm, pi, pm)
        rep = O.replay(case["truth"], [(t, r) for t, r in case["corpus"]], cfg)
        assert rep.tokens_per_iter == case["tokens_per_iter"]
        assert rep.drafted == case["drafted"] and rep.accepted == case["accepted"]
        assert list(rep.stats.as_tuple()) == case["stats"]


def test_c_oracle_replays_golden():
    for case in load_golden("replays.json.gz"):
        wi, wa, wm, pi, pm = case["config"]
        per, stats = C.replay_batch([[(t, r) for t, r in case["corpus"]]], [case["truth"]], [0],
                                    cfg=(1, wi, wa, wm, pi, pm))
        assert per[0] == case["tokens_per_iter"]
        assert stats[0].tolist() == case["stats"]


@pytest.mark.parametrize("row", range(3))
def test_c_oracle_appendix_b_digest(row):
    """Appendix-B replay digest over the full 64x16 trace."""
    g = load_golden("trace_digests.json")[row]
    spec = TraceSpec(num_prompts=64, epochs=2, group_size=16, vocab_size=4096, similarity=g["s"], seed=0)
    tr = generate_trace(spec)
    pids = sorted(tr[1])
    hist = [[(t, r) for t, r in tr[1][p]] for p in pids]
    truths, tprompt = [], []
    for i, p in enumerate(pids):
        for t, _r in tr[2][p]:
            truths.append(t)
            tprompt.append(i)
    per, stats = C.replay_batch(hist, truths, tprompt, threads=4)
    h = hashlib.sha256()
    for tpi in per:
        h.update(json.dumps(tpi).encode())
    assert h.hexdigest() == g["replay_sha"]
    assert stats.sum(axis=0).tolist() == g["stats"]


def test_c_oracle_derived_digest():
    from paper_2508_18588_b200.synth import derive_history
    for g in load_golden("derived_digests.json"):
        hist_h = hashlib.sha256()
        hists, truths = [], []
        for p in range(g["prompts"]):
            rng = np.random.default_rng([g["seed"], p])
            truth = rng.integers(0, g["V"], size=g["L"], dtype=np.int64)
            hist = derive_history(rng, truth, g["s"], g["G"], g["V"])
            for t, _ in hist:
                hist_h.update(np.asarray(t, dtype=np.int64).tobytes())
            hists.append(hist)
            truths.append(truth)
        assert hist_h.hexdigest() == g["history_sha"]
        per, stats = C.replay_batch(hists, truths, list(range(len(truths))), threads=4)
        h = hashlib.sha256()
        for tpi in per:
            h.update(json.dumps(tpi).encode())
        assert h.hexdigest() == g["replay_sha"]
        assert stats.sum(axis=0).tolist() == g["stats"]


def test_oracle_branch0_is_reference_draft(golden):
    """oracle.draft_branches (the checker of hs_lookup_branches): branch 0 equals the reference's
    extract_draft output on the golden corpora, and branch masses are non-increasing."""
    from oracle import hs_oracle as O
    for c in golden("drafts.json.gz")[:60]:
        corpus = [(list(t), float(r)) for t, r in c["corpus"]]
        for q in c["queries"]:
            br, ms = O.draft_branches(corpus, q["prefix"], q["window"], 4)
            assert (br[0] if br else []) == q["tokens"], q
            assert all(a >= b for a, b in zip(ms, ms[1:]))
