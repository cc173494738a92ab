"""Host-side state-machine semantics of the drop-in spec_engine (no GPU needed).

Mirrors pkg/tests/test_spec_engine.py:27-206 and acceptance criterion 2
(test_acceptance.py:99-113); expected values from tests/golden/kats.json.
"""

import itertools
import random

import pytest

from conftest import load_golden
from paper_2508_18588_b200 import spec_engine as S


def window_after(history, init=2, step=2, cap=32):
    streak = 0
    for a in reversed(history):
        if not a:
            break
        streak += 1
    return min(init + step * streak, cap)


def test_kats():
    k = load_golden("kats.json")
    for a in k["aimd"]:
        w = S.AimdWindow(size=a["size"], init=a["init"], add_step=a["add"], max=a["max"])
        assert S.next_window(w, a["all"]).size == a["next"]
    for p in k["prefix"]:
        pol = S.PrefixPolicy(current_len=p["cur"], initial_len=p["init"], min_len=p["min"])
        assert S.choose_prefix(pol, p["found"]).current_len == p["next"]
    for v in k["verify"]:
        assert S.verify(v["draft"], v["truth"]) == v["accepted"]
    for g in k["gate"]:
        assert S.gate_check(S.BatchGate(tuple(g["table"])), g["batch"], g["acc"]) == g["speculate"]


def test_criterion_2_aimd_exhaustive():
    checked = 0
    for n in range(13):
        for hist in itertools.product([False, True], repeat=n):
            w = S.AimdWindow()
            for a in hist:
                w = S.next_window(w, a)
            assert w.size == window_after(list(hist))
            checked += 1
    assert checked == 8191


def test_invariants():
    with pytest.raises(ValueError):
        S.AimdWindow(size=64)
    with pytest.raises(ValueError):
        S.BatchGate(tuple([100] * 5 + [50] * 5))
    with pytest.raises(ValueError):
        S.BatchGate((1,) * 9)
    with pytest.raises(ValueError):
        S.PrefixPolicy(current_len=9, initial_len=7)


def test_stats_rates_and_csv():
    st = S.SpecStats()
    st.record(total=3, speculated=2, accepted=2, verify_pass=True)
    st.record(total=1, speculated=0, accepted=0, verify_pass=False)
    assert st.speculation_rate == 0.5 and st.acceptance_rate == 1.0
    assert st.csv_row(1) == [1, "0.500000", "1.000000", 1, 1]
    assert S.SpecStats.CSV_HEADER[0] == "step"


class ListTree:
    """Duck-typed CPU tree (test double) backed by the Python oracle."""

    def __init__(self, corpus):
        self.corpus = corpus

    def extract_draft(self, prefix, window):
        from oracle import hs_oracle as O
        toks, matched, prio = O.extract_draft(self.corpus, prefix, window)
        return type("D", (), {"tokens": toks, "found": matched > 0})()


def test_step_response_output_equals_truth():
    rng = random.Random(5)
    for _ in range(30):
        truth = [rng.randrange(6) for _ in range(rng.randint(1, 120))]
        corpus = [([rng.randrange(6) for _ in range(rng.randint(1, 120))], 1.0) for _ in range(3)]
        if rng.random() < 0.5:
            corpus.append((list(truth), 0.5))
        cfg = S.SpecConfig()
        ctx = S.ResponseContext(truth=truth, tree=ListTree(corpus), window=cfg.new_window(),
                                prefix=cfg.new_prefix(), stats=S.SpecStats())
        iters = 0
        while not ctx.done:
            S.step_response(ctx)
            iters += 1
        assert ctx.generated == truth
        assert ctx.stats.tokens_total == len(truth)
        assert ctx.stats.verify_passes + ctx.stats.decode_passes == iters
        with pytest.raises(S.ResponseComplete):
            S.step_response(ctx)


def test_replay_disabled_is_one_token_per_iter():
    rep = S.replay_response(list(range(50)), None, S.SpecConfig(enabled=False))
    assert rep.tokens_per_iter == [1] * 50
