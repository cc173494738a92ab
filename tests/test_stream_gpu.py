"""Continuous batching (RolloutEngine.rollout_stream) and migration with KV recompute.

Every sequence's output must equal what the fixed-wave engine produces for it (greedy: batch-invariant
kernels, so lane, admission time and companions do not change a bit), its SpecStats must equal the reference
state machine replayed on that output (oracle), and a rollout evicted mid-way and re-admitted -- its KV
recomputed by prefill on another engine (migration, sim.py:719-779) -- must finish with the same tokens and
the same stats as one that never moved.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    torch.cuda.set_device(0)
    from paper_2508_18588_b200.engine import RolloutEngine
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import TINY, Weights
    from paper_2508_18588_b200.synth import mutate
    w = Weights(TINY, "cuda", seed=3)
    B, P, Tmax = 40, 32, 260
    rng = np.random.default_rng(7)
    prompts = rng.integers(0, TINY.vocab, size=(B, P), dtype=np.int32)
    tl = rng.integers(5, Tmax, size=B).astype(np.int32)
    eng = RolloutEngine(TINY, w, n_slots=B, max_len=P + Tmax + 8, device="cuda")
    base = eng.rollout(prompts, [Tmax] * B, speculate=False)       # greedy reference at full length
    hist = [[(mutate(rng, base.tokens[b].astype(np.int64), 0.7, Tmax, TINY.vocab, 4.0), float(rng.random() < .5))
             for _ in range(6)] for b in range(B)]
    idx = GpuIndex(hist)
    return dict(w=w, B=B, P=P, Tmax=Tmax, prompts=prompts, tl=tl, base=base, hist=hist, idx=idx, TINY=TINY)


def _reqs(S, order=None):
    from paper_2508_18588_b200.engine import SeqRequest
    order = range(S["B"]) if order is None else order
    return [SeqRequest(key=int(b), prompt=S["prompts"][b], target_len=int(S["tl"][b]), slot=int(b)) for b in order]


@pytest.mark.parametrize("lanes,spec", [(8, False), (8, True), (13, True)])
def test_stream_equals_waves_and_reference_stats(setup, lanes, spec):
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.engine import RolloutEngine
    S = setup
    eng = RolloutEngine(S["TINY"], S["w"], n_slots=lanes, max_len=S["P"] + S["Tmax"] + 8, device="cuda",
                        check_every=4)
    order = np.argsort(-S["tl"], kind="stable")                     # longest first (length-aware admission)
    res = eng.rollout_stream(_reqs(S, order), index=S["idx"] if spec else None, speculate=spec, admit_min=1)
    assert sorted(res.tokens) == list(range(S["B"]))
    for b in range(S["B"]):
        assert np.array_equal(res.tokens[b], S["base"].tokens[b, :S["tl"][b]]), b
    if spec:
        truths = [S["base"].tokens[b, :S["tl"][b]] for b in range(S["B"])]
        _per, st = C.replay_batch(S["hist"], truths, list(range(S["B"])))
        got = np.stack([res.stats[b] for b in range(S["B"])])
        assert (got == st).all()
        assert res.iterations < int(S["tl"].max()) * S["B"] / lanes
    assert res.admissions == S["B"] and res.generated == int(S["tl"].sum())


def test_migration_with_kv_recompute(setup):
    """Evict every rollout once it has generated >= 40 tokens, re-admit it on a second engine (KV of
    prompt + generated recomputed by prefill): outputs and stats equal the unmigrated run."""
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.engine import RolloutEngine
    S = setup
    mk = lambda: RolloutEngine(S["TINY"], S["w"], n_slots=10, max_len=S["P"] + S["Tmax"] + 8,  # noqa: E731
                               device="cuda", check_every=4)
    a, b = mk(), mk()

    def on_check(busy, gen_len, it, waiting):
        return [ln for ln in busy if gen_len[ln] >= 40]

    r1 = a.rollout_stream(_reqs(S), index=S["idx"], speculate=True, admit_min=1, on_check=on_check)
    moved = r1.evicted
    assert moved, "no rollout reached the migration threshold"
    assert all(len(m.generated) >= 40 for m in moved)
    r2 = b.rollout_stream(moved, index=S["idx"], speculate=True, admit_min=1)
    toks = {**r1.tokens, **r2.tokens}
    stats = {**r1.stats, **r2.stats}
    assert sorted(toks) == list(range(S["B"]))
    truths = [S["base"].tokens[k, :S["tl"][k]] for k in range(S["B"])]
    _per, st = C.replay_batch(S["hist"], truths, list(range(S["B"])))
    for k in range(S["B"]):
        assert np.array_equal(toks[k], truths[k]), k
        assert (stats[k] == st[k]).all(), k


def test_stream_sampling_equals_waves(setup):
    """Rejection-sampling verify (T = 1) under continuous batching: the Gumbel noise is keyed by (sequence key,
    position), so a sequence samples the same tokens whichever lane and admission time it gets -- outputs
    equal the fixed-wave engine's with the same keys, with speculation on and off."""
    from paper_2508_18588_b200.engine import RolloutEngine
    S = setup
    mk = lambda n: RolloutEngine(S["TINY"], S["w"], n_slots=n, max_len=S["P"] + S["Tmax"] + 8,  # noqa: E731
                                 device="cuda", temperature=1.0, seed=11, check_every=4)
    keys = np.arange(S["B"]) * 7 + 3
    waves = mk(S["B"]).rollout(S["prompts"], [S["Tmax"]] * S["B"], speculate=False, seq_keys=keys)
    reqs = _reqs(S)
    for r, k in zip(reqs, keys):
        r.key = int(k)
    for spec in (False, True):
        res = mk(9).rollout_stream(reqs, index=S["idx"] if spec else None, speculate=spec, admit_min=1)
        for b, k in enumerate(keys):
            assert np.array_equal(res.tokens[int(k)], waves.tokens[b, :S["tl"][b]]), (spec, b)
