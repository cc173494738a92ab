"""GPU parity of the speculation state machine (K2 + K6) against the reference.

Golden sources: tests/golden/replays.json.gz (reference replay_response on
random cases), trace_digests.json (SURVEY Appendix B, 64x16 tracegen traces)
and derived_digests.json ((D) histories, L=2048).
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _sha(per):
    h = hashlib.sha256()
    for tpi in per:
        h.update(json.dumps(tpi).encode())
    return h.hexdigest()


@pytest.fixture(scope="module")
def mods():
    import paper_2508_18588_b200.history as H
    import paper_2508_18588_b200.spec_engine as S
    return H, S


def test_replays_golden(mods):
    H, S = mods
    for case in load_golden("replays.json.gz"):
        wi, wa, wm, pi, pm = case["config"]
        cfg = S.SpecConfig(window_init=wi, window_add=wa, window_max=wm, prefix_init=pi, prefix_min=pm)
        tree = H.build_tree("p", 1, [H.Response("p", 1, t, r) for t, r in case["corpus"]])
        stats = S.SpecStats()
        rep = S.replay_response(case["truth"], tree, cfg, stats=stats)
        assert rep.tokens_per_iter == case["tokens_per_iter"]
        assert rep.drafted == case["drafted"] and rep.accepted == case["accepted"]
        assert [stats.tokens_total, stats.tokens_speculated, stats.tokens_accepted, stats.verify_passes,
                stats.decode_passes] == case["stats"]


def _appendix_b(s):
    from paper_2508_18588_b200.synth import TraceSpec, generate_trace
    tr = generate_trace(TraceSpec(num_prompts=64, epochs=2, group_size=16, vocab_size=4096, similarity=s, seed=0))
    pids = sorted(tr[1])
    hist = [[(t, r) for t, r in tr[1][p]] for p in pids]
    truths, slots = [], []
    for i, p in enumerate(pids):
        for t, _ in tr[2][p]:
            truths.append(t)
            slots.append(i)
    return hist, truths, slots


@pytest.mark.parametrize("row", range(3))
def test_appendix_b_fused(mods, row):
    H, S = mods
    from paper_2508_18588_b200.index import GpuIndex
    g = load_golden("trace_digests.json")[row]
    hist, truths, slots = _appendix_b(g["s"])
    idx = GpuIndex(hist)
    per, st = S.replay_batch(idx, slots, truths, S.SpecConfig())
    assert _sha(per) == g["replay_sha"]
    assert st.sum(axis=0).tolist() == g["stats"]


def test_appendix_b_stepwise_engine(mods):
    """Per-iteration engine (K2 launch + K6 launch per step) == reference replay."""
    H, S = mods
    import torch
    from paper_2508_18588_b200.index import GpuIndex
    g = load_golden("trace_digests.json")[1]
    hist, truths, slots = _appendix_b(g["s"])
    idx = GpuIndex(hist)
    L = max(len(t) for t in truths)
    truth = np.zeros((len(truths), L + 40), dtype=np.int32)
    for i, t in enumerate(truths):
        truth[i, :len(t)] = t
    b = S.SpecBatch(slots, [len(t) for t in truths], S.SpecConfig())
    d_truth = torch.from_numpy(truth).cuda()
    for _ in range(L + 1):
        b.propose(idx)
        b.accept_replay(d_truth, truth.shape[1])
    assert int((b.gen_len.cpu() == b.target_len.cpu()).all())
    gen = b.gen_tok.cpu().numpy()
    for i, t in enumerate(truths):
        assert (gen[i, :len(t)] == t).all()
    assert _sha(b.tokens_per_iter()) == g["replay_sha"]
    assert b.stats.cpu().numpy().sum(axis=0).tolist() == g["stats"]


@pytest.mark.parametrize("pi,pm,wm", [(7, 3, 32), (9, 2, 32), (5, 1, 12)])
def test_stepwise_draft_paths_match_oracle(mods, pi, pm, wm):
    """K2 8-lane-group path (prefixes tabled, <= 8) and warp/SA fallback path vs the C oracle."""
    H, S = mods
    import torch
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.index import GpuIndex
    hist, truths, slots = _appendix_b(0.8)
    truths, slots = truths[:300], slots[:300]
    cfg = S.SpecConfig(window_max=wm, prefix_init=pi, prefix_min=pm)
    idx = GpuIndex(hist, prefix_min=3, prefix_max=7)
    L = max(len(t) for t in truths)
    truth = np.zeros((len(truths), L + 40), dtype=np.int32)
    for i, t in enumerate(truths):
        truth[i, :len(t)] = t
    b = S.SpecBatch(slots, [len(t) for t in truths], cfg)
    d_truth = torch.from_numpy(truth).cuda()
    for _ in range(L + 1):
        b.propose(idx)
        b.accept_replay(d_truth, truth.shape[1])
    per, st = C.replay_batch(hist, truths, slots, cfg=(1, cfg.window_init, cfg.window_add, wm, pi, pm))
    assert b.tokens_per_iter() == per
    assert (b.stats.cpu().numpy() == st).all()


def test_accept_greedy_with_oracle_argmax(mods):
    """K6 greedy: a model whose argmax reproduces the truth lands the same profile."""
    H, S = mods
    import torch
    from paper_2508_18588_b200.index import GpuIndex
    g = load_golden("trace_digests.json")[2]
    hist, truths, slots = _appendix_b(g["s"])
    truths, slots = truths[:256], slots[:256]
    idx = GpuIndex(hist)
    b = S.SpecBatch(slots, [len(t) for t in truths], S.SpecConfig())
    n = len(truths)
    L = max(len(t) for t in truths)
    padded = np.zeros((n, L + 64), dtype=np.int32)
    for i, t in enumerate(truths):
        padded[i, :len(t)] = t
    d_truth = torch.from_numpy(padded).cuda()
    for _ in range(L + 1):
        b.propose(idx)
        # verify rows: row i of seq s = truth[pos + i] (what a perfect model predicts)
        q = (b.draft_len + 1).to(torch.int32)
        q_off = torch.zeros(n, dtype=torch.int32, device="cuda")
        q_off[1:] = torch.cumsum(q, 0)[:-1].to(torch.int32)
        rows = torch.arange(int(q.sum()), device="cuda")
        seq = torch.repeat_interleave(torch.arange(n, device="cuda"), q.long())
        i = rows - q_off[seq].long()
        pos = b.gen_len[seq].long() + i
        argmax = d_truth[seq, pos.clamp(max=padded.shape[1] - 1)].to(torch.int32).contiguous()
        b.accept_greedy(argmax, q_off)
    ref_per, ref_st = S.replay_batch(idx, slots, truths, S.SpecConfig())
    assert b.tokens_per_iter() == ref_per
    assert (b.stats.cpu().numpy() == ref_st).all()


def test_derived_digest(mods):
    H, S = mods
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.synth import derive_history
    for g in load_golden("derived_digests.json"):
        hists, truths = [], []
        for p in range(g["prompts"]):
            rng = np.random.default_rng([g["seed"], p])
            truth = rng.integers(0, g["V"], size=g["L"], dtype=np.int64)
            hists.append(derive_history(rng, truth, g["s"], g["G"], g["V"]))
            truths.append(truth)
        idx = GpuIndex(hists)
        per, st = S.replay_batch(idx, list(range(len(truths))), truths, S.SpecConfig())
        assert _sha(per) == g["replay_sha"]
        assert st.sum(axis=0).tolist() == g["stats"]


def test_large_derived_vs_c_oracle(mods):
    """(D) histories at L=4096, G=8, 32 prompts: GPU == C oracle (bit-exact profiles)."""
    H, S = mods
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.synth import derive_history
    hists, truths = [], []
    for p in range(32):
        rng = np.random.default_rng([99, p])
        truth = rng.integers(0, 151936, size=4096, dtype=np.int64)
        hists.append(derive_history(rng, truth, 0.7, 8, 151936))
        truths.append(truth)
    idx = GpuIndex(hists)
    per, st = S.replay_batch(idx, list(range(32)), truths, S.SpecConfig())
    cper, cst = C.replay_batch(hists, truths, list(range(32)), threads=8)
    assert per == cper
    assert (st == cst).all()


def test_step_response_with_gpu_tree(mods):
    """Reference step_response semantics with the duck-typed GPU tree."""
    H, S = mods
    truth = list(range(1, 11))
    tree = H.build_tree("p", 1, [H.Response("p", 1, list(truth), 1.0)])
    cfg = S.SpecConfig(prefix_init=3, prefix_min=3)
    ctx = S.ResponseContext(truth=truth, tree=tree, window=cfg.new_window(), prefix=cfg.new_prefix(),
                            stats=S.SpecStats())
    for _ in range(3):
        S.step_response(ctx)
    out = S.step_response(ctx)
    assert out.used_speculation and out.accepted == 2 and out.tokens_appended == 3
    assert ctx.window.size == 4
