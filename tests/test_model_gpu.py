"""Numerics of the verify-forward kernels (libhsmodel.so) vs plain PyTorch fp32.

Tolerances: GEMM outputs are bf16-rounded fp32 accumulations -> compared to
an fp32 torch reference within 2^-7 relative + 1e-3 absolute.  Full-model
logits (bf16 path) vs the bf16-emulating CPU restatement within 0.05 absolute
(logit std ~0.8) and vs the plain fp32 reference within 0.25; argmax agreement
is required wherever the reference top-2 margin exceeds that bound.
"""

import numpy as np
import pytest


def _kv_major(q, KVH):
    """[rows, H, hd] -> the kernels' kv-group-major [KVH][rows][G][hd] layout (hm_rope_kv_append's)."""
    M, H, hd = q.shape
    return q.view(M, KVH, H // KVH, hd).transpose(0, 1).contiguous()


pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    torch.cuda.set_device(0)
    return torch


def _gemm(M_, epi, x, w, bias=None, out=None, resid=None, amax=None):
    import paper_2508_18588_b200.model as Mo
    L = Mo.lib()
    M, K = x.shape
    N = w.shape[0]
    Mo.check(L.hm_gemm(epi, x.data_ptr(), K, w.data_ptr(), K, M, N, K,
                       bias.data_ptr() if bias is not None else None,
                       out.data_ptr() if out is not None else None, out.shape[1] if out is not None else 0,
                       resid.data_ptr() if resid is not None else None, resid.shape[1] if resid is not None else 0,
                       amax[0].data_ptr() if amax else None, amax[1].data_ptr() if amax else None, None, 0))


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (1, 256, 128), (300, 384, 1536), (1000, 2048, 1536),
                                   (77, 1536, 8960), (200, 1664, 256)])   # 1664: half-empty last 256-wide tile
def test_gemm_store_bias(torch, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, 0, x, w, bias=b, out=out)
    ref = x.float() @ w.float().T + b.float()
    err = (out.float() - ref).abs()
    assert (err <= ref.abs() * 2 ** -7 + 1e-3).all(), float(err.max())


def test_gemm_rows_are_batch_invariant(torch):
    """A row's bits do not depend on M or on the other rows in its tile."""
    g = torch.Generator(device="cuda").manual_seed(3)
    K, N = 1536, 384
    x = torch.randn(517, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    full = torch.empty(517, N, dtype=torch.bfloat16, device="cuda")
    _gemm(517, 0, x, w, out=full)
    perm = torch.randperm(517, device="cuda", generator=g)
    for rows in (perm[:1], perm[:5], perm[:130], perm):
        sub = x[rows].contiguous()
        o = torch.empty(len(rows), N, dtype=torch.bfloat16, device="cuda")
        _gemm(len(rows), 0, sub, w, out=o)
        assert torch.equal(o, full[rows])


@pytest.mark.parametrize("epi,N", [(0, 2048), (4, 1536)])
def test_gemm_tile_width_is_bit_neutral(torch, epi, N):
    """Decode-sized launches use 128-wide tiles, verify-sized ones 256-wide (N >= 1536): the rows they
    share must be bit-identical (greedy under speculation stays bit-exact)."""
    g = torch.Generator(device="cuda").manual_seed(N + epi)
    K = 1536
    x = torch.randn(3000, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)

    def run(M):   # M = 100: 1 x N/256 tiles < SMs -> 128-wide; M = 3000: 24 x N/256 >= SMs -> 256-wide
        if epi == 0:
            o = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            _gemm(M, 0, x[:M].contiguous(), w, bias=b, out=o)
        else:
            o = torch.empty(M, N, dtype=torch.float32, device="cuda")
            _gemm(M, 4, x[:M].contiguous(), w, resid=o)
        return o

    small, large = run(100), run(3000)
    assert torch.equal(small, large[:100])


@pytest.mark.parametrize("epi,N,K,M", [(0, 2048, 1536, 5110), (4, 1536, 1536, 4999), (4, 1536, 8960, 5110),
                                       (1, 17920, 1536, 1111), (3, 38016, 1536, 700), (2, 1536, 1536, 4737)])
def test_gemm_pair_is_bit_neutral(torch, epi, N, K, M):
    """The CTA-pair kernel (cta_group::2, 256 x 256 tiles over two SMs) gives every row the same bits as the
    1-CTA kernels, and matches fp32 torch; ragged M leaves the last pair tile (and whole peer CTAs) part-empty."""
    import paper_2508_18588_b200.model as Mo
    L = Mo.lib()
    g = torch.Generator(device="cuda").manual_seed(N + K + epi)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)
    r0 = torch.randn(M, N, device="cuda", generator=g) if epi == 2 else None

    def run():
        if epi in (0, 1):
            o = torch.zeros(M, N if epi == 0 else N // 2, dtype=torch.bfloat16, device="cuda")
            _gemm(M, epi, x, w, bias=b if epi == 0 else None, out=o)
            return (o,)
        if epi in (2, 4):
            o = r0.clone() if epi == 2 else torch.zeros(M, N, dtype=torch.float32, device="cuda")
            _gemm(M, epi, x, w, resid=o)
            return (o,)
        av = torch.zeros(M, N // 128, dtype=torch.float32, device="cuda")
        ai = torch.zeros(M, N // 128, dtype=torch.int32, device="cuda")
        _gemm(M, 3, x, w, amax=(av, ai))
        return av, ai

    try:
        Mo.check(L.hm_set_gemm_pair(1))
        paired = run()
        Mo.check(L.hm_set_gemm_pair(0))
        single = run()
    finally:
        Mo.check(L.hm_set_gemm_pair(1))
    for a, c in zip(paired, single):
        assert torch.equal(a, c)
    ref = x.float() @ w.float().T
    if epi == 0:
        ref = ref + b.float()
        assert ((paired[0].float() - ref).abs() <= ref.abs() * 2 ** -7 + 1e-3).all()
    elif epi == 4:
        assert torch.allclose(paired[0], ref, rtol=1e-4, atol=1e-3)
    elif epi == 2:
        assert torch.allclose(paired[0], r0 + ref, rtol=1e-4, atol=1e-3)
    elif epi == 3:
        assert torch.equal(paired[1].view(M, -1, 1)[:, :, 0] // 128, torch.arange(N // 128, device="cuda").expand(M, -1))
        best = ref.view(M, N // 128, 128).max(dim=2).values
        assert torch.allclose(paired[0], best, rtol=1e-4, atol=1e-3)


def test_gemm_swiglu_residual_argmax(torch):
    from paper_2508_18588_b200.model import interleave_gate_up
    g = torch.Generator(device="cuda").manual_seed(5)
    M, K, F = 333, 256, 1024
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    gate = (torch.randn(F, K, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    up = (torch.randn(F, K, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    _gemm(M, 1, x, interleave_gate_up(gate, up), out=act)
    gr, ur = x.float() @ gate.float().T, x.float() @ up.float().T
    ref = torch.nn.functional.silu(gr) * ur
    assert ((act.float() - ref).abs() <= ref.abs() * 2 ** -6 + 2e-3).all()
    # residual
    wd = (torch.randn(K, F, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    res = torch.randn(M, K, device="cuda", generator=g)
    res0 = res.clone()
    _gemm(M, 2, act, wd, resid=res)
    ref2 = res0 + act.float() @ wd.float().T
    assert torch.allclose(res, ref2, rtol=1e-4, atol=1e-3)
    # argmax epilogue over a 4096-vocab head and a head whose last 256-wide tile is half empty
    import paper_2508_18588_b200.model as Mo
    for V in (4096, 1664):
        E = (torch.randn(V, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        nt = V // 128
        av = torch.empty(M, nt, device="cuda")
        ai = torch.empty(M, nt, dtype=torch.int32, device="cuda")
        _gemm(M, 3, x, E, amax=(av, ai))
        out = torch.empty(M, dtype=torch.int32, device="cuda")
        Mo.check(Mo.lib().hm_argmax_reduce(av.data_ptr(), ai.data_ptr(), M, nt, None, out.data_ptr(), 0))
        logits = x.float() @ E.float().T
        top2 = logits.topk(2, dim=1).values
        sure = (top2[:, 0] - top2[:, 1]) > 1e-3
        assert (out.long()[sure] == logits.argmax(1)[sure]).all()


def _attn_ref(torch, q, kc, vc, seqs, H, KVH, hd):
    outs = []
    for (qo, ql, p0, slot) in seqs:
        for i in range(ql):
            pos = p0 + i
            for h in range(H):
                kh = h // (H // KVH)
                k = kc[slot, kh, :pos + 1].float()
                v = vc[slot, kh, :pos + 1].float()
                s = (k @ q[qo + i, h].float()) / np.sqrt(hd)
                outs.append(((qo + i, h), torch.softmax(s, 0) @ v))
    return outs


@pytest.mark.parametrize("H,KVH,hd", [(12, 2, 128), (4, 4, 64)])
def test_attention_varlen_and_invariance(torch, H, KVH, hd):
    import paper_2508_18588_b200.model as Mo
    g = torch.Generator(device="cuda").manual_seed(11)
    slots, max_len = 4, 400
    kc = torch.randn(slots, KVH, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(slots, KVH, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
    # (q_off, q_len, pos0, slot): a decode row, a verify block, a prefill-like block
    seqs = [(0, 1, 70, 0), (1, 5, 129, 1), (6, 33, 300, 2), (39, 12, 0, 3)]
    M = 51
    q = torch.randn(M, H, hd, device="cuda", generator=g).to(torch.bfloat16)

    work = torch.empty(64, dtype=torch.int32, device="cuda")

    def run(sq, persistent=True, tma=True):
        i32 = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
        out = torch.zeros(M, H * hd, dtype=torch.bfloat16, device="cuda")
        meta = [i32([s[j] for s in sq]) for j in range(4)]   # keep alive across the launch
        Mo.check(Mo.lib().hm_attention(_kv_major(q, KVH).data_ptr(), kc.data_ptr(), vc.data_ptr(), KVH * max_len * hd,
                                       meta[0].data_ptr(), meta[1].data_ptr(), meta[2].data_ptr(),
                                       meta[3].data_ptr(), len(sq), max(s[1] for s in sq), H, KVH, hd, max_len,
                                       1.0 / np.sqrt(hd), out.data_ptr(), work.data_ptr() if persistent else None,
                                       0, slots if tma else 0, M, 0))
        torch.cuda.synchronize()
        return out.view(M, H, hd)

    out = run(seqs)                          # default family with the work list + TMA maps
    v2 = run(seqs, persistent=False)         # mma.sync kernel, per-sequence schedule
    assert torch.equal(v2, run(seqs, persistent=False, tma=False))   # its TMA- and cp.async-fed stages agree
    for (row, h), ref in _attn_ref(torch, q, kc, vc, seqs, H, KVH, hd):
        assert torch.allclose(out[row, h].float(), ref, atol=2e-2, rtol=2e-2), (row, h)
        assert torch.allclose(v2[row, h].float(), ref, atol=2e-2, rtol=2e-2), (row, h)
    # the verify block of seq 1 computed one row at a time must be bit-identical
    for i in range(5):
        single = run([(1 + i, 1, 129 + i, 1)])
        assert torch.equal(single[1 + i], out[1 + i])


@pytest.mark.gpu
def test_attention_many_items_per_cta(torch):
    """Several work items per persistent CTA (the warp-specialised verify kernel's
    producer runs ahead across items and wraps the stage ring many times):
    identical to the per-sequence schedule and to one-row-at-a-time decode."""
    import paper_2508_18588_b200.model as Mo
    H, KVH, hd = 12, 2, 128
    rng = np.random.default_rng(5)
    n, slots, max_len = 700, 700, 640
    g = torch.Generator(device="cuda").manual_seed(3)
    kc = torch.randn(slots, KVH, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(slots, KVH, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
    q_len = rng.integers(1, 34, size=n)
    q_off = np.concatenate([[0], np.cumsum(q_len)[:-1]])
    pos0 = rng.integers(0, max_len - 34, size=n)
    M = int(q_len.sum())
    q = torch.randn(M, H, hd, device="cuda", generator=g).to(torch.bfloat16)
    work = torch.empty(2 * M + 2, dtype=torch.int32, device="cuda")   # hm_attention_work_size for the decode run below
    i32 = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int32)).cuda()  # noqa: E731

    def run(qo, ql, p0, sl, persistent):
        out = torch.zeros(M, H * hd, dtype=torch.bfloat16, device="cuda")
        meta = [i32(qo), i32(ql), i32(p0), i32(sl)]
        Mo.check(Mo.lib().hm_attention(_kv_major(q, KVH).data_ptr(), kc.data_ptr(), vc.data_ptr(), KVH * max_len * hd,
                                       meta[0].data_ptr(), meta[1].data_ptr(), meta[2].data_ptr(),
                                       meta[3].data_ptr(), len(ql), int(max(ql)), H, KVH, hd, max_len,
                                       1.0 / np.sqrt(hd), out.data_ptr(), work.data_ptr() if persistent else None,
                                       0, slots, M, 0))
        torch.cuda.synchronize()
        return out

    slot = np.arange(n)
    a = run(q_off, q_len, pos0, slot, True)     # tcgen05 kernel
    b = run(q_off, q_len, pos0, slot, False)    # mma.sync kernel
    assert torch.allclose(a.float(), b.float(), atol=2e-2, rtol=2e-2)
    # every row as its own decode query (q_len 1: the 16-row decode kernel)
    rows = np.arange(M)
    seq_of_row = np.repeat(np.arange(n), q_len)
    dec = run(rows, np.ones(M), pos0[seq_of_row] + rows - q_off[seq_of_row], slot[seq_of_row], True)
    assert torch.equal(a, dec)


def test_tiny_forward_logits_vs_reference(torch):
    from oracle import model_ref as R
    from paper_2508_18588_b200.model import TINY, Forward, KVCache, Weights
    w = Weights(TINY, "cuda", seed=0)
    W = R.weights_fp32(w)
    rng = np.random.default_rng(0)
    T = 48
    toks = rng.integers(0, TINY.vocab, size=T)
    cache = KVCache(TINY, 1, 128, "cuda")
    f = Forward(w, cache, 256, "cuda")
    i32 = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int32)).cuda()  # noqa: E731
    logits = torch.empty(T, TINY.vocab, dtype=torch.bfloat16, device="cuda")
    am = f.run(T, i32(toks), i32(np.arange(T)), i32(np.zeros(T)), i32([0]), i32([T]), i32([0]), i32([0]), 1, T,
               logits_out=logits)
    got = logits.float().cpu()
    emu = R.forward_logits(TINY, W, toks, emulate_bf16=True)
    fp = R.forward_logits(TINY, W, toks, emulate_bf16=False)
    assert (got - emu).abs().max() < 0.05, float((got - emu).abs().max())
    assert (got - fp).abs().max() < 0.25, float((got - fp).abs().max())
    top2 = fp.topk(2, dim=1).values
    sure = (top2[:, 0] - top2[:, 1]) > 0.5
    assert (am.cpu().long()[sure] == fp.argmax(1)[sure]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg_name", ["TINY", "QWEN25_1P5B"])
def test_fused_qkv_rope_matches_unfused(torch, cfg_name):
    """hm_gemm_qkv_rope (QKV GEMM + RoPE + KV append in one epilogue) writes the same bits as hm_gemm followed
    by hm_rope_kv_append, and the residual add in the O / down epilogues the same bits as in the next norm:
    logits, argmax and both KV caches, on a ragged two-sequence batch."""
    import paper_2508_18588_b200.model as Mo
    cfg = getattr(Mo, cfg_name)
    if cfg_name != "TINY":
        cfg = Mo.ModelConfig(**{**cfg.__dict__, "n_layers": 2})
    w = Mo.Weights(cfg, "cuda", seed=1)
    i32 = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int32)).cuda()  # noqa: E731
    rng = np.random.default_rng(2)
    lens, starts = [37, 5], [0, 64]
    T = sum(lens)
    toks = rng.integers(0, cfg.vocab, size=T)
    pos = np.concatenate([np.arange(s, s + n) for s, n in zip(starts, lens)])
    slot = np.concatenate([np.full(n, i) for i, n in enumerate(lens)])
    outs = []
    for fused, resid, res_dtype in ((True, False, "bf16"), (False, False, "bf16"), (True, False, "fp32"),
                                    (True, True, "fp32")):
        cache = Mo.KVCache(cfg, 2, 160, "cuda")
        f = Mo.Forward(w, cache, 64, "cuda", residual=res_dtype)
        f.fused_qkv_rope = fused
        f.residual_in_gemm = resid   # residual add in the O / down GEMM epilogues: the same fp32 adds
        logits = torch.empty(T, cfg.vocab, dtype=torch.bfloat16, device="cuda")
        am = f.run(T, i32(toks), i32(pos), i32(slot), i32([0, lens[0]]), i32(lens), i32(starts), i32([0, 1]), 2,
                   max(lens), logits_out=logits)
        torch.cuda.synchronize()
        outs.append((logits.clone(), am.clone(), cache.k(0).clone(), cache.v(cfg.n_layers - 1).clone()))
    # bf16 residual: fused == unfused; fp32 residual: add in the norm == add in the GEMM epilogue
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    for a, b in zip(outs[2], outs[3]):
        assert torch.equal(a, b)


def test_tiny_engine_spec_equals_greedy_and_reference_replay(torch):
    """Greedy HistoSpec output == plain greedy output (bit-exact), and the engine's
    draft/accept profile == the reference state machine replayed on that output."""
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.engine import RolloutEngine
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import TINY, Weights
    from paper_2508_18588_b200.synth import mutate
    w = Weights(TINY, "cuda", seed=1)
    B, P, T = 24, 32, 200
    eng = RolloutEngine(TINY, w, n_slots=B, max_len=P + T + 8, device="cuda")
    rng = np.random.default_rng(1)
    prompts = rng.integers(0, TINY.vocab, size=(B, P), dtype=np.int32)
    base = eng.rollout(prompts, [T] * B, speculate=False, record_tpi=True)
    assert base.iterations == T
    hist = [[(mutate(rng, base.tokens[b].astype(np.int64), 0.7, T, TINY.vocab, 4.0), float(rng.random() < 0.5))
             for _ in range(8)] for b in range(B)]
    idx = GpuIndex(hist)
    spec = eng.rollout(prompts, [T] * B, slots=np.arange(B), index=idx, speculate=True, record_tpi=True)
    assert np.array_equal(spec.tokens, base.tokens)
    per, st = C.replay_batch(hist, [base.tokens[b] for b in range(B)], list(range(B)))
    assert spec.tokens_per_iter == per
    assert (spec.stats == st).all()
    assert spec.iterations < base.iterations


def test_gumbel_sampling_marginal_matches_softmax(torch):
    """hm_lm_head_sample draws from softmax(logit / T): chi-square over 100k keyed draws."""
    import paper_2508_18588_b200.model as Mo
    g = torch.Generator(device="cuda").manual_seed(9)
    K, V, n = 64, 256, 100000
    x1 = torch.randn(1, K, device="cuda", generator=g).to(torch.bfloat16)
    x = x1.repeat(n, 1).contiguous()
    E = (torch.randn(V, K, device="cuda", generator=g) * 0.3).to(torch.bfloat16)
    T = 1.0
    key0 = torch.arange(n, dtype=torch.int32, device="cuda")
    key1 = torch.full((n,), 17, dtype=torch.int32, device="cuda")
    nt = V // 128
    av = torch.empty(n, nt, device="cuda")
    ai = torch.empty(n, nt, dtype=torch.int32, device="cuda")
    L = Mo.lib()
    Mo.check(L.hm_lm_head_sample(x.data_ptr(), K, E.data_ptr(), K, n, V, K, key0.data_ptr(), key1.data_ptr(), 1234,
                                 T, av.data_ptr(), ai.data_ptr(), None, 0))
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    Mo.check(L.hm_argmax_reduce(av.data_ptr(), ai.data_ptr(), n, nt, None, out.data_ptr(), 0))
    counts = torch.bincount(out.long(), minlength=V).double().cpu()
    p = torch.softmax((x1.float() @ E.float().T)[0] / T, 0).double().cpu()
    exp = p * n
    keep = exp >= 5
    chi2 = float((((counts - exp) ** 2) / exp)[keep].sum())
    dof = int(keep.sum()) - 1
    assert chi2 < dof + 6 * (2 * dof) ** 0.5, (chi2, dof)
    # same keys -> same draws (seeded, independent of batch composition)
    sub = slice(1000, 1100)
    av2, ai2 = av[:100].clone(), ai[:100].clone()
    Mo.check(L.hm_lm_head_sample(x[sub].contiguous().data_ptr(), K, E.data_ptr(), K, 100, V, K,
                                 key0[sub].contiguous().data_ptr(), key1[sub].contiguous().data_ptr(), 1234, T,
                                 av2.data_ptr(), ai2.data_ptr(), None, 0))
    out2 = torch.empty(100, dtype=torch.int32, device="cuda")
    Mo.check(L.hm_argmax_reduce(av2.data_ptr(), ai2.data_ptr(), 100, nt, None, out2.data_ptr(), 0))
    assert torch.equal(out2, out[sub])


def test_gumbel_sampling_large_vocab_no_spurious_winners(torch):
    """V = 151,936 (the Qwen head): one dominant logit (+20 over 0) loses with probability
    (V - 1) e^-20 / (1 + (V - 1) e^-20) = 3.1e-4 per row, i.e. ~2.6 of 8,192 rows.  A Gumbel uniform that
    rounds to 0 or 1 gives an infinite noise value that beats any logit, so a random token wins; with 32-bit
    uniforms that happens on ~0.45% of rows (~37 here).  Every per-tile partial must also be finite."""
    import paper_2508_18588_b200.model as Mo
    K, V, n = 64, 151936, 8192
    x = torch.zeros(n, K, dtype=torch.bfloat16, device="cuda")
    x[:, 0] = 1.0
    E = torch.zeros(V, K, dtype=torch.bfloat16, device="cuda")
    hot = 12345
    E[hot, 0] = 20.0
    key0 = torch.arange(n, dtype=torch.int32, device="cuda")
    key1 = torch.full((n,), 3, dtype=torch.int32, device="cuda")
    nt = V // 128
    av = torch.empty(n, nt, device="cuda")
    ai = torch.empty(n, nt, dtype=torch.int32, device="cuda")
    L = Mo.lib()
    Mo.check(L.hm_lm_head_sample(x.data_ptr(), K, E.data_ptr(), K, n, V, K, key0.data_ptr(), key1.data_ptr(), 77,
                                 1.0, av.data_ptr(), ai.data_ptr(), None, 0))
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    Mo.check(L.hm_argmax_reduce(av.data_ptr(), ai.data_ptr(), n, nt, None, out.data_ptr(), 0))
    assert torch.isfinite(av).all()
    misses = int((out != hot).sum())
    assert misses <= 12, misses     # Poisson(2.6): P(> 12) ~ 1e-5


def test_tiny_engine_rejection_sampling_spec_equals_plain_sampling(torch):
    """T = 1.0: HistoSpec output == plain sampling output with the same seed (Gumbel-max coupling),
    and the accept profile == reference state machine on that output."""
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.engine import RolloutEngine
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import TINY, Weights
    from paper_2508_18588_b200.synth import mutate
    w = Weights(TINY, "cuda", seed=3)
    B, P, T = 16, 24, 160
    eng = RolloutEngine(TINY, w, n_slots=B, max_len=P + T + 8, device="cuda", temperature=1.0, seed=99)
    rng = np.random.default_rng(3)
    prompts = rng.integers(0, TINY.vocab, size=(B, P), dtype=np.int32)
    base = eng.rollout(prompts, [T] * B, speculate=False)
    hist = [[(mutate(rng, base.tokens[b].astype(np.int64), 0.7, T, TINY.vocab, 4.0), 1.0) for _ in range(8)]
            for b in range(B)]
    spec = eng.rollout(prompts, [T] * B, slots=np.arange(B), index=GpuIndex(hist), speculate=True, record_tpi=True)
    assert np.array_equal(spec.tokens, base.tokens)
    per, _ = C.replay_batch(hist, [base.tokens[b] for b in range(B)], list(range(B)))
    assert spec.tokens_per_iter == per
    # sampling is not greedy: outputs differ from the T=0 engine
    greedy = RolloutEngine(TINY, w, n_slots=B, max_len=P + T + 8, device="cuda").rollout(prompts, [T] * B,
                                                                                        speculate=False)
    assert not np.array_equal(greedy.tokens, base.tokens)


def test_qwen7b_shape_rejection_sampling(torch):
    """configs[2]: Qwen2.5-7B shape (untied head, GQA 7, V=152,064) at T=1.0, small batch:
    speculative sampling output == plain sampling output; profile == reference replay."""
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.engine import RolloutEngine
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import QWEN25_7B, Weights
    from paper_2508_18588_b200.synth import mutate
    w = Weights(QWEN25_7B, "cuda", seed=0)
    B, P, T = 4, 48, 96
    eng = RolloutEngine(QWEN25_7B, w, n_slots=B, max_len=P + T + 8, device="cuda", temperature=1.0, seed=5)
    rng = np.random.default_rng(4)
    prompts = rng.integers(0, QWEN25_7B.vocab, size=(B, P), dtype=np.int32)
    base = eng.rollout(prompts, [T] * B, speculate=False)
    hist = [[(mutate(rng, base.tokens[b].astype(np.int64), 0.7, T, QWEN25_7B.vocab, 4.0), 1.0) for _ in range(8)]
            for b in range(B)]
    spec = eng.rollout(prompts, [T] * B, slots=np.arange(B), index=GpuIndex(hist), speculate=True, record_tpi=True)
    assert np.array_equal(spec.tokens, base.tokens)
    per, _ = C.replay_batch(hist, [base.tokens[b] for b in range(B)], list(range(B)))
    assert spec.tokens_per_iter == per
    del eng, w
    torch.cuda.empty_cache()


def test_qwen_shape_engine_spec_equals_greedy(torch):
    """Qwen2.5-1.5B shape, small batch: bit-exact spec == greedy, profile == reference replay."""
    from oracle import hs_oracle_c as C
    from paper_2508_18588_b200.engine import RolloutEngine
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import QWEN25_1P5B, Weights
    from paper_2508_18588_b200.synth import mutate
    w = Weights(QWEN25_1P5B, "cuda", seed=0)
    B, P, T = 8, 64, 160
    eng = RolloutEngine(QWEN25_1P5B, w, n_slots=B, max_len=P + T + 8, device="cuda")
    rng = np.random.default_rng(2)
    prompts = rng.integers(0, QWEN25_1P5B.vocab, size=(B, P), dtype=np.int32)
    base = eng.rollout(prompts, [T] * B, speculate=False)
    hist = [[(mutate(rng, base.tokens[b].astype(np.int64), 0.7, T, QWEN25_1P5B.vocab, 4.0), 1.0)
             for _ in range(8)] for b in range(B)]
    idx = GpuIndex(hist)
    spec = eng.rollout(prompts, [T] * B, slots=np.arange(B), index=idx, speculate=True, record_tpi=True)
    assert np.array_equal(spec.tokens, base.tokens)
    per, st = C.replay_batch(hist, [base.tokens[b] for b in range(B)], list(range(B)))
    assert spec.tokens_per_iter == per
    # outputs are not a degenerate loop
    distinct = len({tuple(base.tokens[b, i:i + 4]) for b in range(B) for i in range(T - 4)}) / (B * (T - 4))
    assert distinct > 0.5, distinct


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["mma_sync", "mma_sync_w8", "tcgen05"])
def test_attention_family_subprocess(family):
    """Each attention kernel family (chosen per process) against the fp32 reference, decode-row
    invariance and spec == greedy, in a fresh interpreter."""
    import os
    import subprocess
    import sys
    env = dict(os.environ)
    env.pop("HM_ATTN_V2", None)
    env.pop("HM_ATTN_W8", None)
    env.pop("HM_ATTN_MMA", None)
    if family in ("mma_sync", "mma_sync_w8"):
        env["HM_ATTN_MMA"] = "1"
    if family == "mma_sync_w8":
        env["HM_ATTN_W8"] = "1"
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "attn_family_check.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
