"""Per-epoch history pipeline kernels (hs_route.cu) and device routing (workers.route_rollouts_device).

hs_pack_rows is checked exactly; hs_mutate_bursts statistically against tracegen's burst semantics
(tracegen.py:78-120: keep fraction s, mean mutate run `burst`, fresh tokens uniform) and exactly at s = 1.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    torch.cuda.set_device(0)
    return torch


def test_pack_rows(torch):
    from paper_2508_18588_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(1)
    n, stride = 97, 301
    src = torch.randint(0, 1 << 30, (n, stride), dtype=torch.int32, device="cuda")
    lens = rng.integers(0, stride + 1, size=n).astype(np.int64)
    order = rng.permutation(n).astype(np.int32)
    off = np.concatenate([[0], np.cumsum(lens[order])[:-1]]).astype(np.int64)
    dst = torch.full((int(lens.sum()) + 5,), -7, dtype=torch.int32, device="cuda")
    d_order, d_len, d_off = (torch.as_tensor(a).cuda() for a in (order, lens[order], off))   # kept alive
    _lib.check(lib.hs_pack_rows(src.data_ptr(), stride, d_order.data_ptr(), d_len.data_ptr(), d_off.data_ptr(),
                                n, dst.data_ptr(), None))
    h = src.cpu().numpy()
    ref = np.concatenate([h[i, :lens[i]] for i in order])
    out = dst.cpu().numpy()
    assert (out[:len(ref)] == ref).all() and (out[len(ref):] == -7).all()


def _mutate(torch, src2d, G, s, seed=5, vocab=1 << 20):
    from paper_2508_18588_b200 import _lib
    n, L = src2d.shape
    off = torch.arange(n + 1, dtype=torch.int64, device="cuda") * L
    dst = torch.empty(n * G * L, dtype=torch.int32, device="cuda")
    rfx = torch.empty(n * G, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().hs_mutate_bursts(src2d.data_ptr(), off.data_ptr(), n, G, float(s), 4.0, vocab, seed,
                                            dst.data_ptr(), rfx.data_ptr(), None))
    return dst.view(n, G, L), rfx.view(n, G)


@pytest.mark.parametrize("s", [0.3, 0.7, 0.9])
def test_mutate_bursts_statistics(torch, s):
    n, G, L = 64, 8, 4096
    src = torch.randint(0, 1 << 20, (n, L), dtype=torch.int32, device="cuda")
    out, rfx = _mutate(torch, src, G, s)
    keep = (out == src[:, None, :]).cpu().numpy()
    assert abs(keep.mean() - s) < 0.02, keep.mean()
    # mean length of mutated runs ~ burst (4)
    flips = np.diff(keep.astype(np.int8), axis=2)
    runs_mut = (flips == -1).sum()
    assert abs((~keep).sum() / max(1, runs_mut) - 4.0) < 0.4
    # members are independent (not all equal), rewards Bernoulli(0.5) in 2^-32 fixed point
    assert not torch.equal(out[:, 0], out[:, 1])
    r = rfx.cpu().numpy()
    assert set(np.unique(r)) <= {0, 1 << 32} and 0.4 < (r > 0).mean() < 0.6
    # deterministic for a seed
    out2, _ = _mutate(torch, src, G, s)
    assert torch.equal(out, out2)


def test_mutate_bursts_edges(torch):
    from paper_2508_18588_b200 import _lib
    src = torch.randint(0, 1000, (3, 50), dtype=torch.int32, device="cuda")
    out, _ = _mutate(torch, src, 2, 1.0)
    assert torch.equal(out[:, 0], src) and torch.equal(out[:, 1], src)
    out0, _ = _mutate(torch, src, 2, 0.0, vocab=1 << 30)
    assert (out0 != src[:, None, :]).float().mean() > 0.99
    with pytest.raises(ValueError):
        _lib.check(_lib.load().hs_mutate_bursts(src.data_ptr(), None, 3, 0, 0.5, 4.0, 10, 0, None, None, None))


def test_route_world1_feeds_index(torch):
    """world = 1: records come back grouped by prompt in key order, tokens intact; the mutated history of the
    routed rollouts indexes and drafts (the bench's epoch pipeline, end to end on one rank)."""
    from paper_2508_18588_b200 import workers as W
    from paper_2508_18588_b200.index import GpuIndex
    B, S, T, G = 24, 4, 256, 8
    toks = torch.randint(0, 5000, (B, T + 33), dtype=torch.int32, device="cuda")
    pids = np.repeat(np.array([7, 3, 11, 5, 2, 9]), S)
    keys = np.arange(B)
    routed = W.route_rollouts_device(toks[:, :T], np.full(B, T), pids, keys, np.full(B, 1 << 32),
                                     {int(p): 0 for p in pids}, 0, 1)
    order = np.lexsort((np.arange(B), pids))
    assert (routed.pids == pids[order]).all() and (routed.keys == keys[order]).all()
    assert torch.equal(routed.tokens.view(B, T), toks[torch.as_tensor(order).cuda(), :T])
    hist, rfx = _mutate(torch, routed.tokens.view(B, T), G, 0.9)
    idx = GpuIndex.from_arrays(hist.reshape(-1), np.arange(B * G + 1) * T, np.arange(B + 1) * G,
                               rfx.reshape(-1).cpu().numpy())
    truth = routed.tokens.view(B, T).cpu().numpy()
    drafts, info = idx.lookup(list(range(B)), [truth[i, 10:17].tolist() for i in range(B)], [8] * B)
    assert info[:, 0].mean() > 0.5      # most 7-grams of a 0.9-similar history are found
