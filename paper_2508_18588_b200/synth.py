"""Synthetic controlled-similarity histories (workload generation, not the hot path).

The reference synthesizes epoch-to-epoch token similarity with geometric
copy/mutate bursts (`rhymesim/tracegen.py:78-162`).  The bench and the parity
tests need byte-identical inputs on the GPU box, where the reference is not
installed, so this module re-derives the same numpy `Generator` call sequence.
`tests/golden/trace_digests.json` pins the output against the reference's own
generator (sha256 over the token lists).

Two similarity definitions are provided:
  (T) `generate_trace`: tracegen semantics -- each epoch's group members are
      s-mutations of the previous epoch's member 0.
  (D) `derive_history`: each of the G history members is an independent
      s-mutation of the current rollout (`_derive_tokens(rng, truth, s, ...)`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class TraceSpec:
    """Knobs of the reference generator (tracegen.py:35-76), same names/defaults."""

    num_prompts: int
    epochs: int
    group_size: int = 16
    vocab_size: int = 32768
    len_mu: float = math.log(300.0)
    len_sigma: float = 0.8
    similarity: float = 0.93
    similarity_schedule: list | None = None
    growth_mean: float = 1.0
    rank_noise: float = 0.95
    length_jitter: float = 0.08
    burst_mean: float = 4.0
    high_reward_frac: float = 0.5
    seed: int = 0

    def sim_at(self, epoch: int) -> float:
        if self.similarity_schedule is not None:
            return self.similarity_schedule[epoch - 1]
        return self.similarity

    def pid(self, index: int) -> str:
        width = max(4, len(str(self.num_prompts - 1)))
        return f"p{index:0{width}d}"


def keep_mask(rng: np.random.Generator, n: int, s: float, burst: float) -> np.ndarray:
    """Alternating geometric keep/mutate runs with mean keep fraction s (tracegen.py:78-97)."""
    mean_keep = burst * s / (1.0 - s)
    p_keep = min(1.0, 1.0 / mean_keep)
    p_mut = min(1.0, 1.0 / burst)
    starts_kept = bool(rng.random() < s)
    runs = max(4, int(2.0 * n / (mean_keep + burst)) + 4)
    p_first, p_second = (p_keep, p_mut) if starts_kept else (p_mut, p_keep)
    while True:
        a = rng.geometric(p_first, size=runs)
        b = rng.geometric(p_second, size=runs)
        lens = np.empty(2 * runs, dtype=np.int64)
        lens[0::2], lens[1::2] = a, b
        if int(lens.sum()) >= n:
            break
        runs *= 2
    flags = np.empty(2 * runs, dtype=bool)
    flags[0::2], flags[1::2] = starts_kept, not starts_kept
    return np.repeat(flags, lens)[:n]


def mutate(rng, parent: np.ndarray, s: float, target_len: int, vocab: int, burst: float) -> np.ndarray:
    """s-similar copy of `parent` resized to target_len (tracegen.py:100-120)."""
    n = min(len(parent), target_len)
    if s >= 1.0:
        body = parent[:n].copy()
    elif s <= 0.0:
        body = rng.integers(0, vocab, size=n, dtype=np.int64)
    else:
        mask = keep_mask(rng, n, s, burst)
        body = np.where(mask, parent[:n], rng.integers(0, vocab, size=n, dtype=np.int64))
    if target_len > n:
        body = np.concatenate([body, rng.integers(0, vocab, size=target_len - n, dtype=np.int64)])
    return body


def generate_trace(spec: TraceSpec):
    """{epoch: {prompt_id: [(tokens(np.int64), reward)]}} in group order (tracegen.py:123-162)."""
    out = {e: {} for e in range(1, spec.epochs + 1)}
    ar = spec.rank_noise ** 0.125
    drift = math.sqrt(max(0.0, 1.0 - ar * ar))
    for p in range(spec.num_prompts):
        rng = np.random.default_rng([spec.seed, p])
        pid = spec.pid(p)
        z = rng.standard_normal()
        first_len = max(1, int(round(math.exp(spec.len_mu + spec.len_sigma * z))))
        parent = rng.integers(0, spec.vocab_size, size=first_len, dtype=np.int64)
        for e in range(1, spec.epochs + 1):
            median = math.exp(spec.len_mu + (e - 1) * math.log(spec.growth_mean) + spec.len_sigma * z)
            s = spec.sim_at(e)
            grp = []
            for _ in range(spec.group_size):
                jit = math.exp(spec.length_jitter * rng.standard_normal()) if spec.length_jitter > 0 else 1.0
                tgt = max(1, int(round(median * jit)))
                toks = mutate(rng, parent, s, tgt, spec.vocab_size, spec.burst_mean)
                rew = 1.0 if rng.random() < spec.high_reward_frac else 0.0
                grp.append((toks, rew))
            parent = np.asarray(grp[0][0], dtype=np.int64)
            out[e][pid] = grp
            z = ar * z + drift * rng.standard_normal()
    return out


def derive_history(rng, truth: np.ndarray, s: float, group: int, vocab: int,
                   burst: float = 4.0, length: int | None = None):
    """(D) definition: G independent s-mutations of the current rollout, rewards Bernoulli(0.5)."""
    length = len(truth) if length is None else length
    hist = []
    for _ in range(group):
        toks = mutate(rng, np.asarray(truth, dtype=np.int64), s, length, vocab, burst)
        rew = 1.0 if rng.random() < 0.5 else 0.0
        hist.append((toks, rew))
    return hist
