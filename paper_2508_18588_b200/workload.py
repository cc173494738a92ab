"""Synthetic workloads of BASELINE.json configs (deterministic, seeded).

configs[1] (bench default): Qwen2.5-1.5B-shaped policy, 512 prompts x 8
samples, 4k-token rollouts, greedy verify, 1 GPU.  Histories follow the (D)
definition of SURVEY.md 8(d): each of the G = 8 previous-epoch responses of a
prompt is an independent s-mutation (burst 4) of the prompt's current greedy
rollout; rewards Bernoulli(0.5) in {0, 1}.  Under greedy decoding the 8
samples of a prompt share their prompt tokens, so they produce the same
rollout; the engine still runs all 8 (no deduplication).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .synth import mutate


@dataclass
class ReplayWorkload:
    """History + truths for the HistoSpec bookkeeping path (the reference's own path)."""

    prompts: int = 512
    samples: int = 8
    length: int = 4096
    vocab: int = 151936
    similarity: float = 0.7
    group: int = 8
    seed: int = 0
    shard: int = 0   # rank offset: prompts of shard k are disjoint from shard j

    def generate(self):
        """Flat arrays: history text (int32), resp_off, slot_resp_off, reward_fx; truths + slots."""
        P, G, L = self.prompts, self.group, self.length
        hist = np.empty((P, G, L), dtype=np.int32)
        rewards = np.empty((P, G), dtype=np.float64)
        truths = np.empty((P, L), dtype=np.int32)
        for p in range(P):
            rng = np.random.default_rng([self.seed, self.shard * P + p])
            truth = rng.integers(0, self.vocab, size=L, dtype=np.int64)
            truths[p] = truth
            for g in range(G):
                hist[p, g] = mutate(rng, truth, self.similarity, L, self.vocab, 4.0)
                rewards[p, g] = 1.0 if rng.random() < 0.5 else 0.0
        resp_off = np.arange(P * G + 1, dtype=np.int64) * L
        slot_resp_off = np.arange(P + 1, dtype=np.int64) * G
        reward_fx = (rewards.reshape(-1) * float(1 << 32)).astype(np.int64)
        # every sample of prompt p replays the prompt's rollout
        truth_rows = np.repeat(truths, self.samples, axis=0)
        truth_slots = np.repeat(np.arange(P, dtype=np.int32), self.samples)
        return {"hist_tokens": hist.reshape(-1), "resp_off": resp_off, "slot_resp_off": slot_resp_off,
                "reward_fx": reward_fx, "rewards": rewards.reshape(-1), "truths": truth_rows,
                "truth_slots": truth_slots}


def history_lists(data):
    """Per-slot [(tokens, reward)] lists (for the oracle / drop-in API)."""
    P = len(data["slot_resp_off"]) - 1
    ro, so = data["resp_off"], data["slot_resp_off"]
    out = []
    for p in range(P):
        out.append([(data["hist_tokens"][ro[r]:ro[r + 1]], float(data["rewards"][r]))
                    for r in range(so[p], so[p + 1])])
    return out
