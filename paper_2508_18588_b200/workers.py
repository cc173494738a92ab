"""Data-parallel rollout workers: prompt -> rank assignment and the epoch-boundary collectives.

One process per GPU; prompts are independent (per-prompt histories, per-
sequence state), so the rollout step itself has no collective.
Two exchanges happen at epoch boundaries only:

  * `broadcast_weights`: the updated policy from rank 0 (NCCL broadcast).
  * `route_rollouts`: finished rollouts move to the rank that owns their prompt
    in the next step, so that rank can ingest them as history (all-to-all-v of
    int32 tokens + lengths + rewards).

Prompt -> rank assignment follows HistoPipe (rhymesim/scheduler.py): prompts
are ranked by last-epoch median length and split into equal groups (remainder
to the longest groups, :22-25, :45-76), and the group -> worker order
alternates ascending / descending between consecutive steps (:79-88).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition_sizes(total: int, groups: int) -> list:
    """Equal split; the remainder goes to the last (longest) groups (scheduler.py:22-25)."""
    base, rem = divmod(total, groups)
    return [base + (1 if i >= groups - rem else 0) for i in range(groups)]


@dataclass
class Group:
    index: int
    prompt_ids: list
    representative_len: float


def build_groups(medians: dict, n_groups: int) -> list:
    """Rank prompts by (median length, id) and cut into equal groups (scheduler.py:45-76)."""
    if n_groups < 1:
        raise ValueError("need at least 1 group")
    if len(medians) < n_groups:
        raise ValueError(f"fewer prompts ({len(medians)}) than groups ({n_groups})")
    ranked = sorted(medians, key=lambda pid: (float(medians[pid]), pid))
    out, i = [], 0
    for g, size in enumerate(partition_sizes(len(ranked), n_groups)):
        members = ranked[i:i + size]
        i += size
        out.append(Group(g, members, sum(float(medians[p]) for p in members) / len(members)))
    return out


def assignment_order(step: int, n_groups: int) -> list:
    """Group served by each worker slot: ascending on odd steps, descending on even (scheduler.py:79-88)."""
    if step < 1:
        raise ValueError("step_index starts at 1")
    order = list(range(n_groups))
    return order if step % 2 == 1 else order[::-1]


def assign_prompts(medians: dict, n_ranks: int, step: int) -> dict:
    """{rank: [prompt ids]} for this step."""
    groups = build_groups(medians, n_ranks)
    order = assignment_order(step, n_ranks)
    return {rank: groups[order[rank]].prompt_ids for rank in range(n_ranks)}


def owner_map(assignment: dict) -> dict:
    return {pid: rank for rank, pids in assignment.items() for pid in pids}


def broadcast_weights(weights, src: int = 0, group=None) -> None:
    """Broadcast every weight tensor of a model.Weights in place (NCCL over NVLink)."""
    import torch.distributed as dist
    tensors = [weights.embed] + ([] if weights.cfg.tied else [weights.lm_head]) + [weights.final_ln]
    for layer in weights.layers:
        tensors += [layer[k] for k in ("ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wd")]
    for t in tensors:
        dist.broadcast(t, src=src, group=group)


def route_rollouts(rollouts: list, next_owner: dict, rank: int, world: int, device="cpu", group=None) -> list:
    """Send each finished rollout to the rank that owns its prompt next step.

    rollouts: [(prompt_id_int, tokens int32 array, reward float)] produced on this rank.
    Returns the rollouts this rank receives (including its own that stay),
    ordered by (source rank, original order) -- deterministic.
    """
    import torch
    import torch.distributed as dist
    if world == 1:
        return [r for r in rollouts if next_owner[r[0]] == rank]
    per_dst = [[] for _ in range(world)]
    for r in rollouts:
        per_dst[next_owner[r[0]]].append(r)
    # payload per record: [pid, len, reward_fx_hi, reward_fx_lo, tokens...] (int32)
    payloads = []
    for d in range(world):
        parts = []
        for pid, toks, rew in per_dst[d]:
            fx = int(round(float(rew) * (1 << 32)))
            hdr = np.array([int(pid), len(toks), (fx >> 32) & 0xFFFFFFFF, fx & 0xFFFFFFFF], dtype=np.int64)
            parts.append(hdr.astype(np.uint32).view(np.int32))
            parts.append(np.asarray(toks, dtype=np.int32))
        payloads.append(np.concatenate(parts) if parts else np.zeros(0, np.int32))
    send_sizes = torch.tensor([len(p) for p in payloads], dtype=torch.int64, device=device)
    recv_sizes = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_to_all_single(recv_sizes, send_sizes, group=group)
    send = torch.from_numpy(np.concatenate(payloads) if sum(map(len, payloads)) else np.zeros(0, np.int32)).to(device)
    recv = torch.empty(int(recv_sizes.sum()), dtype=torch.int32, device=device)
    dist.all_to_all_single(recv, send, output_split_sizes=recv_sizes.tolist(),
                           input_split_sizes=send_sizes.tolist(), group=group)
    flat = recv.cpu().numpy()
    out, i = [], 0
    while i < len(flat):
        pid, n = int(flat[i]), int(flat[i + 1])
        fx = ((int(flat[i + 2]) & 0xFFFFFFFF) << 32) | (int(flat[i + 3]) & 0xFFFFFFFF)
        if fx >= 1 << 63:
            fx -= 1 << 64
        out.append((pid, flat[i + 4:i + 4 + n].copy(), fx / float(1 << 32)))
        i += 4 + n
    return out
