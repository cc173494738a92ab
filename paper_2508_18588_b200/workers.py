"""Data-parallel rollout workers: prompt -> rank assignment and the epoch-boundary collectives.

One process per GPU; prompts are independent (per-prompt histories, per-
sequence state), so the rollout step itself has no collective.
Two exchanges happen at epoch boundaries only:

  * `broadcast_weights`: the updated policy from rank 0 (NCCL broadcast).
  * `route_rollouts_device`: finished rollouts move, without leaving HBM, to
    the rank that owns their prompt in the next step, so that rank can ingest
    them as history (hs_pack_rows + all-to-all-v of int32 tokens and an int64
    (prompt, key, length, reward) record table).  `route_rollouts` is the
    host-list form of the same exchange (API glue and tests).

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
    """Broadcast the policy from `src` in place: one NCCL call over the weights' flat buffer (model.Weights.flat).

    Replaces round 1's ~200 per-tensor broadcasts (launch-latency bound, ~390 GB/s for 3.1 GB)."""
    import torch.distributed as dist
    dist.broadcast(weights.flat, src=src, group=group)


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


# ---------------------------------------------------------------- device-resident routing (epoch pipeline)

@dataclass
class RoutePlan:
    order: np.ndarray        # record indices in send order (by destination, then prompt, then input order)
    dest: np.ndarray         # destination rank of each record (input order)
    counts: np.ndarray       # [world] records per destination
    tok_counts: np.ndarray   # [world] tokens per destination
    dst_off: np.ndarray      # [n] offset of each sent record (send order) in the flat send buffer


def plan_routes(pids, lengths, next_owner: dict, world: int) -> RoutePlan:
    """Host side of the exchange: destination of every record and the send layout (deterministic)."""
    pids = np.asarray(pids, dtype=np.int64)
    lengths = np.asarray(lengths, dtype=np.int64)
    dest = np.array([next_owner[int(p)] for p in pids], dtype=np.int64)
    if len(dest) and (dest.min() < 0 or dest.max() >= world):
        raise ValueError("next_owner maps a prompt outside [0, world)")
    order = np.lexsort((np.arange(len(pids)), pids, dest)) if len(pids) else np.zeros(0, np.int64)
    counts = np.bincount(dest, minlength=world).astype(np.int64)
    tok_counts = np.bincount(dest, weights=lengths, minlength=world).astype(np.int64)
    ls = lengths[order]
    dst_off = np.concatenate([[0], np.cumsum(ls)[:-1]]).astype(np.int64) if len(ls) else np.zeros(0, np.int64)
    return RoutePlan(order, dest, counts, tok_counts, dst_off)


def exchange_route_meta(plan: RoutePlan, meta: np.ndarray, device, group=None):
    """All-to-all of the per-destination (records, tokens) counts and of the [n, 4] int64 record table
    (prompt id, sequence key, length, reward fixed point) in send order.  Returns (recv counts [world, 2],
    recv table [m, 4]) as numpy -- the receiver's resp_off / slots / rewards for hs_index_build."""
    import torch
    import torch.distributed as dist
    world = len(plan.counts)
    cnt = torch.as_tensor(np.stack([plan.counts, plan.tok_counts], axis=1)).to(device)
    rcnt = torch.empty_like(cnt)
    dist.all_to_all_single(rcnt, cnt, group=group)
    rc = rcnt.cpu().numpy()
    send = torch.as_tensor(np.ascontiguousarray(meta[plan.order])).reshape(-1, 4).to(device)
    recv = torch.empty((int(rc[:, 0].sum()), 4), dtype=torch.int64, device=device)
    dist.all_to_all_single(recv, send, output_split_sizes=rc[:, 0].tolist(),
                           input_split_sizes=plan.counts.tolist(), group=group)
    return rc.reshape(world, 2), recv.cpu().numpy()


@dataclass
class RoutedRollouts:
    """Rollouts received for the next epoch, slot-major (one record per slot), ready for GpuIndex.from_arrays."""
    tokens: object           # torch int32 [sum(lengths)] on the device
    resp_off: np.ndarray     # int64 [n + 1]
    pids: np.ndarray         # int64 [n]
    keys: np.ndarray         # int64 [n] sequence keys (prompt, sample)
    reward_fx: np.ndarray    # int64 [n]


def route_rollouts_device(tokens, lengths, pids, keys, reward_fx, next_owner: dict, rank: int, world: int,
                          stream=None, group=None) -> RoutedRollouts:
    """Send each finished rollout (row i of the device matrix `tokens` [n, stride], first lengths[i] tokens) to
    the rank owning its prompt next step; return what this rank receives, in (source rank, prompt, input)
    order.  Tokens stay in HBM: hs_pack_rows gathers the send buffer, NCCL moves it (all-to-all-v)."""
    import ctypes  # noqa: F401
    import torch
    import torch.distributed as dist
    from . import _lib
    lib = _lib.load()
    dev = tokens.device
    n = tokens.shape[0]
    lengths = np.asarray(lengths, dtype=np.int64)
    plan = plan_routes(pids, lengths, next_owner, world)
    meta = np.stack([np.asarray(pids, np.int64), np.asarray(keys, np.int64), lengths,
                     np.asarray(reward_fx, np.int64)], axis=1) if n else np.zeros((0, 4), np.int64)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev), torch.cuda.stream(s):
        total = int(lengths.sum())
        send = torch.empty(max(1, total), dtype=torch.int32, device=dev)
        rows = torch.as_tensor(plan.order.astype(np.int32)).to(dev, non_blocking=True)
        lens = torch.as_tensor(lengths[plan.order]).to(dev, non_blocking=True)
        offs = torch.as_tensor(plan.dst_off).to(dev, non_blocking=True)
        _lib.check(lib.hs_pack_rows(tokens.data_ptr(), tokens.stride(0), rows.data_ptr(), lens.data_ptr(),
                                    offs.data_ptr(), n, send.data_ptr(), s.cuda_stream))
        if world == 1:
            m = meta[plan.order]
            recv = send[:total]
        else:
            rc, m = exchange_route_meta(plan, meta, dev, group)
            recv = torch.empty(max(1, int(rc[:, 1].sum())), dtype=torch.int32, device=dev)
            dist.all_to_all_single(recv, send[:total], output_split_sizes=rc[:, 1].tolist(),
                                   input_split_sizes=plan.tok_counts.tolist(), group=group)
            recv = recv[:int(rc[:, 1].sum())]
    resp_off = np.concatenate([[0], np.cumsum(m[:, 2])]).astype(np.int64)
    return RoutedRollouts(recv, resp_off, m[:, 0].copy(), m[:, 1].copy(), m[:, 3].copy())


# ---------------------------------------------------------------- HistoPipe two-tier allocation + migration
# Semantics of rhymesim/scheduler.py:120-330 (ProfileCostModel, cal_wks, plan_allocation, beta_from_history,
# migration_decision), restated for the GPU workers: a "worker" is one GPU running the continuous-batching
# engine, and tau(len, k) comes from the engine's own measured iteration costs (bench.py --workload longtail
# writes the profile CSV, profiles/r02_tau_profile_*.csv).

@dataclass
class TauProfile:
    """tau(length, workers) over a measured (length x workers) grid: bilinear inside, clamped outside
    (scheduler.py:120-170).  `accepted_per_pass` divides every estimate (speculation lands 1 + a tokens/pass)."""
    lengths: list
    workers: list
    seconds: list                 # [length index][worker index]
    accepted_per_pass: float = 0.0

    @classmethod
    def from_rows(cls, rows, accepted_per_pass: float = 0.0):
        """rows: iterable of (len, dp, seconds); the grid must be complete."""
        cell = {(float(l), int(k)): float(t) for l, k, t in rows}
        ls = sorted({l for l, _ in cell})
        ks = sorted({k for _, k in cell})
        missing = [(l, k) for l in ls for k in ks if (l, k) not in cell]
        if missing:
            raise ValueError(f"profile grid is incomplete: missing {missing[0]}")
        return cls(ls, ks, [[cell[(l, k)] for k in ks] for l in ls], accepted_per_pass)

    @classmethod
    def from_csv(cls, path, accepted_per_pass: float = 0.0):
        import csv
        with open(path, newline="") as fh:
            rd = csv.DictReader(fh)
            if rd.fieldnames is None or not {"len", "dp", "seconds"} <= set(rd.fieldnames):
                raise ValueError("profile CSV needs columns ['dp', 'len', 'seconds']")
            return cls.from_rows(((r["len"], r["dp"], r["seconds"]) for r in rd), accepted_per_pass)

    def to_csv(self, path):
        with open(path, "w") as fh:
            fh.write("len,dp,seconds\n")
            for i, l in enumerate(self.lengths):
                for j, k in enumerate(self.workers):
                    fh.write(f"{l:g},{k},{self.seconds[i][j]:.6f}\n")

    @staticmethod
    def _bracket(axis, x):
        if x <= axis[0]:
            return 0, 0, 0.0
        if x >= axis[-1]:
            return len(axis) - 1, len(axis) - 1, 0.0
        import bisect
        hi = bisect.bisect_left(axis, x)
        if axis[hi] == x:
            return hi, hi, 0.0
        return hi - 1, hi, (x - axis[hi - 1]) / (axis[hi] - axis[hi - 1])

    def tau(self, length: float, workers: int) -> float:
        i0, i1, a = self._bracket(self.lengths, float(length))
        j0, j1, b = self._bracket([float(k) for k in self.workers], float(workers))
        s = self.seconds
        lo = s[i0][j0] + (s[i0][j1] - s[i0][j0]) * b
        hi = s[i1][j0] + (s[i1][j1] - s[i1][j0]) * b
        return (lo + (hi - lo) * a) / (1.0 + self.accepted_per_pass)


def workers_for_gradient(d, lens, t0, model, min_wks=1, max_wks=None):
    """Fewest workers per group so that group i finishes by t0 + i * d (cal_wks, scheduler.py:173-206).
    Returns (total, plan), or (inf, []) when a group misses its deadline even at max_wks."""
    import math
    max_wks = len(lens) if max_wks is None else max_wks
    plan = []
    for i, length in enumerate(lens):
        k = next((k for k in range(min_wks, max_wks + 1) if model.tau(length, k) <= t0 + i * d), None)
        if k is None:
            return math.inf, []
        plan.append(k)
    return sum(plan), plan


@dataclass
class AllocationPlan:
    per_group_workers: list
    gradient_d: float
    t0: float
    feasible: bool


def plan_allocation(lens, wks: int, t_train: float, model, min_wks: int = 1, max_wks: int | None = None,
                    precision: float = 1.0) -> AllocationPlan:
    """Smallest finish-time gradient d (binary search) whose per-group worker counts fit in `wks`
    (scheduler.py:224-266).  t0 = the shortest group's best time, floored at the training time."""
    n = len(lens)
    if n < 2:
        raise ValueError("plan_allocation needs at least 2 groups")
    if any(a > b for a, b in zip(lens, lens[1:])):
        raise ValueError("lens must be sorted ascending")
    if max_wks is None:
        max_wks = max(min_wks, wks - (n - 1))
    if wks < n * min_wks:
        return AllocationPlan([], 0.0, t_train, False)
    t0 = max(model.tau(lens[0], max_wks), t_train)
    hi = max(0.0, (model.tau(lens[-1], min_wks) - t0) / (n - 1))
    lo = 0.0
    total, plan = workers_for_gradient(hi, lens, t0, model, min_wks, max_wks)
    if total > wks:
        return AllocationPlan([], hi, t0, False)
    best = (plan, hi)
    while hi - lo > precision:
        mid = 0.5 * (lo + hi)
        total, plan = workers_for_gradient(mid, lens, t0, model, min_wks, max_wks)
        if total > wks:
            lo = mid
        else:
            best, hi = (plan, mid), mid
    return AllocationPlan(best[0], best[1], t0, True)


def plan_makespan(lens, wks: int, model, min_wks: int = 1) -> AllocationPlan:
    """Rollout-only variant of the two-tier allocation: the per-group worker counts that minimise the slowest
    group's tau (every group's deadline is the same T: workers_for_gradient with d = 0, T the smallest
    candidate whose plan fits in `wks`).  plan_allocation's staggered deadlines t0 + i * d exist to overlap
    short groups' training with long groups' rollouts (scheduler.py:224-266); a rollout-throughput
    benchmark with no training stage wants them all to finish together."""
    n = len(lens)
    if n < 1 or wks < n * min_wks:
        return AllocationPlan([], 0.0, 0.0, False)
    hi_k = max(min_wks, wks - (n - 1) * min_wks)
    cands = sorted({model.tau(l, k) for l in lens for k in range(min_wks, hi_k + 1)})
    for T in cands:
        total, plan = workers_for_gradient(0.0, lens, T, model, min_wks, hi_k)
        if total <= wks:
            # hand spare workers to the groups that gain most (longest first)
            spare = wks - total
            for i in sorted(range(n), key=lambda i: -lens[i]):
                while spare > 0 and model.tau(lens[i], plan[i] + 1) < model.tau(lens[i], plan[i]):
                    plan[i] += 1
                    spare -= 1
            return AllocationPlan(plan, 0.0, T, True)
    return AllocationPlan([], 0.0, 0.0, False)


def assign_with_plan(groups: list, per_group_workers: list, step: int) -> dict:
    """{rank: prompt ids}: group i gets per_group_workers[i] consecutive ranks (the group order alternates
    with the step, scheduler.py:79-88); a group's prompts, in length order, are dealt round-robin over its
    ranks so every rank of a group sees the same length mix."""
    order = assignment_order(step, len(groups))
    out, rank = {}, 0
    for slot in range(len(groups)):
        g = order[slot]
        k = per_group_workers[g]
        ranks = list(range(rank, rank + k))
        for r in ranks:
            out[r] = []
        for i, pid in enumerate(groups[g].prompt_ids):
            out[ranks[i % k]].append(pid)
        rank += k
    return out


def beta_from_history(growth_rates) -> float:
    """Length-growth threshold: nearest-rank 75th percentile, at least 1.1 (scheduler.py:269-275)."""
    import math
    if not growth_rates:
        return 1.1
    r = sorted(growth_rates)
    return max(r[max(math.ceil(0.75 * len(r)), 1) - 1], 1.1)


@dataclass
class MigrationPolicy:
    alpha_pct: float = 10.0
    beta: float = 1.1
    beta_floor: float = 1.1

    def __post_init__(self):
        if not 0.0 < self.alpha_pct < 100.0:
            raise ValueError("alpha_pct must be in (0, 100)")
        self.beta = max(self.beta, self.beta_floor)


def migration_decision(group_index: int, group_max_hist_len: float, generated_len: int, completed: int,
                       total: int, policy: MigrationPolicy, n_groups: int, active_group_loads: dict):
    """("none" | "intra_step" | "inter_step", target group) for one straggler (scheduler.py:304-330): it must be
    among the group's last alpha% and longer than beta x the group's longest history; short/medium groups hand
    it to the least-loaded other active group, long groups defer it to the next step."""
    import math
    if total - completed > max(1, math.floor(policy.alpha_pct / 100.0 * total)):
        return "none", None
    if generated_len <= policy.beta * group_max_hist_len:
        return "none", None
    if group_index < n_groups / 2:
        cands = sorted((load, g) for g, load in active_group_loads.items() if g != group_index)
        if cands:
            return "intra_step", cands[0][1]
    return "inter_step", None


class MigrationBroker:
    """Hands straggler rollouts between GPU workers mid-step (intra-step migration, sim.py:719-779) through
    the process group's key-value store: a sender posts the evicted rollout's state (tokens generated so far,
    AIMD window, prefix length, SpecStats -- engine.SeqRequest) to the receiver's mailbox; the receiver's
    engine polls it between CUDA-graph replays and re-admits the rollout, recomputing its KV by prefill.

    Termination: a worker may stop only when every worker is idle and every posted rollout was taken
    (an idle worker marks itself busy before it takes a message, so the check cannot pass in between)."""

    def __init__(self, store, rank: int, world: int, tag: str = "mig"):
        self.store, self.rank, self.world, self.tag = store, rank, world, tag
        self.read = 0
        self.store.set(f"{tag}/idle/{rank}", "0")

    def post(self, dst: int, req) -> None:
        import pickle
        self.store.add(f"{self.tag}/posted", 1)
        n = self.store.add(f"{self.tag}/box/{dst}/n", 1) - 1
        self.store.set(f"{self.tag}/box/{dst}/{n}", pickle.dumps(req))

    def poll(self) -> list:
        import pickle
        n = self.store.add(f"{self.tag}/box/{self.rank}/n", 0)
        out = []
        while self.read < n:
            key = f"{self.tag}/box/{self.rank}/{self.read}"
            self.store.wait([key])
            out.append(pickle.loads(self.store.get(key)))
            self.read += 1
        if out:
            self.store.set(f"{self.tag}/idle/{self.rank}", "0")
            self.store.add(f"{self.tag}/taken", len(out))
        return out

    def publish_load(self, remaining_tokens: float) -> None:
        self.store.set(f"{self.tag}/load/{self.rank}", repr(float(remaining_tokens)))

    def loads(self) -> dict:
        out = {}
        for r in range(self.world):
            key = f"{self.tag}/load/{r}"
            if self.store.check([key]):
                out[r] = float(self.store.get(key))
        return out

    def keep_alive(self) -> bool:
        """Called by an idle engine: True while another worker may still hand it work."""
        self.store.set(f"{self.tag}/idle/{self.rank}", "1")
        if self.store.add(f"{self.tag}/box/{self.rank}/n", 0) > self.read:
            return True
        idle = all(self.store.get(f"{self.tag}/idle/{r}") == b"1" for r in range(self.world)
                   if self.store.check([f"{self.tag}/idle/{r}"]))
        if not idle:
            return True
        return self.store.add(f"{self.tag}/posted", 0) != self.store.add(f"{self.tag}/taken", 0)
