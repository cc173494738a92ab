"""Drop-in for `rhymesim.spec_engine` plus the batched GPU speculation engine.

Reference-compatible names (same fields, defaults, invariants and errors as
`/root/reference/pkg/src/rhymesim/spec_engine.py`): AimdWindow, next_window,
PrefixPolicy, choose_prefix, BatchGate, gate_check, verify, SpecStats,
SpecConfig, ResponseContext, StepOutcome, step_response, ResponseReplay,
replay_response, ResponseComplete and the default constants.

GPU path: `replay_response` on a GPU `SuffixTree` runs the fused K2+K6 replay
kernel (`hs_replay_fused`); `SpecBatch` holds the per-sequence state of a
whole rollout batch on the device (SoA) and drives `hs_draft` (K2) and
`hs_accept_replay` / `hs_accept_greedy` (K6) for the rollout engine.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib

WINDOW_INIT = 2          # spec_engine.py:22
WINDOW_ADD = 2           # :23
WINDOW_MAX = 32          # :24
PREFIX_INIT = 7          # :25
PREFIX_MIN = 3           # :26
GATE_BUCKETS = 10        # :27
GATE_DEFAULT_MAX_BATCH = 8192  # :28


class ResponseComplete(RuntimeError):
    """Stepping a response that already has its full length (spec_engine.py:31-32)."""


@dataclass(frozen=True)
class AimdWindow:
    size: int = WINDOW_INIT
    init: int = WINDOW_INIT
    add_step: int = WINDOW_ADD
    max: int = WINDOW_MAX

    def __post_init__(self):
        if not 1 <= self.init <= self.size <= self.max:
            raise ValueError(f"window invariant violated: {self}")


def next_window(window: AimdWindow, all_accepted: bool) -> AimdWindow:
    """Additive increase on a fully accepted draft, reset to init otherwise (:49-53)."""
    size = min(window.size + window.add_step, window.max) if all_accepted else window.init
    return replace(window, size=size)


@dataclass(frozen=True)
class PrefixPolicy:
    current_len: int = PREFIX_INIT
    initial_len: int = PREFIX_INIT
    min_len: int = PREFIX_MIN

    def __post_init__(self):
        if not 1 <= self.min_len <= self.current_len <= self.initial_len:
            raise ValueError(f"prefix invariant violated: {self}")


def choose_prefix(policy: PrefixPolicy, found_match: bool) -> PrefixPolicy:
    """Reset to the initial length on a hit, shrink by one (floored) on a miss (:69-72)."""
    cur = policy.initial_len if found_match else max(policy.current_len - 1, policy.min_len)
    return replace(policy, current_len=cur)


@dataclass(frozen=True)
class BatchGate:
    table: tuple = (GATE_DEFAULT_MAX_BATCH,) * GATE_BUCKETS

    def __post_init__(self):
        if len(self.table) != GATE_BUCKETS:
            raise ValueError(f"gate table needs {GATE_BUCKETS} buckets, got {len(self.table)}")
        if any(b < a for a, b in zip(self.table, self.table[1:])):
            raise ValueError("gate table must be non-decreasing in acceptance bucket")


def gate_check(gate: BatchGate, current_batch: int, recent_acceptance: float) -> bool:
    """Speculate iff the batch fits the acceptance decile's cap (:93-97)."""
    bucket = max(0, min(int(recent_acceptance * GATE_BUCKETS), GATE_BUCKETS - 1))
    return current_batch <= gate.table[bucket]


def verify(draft, truth) -> int:
    """Longest common prefix length (:100-107)."""
    n = 0
    for d, t in zip(draft, truth):
        if d != t:
            break
        n += 1
    return n


class SpecStats:
    """Lock-protected counters (:110-147); `absorb` adds a device stats array."""

    __slots__ = ("_lock", "tokens_total", "tokens_speculated", "tokens_accepted",
                 "verify_passes", "decode_passes")
    CSV_HEADER = ["step", "speculation_rate", "acceptance_rate", "verify_passes", "decode_passes"]

    def __init__(self):
        self._lock = threading.Lock()
        self.tokens_total = self.tokens_speculated = self.tokens_accepted = 0
        self.verify_passes = self.decode_passes = 0

    def record(self, *, total: int, speculated: int, accepted: int, verify_pass: bool) -> None:
        with self._lock:
            self.tokens_total += total
            self.tokens_speculated += speculated
            self.tokens_accepted += accepted
            if verify_pass:
                self.verify_passes += 1
            else:
                self.decode_passes += 1

    def absorb(self, rows) -> None:
        """Add per-sequence device counters [n, 5] (total, spec, acc, verify, decode)."""
        tot = np.asarray(rows, dtype=np.int64).reshape(-1, 5).sum(axis=0)
        with self._lock:
            self.tokens_total += int(tot[0])
            self.tokens_speculated += int(tot[1])
            self.tokens_accepted += int(tot[2])
            self.verify_passes += int(tot[3])
            self.decode_passes += int(tot[4])

    @property
    def speculation_rate(self) -> float:
        return self.tokens_accepted / self.tokens_total if self.tokens_total else 0.0

    @property
    def acceptance_rate(self) -> float:
        return self.tokens_accepted / self.tokens_speculated if self.tokens_speculated else 0.0

    def csv_row(self, step: int) -> list:
        return [step, f"{self.speculation_rate:.6f}", f"{self.acceptance_rate:.6f}",
                self.verify_passes, self.decode_passes]


@dataclass
class SpecConfig:
    """Mirrors the `spec.*` config keys one to one (:150-171)."""

    enabled: bool = True
    window_init: int = WINDOW_INIT
    window_add: int = WINDOW_ADD
    window_max: int = WINDOW_MAX
    prefix_init: int = PREFIX_INIT
    prefix_min: int = PREFIX_MIN
    gate_table: tuple = (GATE_DEFAULT_MAX_BATCH,) * GATE_BUCKETS

    def new_window(self) -> AimdWindow:
        return AimdWindow(size=self.window_init, init=self.window_init, add_step=self.window_add,
                          max=self.window_max)

    def new_prefix(self) -> PrefixPolicy:
        return PrefixPolicy(current_len=self.prefix_init, initial_len=self.prefix_init,
                            min_len=self.prefix_min)

    def gate(self) -> BatchGate:
        return BatchGate(tuple(self.gate_table))

    def c_struct(self) -> _lib.HsSpecConfig:
        self.new_window()
        self.new_prefix()
        if self.window_max > _lib.HS_MAX_WINDOW:
            raise ValueError(f"window_max must be <= {_lib.HS_MAX_WINDOW} on the GPU path")
        return _lib.HsSpecConfig(int(bool(self.enabled)), self.window_init, self.window_add,
                                 self.window_max, self.prefix_init, self.prefix_min)


@dataclass
class ResponseContext:
    truth: list
    tree: object
    window: AimdWindow
    prefix: PrefixPolicy
    stats: SpecStats
    speculate: bool = True
    generated: list = field(default_factory=list)

    @property
    def done(self) -> bool:
        return len(self.generated) >= len(self.truth)


@dataclass
class StepOutcome:
    tokens_appended: int
    drafted: int
    accepted: int
    used_speculation: bool
    done: bool


def step_response(ctx: ResponseContext) -> StepOutcome:
    """One engine iteration for one response (spec_engine.py:200-240).

    The tree is duck-typed (`extract_draft(prefix, window)`), so a GPU
    `SuffixTree` runs the lookup kernel here.
    """
    if ctx.done:
        raise ResponseComplete(f"response already complete at {len(ctx.truth)} tokens")
    pos = len(ctx.generated)
    looked = ctx.speculate and ctx.tree is not None and pos >= ctx.prefix.current_len
    draft, found = [], False
    if looked:
        res = ctx.tree.extract_draft(ctx.generated[pos - ctx.prefix.current_len:], ctx.window.size)
        draft, found = list(res.tokens), res.found
    if not draft:
        ctx.generated.append(ctx.truth[pos])
        ctx.stats.record(total=1, speculated=0, accepted=0, verify_pass=False)
        if looked:
            ctx.prefix = choose_prefix(ctx.prefix, found)
        return StepOutcome(1, 0, 0, False, ctx.done)
    rest = ctx.truth[pos:]
    acc = verify(draft, rest)
    landed = min(acc, len(rest))
    ctx.generated.extend(rest[:landed])
    bonus = 0
    if not ctx.done:
        ctx.generated.append(ctx.truth[pos + landed])
        bonus = 1
    ctx.stats.record(total=landed + bonus, speculated=len(draft), accepted=landed, verify_pass=True)
    ctx.window = next_window(ctx.window, acc == len(draft))
    ctx.prefix = choose_prefix(ctx.prefix, True)
    return StepOutcome(landed + bonus, len(draft), landed, True, ctx.done)


@dataclass
class ResponseReplay:
    tokens_per_iter: list
    drafted: int
    accepted: int

    @property
    def iterations(self) -> int:
        return len(self.tokens_per_iter)

    @property
    def total_tokens(self) -> int:
        return sum(self.tokens_per_iter)


def _is_gpu_tree(tree) -> bool:
    return getattr(tree, "index", None) is not None and hasattr(tree, "slot")


def replay_response(truth, tree, config: SpecConfig, stats: SpecStats | None = None,
                    speculate: bool = True) -> ResponseReplay:
    """Run one response to completion (spec_engine.py:260-279).

    With a GPU tree the whole replay is one `hs_replay_fused` launch.
    """
    stats = stats if stats is not None else SpecStats()
    spec = speculate and config.enabled
    if spec and _is_gpu_tree(tree) and tree.total_tokens > 0 and config.window_max <= _lib.HS_MAX_WINDOW:
        per, rows = replay_batch(tree.index, [tree.slot], [truth], config)
        stats.absorb(rows)
        r = rows[0]
        return ResponseReplay(per[0], int(r[1]), int(r[2]))
    ctx = ResponseContext(truth=list(truth), tree=tree if spec else None, window=config.new_window(),
                          prefix=config.new_prefix(), stats=stats, speculate=spec)
    per, drafted, accepted = [], 0, 0
    while not ctx.done:
        out = step_response(ctx)
        per.append(out.tokens_appended)
        drafted += out.drafted
        accepted += out.accepted
    return ResponseReplay(per, drafted, accepted)


# ---------------------------------------------------------------- batched GPU engine


def replay_batch(index, slots, truths, config: SpecConfig, speculate=None, stream=None):
    """Replay many responses at once (one warp per response, one launch).

    Returns (tokens_per_iter list per response, stats [n, 5] numpy:
    total, speculated, accepted, verify_passes, decode_passes).
    """
    torch = _lib.require_cuda()
    n = len(truths)
    lens = np.array([len(t) for t in truths], dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    cat = np.concatenate([np.asarray(t, dtype=np.int32) for t in truths]) if n else np.zeros(1, np.int32)
    spec = np.ones(n, dtype=np.uint8) if speculate is None else np.asarray(speculate, dtype=np.uint8)
    dev = index.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev), torch.cuda.stream(s):
        d = ReplayBuffers.from_host(cat, off, np.asarray(slots, dtype=np.int32), spec, dev)
        d.run(index, config, s)
        tpi = d.tpi.cpu().numpy()
        niter = d.n_iter.cpu().numpy()
        st = d.stats.cpu().numpy()
    per = [tpi[off[i]:off[i] + niter[i]].tolist() for i in range(n)]
    return per, st


@dataclass
class ReplayBuffers:
    """Device inputs/outputs of `hs_replay_fused` (inputs resident in HBM)."""

    truth: object
    truth_off: object
    slots: object
    speculate: object
    tpi: object
    n_iter: object
    stats: object

    @classmethod
    def from_host(cls, cat, off, slots, spec, dev):
        import torch
        n = len(off) - 1
        return cls(
            truth=torch.from_numpy(np.ascontiguousarray(cat, dtype=np.int32)).to(dev),
            truth_off=torch.from_numpy(np.ascontiguousarray(off, dtype=np.int64)).to(dev),
            slots=torch.from_numpy(np.ascontiguousarray(slots, dtype=np.int32)).to(dev),
            speculate=torch.from_numpy(np.ascontiguousarray(spec, dtype=np.uint8)).to(dev),
            tpi=torch.zeros(max(int(off[-1]), 1), dtype=torch.int32, device=dev),
            n_iter=torch.zeros(max(n, 1), dtype=torch.int32, device=dev),
            stats=torch.zeros((max(n, 1), 5), dtype=torch.int64, device=dev),
        )

    def run(self, index, config: SpecConfig, stream) -> None:
        n = self.truth_off.numel() - 1
        _lib.check(_lib.load().hs_replay_fused(
            ctypes.byref(index.view), n, self.slots.data_ptr(), self.truth.data_ptr(),
            self.truth_off.data_ptr(), self.speculate.data_ptr(), self.tpi.data_ptr(), self.n_iter.data_ptr(),
            self.stats.data_ptr(), config.c_struct(), stream.cuda_stream))


class SpecBatch:
    """Device-resident HistoSpec state of a rollout batch (SoA, one row per sequence).

    Fields mirror ResponseContext (spec_engine.py:174-187) for n sequences:
    gen_tok/gen_len (generated response tokens), window (AimdWindow.size),
    prefix_len (PrefixPolicy.current_len), stats [n, 5], plus the current
    draft.  `propose` is K2, `accept_replay` / `accept_greedy` are K6.
    """

    def __init__(self, slots, target_len, config: SpecConfig, speculate=None, device=None,
                 max_len: int | None = None, record_tpi: bool = True):
        torch = _lib.require_cuda()
        self.config = config
        self.c_cfg = config.c_struct()
        n = len(slots)
        self.n = n
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        tl = np.asarray(target_len, dtype=np.int32)
        self.max_len = int(max_len if max_len is not None else (tl.max() if n else 1))
        W = _lib.HS_MAX_WINDOW
        i32 = dict(dtype=torch.int32, device=dev)
        self.slots = torch.as_tensor(np.asarray(slots, dtype=np.int32)).to(dev)
        self.target_len = torch.from_numpy(tl).to(dev)
        spec = np.ones(n, np.uint8) if speculate is None else np.asarray(speculate, dtype=np.uint8)
        if not config.enabled:
            spec[:] = 0
        self.speculate = torch.from_numpy(spec).to(dev)
        self.gen_stride = self.max_len + W + 1
        self.gen_tok = torch.zeros((n, self.gen_stride), **i32)
        self.gen_len = torch.zeros(n, **i32)
        self.window = torch.full((n,), config.window_init, **i32)
        self.prefix_len = torch.full((n,), config.prefix_init, **i32)
        self.stats = torch.zeros((n, 5), dtype=torch.int64, device=dev)
        self.draft_tok = torch.zeros((n, W), **i32)
        self.draft_len = torch.zeros(n, **i32)
        self.looked = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.found = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.n_iter = torch.zeros(n, **i32)
        self.tpi = torch.zeros((n, self.max_len), **i32) if record_tpi else None

    def propose(self, index, stream=None) -> None:
        """K2: draft for every sequence (spec_engine.py:206-215)."""
        torch = _lib.require_cuda()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if index is None:
            self.draft_len.zero_()
            self.looked.zero_()
            self.found.zero_()
            return
        c = self.config
        _lib.check(_lib.load().hs_draft(
            ctypes.byref(index.view), self.n, self.slots.data_ptr(), self.gen_tok.data_ptr(), self.gen_stride,
            self.gen_len.data_ptr(), self.prefix_len.data_ptr(), self.window.data_ptr(),
            self.speculate.data_ptr(), c.prefix_min, c.prefix_init, c.window_max, self.draft_tok.data_ptr(),
            self.draft_tok.shape[1], self.draft_len.data_ptr(), self.looked.data_ptr(), self.found.data_ptr(),
            s.cuda_stream))

    def accept_replay(self, truth, truth_stride: int, stream=None) -> None:
        """K6 with supplied truth rows [n, truth_stride]."""
        torch = _lib.require_cuda()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        tpi = self.tpi.data_ptr() if self.tpi is not None else None
        _lib.check(_lib.load().hs_accept_replay(
            self.n, truth.data_ptr(), truth_stride, self.target_len.data_ptr(), self.draft_tok.data_ptr(),
            self.draft_tok.shape[1], self.draft_len.data_ptr(), self.looked.data_ptr(), self.found.data_ptr(),
            self.gen_tok.data_ptr(), self.gen_stride, self.gen_len.data_ptr(), self.window.data_ptr(),
            self.prefix_len.data_ptr(), self.stats.data_ptr(), tpi, self.max_len, self.n_iter.data_ptr(),
            self.c_cfg, s.cuda_stream))

    def accept_greedy(self, argmax, q_off, stream=None) -> None:
        """K6 with truth = argmax of the verify rows (row q_off[s] + i)."""
        torch = _lib.require_cuda()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        tpi = self.tpi.data_ptr() if self.tpi is not None else None
        _lib.check(_lib.load().hs_accept_greedy(
            self.n, argmax.data_ptr(), q_off.data_ptr(), self.target_len.data_ptr(), self.draft_tok.data_ptr(),
            self.draft_tok.shape[1], self.draft_len.data_ptr(), self.looked.data_ptr(), self.found.data_ptr(),
            self.gen_tok.data_ptr(), self.gen_stride, self.gen_len.data_ptr(), self.window.data_ptr(),
            self.prefix_len.data_ptr(), self.stats.data_ptr(), tpi, self.max_len, self.n_iter.data_ptr(),
            self.c_cfg, s.cuda_stream))

    def tokens_per_iter(self):
        tpi = self.tpi.cpu().numpy()
        n_it = self.n_iter.cpu().numpy()
        return [tpi[i, :n_it[i]].tolist() for i in range(self.n)]
