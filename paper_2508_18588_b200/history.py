"""Drop-in for `rhymesim.history` backed by the GPU suffix-array index.

Same public names, signatures, error types and snapshot semantics as the
reference module (`/root/reference/pkg/src/rhymesim/history.py`):

  Response, DraftResult, Cursor, SuffixTree, build_tree, HistoryStore,
  MemoryStats, StaleEpochError, TERMINAL, DEFAULT_VOCAB_SIZE

A `SuffixTree` here is an immutable view of one slot of a `GpuIndex`
(K1, `index.py`); its query methods run the K2 lookup kernels (n = 1).  The
store additionally offers `ingest_epoch_batch`, which builds every prompt of
an epoch in one GPU index (the rollout engine's path).

Deliberate differences: token ids must be non-negative int32;
rewards are held in int64 fixed point with 2^-32 resolution (exact for the
reference's dyadic test rewards and tracegen's {0, 1}); `approx_bytes`
reports device bytes of the slot's share of the index.
"""

from __future__ import annotations

import threading
from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass, field

from . import _lib
from .index import GpuIndex, fx_to_float

DEFAULT_VOCAB_SIZE = 32768
TERMINAL = None   # end-of-response marker of the reference; the GPU text uses -1


class StaleEpochError(ValueError):
    """Ingest of an epoch that is not newer than the prompt's latest request (history.py:31-32)."""


@dataclass
class Response:
    prompt_id: str
    epoch: int
    tokens: list
    reward: float

    @property
    def generated_len(self) -> int:
        return len(self.tokens)


@dataclass
class DraftResult:
    tokens: list
    matched_prefix_len: int
    source_priority: float

    @property
    def found(self) -> bool:
        # a match with an empty draft still counts as found (history.py:57-59)
        return self.matched_prefix_len > 0


@dataclass
class _Root:
    priority: float


class Cursor:
    """Matched position: `priority` is the reward mass below it (history.py:93-111)."""

    __slots__ = ("tree", "priority", "_at_node", "depth")

    def __init__(self, tree, priority: float, at_node: bool, depth: int):
        self.tree = tree
        self.priority = priority
        self._at_node = at_node
        self.depth = depth

    def at_node(self) -> bool:
        return self._at_node


class SuffixTree:
    """One prompt's previous-epoch history (a slot of a GPU index)."""

    def __init__(self, prompt_id: str, epoch: int, index: GpuIndex | None = None, slot: int = 0,
                 total_reward: float = 0.0):
        self.prompt_id = prompt_id
        self.epoch = epoch
        self._index = index
        self._slot = slot
        self.total_reward = total_reward
        if index is None:
            self.total_tokens, self.node_count, root = 0, 1, 0.0
        else:
            self.total_tokens = index.slot_tokens[slot]
            self.node_count = index.node_counts[slot]
            root = fx_to_float(index.slot_root_mass_fx[slot])
        self.root = _Root(root)

    @property
    def index(self) -> GpuIndex | None:
        return self._index

    @property
    def slot(self) -> int:
        return self._slot

    def _lookup(self, prefix, window):
        if self._index is None or self.total_tokens == 0:
            return None
        drafts, info = self._index.lookup([self._slot], [list(prefix)], [window])
        return drafts[0], info[0]

    def match_prefix(self, prefix) -> Cursor | None:
        if not prefix:
            raise ValueError("prefix must be non-empty")             # history.py:285-286
        res = self._lookup(prefix, 0)
        if res is None or not res[1][0]:
            return None
        info = res[1]
        return Cursor(self, fx_to_float(int(info[2])), bool(info[3]), int(info[5]))

    def extract_draft(self, prefix, window: int) -> DraftResult:
        if window < 1:
            raise ValueError("window must be >= 1")                  # history.py:307-308
        if not prefix:
            raise ValueError("prefix must be non-empty")
        res = self._lookup(prefix, window)
        if res is None or not res[1][0]:
            return DraftResult(tokens=[], matched_prefix_len=0, source_priority=0.0)
        draft, info = res
        return DraftResult(tokens=draft, matched_prefix_len=len(prefix),
                           source_priority=fx_to_float(int(info[2])))

    def approx_bytes(self) -> int:
        if self._index is None or self._index.n_tokens == 0:
            return 64
        share = self.total_tokens / max(1, self._index.n_tokens)
        return max(64, int(self._index.device_bytes * share))


def _corpus(prompt_id: str, responses) -> list:
    corpus = []
    for resp in responses:
        if resp.prompt_id != prompt_id:
            raise ValueError(f"response prompt {resp.prompt_id!r} != tree prompt {prompt_id!r}")
        corpus.append((resp.tokens, resp.reward))
    return corpus


def build_tree(prompt_id: str, epoch: int, responses) -> SuffixTree:
    """One-prompt GPU index (history.py:343-355); empty list -> root-only tree."""
    corpus = _corpus(prompt_id, responses)
    total = sum(float(r) for _t, r in corpus)
    index = GpuIndex([corpus])
    return SuffixTree(prompt_id, epoch, index, 0, total)


def build_trees(items, prefix_min: int = 3, prefix_max: int = 7, stream=None) -> dict:
    """Batched build: {prompt_id: (epoch, responses)} -> {prompt_id: SuffixTree} sharing one index."""
    pids = list(items)
    slots = [_corpus(pid, items[pid][1]) for pid in pids]
    index = GpuIndex(slots, prefix_min=prefix_min, prefix_max=prefix_max, stream=stream)
    return {pid: SuffixTree(pid, items[pid][0], index, i, sum(float(r) for _t, r in slots[i]))
            for i, pid in enumerate(pids)}


@dataclass
class MemoryStats:
    prompt_count: int
    total_nodes: int
    total_tokens: int
    approx_bytes: int


@dataclass
class _PromptSlot:
    tree: SuffixTree | None = None
    latest_requested: int = -1
    lock: threading.Lock = field(default_factory=threading.Lock)


class HistoryStore:
    """Latest-epoch GPU index per prompt, built off the caller's thread.

    Semantics of history.py:373-454: `ingest_epoch` rejects epochs not newer
    than the latest request (StaleEpochError), readers keep the previous
    snapshot until the build lands, and a late build never replaces a newer
    visible epoch.  Builds run on per-thread CUDA side streams and are
    synchronized before the snapshot swap.
    """

    def __init__(self, workers: int = 2, prefix_min: int = 3, prefix_max: int = 7, device=None):
        self._slots: dict[str, _PromptSlot] = {}
        self._slots_lock = threading.Lock()
        self._pool = ThreadPoolExecutor(max_workers=workers, thread_name_prefix="gpu-history")
        self._pending: set[Future] = set()
        self._pending_lock = threading.Lock()
        self._prefix = (prefix_min, prefix_max)
        self._device = device
        self._tls = threading.local()

    def _slot(self, prompt_id: str) -> _PromptSlot:
        with self._slots_lock:
            slot = self._slots.get(prompt_id)
            if slot is None:
                slot = self._slots[prompt_id] = _PromptSlot()
            return slot

    def _claim(self, prompt_id: str, epoch: int) -> _PromptSlot:
        slot = self._slot(prompt_id)
        with slot.lock:
            if epoch <= slot.latest_requested:
                raise StaleEpochError(
                    f"epoch {epoch} for prompt {prompt_id!r} is not newer than "
                    f"already-ingested epoch {slot.latest_requested}")
            slot.latest_requested = epoch
        return slot

    def _track(self, fut: Future) -> Future:
        with self._pending_lock:
            self._pending.add(fut)
        fut.add_done_callback(self._untrack)
        return fut

    def _untrack(self, fut: Future) -> None:
        with self._pending_lock:
            self._pending.discard(fut)

    def _stream(self):
        torch = _lib.require_cuda()
        st = getattr(self._tls, "stream", None)
        if st is None:
            dev = self._device if self._device is not None else torch.cuda.current_device()
            torch.cuda.set_device(dev)
            st = self._tls.stream = torch.cuda.Stream(device=dev)
        return st

    @staticmethod
    def _swap(slot: _PromptSlot, tree: SuffixTree) -> None:
        with slot.lock:
            if slot.tree is None or slot.tree.epoch < tree.epoch:
                slot.tree = tree

    def ingest_epoch(self, prompt_id: str, epoch: int, responses) -> Future:
        slot = self._claim(prompt_id, epoch)
        responses = list(responses)

        def job():
            items = {prompt_id: (epoch, responses)}
            tree = build_trees(items, *self._prefix, stream=self._stream())[prompt_id]
            self._swap(slot, tree)

        return self._track(self._pool.submit(job))

    def ingest_epoch_batch(self, items) -> Future:
        """{prompt_id: (epoch, responses)} -> one GPU index for all of them."""
        claimed = {pid: self._claim(pid, ep) for pid, (ep, _r) in items.items()}
        items = {pid: (ep, list(r)) for pid, (ep, r) in items.items()}

        def job():
            trees = build_trees(items, *self._prefix, stream=self._stream())
            for pid, tree in trees.items():
                self._swap(claimed[pid], tree)

        return self._track(self._pool.submit(job))

    def get_tree(self, prompt_id: str) -> SuffixTree | None:
        with self._slots_lock:
            slot = self._slots.get(prompt_id)
        return slot.tree if slot is not None else None

    def flush(self) -> None:
        while True:
            with self._pending_lock:
                pending = list(self._pending)
            if not pending:
                return
            for fut in pending:
                fut.result()

    def memory_stats(self) -> MemoryStats:
        with self._slots_lock:
            slots = list(self._slots.values())
        count = nodes = tokens = approx = 0
        for slot in slots:
            tree = slot.tree
            if tree is None:
                continue
            count += 1
            nodes += tree.node_count
            tokens += tree.total_tokens
            approx += tree.approx_bytes()
        return MemoryStats(count, nodes, tokens, approx)

    def close(self) -> None:
        self._pool.shutdown(wait=True)
