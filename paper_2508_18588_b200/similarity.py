"""Token-similarity replay on the GPU (reference `rhymesim/tracegen.py:288-353`).

`token_similarity_replay(trace, epoch_pair, prefix_len)` keeps the reference's
signature, result type and error behaviour.  The previous epoch's responses
are indexed per prompt by K1 (`GpuIndex`, one slot per prompt), and
`hs_similarity_replay` replays every current response in one launch, one warp
per response: each step is a binary search of the remaining response over the
slot's suffix array (the longest continuation over all occurrences of the last
`prefix_len` tokens is the insertion point's neighbour LCP minus `prefix_len`).
By default (`hs_similarity_replay_isa`) a search after an accepted run starts at
the rank (inverse suffix array) of the matched suffix advanced by the run, which
shares the next query's first `prefix_len` tokens: a short gallop replaces most
of the binary search.  There is no CPU fallback: without CUDA the call raises.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .index import GpuIndex


# HS_SIM_SEARCH = "isa" (default, 2.0x faster on the configs[1] epoch): ISA-seeded searches
# (hs_similarity_replay_isa); "plain": plain binary searches (hs_similarity_replay, whose kernel variant the
# library's own A/B switch HS_SIM_VARIANT selects).  Any other value is an error, not a silent fallback.
_SEARCHES = ("isa", "plain")


def _search_mode() -> str:
    mode = os.environ.get("HS_SIM_SEARCH", "isa")
    if mode not in _SEARCHES:
        raise ValueError(f"HS_SIM_SEARCH must be one of {_SEARCHES}, got {mode!r}")
    return mode


@dataclass(frozen=True)
class ReplayResult:
    """Token accounting from the prefix-search replay of one epoch pair (tracegen.py:288-303)."""

    accepted: int
    total: int
    warmup: int

    @property
    def acceptance(self) -> float:
        return self.accepted / self.total if self.total else 0.0

    @property
    def acceptance_after_warmup(self) -> float:
        effective = self.total - self.warmup
        return self.accepted / effective if effective > 0 else 0.0


def _epoch(trace, epoch):
    """{prompt_id: [tokens, ...]} of one epoch from a reference `Trace`, or a
    `synth.generate_trace` dict {epoch: {prompt_id: [(tokens, reward), ...]}}."""
    if hasattr(trace, "epoch_responses"):
        group = trace.epoch_responses(epoch)           # raises KeyError like the reference (tracegen.py:183-186)
    else:
        if epoch not in trace:
            raise KeyError(f"trace has no epoch {epoch}")
        group = trace[epoch]
    return {pid: [r.tokens if hasattr(r, "tokens") else r[0] for r in rs] for pid, rs in group.items()}


def replay_against_index(index: GpuIndex, d_tokens, resp_off, slot_of_resp, prefix_len: int, stream=None):
    """Per-response accepted counts (int64 device tensor) for responses already in HBM.

    d_tokens: int32 device tensor of concatenated responses; resp_off: int64
    device tensor [n + 1]; slot_of_resp: int32 device tensor [n] (slot of
    `index` holding that prompt's previous epoch)."""
    torch = _lib.require_cuda()
    if prefix_len < 1:
        raise ValueError("prefix_len must be >= 1")        # tracegen.py:322-323
    mode = _search_mode()
    n = int(slot_of_resp.numel())
    dev = d_tokens.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    lib = _lib.load()
    with torch.cuda.device(dev), torch.cuda.stream(s):
        # allocated on s (the kernel writes every entry), so no fill on another stream can race it
        out = torch.empty(n, dtype=torch.int64, device=dev)
        if mode == "isa":
            cached = getattr(index, "_isa", None)
            if cached is None:
                isa = torch.empty(max(1, index.view.n_text), dtype=torch.int32, device=dev)
                _lib.check(lib.hs_index_inverse_sa(ctypes.byref(index.view), isa.data_ptr(), s.cuda_stream))
                ready = torch.cuda.Event()
                ready.record(s)
                index._isa = (isa, ready)      # 4 B per indexed token, kept with the index
            else:
                # built on another stream by an earlier call: order this stream after the build
                isa, ready = cached
                s.wait_event(ready)
            _lib.check(lib.hs_similarity_replay_isa(
                ctypes.byref(index.view), isa.data_ptr(), n, d_tokens.data_ptr(), resp_off.data_ptr(),
                slot_of_resp.data_ptr(), int(prefix_len), out.data_ptr(), s.cuda_stream))
        else:
            _lib.check(lib.hs_similarity_replay(
                ctypes.byref(index.view), n, d_tokens.data_ptr(), resp_off.data_ptr(), slot_of_resp.data_ptr(),
                int(prefix_len), out.data_ptr(), s.cuda_stream))
    return out


def token_similarity_replay(trace, epoch_pair: tuple[int, int], prefix_len: int, device=None) -> ReplayResult:
    """Replay each current response against the previous epoch's responses (tracegen.py:306-353)."""
    if prefix_len < 1:
        raise ValueError("prefix_len must be >= 1")
    torch = _lib.require_cuda()
    prev = _epoch(trace, epoch_pair[0])
    cur = _epoch(trace, epoch_pair[1])
    common = sorted(set(prev) & set(cur))
    total = warmup = 0
    slots, cur_tok, cur_slot = [], [], []
    for pid in common:
        # empty history responses hold no prefix_len-gram (tracegen.py:331); the index rejects them
        hist = [(np.asarray(t, dtype=np.int64), 0.0) for t in prev[pid] if len(t) > 0]
        slot = len(slots) if hist else -1
        if hist:
            slots.append(hist)
        for t in cur[pid]:
            total += len(t)
            warmup += min(prefix_len, len(t))
            if slot >= 0 and len(t) > prefix_len:
                cur_tok.append(np.asarray(t, dtype=np.int64))
                cur_slot.append(slot)
    if not cur_tok:
        return ReplayResult(accepted=0, total=total, warmup=warmup)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    flat = np.concatenate(cur_tok)
    if flat.min() < 0 or flat.max() > np.iinfo(np.int32).max:
        raise ValueError("token ids must be in [0, 2^31)")
    off = np.zeros(len(cur_tok) + 1, dtype=np.int64)
    np.cumsum([len(t) for t in cur_tok], out=off[1:])
    index = GpuIndex(slots, device=dev)
    d_tok = torch.from_numpy(flat.astype(np.int32)).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    d_slot = torch.from_numpy(np.asarray(cur_slot, dtype=np.int32)).to(dev)
    acc = replay_against_index(index, d_tok, d_off, d_slot, prefix_len)
    return ReplayResult(accepted=int(acc.sum().item()), total=total, warmup=warmup)
