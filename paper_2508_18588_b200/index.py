"""GPU-resident history index over many prompt slots (K1), plus batched lookups.

One `GpuIndex` covers a batch of slots (one slot = one prompt's previous-epoch
responses).  HBM layout (all slot-major):

  text   int32 [sum(len) + n_resp + pad]  tokens, -1 after every response
  sa     int32 [sum(len)]                 suffix array
  lcp    int32 [sum(len) + 1]             -1 at slot boundaries
  wsum   int64 [sum(len) + 1]             prefix sums of reward fixed point (2^-32)
  heavy  int32 [sum(len)]                 heavy (greedy) continuation per LCP node
  table  (8 + 8) B x 2^k                 (slot, m, m-gram) -> heavy pos [+ tag]; mass in a parallel array

Replaces `rhymesim/history.py:343-355 build_tree` (+ `SuffixTree.add_response`
/ `finalize`, :148-279) for many prompts in one launch sequence.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib

FX_SCALE = float(1 << _lib.HS_REWARD_FRAC_BITS)
_FX_LIMIT = float(1 << 30)


def reward_to_fx(reward: float) -> int:
    r = float(reward)
    if not math.isfinite(r):
        raise ValueError(f"reward must be finite, got {reward!r}")   # history.py:152-153
    if abs(r) >= _FX_LIMIT:
        raise ValueError(f"|reward| must be < 2^30 for the fixed-point index, got {reward!r}")
    return int(round(r * FX_SCALE))


def fx_to_float(x: int) -> float:
    return float(x) / FX_SCALE


class GpuIndex:
    """Suffix-array index of several slots, built on `stream` (default: current)."""

    def __init__(self, slots, prefix_min: int = 3, prefix_max: int = 7, device=None, stream=None,
                 keep_workspace: bool = False):
        """Build from host lists: slots[s] = [(tokens, reward), ...]."""
        torch = _lib.require_cuda()
        lens, rewards, toks, slot_resp_off = [], [], [], [0]
        for corpus in slots:
            for tokens, reward in corpus:
                arr = np.asarray(tokens, dtype=np.int64)
                if arr.ndim != 1 or arr.size == 0:
                    raise ValueError("cannot index an empty response")       # history.py:150-151
                if arr.min() < 0 or arr.max() >= 2 ** 31 - 1:
                    raise ValueError("token ids must be in [0, 2^31-1)")
                lens.append(arr.size)
                rewards.append(reward_to_fx(reward))
                toks.append(arr.astype(np.int32))
            slot_resp_off.append(slot_resp_off[-1] + len(corpus))
        resp_off = np.zeros(len(lens) + 1, dtype=np.int64)
        if lens:
            resp_off[1:] = np.cumsum(lens)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        host_tok = torch.from_numpy(np.concatenate(toks) if toks else np.zeros(1, np.int32))
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.device(dev), torch.cuda.stream(s):
            d_tok = host_tok.to(dev)
        self._build(d_tok, resp_off, np.asarray(slot_resp_off, dtype=np.int64),
                    np.asarray(rewards if rewards else [0], dtype=np.int64), prefix_min, prefix_max, dev, s,
                    keep_workspace)

    @classmethod
    def from_arrays(cls, d_tokens, resp_off, slot_resp_off, reward_fx, prefix_min=3, prefix_max=7, stream=None,
                    keep_workspace=False):
        """Build from device tokens (int32, already in HBM) + small host metadata arrays."""
        torch = _lib.require_cuda()
        self = cls.__new__(cls)
        s = stream if stream is not None else torch.cuda.current_stream(d_tokens.device)
        self._build(d_tokens, np.asarray(resp_off, dtype=np.int64), np.asarray(slot_resp_off, dtype=np.int64),
                    np.asarray(reward_fx, dtype=np.int64), prefix_min, prefix_max, d_tokens.device, s,
                    keep_workspace)
        return self

    def _build(self, d_tok, resp_off, slot_resp_off, reward_fx, prefix_min, prefix_max, dev, s, keep_workspace):
        torch = _lib.require_cuda()
        lib = _lib.load()
        self.device = dev
        self.prefix_min, self.prefix_max = int(prefix_min), int(min(prefix_max, _lib.HS_MAX_TABLE_PREFIX))
        n_resp = len(resp_off) - 1
        n_slots = len(slot_resp_off) - 1
        lens = np.diff(resp_off)
        self.n_tokens = int(resp_off[-1])
        self.n_slots = n_slots
        self._resp_off = resp_off
        self._slot_resp_off = slot_resp_off
        self._reward_fx = reward_fx
        self.max_len = int(lens.max()) if n_resp else 1
        tok_at = resp_off[slot_resp_off]
        self.slot_tokens = [int(x) for x in np.diff(tok_at)]
        w = reward_fx[:n_resp].astype(object) * lens.astype(object) if n_resp else np.zeros(0, dtype=object)
        csum = np.concatenate([[0], np.cumsum(w)]) if n_resp else np.zeros(1, dtype=object)
        self.slot_root_mass_fx = [int(csum[slot_resp_off[i + 1]] - csum[slot_resp_off[i]]) for i in range(n_slots)]
        plan = _lib.HsIndexPlan()
        _lib.check(lib.hs_index_plan(self.n_tokens, n_resp, n_slots, self.max_len, self.prefix_min,
                                     self.prefix_max, ctypes.byref(plan)))
        with torch.cuda.device(dev), torch.cuda.stream(s):
            self.tokens = d_tok
            self.index_buf = torch.empty(max(plan.index_bytes, 256), dtype=torch.uint8, device=dev)
            ws = torch.empty(max(plan.workspace_bytes, 256), dtype=torch.uint8, device=dev)
            self.view = _lib.HsIndexView()
            _lib.check(lib.hs_index_build(
                d_tok.data_ptr(), self.n_tokens, resp_off.ctypes.data, n_resp,
                slot_resp_off.ctypes.data, n_slots, reward_fx.ctypes.data,
                self.prefix_min, self.prefix_max, self.index_buf.data_ptr(), self.index_buf.numel(),
                ws.data_ptr(), ws.numel(), ctypes.byref(self.view), s.cuda_stream))
            tb = ctypes.c_size_t(0)
            _lib.check(lib.hs_index_table_bytes(ctypes.byref(self.view), ctypes.byref(tb)))
            self.table_buf = torch.empty(tb.value, dtype=torch.uint8, device=dev)
            _lib.check(lib.hs_index_build_table(ctypes.byref(self.view), self.table_buf.data_ptr(),
                                                self.table_buf.numel(), s.cuda_stream))
            self._node_counts = None
            if keep_workspace:
                self.ws = ws
            else:
                # readers never touch the workspace; keep it alive until the table build has run
                ws.record_stream(s)
                self.ws = None
                self.view.ws = None
                self.view.ws_bytes = 0
        self.device_bytes = self.index_buf.numel() + self.table_buf.numel() + self.tokens.numel() * 4

    @property
    def node_counts(self):
        """Reference-equivalent node count per slot (history.py node_count)."""
        if self._node_counts is None:
            counts = [1] * self.n_slots
            if self.n_slots and self.n_tokens:
                off = self.view.slot_stats - self.index_buf.data_ptr()
                st = self.index_buf[off:off + 16 * self.n_slots].cpu().numpy().view(np.int64)
                counts = [int(st[2 * i]) if self.slot_tokens[i] else 1 for i in range(self.n_slots)]
            self._node_counts = counts
        return self._node_counts

    # ------------------------------------------------------------------ lookups
    def lookup(self, slots, prefixes, windows, use_table: bool = False, stream=None):
        """Batched general lookup.  Returns (draft lists, info [n,6] int64 numpy).

        info columns: found, draft_len, mass_fx, at_node, heavy_pos, locus_depth.
        """
        torch = _lib.require_cuda()
        n = len(prefixes)
        if n == 0:
            return [], np.zeros((0, 6), dtype=np.int64)
        stride = max(1, max(len(p) for p in prefixes))
        pre = np.zeros((n, stride), dtype=np.int32)
        plen = np.zeros(n, dtype=np.int32)
        for i, p in enumerate(prefixes):
            if len(p) == 0:
                raise ValueError("prefix must be non-empty")   # history.py:285-286
            pre[i, :len(p)] = p
            plen[i] = len(p)
        win = np.asarray(windows, dtype=np.int32)
        if (win < 0).any():
            raise ValueError("window must be >= 0")
        ostride = max(1, int(win.max()))
        dev = self.device
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.device(dev), torch.cuda.stream(s):
            d_slot = torch.as_tensor(np.asarray(slots, dtype=np.int32)).to(dev)
            d_pre = torch.from_numpy(pre).to(dev)
            d_plen = torch.from_numpy(plen).to(dev)
            d_win = torch.from_numpy(win).to(dev)
            d_out = torch.zeros((n, ostride), dtype=torch.int32, device=dev)
            d_info = torch.zeros((n, 6), dtype=torch.int64, device=dev)
            _lib.check(_lib.load().hs_lookup_batch(
                ctypes.byref(self.view), n, d_slot.data_ptr(), d_pre.data_ptr(), stride, d_plen.data_ptr(),
                d_win.data_ptr(), d_out.data_ptr(), ostride, d_info.data_ptr(), int(use_table), s.cuda_stream))
            out = d_out.cpu().numpy()
            info = d_info.cpu().numpy()
        drafts = [out[i, :info[i, 1]].tolist() for i in range(n)]
        return drafts, info

    def lookup_branches(self, slots, prefixes, windows, width: int = 4, stream=None):
        """Draft-tree candidate branches per query (hs_lookup_branches): a list of up to `width` drafts per query
        (branch 0 = extract_draft's draft, then the runner-up first tokens with their greedy continuations)
        and their first-token masses in reward fixed point."""
        torch = _lib.require_cuda()
        n = len(prefixes)
        if n == 0:
            return [], []
        stride = max(1, max(len(p) for p in prefixes))
        pre = np.zeros((n, stride), dtype=np.int32)
        plen = np.zeros(n, dtype=np.int32)
        for i, p in enumerate(prefixes):
            if len(p) == 0:
                raise ValueError("prefix must be non-empty")
            pre[i, :len(p)] = p
            plen[i] = len(p)
        win = np.asarray(windows, dtype=np.int32)
        if (win < 1).any():
            raise ValueError("window must be >= 1")
        ostride = int(win.max())
        dev = self.device
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.device(dev), torch.cuda.stream(s):
            d_slot = torch.as_tensor(np.asarray(slots, dtype=np.int32)).to(dev)
            d_pre = torch.from_numpy(pre).to(dev)
            d_plen = torch.from_numpy(plen).to(dev)
            d_win = torch.from_numpy(win).to(dev)
            d_out = torch.zeros((n, width, ostride), dtype=torch.int32, device=dev)
            d_len = torch.zeros((n, width), dtype=torch.int32, device=dev)
            d_mass = torch.zeros((n, width), dtype=torch.int64, device=dev)
            _lib.check(_lib.load().hs_lookup_branches(
                ctypes.byref(self.view), n, d_slot.data_ptr(), d_pre.data_ptr(), stride, d_plen.data_ptr(),
                d_win.data_ptr(), int(width), d_out.data_ptr(), ostride, d_len.data_ptr(), d_mass.data_ptr(),
                s.cuda_stream))
            out, lens, mass = d_out.cpu().numpy(), d_len.cpu().numpy(), d_mass.cpu().numpy()
        branches = [[out[i, b, :lens[i, b]].tolist() for b in range(width) if lens[i, b] > 0] for i in range(n)]
        masses = [[int(mass[i, b]) for b in range(width) if lens[i, b] > 0] for i in range(n)]
        return branches, masses

