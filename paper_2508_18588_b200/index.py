"""GPU-resident history index over many prompt slots (K1), plus batched lookups.

One `GpuIndex` covers a batch of slots (one slot = one prompt's previous-epoch
responses).  HBM layout (all slot-major):

  text   int32 [sum(len) + n_resp + pad]  tokens, -1 after every response
  sa     int32 [sum(len)]                 suffix array
  lcp    int32 [sum(len) + 1]             -1 at slot boundaries
  wsum   int64 [sum(len) + 1]             prefix sums of reward fixed point (2^-32)
  heavy  int32 [sum(len)]                 heavy (greedy) continuation per LCP node
  table  16 B x 2^k                       (slot, m, m-gram) -> (heavy pos, mass)

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
        torch = _lib.require_cuda()
        lib = _lib.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.prefix_min, self.prefix_max = int(prefix_min), int(min(prefix_max, _lib.HS_MAX_TABLE_PREFIX))
        n_slots = len(slots)
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
        n_resp = len(lens)
        resp_off = np.zeros(n_resp + 1, dtype=np.int64)
        if n_resp:
            resp_off[1:] = np.cumsum(lens)
        self.n_tokens = int(resp_off[-1])
        self.n_slots = n_slots
        self._resp_off = resp_off
        self._slot_resp_off = np.asarray(slot_resp_off, dtype=np.int64)
        self._reward_fx = np.asarray(rewards if rewards else [0], dtype=np.int64)
        self.max_len = int(max(lens)) if lens else 1
        # per-slot host summaries
        self.slot_tokens = [int(resp_off[self._slot_resp_off[s + 1]] - resp_off[self._slot_resp_off[s]])
                            for s in range(n_slots)]
        self.slot_root_mass_fx = []
        for s in range(n_slots):
            a, b = self._slot_resp_off[s], self._slot_resp_off[s + 1]
            self.slot_root_mass_fx.append(int(sum(self._reward_fx[r] * lens[r] for r in range(a, b))))

        plan = _lib.HsIndexPlan()
        _lib.check(lib.hs_index_plan(self.n_tokens, n_resp, n_slots, self.max_len, self.prefix_min,
                                     self.prefix_max, ctypes.byref(plan)))
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device), torch.cuda.stream(s):
            host_tok = torch.from_numpy(np.concatenate(toks) if toks else np.zeros(1, np.int32))
            self.tokens = host_tok.to(self.device, non_blocking=False)
            self.index_buf = torch.empty(max(plan.index_bytes, 256), dtype=torch.uint8, device=self.device)
            ws = torch.empty(max(plan.workspace_bytes, 256), dtype=torch.uint8, device=self.device)
            self.view = _lib.HsIndexView()
            _lib.check(lib.hs_index_build(
                self.tokens.data_ptr(), self.n_tokens, resp_off.ctypes.data, n_resp,
                self._slot_resp_off.ctypes.data, n_slots, self._reward_fx.ctypes.data,
                self.prefix_min, self.prefix_max, self.index_buf.data_ptr(), self.index_buf.numel(),
                ws.data_ptr(), ws.numel(), ctypes.byref(self.view), s.cuda_stream))
            tb = ctypes.c_size_t(0)
            _lib.check(lib.hs_index_table_bytes(ctypes.byref(self.view), ctypes.byref(tb)))
            self.table_buf = torch.empty(tb.value, dtype=torch.uint8, device=self.device)
            _lib.check(lib.hs_index_build_table(ctypes.byref(self.view), self.table_buf.data_ptr(),
                                                self.table_buf.numel(), s.cuda_stream))
            s.synchronize()
        self.node_counts = [1] * n_slots
        if n_slots and self.n_tokens:
            off = self.view.slot_stats - self.index_buf.data_ptr()
            st = self.index_buf[off:off + 16 * n_slots].view(torch.int64).cpu().numpy()
            self.node_counts = [int(st[2 * i]) for i in range(n_slots)]
        # reference counts the root even for an empty slot
        self.node_counts = [c if self.slot_tokens[i] else 1 for i, c in enumerate(self.node_counts)]
        self.keep_workspace = keep_workspace
        self.ws = ws if keep_workspace else None
        if not keep_workspace:
            self.view.ws = None
            self.view.ws_bytes = 0
        del ws
        self.device_bytes = self.index_buf.numel() + self.table_buf.numel() + self.tokens.numel() * 4

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
