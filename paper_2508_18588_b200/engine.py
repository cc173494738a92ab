"""Greedy HistoSpec rollout engine (one process per GPU).

Replaces the reference simulator's replay loop (`sim._make_tasks` ->
`replay_response`, rhymesim/sim.py:344-377; spec_engine.py:200-279) with real
forward passes.  One engine iteration for every live sequence:

  K2 hs_draft                      drafts from the previous epoch's index
  hm_build_verify_batch            rows [last token, d_1..d_k] per sequence
  verify forward (model.Forward)   tcgen05 GEMMs, attention, fused LM-head argmax
  K6 hs_accept_greedy              LCP accept + bonus + AIMD + prefix + stats
                                   (KV rollback = gen_len update)

With speculation off the same loop decodes one token per sequence per
iteration, so "spec on" and "spec off" differ only in the rows fed to the
same batch-invariant kernels -- their outputs must agree bit for bit.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .model import Forward, KVCache, ModelConfig, Weights, check, lib
from .spec_engine import SpecBatch, SpecConfig


def launch_count() -> int:
    """Kernel launches issued by this repo's two libraries so far (process-wide)."""
    return int(_lib.load().hs_launch_count()) + int(lib().hm_launch_count())


@dataclass
class RolloutResult:
    tokens: np.ndarray            # [B, T] generated response tokens
    stats: np.ndarray             # [B, 5] total, speculated, accepted, verify, decode
    iterations: int
    rows: int                     # sum of verify rows over iterations (incl. prefill rows)
    gpu_ms: float
    tokens_per_iter: list = field(default_factory=list)
    flops: float = 0.0
    kv_bytes: float = 0.0
    qlen_hist: np.ndarray = None  # [1 + max_q] count of (sequence, iteration) verify blocks by rows

    @property
    def generated(self) -> int:
        return int(self.stats[:, 0].sum())


class RolloutEngine:
    def __init__(self, cfg: ModelConfig, weights: Weights, n_slots: int, max_len: int, device,
                 spec: SpecConfig | None = None, prefill_rows: int = 16384, use_graphs: bool = True,
                 check_every: int = 8, temperature: float = 0.0, seed: int = 0, attention: str | None = None,
                 tp_group=None):
        """tp_group: the process group of a tensor-parallel pair; `weights` is then this GPU's shard
        (Weights(tp_rank, tp_size)) and `cfg` its local shape (weights.cfg)."""
        import torch
        # attention kernel family ("tcgen05" or "mma_sync"; None: the library default), set per rollout
        self.attention = attention
        self.use_graphs, self.check_every = use_graphs, check_every
        self.graph_launches = 0   # kernels executed by graph replays (not seen by the C launch counters)
        self.cfg, self.w, self.device = cfg, weights, torch.device(device)
        self.spec = spec or SpecConfig()
        self.n_slots, self.max_len = n_slots, max_len
        self.cache = KVCache(cfg, n_slots, max_len + self.spec.window_max + 2, self.device)
        self.max_q = 1 + self.spec.window_max
        self.fwd = Forward(weights, self.cache, max(prefill_rows, n_slots * self.max_q), self.device)
        # T = 0: greedy verify (argmax); T > 0: rejection-sampling verify by Gumbel-max coupling --
        # accept a point-mass draft x iff the row's sample equals x (probability p(x)), else emit the
        # sample, which is then distributed as p restricted to tokens != x (hm_lm_head_sample)
        self.fwd.temperature, self.fwd.seed = float(temperature), int(seed)
        if tp_group is not None:
            from .tp import TensorParallel
            self.fwd.tp = TensorParallel(tp_group, self.fwd.max_rows, cfg.d_model, self.device, dtype=self.fwd.x.dtype)
        self.prefill_rows = prefill_rows
        i32 = dict(dtype=torch.int32, device=self.device)
        R = self.fwd.max_rows
        self.tokens = torch.empty(R, **i32)
        self.pos = torch.empty(R, **i32)
        self.row_slot = torch.empty(R, **i32)
        self.row_key = torch.empty(R, **i32)     # per-row sampling key: the row's sequence key
        self.q_off = torch.empty(n_slots, **i32)
        self.q_len = torch.empty(n_slots, **i32)
        self.pos0 = torch.empty(n_slots, **i32)
        self.d_m = torch.zeros(1, **i32)
        self.kv_slot = torch.arange(n_slots, **i32)

    # -------------------------------------------------------------- phases
    def prefill(self, prompts, state: SpecBatch, seq_key=None):
        """Prompt forward in chunks; the last prompt row's argmax is response token 0."""
        import torch
        B, P = prompts.shape
        first = torch.empty(B, dtype=torch.int32, device=self.device)
        per = max(1, self.prefill_rows // P)
        rows = 0
        for a in range(0, B, per):
            b = min(B, a + per)
            n = b - a
            M = n * P
            self.tokens[:M] = prompts[a:b].reshape(-1)
            self.pos[:M] = torch.arange(P, dtype=torch.int32, device=self.device).repeat(n)
            self.row_slot[:M] = self.kv_slot[a:b].repeat_interleave(P)
            self.row_key[:M] = (seq_key if seq_key is not None else self.kv_slot)[a:b].repeat_interleave(P)
            self.q_off[:n] = torch.arange(n, dtype=torch.int32, device=self.device) * P
            self.q_len[:n] = P
            self.pos0[:n] = 0
            am = self.fwd.run(M, self.tokens, self.pos, self.row_slot, self.q_off, self.q_len, self.pos0,
                              self.kv_slot[a:b], n, P, row_key=self.row_key)
            first[a:b] = am.view(n, P)[:, P - 1]
            rows += M
        # iteration 0 of every response: a plain decode (pos 0 < prefix length)
        state.draft_len.zero_()
        state.looked.zero_()
        q_off = torch.arange(B, dtype=torch.int32, device=self.device)
        state.accept_greedy(first, q_off)
        return rows

    # -------------------------------------------------------------- continuous batching
    def _prefill_rows(self, reqs, lanes, seq_keys):
        """Admission prefill: KV of every request's context (prompt + generated[:-1]) into its lane's slot, in
        forwards of <= prefill_rows rows whose entries are chunks of <= `chunk` rows (one attention entry
        per chunk, positions continuing the sequence).  Returns (first-token argmax per request, -1 for
        migrated ones; device int32 [n]), rows."""
        import torch
        dev = self.device
        chunk = 2048
        ent = []   # (request i, start, length)
        ctx = []
        for i, r in enumerate(reqs):
            g = 0 if r.generated is None else len(r.generated)
            c = np.asarray(r.prompt, np.int32) if g == 0 else np.concatenate(
                [np.asarray(r.prompt, np.int32), np.asarray(r.generated[:g - 1], np.int32)])
            ctx.append(c)
            for a in range(0, len(c), chunk):
                ent.append((i, a, min(chunk, len(c) - a)))
        first = torch.full((len(reqs),), -1, dtype=torch.int32, device=dev)
        rows = 0
        e = 0
        while e < len(ent):
            batch, m = [], 0
            while e < len(ent) and (not batch or m + ent[e][2] <= self.prefill_rows):
                batch.append(ent[e])
                m += ent[e][2]
                e += 1
            toks = np.concatenate([ctx[i][a:a + n] for i, a, n in batch]).astype(np.int32)
            pos = np.concatenate([np.arange(a, a + n, dtype=np.int32) for i, a, n in batch])
            rslot = np.concatenate([np.full(n, lanes[i], np.int32) for i, a, n in batch])
            rkey = np.concatenate([np.full(n, seq_keys[i], np.int32) for i, a, n in batch])
            qlen = np.array([n for _, _, n in batch], np.int32)
            qoff = np.concatenate([[0], np.cumsum(qlen)[:-1]]).astype(np.int32)
            pos0 = np.array([a for _, a, _ in batch], np.int32)
            kvs = np.array([lanes[i] for i, _, _ in batch], np.int32)
            nb = len(batch)
            self.tokens[:m] = torch.from_numpy(toks).to(dev, non_blocking=True)
            self.pos[:m] = torch.from_numpy(pos).to(dev, non_blocking=True)
            self.row_slot[:m] = torch.from_numpy(rslot).to(dev, non_blocking=True)
            self.row_key[:m] = torch.from_numpy(rkey).to(dev, non_blocking=True)
            q_off = torch.from_numpy(qoff).to(dev, non_blocking=True)
            q_len = torch.from_numpy(qlen).to(dev, non_blocking=True)
            p0 = torch.from_numpy(pos0).to(dev, non_blocking=True)
            kv = torch.from_numpy(kvs).to(dev, non_blocking=True)
            am = self.fwd.run(m, self.tokens, self.pos, self.row_slot, q_off, q_len, p0, kv, nb, int(qlen.max()),
                              row_key=self.row_key)
            # fresh requests whose context ends in this forward: their first response token
            last = {}
            for j, (i, a, n) in enumerate(batch):
                if reqs[i].generated is None and a + n == len(ctx[i]):
                    last[i] = int(qoff[j]) + n - 1
            if last:
                idx = torch.as_tensor(list(last.values()), dtype=torch.long).to(dev, non_blocking=True)
                dst = torch.as_tensor(list(last.keys()), dtype=torch.long).to(dev, non_blocking=True)
                first.index_copy_(0, dst, am.index_select(0, idx))
            rows += m
        return first, rows

    def rollout_stream(self, requests, index=None, speculate=True, admit_min=None, on_check=None, inbox=None,
                       keep_alive=None, max_target=None, on_evict=None):
        """Continuous batching: every engine lane runs a sequence; finished lanes are refilled from the
        request queue (in the given order -- the caller puts the predicted-longest first) by an admission
        prefill between CUDA-graph replays, so a long tail does not idle the batch.

        on_check(busy: {lane: key}, gen_len: np.ndarray, iteration, waiting) -> lanes to evict, called every
        `check_every` iterations with the lanes' progress (one chunk old): their state leaves as SeqRequest
        (migration with KV recompute).  inbox() -> SeqRequests that arrived (migrated in from other
        workers) is polled at every check; while keep_alive() is true an idle engine keeps polling.
        max_target bounds the target length of requests that may still arrive.  on_evict(req) receives each
        evicted rollout as soon as its state is read (otherwise they are returned in StreamResult.evicted).
        """
        import collections
        import torch
        from .spec_engine import SpecBatch
        if self.attention is not None:
            from .model import set_attention_family
            set_attention_family(self.attention)
        reqs = list(requests)
        n = self.n_slots
        dev = self.device
        cfgs = self.spec
        max_t = max([int(r.target_len) for r in reqs] + [1, int(max_target or 0)])
        max_ctx = max([len(r.prompt) + int(r.target_len) for r in reqs] + [1])
        if max_ctx > self.max_len:
            raise ValueError("prompt + target exceeds max_len")
        spec_on = bool(speculate and index is not None and cfgs.enabled)
        state = SpecBatch(np.full(n, -1, np.int32), np.zeros(n, np.int32), cfgs, speculate=np.zeros(n, np.uint8),
                          device=dev, max_len=max_t, record_tpi=False)
        i32 = dict(dtype=torch.int32, device=dev)
        prompt_len = torch.zeros(n, **i32)
        seq_key = torch.zeros(n, **i32)
        acc = torch.zeros(4, dtype=torch.int64, device=dev)
        qhist = torch.zeros(self.max_q + 1, dtype=torch.int64, device=dev)
        q_cap = self.max_q if spec_on else 1
        R = min(self.fwd.max_rows, n * q_cap)
        L = lib()
        st = torch.cuda.current_stream(dev)

        def iteration():
            s = torch.cuda.current_stream(dev)
            if spec_on:
                state.propose(index, s)
            check(L.hm_build_verify_batch(
                n, state.gen_tok.data_ptr(), state.gen_stride, state.gen_len.data_ptr(), state.target_len.data_ptr(),
                prompt_len.data_ptr(), state.draft_tok.data_ptr(), state.draft_tok.shape[1],
                state.draft_len.data_ptr(), self.kv_slot.data_ptr(), self.tokens.data_ptr(), self.pos.data_ptr(),
                self.row_slot.data_ptr(), self.q_off.data_ptr(), self.q_len.data_ptr(), self.pos0.data_ptr(),
                self.d_m.data_ptr(), acc.data_ptr(), qhist.data_ptr(), qhist.numel(), seq_key.data_ptr(),
                self.row_key.data_ptr(), s.cuda_stream))
            am = self.fwd.run(R, self.tokens, self.pos, self.row_slot, self.q_off, self.q_len, self.pos0,
                              self.kv_slot, n, q_cap, stream=s, m_dev=self.d_m, row_key=self.row_key)
            state.accept_greedy(am, self.q_off, s)

        lib_hs = _lib.load()
        admit_min = max(1, n // 32) if admit_min is None else int(admit_min)
        queue = collections.deque(reqs)
        busy = {}                      # lane -> request
        free = list(range(n))[::-1]
        out_tok, out_stats, evicted = {}, {}, []
        prefill_rows = admissions = 0
        busy_iters = 0
        graph = None
        per_iter = 0
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(st)
        it_host = 0

        def admit(batch_reqs):
            nonlocal prefill_rows, admissions
            for r in batch_reqs:   # requests that arrive later (inbox) are checked here too
                if len(r.prompt) + int(r.target_len) > self.max_len or int(r.target_len) > max_t:
                    raise ValueError(f"request {r.key}: prompt + target exceeds the engine's max_len / max_target")
            lanes = [free.pop() for _ in batch_reqs]
            keys = [int(r.key) for r in batch_reqs]
            first, rows = self._prefill_rows(batch_reqs, lanes, keys)
            prefill_rows += rows
            admissions += len(batch_reqs)
            gen = [np.zeros(0, np.int32) if r.generated is None else np.asarray(r.generated, np.int32)
                   for r in batch_reqs]
            off = np.concatenate([[0], np.cumsum([len(g) for g in gen])]).astype(np.int64)
            fresh = np.array([r.generated is None for r in batch_reqs])
            stats = np.stack([np.array([1, 0, 0, 0, 1], np.int64) if r.stats is None else
                              np.asarray(r.stats, np.int64) for r in batch_reqs])
            win = np.array([cfgs.window_init if r.window is None else r.window for r in batch_reqs], np.int32)
            pre = np.array([cfgs.prefix_init if r.prefix_len is None else r.prefix_len for r in batch_reqs], np.int32)
            spec = np.array([int(spec_on and r.slot >= 0) for r in batch_reqs], np.uint8)
            h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=True)  # noqa: E731
            d = dict(lane=h(np.array(lanes, np.int32)), tok=h(np.concatenate(gen + [np.zeros(1, np.int32)])),
                     off=h(off), first_row=h(np.where(fresh, np.arange(len(lanes)), -1).astype(np.int32)),
                     target=h(np.array([r.target_len for r in batch_reqs], np.int32)),
                     slot=h(np.array([r.slot for r in batch_reqs], np.int32)), spec=h(spec), win=h(win), pre=h(pre),
                     stats=h(stats), plen=h(np.array([len(r.prompt) for r in batch_reqs], np.int32)),
                     key=h(np.array(keys, np.int32)))
            _lib.check(lib_hs.hs_lane_admit(
                len(lanes), d["lane"].data_ptr(), d["tok"].data_ptr(), d["off"].data_ptr(), first.data_ptr(),
                d["first_row"].data_ptr(), d["target"].data_ptr(), d["slot"].data_ptr(), d["spec"].data_ptr(),
                d["win"].data_ptr(), d["pre"].data_ptr(), d["stats"].data_ptr(), d["plen"].data_ptr(),
                d["key"].data_ptr(), state.gen_tok.data_ptr(), state.gen_stride, state.gen_len.data_ptr(),
                state.target_len.data_ptr(), state.slots.data_ptr(), state.speculate.data_ptr(),
                state.window.data_ptr(), state.prefix_len.data_ptr(), state.stats.data_ptr(),
                state.draft_len.data_ptr(), state.looked.data_ptr(), state.found.data_ptr(), prompt_len.data_ptr(),
                seq_key.data_ptr(), st.cuda_stream))
            for ln, r in zip(lanes, batch_reqs):
                busy[ln] = r

        pin = dict(dtype=torch.int32, device="cpu", pin_memory=True)
        h_len = [torch.empty(n, **pin) for _ in range(2)]
        h_tgt = [torch.empty(n, **pin) for _ in range(2)]
        harvests = []              # (event, keys, lanes, pinned tokens [k, stride], pinned stats [k, 5])

        def start_harvest(lanes):
            """Finished lanes: their rows leave the device asynchronously; the lanes are free at once (any
            later admission into them is stream-ordered after these copies)."""
            li = torch.as_tensor(lanes, dtype=torch.long).to(dev, non_blocking=True)
            toks = torch.empty((len(lanes), state.gen_stride), **pin)
            sts = torch.empty((len(lanes), 5), dtype=torch.int64, device="cpu", pin_memory=True)
            toks.copy_(state.gen_tok.index_select(0, li), non_blocking=True)
            sts.copy_(state.stats.index_select(0, li), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
            reqs_ = [busy.pop(ln) for ln in lanes]
            free.extend(lanes)
            harvests.append((ev, reqs_, toks, sts))

        def finish_harvests(block=False):
            while harvests and (block or harvests[0][0].query()):
                ev, reqs_, toks, sts = harvests.pop(0)
                ev.synchronize()
                t, a = toks.numpy(), sts.numpy()
                for j, r in enumerate(reqs_):
                    out_tok[r.key] = t[j, :r.target_len].copy()
                    out_stats[r.key] = a[j].copy()

        def evict(lanes):
            """Migration: the lanes' state leaves as SeqRequest (synchronous; `on_check` callers only)."""
            li = torch.as_tensor(lanes, dtype=torch.long).to(dev)
            toks = state.gen_tok.index_select(0, li).cpu().numpy()
            sts = state.stats.index_select(0, li).cpu().numpy()
            win = state.window.index_select(0, li).cpu().numpy()
            pre = state.prefix_len.index_select(0, li).cpu().numpy()
            gl = state.gen_len.index_select(0, li).cpu().numpy()
            state.target_len.index_fill_(0, li, 0)     # the lane stops decoding
            for j, ln in enumerate(lanes):
                r = busy.pop(ln)
                req = SeqRequest(r.key, r.prompt, r.target_len, r.slot, toks[j, :gl[j]].copy(), int(win[j]),
                                 int(pre[j]), sts[j].copy())
                if on_evict is not None:
                    on_evict(req)
                else:
                    evicted.append(req)
                free.append(ln)

        # The host reads the lanes' progress one chunk late: chunk c + 1 is queued before chunk c's gen_len
        # copy is waited on, so the GPU never drains at a check (a finished lane idles at most two chunks).
        chunk = 0
        pending = None
        import time as _time
        while True:
            if inbox is not None:
                queue.extend(inbox())
            if not (queue or busy or pending is not None):
                if keep_alive is None or not keep_alive():
                    break
                _time.sleep(0.002)
                continue
            if queue and free and (len(free) >= admit_min or not busy or len(queue) <= len(free)):
                k = min(len(free), len(queue))
                admit([queue.popleft() for _ in range(k)])
            if busy and graph is None and self.use_graphs:
                iteration()            # eager first iteration (kernel attributes), then capture
                it_host += 1
                busy_iters += len(busy)
                graph = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(dev)
                side.wait_stream(st)
                c0 = launch_count()
                with torch.cuda.graph(graph, stream=side):
                    iteration()
                per_iter = launch_count() - c0
                self.graph_launches -= per_iter
                st.wait_stream(side)
            snap = None
            if busy:
                for _ in range(self.check_every):
                    if self.use_graphs:
                        graph.replay()
                        self.graph_launches += per_iter
                    else:
                        iteration()
                it_host += self.check_every
                busy_iters += self.check_every * len(busy)
                b = chunk & 1
                h_len[b].copy_(state.gen_len, non_blocking=True)
                h_tgt[b].copy_(state.target_len, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(st)
                snap = (ev, b, dict(busy))
                chunk += 1
            if pending is not None:
                ev, b, was_busy = pending
                ev.synchronize()
                gl, tl = h_len[b].numpy(), h_tgt[b].numpy()
                done = [ln for ln, r in was_busy.items() if busy.get(ln) is r and gl[ln] >= tl[ln]]
                if done:
                    start_harvest(done)
                if on_check is not None and busy:
                    # lanes still running the request the snapshot saw (a refilled lane's gen_len is stale)
                    live = {ln: busy[ln].key for ln in busy if was_busy.get(ln) is busy[ln] and gl[ln] < tl[ln]}
                    ev_l = [ln for ln in (on_check(live, gl, it_host, len(queue)) or []) if ln in live]
                    if ev_l:
                        evict(ev_l)
            finish_harvests()
            pending = snap
        finish_harvests(block=True)
        ev1.record(st)
        torch.cuda.synchronize(dev)
        a = acc.cpu().numpy()
        cfg = self.cfg
        rows = int(a[0])
        flops = 2.0 * (cfg.body_params() + cfg.vocab * cfg.d_model) * (rows + prefill_rows) \
            + 4.0 * cfg.n_layers * cfg.n_heads * cfg.head_dim * float(a[2])
        qh = qhist.cpu().numpy()
        qh[0] = 0
        res = StreamResult(out_tok, out_stats, evicted, int(a[1]), ev0.elapsed_time(ev1), rows, prefill_rows,
                           admissions, flops, float(cfg.kv_bytes_per_token) * float(a[3]), qh, busy_iters)
        res.weight_bytes = float(self.w.nbytes())
        return res

    def rollout(self, prompts, target_len, slots=None, index=None, speculate=True, record_tpi=False,
                recent_acceptance=None, seq_keys=None):
        """Generate target_len[b] tokens for each prompt row b (greedy), drafting from `index`.

        prompts: [B, P] int32 (host numpy or device tensor); slots[b]: history slot of b in index.
        seq_keys[b]: the sampling key of sequence b (T > 0; default b), so a sequence's samples do not
        depend on the batch row or KV slot it runs in.
        recent_acceptance: the worker's cumulative acceptance rate; when given, the batch gate
        decides whether this batch speculates at all (spec_engine.gate_check, as sim.py:346-352).
        """
        import torch
        from .spec_engine import gate_check
        if self.attention is not None:
            from .model import set_attention_family
            set_attention_family(self.attention)
        prompts = torch.as_tensor(prompts, dtype=torch.int32).to(self.device)
        B, P = prompts.shape
        if recent_acceptance is not None and not gate_check(self.spec.gate(), B, recent_acceptance):
            speculate = False
        self.last_speculated = bool(speculate and index is not None and self.spec.enabled)
        if B > self.n_slots:
            raise ValueError(f"batch {B} > engine slots {self.n_slots}")
        tl = np.asarray(target_len, dtype=np.int32)
        if P + int(tl.max()) > self.max_len:
            raise ValueError("prompt + target exceeds max_len")
        slots = np.zeros(B, np.int32) if slots is None else np.asarray(slots, dtype=np.int32)
        spec_on = bool(speculate and index is not None and self.spec.enabled)
        state = SpecBatch(slots, tl, self.spec, speculate=np.full(B, int(spec_on), np.uint8), device=self.device,
                          max_len=int(tl.max()), record_tpi=record_tpi)
        prompt_len = torch.full((B,), P, dtype=torch.int32, device=self.device)
        seq_key = torch.as_tensor(np.arange(B, dtype=np.int32) if seq_keys is None
                                  else np.asarray(seq_keys, dtype=np.int32)).to(self.device)
        st = torch.cuda.current_stream(self.device)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        L = lib()
        ev0.record(st)
        rows = self.prefill(prompts, state, seq_key)
        # device-side counters (accumulated by hm_build_verify_batch): rows, iterations, sum over rows of
        # (pos + 1), over sequences of (ctx + q); prefill rows are added here
        acc = torch.tensor([0, 0, B * P * (P + 1) // 2, B * P], dtype=torch.int64, device=self.device)
        qhist = torch.zeros(self.max_q + 1, dtype=torch.int64, device=self.device)
        # launch geometry of the captured iteration: one row per sequence without speculation (decode-sized
        # GEMM tiles and attention tiles), up to 1 + window rows per sequence with it
        q_cap = self.max_q if spec_on else 1
        R = min(self.fwd.max_rows, B * q_cap)

        def iteration():
            # one engine iteration, fully device-driven (row count lives in d_m): graph-capturable
            s = torch.cuda.current_stream(self.device)
            if spec_on:
                state.propose(index, s)
            check(L.hm_build_verify_batch(
                B, state.gen_tok.data_ptr(), state.gen_stride, state.gen_len.data_ptr(), state.target_len.data_ptr(),
                prompt_len.data_ptr(), state.draft_tok.data_ptr(), state.draft_tok.shape[1],
                state.draft_len.data_ptr(), self.kv_slot.data_ptr(), self.tokens.data_ptr(), self.pos.data_ptr(),
                self.row_slot.data_ptr(), self.q_off.data_ptr(), self.q_len.data_ptr(), self.pos0.data_ptr(),
                self.d_m.data_ptr(), acc.data_ptr(), qhist.data_ptr(), qhist.numel(), seq_key.data_ptr(),
                self.row_key.data_ptr(), s.cuda_stream))
            am = self.fwd.run(R, self.tokens, self.pos, self.row_slot, self.q_off, self.q_len, self.pos0,
                              self.kv_slot, B, q_cap, stream=s, m_dev=self.d_m, row_key=self.row_key)
            state.accept_greedy(am, self.q_off, s)

        # first decode iteration eagerly (initializes kernel attributes), then replay a captured graph
        iteration()
        if self.use_graphs:
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.device)
            side.wait_stream(st)
            c0 = launch_count()
            with torch.cuda.graph(graph, stream=side):
                iteration()
            per_iter = launch_count() - c0
            self.graph_launches -= per_iter   # captured, not executed
            st.wait_stream(side)

            def run():
                graph.replay()
                self.graph_launches += per_iter
        else:
            run = iteration
        while int(self.d_m.item()) > 0:
            for _ in range(self.check_every if self.use_graphs else 1):
                run()
        ev1.record(st)
        torch.cuda.synchronize(self.device)
        gpu_ms = ev0.elapsed_time(ev1)
        gen = state.gen_tok[:, :int(tl.max())].cpu().numpy()
        stats = state.stats.cpu().numpy()
        a = acc.cpu().numpy()
        rows += int(a[0])
        iters = 1 + int(a[1])
        cfg = self.cfg
        flops = (2.0 * (cfg.body_params() + cfg.vocab * cfg.d_model) * rows
                 + 4.0 * cfg.n_layers * cfg.n_heads * cfg.head_dim * float(a[2]))
        kv_bytes = float(cfg.kv_bytes_per_token) * float(a[3])
        qh = qhist.cpu().numpy()
        qh[0] = 0   # finished sequences
        res = RolloutResult(tokens=gen, stats=stats, iterations=iters, rows=rows, gpu_ms=gpu_ms, flops=flops,
                            kv_bytes=kv_bytes, qlen_hist=qh)
        res.d_tokens = state.gen_tok[:, :int(tl.max())]   # device copy (epoch pipeline: routed without a host trip)
        per = max(1, self.prefill_rows // P)
        res.forwards = (iters - 1) + (B + per - 1) // per   # decode/verify forwards + prefill chunks
        res.weight_bytes = float(self.w.nbytes())
        if record_tpi:
            res.tokens_per_iter = state.tokens_per_iter()
        return res


@dataclass
class SeqRequest:
    """One sequence for the continuous-batching engine (RolloutEngine.rollout_stream).

    A fresh rollout has `generated` None.  A migrated one (sim.py:719-779) carries the
    tokens it generated so far plus its HistoSpec state (AIMD window, prefix length, SpecStats): admission
    recomputes the KV of prompt + generated[:-1] by prefill and the rollout continues where it stopped.
    """
    key: int                      # global sequence key: sampling key and result id
    prompt: np.ndarray            # int32 prompt tokens
    target_len: int               # response length to generate
    slot: int = -1                # history slot in the index (-1: no history)
    generated: np.ndarray | None = None
    window: int | None = None
    prefix_len: int | None = None
    stats: np.ndarray | None = None


@dataclass
class StreamResult:
    tokens: dict                  # key -> int32 response tokens
    stats: dict                   # key -> int64 [5] SpecStats
    evicted: list                 # SeqRequest of sequences handed out by `on_check` (migration)
    iterations: int
    gpu_ms: float
    rows: int                     # verify / decode rows
    prefill_rows: int
    admissions: int
    flops: float = 0.0
    kv_bytes: float = 0.0
    qlen_hist: np.ndarray = None
    busy_lane_iters: int = 0      # sum over iterations of busy lanes (occupancy = / (iterations * lanes))

    @property
    def generated(self) -> int:
        return int(sum(int(v[0]) for v in self.stats.values()))


def profile_forward(engine: RolloutEngine, B: int, ctx: int, q, launch_rows=None, launch_q=None):
    """One verify forward of B sequences at context `ctx`, each launch bracketed by CUDA events.

    q: rows per sequence -- an int, or a length-B array of per-sequence verify
    block sizes (e.g. sampled from RolloutResult.qlen_hist).
    launch_rows / launch_q: launch geometry as the engine's captured iteration uses it (rows sized for
    the worst case, live count on the device; max rows per sequence); default: the exact sizes.
    Returns ({label: (total_ms, launches)}, M).  Used by bench.py for the
    per-kernel roofline (times measured live, not under a profiler).
    """
    import torch
    dev = engine.device
    ql = np.full(B, int(q), np.int32) if np.isscalar(q) else np.asarray(q, dtype=np.int32)
    M = int(ql.sum())
    qmax = int(ql.max())
    i32 = dict(dtype=torch.int32, device=dev)
    tokens = torch.randint(0, engine.cfg.vocab, (M,), **i32)
    q_len = torch.as_tensor(ql).to(dev)
    q_off = torch.as_tensor(np.concatenate([[0], np.cumsum(ql)[:-1]]).astype(np.int32)).to(dev)
    row_slot = torch.arange(B, **i32).repeat_interleave(q_len)
    pos = torch.arange(M, **i32) - q_off.repeat_interleave(q_len) + ctx
    pos0 = torch.full((B,), ctx, **i32)
    kv = torch.arange(B, **i32)
    R, qcap, m_dev = M, qmax, None
    if launch_rows is not None:
        R, qcap = max(launch_rows, M), max(launch_q or qmax, qmax)
        pad = R - M
        tokens = torch.cat([tokens, torch.zeros(pad, **i32)])
        pos = torch.cat([pos, torch.zeros(pad, **i32)])
        row_slot = torch.cat([row_slot, torch.zeros(pad, **i32)])
        m_dev = torch.tensor([M], **i32)
    engine.fwd.run(R, tokens, pos, row_slot, q_off, q_len, pos0, kv, B, qcap, m_dev=m_dev)   # warm
    prof = []
    # hold the stream with a ~50 ms spin so the host enqueues every launch (and its events) before the first
    # one runs: the kernels then run back to back, as in the engine's CUDA graphs, and no event interval
    # includes the host's per-launch cost
    torch.cuda.synchronize(dev)
    torch.cuda._sleep(100_000_000)
    engine.fwd.run(R, tokens, pos, row_slot, q_off, q_len, pos0, kv, B, qcap, m_dev=m_dev, prof=prof)
    torch.cuda.synchronize(dev)
    out = {}
    for label, e0, e1 in prof:
        t, n = out.get(label, (0.0, 0))
        out[label] = (t + e0.elapsed_time(e1), n + 1)
    return out, M


def smoke():
    """Tiny-model greedy rollout: speculation on == off, bit for bit (called by __graft_entry__.smoke)."""
    import torch
    from .index import GpuIndex
    from .model import TINY
    from .synth import mutate
    dev = torch.device("cuda", 0)
    w = Weights(TINY, dev, seed=0)
    eng = RolloutEngine(TINY, w, n_slots=16, max_len=256, device=dev)
    rng = np.random.default_rng(0)
    prompts = rng.integers(0, TINY.vocab, size=(16, 32), dtype=np.int32)
    base = eng.rollout(prompts, [128] * 16, speculate=False)
    hist = [[(mutate(rng, base.tokens[b].astype(np.int64), 0.8, 128, TINY.vocab, 4.0), 1.0) for _ in range(4)]
            for b in range(16)]
    idx = GpuIndex(hist)
    spec = eng.rollout(prompts, [128] * 16, slots=np.arange(16), index=idx, speculate=True)
    assert (spec.tokens == base.tokens).all(), "speculative output differs from greedy decode"
    assert spec.iterations < base.iterations
