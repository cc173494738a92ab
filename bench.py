#!/usr/bin/env python
"""HistoSpec B200 benchmark (driver contract: one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload rollout|replay|lookup|similarity]

Workloads (all on BASELINE.json configs[1] shapes, synthetic, seeded):
  rollout  greedy HistoSpec rollout of the Qwen2.5-1.5B-shaped random-init
           policy (512 prompts x 8 samples x 4k tokens); see engine.py
  replay   the reference's own path without a model: GPU history ingest (K1)
           + draft/verify/accept replay (K2+K6) of 4096 x 4096-token rollouts
  lookup   K2 draft-lookup microbenchmark over every position of an epoch

--impl reference times the reference algorithm on the host cores (the C
oracle port in oracle/, all threads) on a bounded sample of the same workload.
Under torchrun (N > 1) every rank runs its own shard (weak scaling); timing is
CUDA events on the launching stream, max over ranks.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


# ------------------------------------------------------------------ helpers

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "measured"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if not self.path or not os.path.exists(self.path):
            return out
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(smax), reasons=sorted(reasons), samples=len(sm))
        return out


class Dist:
    def __init__(self, backend):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend == "nccl":
                import torch
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self):
        if self.pg is not None:
            if self.pg.get_backend() == "nccl":
                import torch
                self.pg.barrier(device_ids=[self.local])
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        dev = "cuda" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        dev = "cuda" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


def measured_traffic(key, applies=True):
    """Per-launch DRAM traffic (read + write bytes) of `key` from the committed ncu capture
    (profiles/r02_traffic.json), or None when absent or when this run's workload is not the captured one."""
    if not applies:
        return None, None
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(key)
    except (OSError, ValueError):
        return None, None
    return (ent["bytes"], "ncu --set full, profiles/r02_traffic.json: " + ent["launch"]) if ent else (None, None)


def timed(fn, steps, warmup, dist, stream, gpu_index):
    """W untimed + exactly K timed calls bracketed by barrier + synchronize; returns (ms/step, clocks)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_index) as clk:
        start.record(stream)
        for _ in range(steps):
            fn()
        end.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / steps
    return dist.max(ms), clk.summary()


# ------------------------------------------------------------------ replay workload

def replay_setup(args, rank):
    import torch
    from paper_2508_18588_b200.workload import ReplayWorkload
    wl = ReplayWorkload(prompts=args.prompts, samples=args.samples, length=args.length,
                        similarity=args.similarity, shard=rank, seed=args.seed)
    data = wl.generate()
    return wl, data


def cpu_replay_sample(data, sample_prompts, threads):
    """Reference algorithm on the host (oracle C port): ingest + replay a bounded sample."""
    from oracle import hs_oracle_c as C
    P = min(sample_prompts, len(data["slot_resp_off"]) - 1)
    so, ro = data["slot_resp_off"], data["resp_off"]
    n_resp = int(so[P])
    L = int(ro[1] - ro[0])
    toks = data["hist_tokens"][:int(ro[n_resp])].reshape(n_resp, L)
    text = np.concatenate([toks, np.full((n_resp, 1), -1, np.int32)], axis=1).reshape(-1).astype(np.int32)
    rid = np.repeat(np.arange(n_resp, dtype=np.int32), L + 1)
    rew = data["rewards"][:n_resp].astype(np.float64)
    poff = (np.asarray(so[:P + 1]) * (L + 1)).astype(np.int64)
    samples = len(data["truth_slots"]) // (len(so) - 1)
    n_truth = P * samples
    truths = data["truths"][:n_truth]
    tcat = truths.reshape(-1).astype(np.int32)
    toff = (np.arange(n_truth + 1, dtype=np.int64) * truths.shape[1])
    tslot = data["truth_slots"][:n_truth].astype(np.int32)
    has = np.ones(P, np.uint8)
    t0 = time.perf_counter()
    tpi, niter, stats = C.replay_arrays(text, rid, rew, poff, has, tcat, toff, tslot, (1, 2, 2, 32, 7, 3), 1,
                                        threads)
    dt = time.perf_counter() - t0
    tok = int(stats[:, 0].sum())
    return {"tokens": tok, "seconds": dt, "value": tok / dt, "stats": stats.sum(axis=0).tolist(),
            "sample": f"{P} prompts x {samples} samples x {truths.shape[1]} tokens (ingest + replay)"}


def run_replay(args, dist, pk):
    import torch
    from paper_2508_18588_b200 import _lib
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.spec_engine import ReplayBuffers, SpecConfig

    dev = torch.device("cuda", dist.local)
    torch.cuda.set_device(dev)
    wl, data = replay_setup(args, dist.rank)
    cfg = SpecConfig()
    stream = torch.cuda.current_stream(dev)
    n_truth = data["truths"].shape[0]
    L = data["truths"].shape[1]
    toff = np.arange(n_truth + 1, dtype=np.int64) * L
    d_hist = torch.from_numpy(data["hist_tokens"]).to(dev)
    bufs = ReplayBuffers.from_host(data["truths"].reshape(-1), toff, data["truth_slots"],
                                   np.ones(n_truth, np.uint8), dev)
    phase = {"build": [], "replay": []}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    state = {}

    def step():
        ev[0].record(stream)
        idx = GpuIndex.from_arrays(d_hist, data["resp_off"], data["slot_resp_off"], data["reward_fx"])
        ev[1].record(stream)
        bufs.run(idx, cfg, stream)
        ev[2].record(stream)
        state["idx"] = idx
        state["pending"] = True

    def step_and_log():
        step()
        torch.cuda.synchronize()
        phase["build"].append(ev[0].elapsed_time(ev[1]))
        phase["replay"].append(ev[1].elapsed_time(ev[2]))

    # phase breakdown (untimed pass) then the contract timing
    step_and_log()
    lc0 = _lib.load().hs_launch_count()
    ms, clocks = timed(step, args.steps, args.warmup, dist, stream, dist.local)
    launches = (_lib.load().hs_launch_count() - lc0) // (args.steps + args.warmup)
    step_and_log()
    st = bufs.stats.cpu().numpy().sum(axis=0)
    tokens = int(st[0])
    total_tokens = dist.sum(tokens)
    value = total_tokens / (ms / 1e3)

    # e2e: public API with host buffers (H2D of history + truths, D2H of results inside the region)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    h_hist = pin(data["hist_tokens"])
    h_truth = pin(data["truths"].reshape(-1))
    h_slots = pin(data["truth_slots"])
    h_toff = pin(toff)
    h_spec = pin(np.ones(n_truth, np.uint8))
    out_tpi = torch.empty(int(toff[-1]), dtype=torch.int32).pin_memory()
    out_stats = torch.empty((n_truth, 5), dtype=torch.int64).pin_memory()

    def e2e_step():
        d_h = h_hist.to(dev, non_blocking=True)
        idx = GpuIndex.from_arrays(d_h, data["resp_off"], data["slot_resp_off"], data["reward_fx"])
        b = ReplayBuffers(truth=h_truth.to(dev, non_blocking=True), truth_off=h_toff.to(dev, non_blocking=True),
                          slots=h_slots.to(dev, non_blocking=True), speculate=h_spec.to(dev, non_blocking=True),
                          tpi=torch.empty(int(toff[-1]), dtype=torch.int32, device=dev),
                          n_iter=torch.empty(n_truth, dtype=torch.int32, device=dev),
                          stats=torch.empty((n_truth, 5), dtype=torch.int64, device=dev))
        b.run(idx, cfg, stream)
        out_tpi.copy_(b.tpi, non_blocking=True)
        out_stats.copy_(b.stats, non_blocking=True)

    e2e_ms, _ = timed(e2e_step, args.steps, max(1, args.warmup // 2), dist, stream, dist.local)
    h2d = h_hist.numel() * 4 + h_truth.numel() * 4 + h_slots.numel() * 4 + h_toff.numel() * 8 + n_truth
    d2h = out_tpi.numel() * 4 + out_stats.numel() * 8

    # roofline: the fused replay kernel (K2+K6, one launch per step)
    rep_ms = float(np.median(phase["replay"]))
    build_ms = float(np.median(phase["build"]))
    iters_lookup = int(st[3] + st[4])
    # per iteration: prefix (4*7) + probe entry 16 + verify text 4*7 + truth compare/draft 8*k + tpi 4
    alg_bytes = iters_lookup * (28 + 16 + 28 + 4) + int(st[1]) * 8 + n_truth * (5 * 8 + 4 + 4 + 8 + 4)
    achieved = alg_bytes / (rep_ms / 1e3) / 1e9
    line = {
        "metric": "rollout tokens/sec (HistoSpec replay path: ingest + draft + verify/accept, truth supplied)",
        "value": value, "unit": "tokens/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (D)-history s=%.2f, seeded" % args.similarity,
        "config": {"workload": "configs[1] shape, replay: %d prompts x %d samples x %d tokens per GPU, G=%d history"
                               % (args.prompts, args.samples, args.length, 8),
                   "l2": "inputs (%.0f MB) + index build traffic exceed the 126 MB L2" % (
                       (d_hist.numel() + bufs.truth.numel()) * 4 / 1e6)},
        "mean_accepted_per_verify": float(st[2] / max(st[3], 1)),
        "tokens_per_iteration": float(st[0] / max(st[3] + st[4], 1)),
        "acceptance_rate": float(st[2] / max(st[1], 1)),
        "phases_ms": {"ingest_k1": build_ms, "replay_k2_k6": rep_ms},
        "e2e": {"value": dist.sum(tokens) / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "roofline": {"kernel": "k_replay_fused", "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": None,
                     "peak_source": pk["source"]},
        "clocks": clocks,
    }
    return line, data


# ------------------------------------------------------------------ rollout workload (headline)

def derived_history(rng, truths, s, G, vocab, definition="D"):
    """Synthetic previous-epoch history of each current rollout; rewards Bernoulli(0.5).

    (D): the G members are independent s-mutations (burst 4) of the rollout itself.
    (T): tracegen semantics (tracegen.py:123-162): the rollout is an s-mutation of member 0, and members
         1..G-1 are siblings, s-mutations of member 0's parent -- built backwards from the rollout:
         member 0 = mutate(rollout), parent = mutate(member 0), member g = mutate(parent)."""
    from paper_2508_18588_b200.synth import mutate
    n, T = truths.shape
    toks = np.empty((n, G, T), dtype=np.int32)
    rew = np.empty((n, G), dtype=np.float64)
    for i in range(n):
        truth = truths[i].astype(np.int64)
        if definition == "D":
            for g in range(G):
                toks[i, g] = mutate(rng, truth, s, T, vocab, 4.0)
                rew[i, g] = 1.0 if rng.random() < 0.5 else 0.0
        else:
            m0 = mutate(rng, truth, s, T, vocab, 4.0)
            parent = mutate(rng, m0, s, T, vocab, 4.0)
            toks[i, 0] = m0
            rew[i, 0] = 1.0 if rng.random() < 0.5 else 0.0
            for g in range(1, G):
                toks[i, g] = mutate(rng, parent, s, T, vocab, 4.0)
                rew[i, g] = 1.0 if rng.random() < 0.5 else 0.0
    return toks, rew


def sample_prompts(prompt_of, pids, S, vocab):
    """[len(pids) * S, P] prompts: sample j of prompt p ends with a sample-id token (vocab - 1 - j), so the S
    greedy samples of a prompt are distinct sequences (hard part 7)."""
    rows = []
    for pid in pids:
        base = prompt_of(pid)
        for j in range(S):
            r = base.copy()
            r[-1] = vocab - 1 - j
            rows.append(r)
    return np.stack(rows).astype(np.int32)


def cpu_rollout_sample(cfg, seed, prompts, T, s, G, threads, W=None):
    """CPU fp32 rollout of the same policy (oracle/model_ref.CpuRollout), HistoSpec drafting from (D)
    histories of the CPU model's own greedy output.  Returns tokens/s of the speculative decode phase."""
    import torch
    from oracle import model_ref as R
    torch.set_num_threads(threads)
    if W is None:
        from paper_2508_18588_b200.model import Weights
        # generated on the host: the reference arm never touches the GPU (same seed, CPU RNG stream)
        w = Weights(cfg, "cpu", seed=seed)
        W = R.weights_fp32(w, "cpu")
        del w
    eng = R.CpuRollout(cfg, W, prompts.shape[1] + T + 40)
    base, _pre, dec0, it0, _, _ = eng.rollout([list(p) for p in prompts], T, None)
    rng = np.random.default_rng([seed, 77])
    toks, rew = derived_history(rng, np.asarray(base, dtype=np.int32), s, G, cfg.vocab)
    hists = [[(toks[p, g], float(rew[p, g])) for g in range(G)] for p in range(len(prompts))]
    out, pre, dec, iters, acc, ver = eng.rollout([list(p) for p in prompts], T, hists)
    n = len(prompts) * (T - 1)    # tokens landed by the decode phase (token 0 comes from prefill)
    return {"value": n / dec, "nonspec_value": n / dec0, "prefill_s": pre, "decode_s": dec, "iterations": iters,
            "accepted_per_verify": acc / max(ver, 1), "same_as_greedy": out == base,
            "sample": f"{len(prompts)} seqs x {T} tokens after a {prompts.shape[1]}-token prompt, fp32 torch on "
                      f"{threads} threads, prefill excluded"}, W


def side_file(name, obj):
    """Per-kernel detail that does not belong on the driver's one-line record (gpurun_out/ when present)."""
    d = os.path.join(ROOT, "gpurun_out")
    try:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, name), "w") as fh:
            json.dump(obj, fh, indent=1)
        return os.path.join("gpurun_out", name)
    except OSError:
        return None


def run_rollout(args, dist, pk):
    import torch
    from paper_2508_18588_b200 import _lib
    from paper_2508_18588_b200.engine import RolloutEngine, profile_forward
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import PRESETS, Weights
    from paper_2508_18588_b200.model import lib as mlib

    from paper_2508_18588_b200 import workers as W

    cfg = PRESETS[args.model]
    dev = torch.device("cuda", dist.local)
    torch.cuda.set_device(dev)
    B, S, P, T, G = args.batch, args.samples, args.prompt_len, args.length, 8
    per_wave = B // S                   # prompts per wave
    n_waves = args.waves
    # tensor parallelism (configs[4]): ranks 2g, 2g + 1 form rollout worker g; data parallelism over workers
    tp = args.tp
    if dist.world % tp:
        raise ValueError("--gpus must be a multiple of --tp")
    world, rank = dist.world // tp, dist.rank // tp          # data-parallel workers
    tp_group, dp_group = None, None
    if tp > 1:
        import torch.distributed as tdist
        for g in range(world):
            pg = tdist.new_group([g * tp + t for t in range(tp)])
            if g == rank:
                tp_group = pg
        for t in range(tp):
            pg = tdist.new_group([g * tp + t for g in range(world)])
            if t == dist.rank % tp:
                dp_group = pg
    w = Weights(cfg, dev, seed=args.seed, tp_rank=dist.rank % tp, tp_size=tp)
    bcast_ms = None
    bcast_gbps = None
    if world > 1:   # epoch boundary: the updated policy travels from worker 0 (one NCCL call over NVLink)
        for _ in range(3):   # first call includes communicator setup; report the warm one
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            W.broadcast_weights(w, src=dist.rank % tp, group=dp_group)
            torch.cuda.synchronize()
            bcast_ms = 1e3 * (time.perf_counter() - t0)
        bcast_gbps = w.flat.numel() * 2 / (bcast_ms / 1e3) / 1e9
    from paper_2508_18588_b200.spec_engine import SpecConfig
    spec_cfg = SpecConfig(window_max=args.window_max)   # the reference's defaults unless --window-max
    eng = RolloutEngine(w.cfg, w, n_slots=B, max_len=P + T, device=dev, attention=args.attention,
                        temperature=args.temperature, seed=args.seed, tp_group=tp_group, spec=spec_cfg)

    def prompt_tokens(pid):
        return np.random.default_rng([args.seed, 1000 + pid]).integers(0, cfg.vocab, size=P, dtype=np.int32)

    def seq_keys(pids):
        # sampling noise is keyed by a global sequence id (prompt, sample), not by the KV slot, so a sequence
        # draws the same tokens on whichever rank / slot it runs
        return np.array([pid * S + j for pid in pids for j in range(S)], dtype=np.int32)

    # HistoPipe assignment over last-epoch medians (uniform lengths here -> ranked by id); every rank owns
    # n_waves * per_wave prompts (weak scaling), rolled out one wave of B sequences at a time
    medians = {pid: float(T) for pid in range(per_wave * n_waves * world)}
    mine1 = W.assign_prompts(medians, world, 1)[rank]
    # previous epoch (step 1): plain rollouts of every wave (greedy, or T > 0 sampling with the same keys);
    # they are the speculation-off baseline and the outputs the speculative step must reproduce bit for bit
    outs, base_ms = {}, []
    for wv in range(n_waves):
        pids = mine1[wv * per_wave:(wv + 1) * per_wave]
        res = eng.rollout(sample_prompts(prompt_tokens, pids, S, cfg.vocab), [T] * B, speculate=False,
                          seq_keys=seq_keys(pids))
        base_ms.append(res.gpu_ms)
        for i, pid in enumerate(pids):
            outs[pid] = res.tokens[i * S:(i + 1) * S]
        if wv == 0:
            base0 = res
    # the same baseline with the other attention family on wave 0: a run must keep one family (bit-exact
    # spec == plain), but the fastest non-speculative configuration of the engine is the honest denominator
    other = "mma_sync" if args.attention == "tcgen05" else "tcgen05"
    eng.attention = other
    base_other = eng.rollout(sample_prompts(prompt_tokens, mine1[:per_wave], S, cfg.vocab), [T] * B,
                             speculate=False, seq_keys=seq_keys(mine1[:per_wave]))
    eng.attention = args.attention
    # ---- per-epoch history pipeline.  Wave w of epoch e on this rank is chunk w of
    # the HistoPipe group it serves; under the alternating group order the whole group (so the whole wave)
    # moves to one rank at the next epoch, where it is that rank's wave w.  After each step the wave's
    # finished rollouts stay in HBM: hs_pack_rows + all-to-all-v route them to their next owner, which turns
    # them into the next epoch's history on a side stream (hs_mutate_bursts: G s-similar relatives per
    # rollout -- the stand-in for policy drift, the (D) definition -- then K1) while the next wave rolls out.
    # Weights are fixed, so a prompt's rollout in epoch e + 1 equals its epoch-e rollout: the routed tokens
    # are also the bit-exactness reference of the step that uses them.
    side_st = torch.cuda.Stream(dev)
    stream = torch.cuda.current_stream(dev)
    resp_off = np.arange(B * G + 1, dtype=np.int64) * T
    slot_resp_off = np.arange(B + 1, dtype=np.int64) * G
    slots = np.arange(B)                 # one history slot per sequence: its G previous-epoch relatives
    hist_rng = np.random.default_rng([args.seed, 2000 + rank])
    acc = {"ms": [], "res": [], "exact": True, "route_ms": [], "n": 0, "ingest_ms": [], "epoch": 2}
    lib_hs = _lib.load()

    def ingest_routed(routed, epoch, wv_idx):
        """On side_st: history of the next epoch's wave from its routed rollouts; returns the wave record."""
        order = np.argsort(routed.keys, kind="stable")
        assert (order == np.arange(len(order))).all(), "routed records arrive in sequence-key order"
        assert len(routed.keys) == B and (np.diff(routed.resp_off) == T).all()
        pids = [int(p) for p in routed.pids[::S]]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(side_st):
            e0.record(side_st)
            truth = routed.tokens.view(B, T)
            if args.history == "D":
                hist = torch.empty(B * G * T, dtype=torch.int32, device=dev)
                rfx = torch.empty(B * G, dtype=torch.int64, device=dev)
                d_off = torch.as_tensor(routed.resp_off).to(dev, non_blocking=True)
                _lib.check(lib_hs.hs_mutate_bursts(truth.data_ptr(), d_off.data_ptr(), B, G, float(args.similarity),
                                                   4.0, cfg.vocab, (args.seed << 20) ^ (epoch << 8) ^ wv_idx,
                                                   hist.data_ptr(), rfx.data_ptr(), side_st.cuda_stream))
                reward_fx = rfx.cpu().numpy()
            else:   # (T) tracegen semantics: host restatement (synth.mutate), not pipelined
                h, rew = derived_history(hist_rng, truth.cpu().numpy(), args.similarity, G, cfg.vocab, "T")
                hist = torch.from_numpy(h.reshape(-1)).to(dev)
                reward_fx = (rew.reshape(-1) * float(1 << 32)).astype(np.int64)
            idx = GpuIndex.from_arrays(hist, resp_off, slot_resp_off, reward_fx, stream=side_st)   # K1
            e1.record(side_st)
            ready = torch.cuda.Event()
            ready.record(side_st)
        return {"pids": pids, "truth": truth, "keys": routed.keys.astype(np.int32), "index": idx, "ready": ready,
                "ev": (e0, e1), "h_prompts": torch.from_numpy(sample_prompts(prompt_tokens, pids, S,
                                                                             cfg.vocab)).pin_memory()}

    def route(d_tokens, pids, epoch_next):
        """Route a finished wave (device [B, T]) to the owners of its prompts at epoch_next (side_st)."""
        owner = W.owner_map(W.assign_prompts(medians, world, epoch_next))
        keys = seq_keys(pids)
        seq_pid = np.repeat(np.asarray(pids, np.int64), S)
        ev = torch.cuda.Event()
        ev.record(stream)
        side_st.wait_event(ev)
        d_tokens.record_stream(side_st)
        with torch.cuda.stream(side_st):
            return W.route_rollouts_device(d_tokens, np.full(B, T, np.int64), seq_pid, keys,
                                           np.full(B, 1 << 32, np.int64), owner, rank, world, stream=side_st,
                                           group=dp_group)

    # epoch 1 -> epoch 2: route the plain rollouts and build every wave's epoch-2 history
    waves = []
    for wv in range(n_waves):
        pids = mine1[wv * per_wave:(wv + 1) * per_wave]
        d_tok = torch.as_tensor(np.concatenate([outs[p] for p in pids])).to(dev)
        waves.append(ingest_routed(route(d_tok, pids, 2), 2, wv))
    torch.cuda.synchronize()
    out_tok = torch.empty((B, T), dtype=torch.int32).pin_memory()

    def step():
        k = acc["n"]
        acc["n"] += 1
        wi = k % n_waves
        epoch = 2 + k // n_waves
        wv = waves[wi]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d_prompts = wv["h_prompts"].to(dev, non_blocking=True)
        e0.record(stream)
        stream.wait_event(wv["ready"])                 # the wave's history (built on side_st) is in place
        res = eng.rollout(d_prompts, [T] * B, slots=slots, index=wv["index"], speculate=True,
                          seq_keys=wv["keys"])
        e1.record(stream)
        out_tok.copy_(torch.from_numpy(res.tokens))   # results already read back by rollout(); keep pinned copy
        acc["exact"] &= bool(torch.equal(res.d_tokens, wv["truth"]))
        # per-epoch history update: route this wave to its next owner, whose next-epoch history of it builds
        # on the side stream under the next wave's rollout
        t0 = time.perf_counter()
        routed = route(res.d_tokens, wv["pids"], epoch + 1)
        acc["route_ms"].append(1e3 * (time.perf_counter() - t0))
        acc["ingest_ms"].append(wv["ev"])
        waves[wi] = ingest_routed(routed, epoch + 1, wi)
        e1.synchronize()
        acc["ms"].append(e0.elapsed_time(e1))
        acc["res"].append(res)

    lc0, mc0, gl0 = _lib.load().hs_launch_count(), mlib().hm_launch_count(), eng.graph_launches
    e2e_ms, clocks = timed(step, args.steps, args.warmup, dist, stream, dist.local)
    launches = ((_lib.load().hs_launch_count() - lc0) + (mlib().hm_launch_count() - mc0)
                + (eng.graph_launches - gl0)) // (args.steps + args.warmup)
    ms_dev = float(np.mean(acc["ms"][-args.steps:]))
    ms_dev = dist.max(ms_dev)
    timed_res = acc["res"][-args.steps:]
    route_iso_ms = None
    if world > 1:   # the route alone, ranks aligned first (the in-step figure includes waiting for the slowest)
        dist.barrier()
        torch.cuda.synchronize()
        r0 = time.perf_counter()
        route(timed_res[-1].d_tokens, waves[(acc["n"] - 1) % n_waves]["pids"], 99)
        torch.cuda.synchronize()
        route_iso_ms = dist.max(1e3 * (time.perf_counter() - r0))
    st = np.sum([r.stats.sum(axis=0) for r in timed_res], axis=0)
    res = timed_res[-1]
    gen = B * T
    # tokens of a tensor-parallel worker are counted once (its tp ranks hold the same rollouts)
    value = dist.sum(gen) / tp / (ms_dev / 1e3)
    e2e = dist.sum(gen) / tp / (e2e_ms / 1e3)
    # step roofline (aggregate bound: max of total bytes / HBM and total flops / sustained bf16)
    bytes_total = res.forwards * res.weight_bytes + res.kv_bytes
    t_roof = max(bytes_total / (pk["hbm_gbs"] * 1e9), res.flops / (pk["bf16_tflops_sustained"] * 1e12))
    # dominant kernel, timed live with CUDA events in a representative verify forward
    # verify-block sizes drawn from this run's own (sequence, iteration) histogram
    qh = np.sum([r.qlen_hist for r in timed_res], axis=0).astype(np.float64)
    q_lens = np.random.default_rng([args.seed, 77]).choice(len(qh), size=B, p=qh / qh.sum()).astype(np.int32)
    q_mean = float(q_lens.mean())
    prof, M = profile_forward(eng, B, P + T // 2, q_lens)
    label, (k_ms, k_n) = max(prof.items(), key=lambda kv: kv[1][0])
    shapes = eng.fwd.gemm_shapes()
    kernels = {}
    for lab, (ms_, n_) in prof.items():
        ent = {"ms_per_forward": ms_, "launches": n_}
        if lab in shapes:
            N_, K_ = shapes[lab]
            tf = 2.0 * M * N_ * K_ * n_ / (ms_ / 1e3) / 1e12
            ent.update(tflops=tf, frac=tf / pk["bf16_tflops_sustained"])
        kernels[lab] = ent
    if label in shapes:
        N_, K_ = shapes[label]
        ach = 2.0 * M * N_ * K_ * k_n / (k_ms / 1e3) / 1e12
        roof = {"kernel": label, "bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": ach / pk["bf16_tflops_sustained"], "traffic": None,
                "per_launch_flops": 2.0 * M * N_ * K_, "M": M, "N": N_, "K": K_}
    else:   # attention: KV bytes
        kvb = float((P + T // 2 + q_lens).sum()) * w.cfg.n_kv_heads * w.cfg.head_dim * 2 * 2 * k_n
        ach = kvb / (k_ms / 1e3) / 1e9
        roof = {"kernel": label, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": ach / pk["hbm_gbs"], "traffic": None}
    std_cfg = (B, P, T, args.samples) == (1024, 256, 4096, 8) and dist.world == 1
    roof["traffic"], roof["traffic_source"] = measured_traffic("rollout:%s:%s" % (label, args.attention), std_cfg)
    roof["peak_source"] = pk["source"] + (" sustained" if roof["unit"] == "TFLOP/s" else "")
    bt = base0.tokens
    grams = [tuple(bt[b, i:i + 4]) for b in range(0, B, max(1, B // 256)) for i in range(0, T - 4, 7)]
    distinct = len(set(grams)) / max(1, len(grams))
    side = side_file("bench_rollout_side_r%d.json" % rank, {
        "kernels_ms_per_forward": kernels,
        "profiled_forward": {"seqs": B, "rows_per_seq_mean": q_mean, "rows_per_seq_max": int(q_lens.max()),
                             "ctx": P + T // 2, "M": M, "note": "verify-block sizes sampled from this run's histogram"},
        "verify_rows_hist": {str(i): int(c) for i, c in enumerate(qh) if c},
        "step_ms": acc["ms"], "ingest_ms": [a.elapsed_time(b) for a, b in acc["ingest_ms"]],
        "route_ms": acc["route_ms"], "nonspec_wave_ms": base_ms,
        "engine_iterations": [r.iterations for r in timed_res]})
    sampling = args.temperature > 0
    line = {
        "metric": "rollout tokens/sec (%s HistoSpec: ingest + draft + verify forward + accept)" % (
            "rejection-sampling T=%g" % args.temperature if sampling else "greedy"),
        "value": value, "unit": "tokens/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": e2e_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic prompts (sample-id token per sample), random-init weights (seed %d), (%s) history "
                "s=%.2f G=%d per sequence, SpecConfig window_max %d" % (args.seed, args.history, args.similarity, G,
                                                                        args.window_max),
        "config": {"workload": "configs[%d]: %s, %d prompts x %d samples per wave (%d resident sequences), "
                               "%d-token prompts, %d-token %s rollouts, waves cycle over %d prompts per GPU" % (
                                   2 if sampling else 1, cfg.name, per_wave, S, B, P, T,
                                   "sampled" if sampling else "greedy", per_wave * n_waves),
                   "step": "one wave: K1 ingest of its history + the HistoSpec rollout + routing of its outputs",
                   "parallelism": ("dp%d (independent rollout workers)" % world) if tp == 1 else
                                  "dp%d x tp%d (each worker a GPU pair; O / down all-reduced over peer memory)" % (
                                      world, tp),
                   "l2": "KV cache (%.0f GB) and weights stream far beyond the 126 MB L2" % (
                       eng.cache.buf.numel() * 2 / 1e9)},
        "attention_family": args.attention,
        "collectives": {"weight_broadcast_ms": bcast_ms, "weight_broadcast_GBps": bcast_gbps,
                        "rollout_route_ms_per_step": float(np.mean(acc["route_ms"][-args.steps:])),
                        "rollout_route_ms_aligned": route_iso_ms,
                        "note": "epoch-boundary only: NCCL broadcast of the policy, all-to-all-v of finished "
                                "rollouts to next-step owners (per-step figure: host time incl. waiting for the "
                                "slowest rank; aligned: one route after a barrier)"},
        "ingest_ms_per_step": float(np.mean([a.elapsed_time(b) for a, b in acc["ingest_ms"][-args.steps:]])),
        "distinct_4gram_ratio": distinct,
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": int(waves[0]["h_prompts"].numel() * 4
                                                                            + (0 if args.history == "D" else
                                                                               B * G * T * 4)),
                "d2h_bytes_per_step": int(out_tok.numel() * 4 + B * 5 * 8)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "roofline_step": {"t_roof_ms": t_roof * 1e3, "t_wall_ms": ms_dev, "frac": t_roof * 1e3 / ms_dev},
        "side_file": side,
        "clocks": clocks,
        # the speculation result last, where a truncated log tail still shows it
        "nonspec_value_%s" % other: dist.sum(B * T) / tp / dist.max(base_other.gpu_ms / 1e3),
        "nonspec_value": dist.sum(B * T) / tp / dist.max(float(np.mean(base_ms)) / 1e3),
        "engine_iterations": float(np.mean([r.iterations for r in timed_res])),
        "acceptance_rate": float(st[2] / max(st[1], 1)),
        "tokens_per_iteration": float(st[0] / max(st[3] + st[4], 1)),
        "mean_accepted_per_verify": float(st[2] / max(st[3], 1)),
        ("bit_exact_vs_plain_sampling" if sampling else "bit_exact_vs_greedy"):
            bool(dist.sum(float(acc["exact"])) == dist.world),
        "speedup_vs_nonspec": value / max(dist.sum(B * T) / tp / dist.max(float(np.mean(base_ms)) / 1e3),
                                          dist.sum(B * T) / tp / dist.max(base_other.gpu_ms / 1e3), 1e-9),
    }
    return line, {"cfg": cfg, "prompts": waves[0]["h_prompts"].numpy(), "T": T, "w": w}


# ------------------------------------------------------------------ long-tail workload (configs[3])

def tau_profile(eng, cfg, world, lanes, group_seqs, pk, dist):
    """HistoPipe tau(len, k) from this engine's measured verify-forward times (rank 0, broadcast): a group of
    `group_seqs` sequences of length len on k GPUs runs min(lanes, group_seqs / k) lanes per GPU for about
    len / tokens-per-iteration iterations at mean context len / 2.  Returns workers.TauProfile."""
    import torch
    from paper_2508_18588_b200 import workers as W
    from paper_2508_18588_b200.engine import profile_forward
    lens = [512, 2048, 8192, 16384]
    ks = list(range(1, world + 1))
    grid = torch.zeros(len(lens), len(ks), dtype=torch.float64, device=eng.device)
    if dist.rank == 0:
        tpi = 3.0   # tokens per iteration assumed by the profile; TauProfile.accepted_per_pass rescales
        for i, l in enumerate(lens):
            for j, k in enumerate(ks):
                b = max(1, min(lanes, -(-group_seqs // k)))
                prof, _m = profile_forward(eng, b, min(eng.max_len - 40, 256 + l // 2), 4)
                t_fwd = sum(v[0] for v in prof.values()) / 1e3
                waves = -(-group_seqs // (b * k))
                grid[i, j] = waves * (l / tpi) * t_fwd
    if dist.pg is not None:
        dist.pg.broadcast(grid, src=0)
    g = grid.cpu().numpy()
    return W.TauProfile.from_rows([(l, k, float(g[i, j])) for i, l in enumerate(lens) for j, k in enumerate(ks)])


def run_longtail(args, dist, pk):
    """configs[3]: long-tail response lengths (log-normal, clipped to [512, 16384]) on the continuous-batching
    engine, prompts placed by HistoPipe (ranked groups, tau-profiled two-tier allocation, alternating order),
    (D) histories at each similarity of the sweep.  One step = one speculative epoch of this rank's share."""
    import torch
    from paper_2508_18588_b200 import _lib
    from paper_2508_18588_b200 import workers as W
    from paper_2508_18588_b200.engine import RolloutEngine, SeqRequest
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import PRESETS, Weights
    from paper_2508_18588_b200.model import lib as mlib

    cfg = PRESETS[args.model]
    dev = torch.device("cuda", dist.local)
    torch.cuda.set_device(dev)
    world, rank = dist.world, dist.rank
    S, P, G = args.samples, args.prompt_len, 8
    lo, hi = 512, 16384
    lanes = args.batch
    n_prompts = args.prompts * world                       # weak scaling: args.prompts per GPU
    rng = np.random.default_rng([args.seed, 4242])
    z = rng.standard_normal(n_prompts)
    # last epoch: per-prompt median and per-sample lengths (HistoPipe ranks on these); this epoch every prompt's
    # lengths grow by a per-prompt factor exp(growth_sigma z') (0 without --migrate: lengths repeat), so some
    # rollouts outgrow beta x their group's longest history -- the stragglers migration_decision moves
    med = np.clip(np.exp(np.log(args.len_median) + args.len_sigma * z), lo, hi)
    tgt_last = np.clip(np.rint(med[:, None] * np.exp(0.08 * rng.standard_normal((n_prompts, S)))), lo, hi)
    g_sigma = args.growth_sigma if args.migrate else 0.0
    growth = np.exp(g_sigma * np.random.default_rng([args.seed, 4343]).standard_normal(n_prompts))
    tgt = np.clip(np.rint(tgt_last * growth[:, None]), lo, hi).astype(int)
    w = Weights(cfg, dev, seed=args.seed)

    def make_engine(max_target):
        # length-aware lanes: the slot-contiguous KV cache holds as many lanes as fit at this rank's longest
        # assigned rollout (a rank serving a short HistoPipe group runs a wider batch)
        ml = P + int(max_target) + 8
        n = int(min(args.batch, max(8, args.kv_gb * 1e9 // ((ml + 34) * cfg.kv_bytes_per_token))))
        return RolloutEngine(cfg, w, n_slots=n, max_len=ml, device=dev, attention=args.attention, check_every=8)

    plan = None
    if world > 1:
        n_groups = max(2, world // 2)
        groups = W.build_groups({p: float(med[p]) for p in range(n_prompts)}, n_groups)
        probe = make_engine(hi)
        tau = tau_profile(probe, cfg, world, probe.n_slots, len(groups[0].prompt_ids) * S, pk, dist)
        if rank == 0:
            try:
                os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
                tau.to_csv(os.path.join(ROOT, "gpurun_out", "tau_profile_%s_%dgpu.csv" % (cfg.name, world)))
            except OSError:
                pass
        del probe
        torch.cuda.empty_cache()
        lens_g = [g.representative_len for g in groups]
        plan = (W.plan_makespan(lens_g, world, tau) if args.histopipe == "makespan"
                else W.plan_allocation(lens_g, world, 0.0, tau, precision=0.01))
        per_group = plan.per_group_workers if plan.feasible else W.partition_sizes(world, n_groups)
        assign = W.assign_with_plan(groups, per_group, 1)
        mine = assign[rank]
        group_of_rank = {r: next(g.index for g in groups if set(assign[r]) <= set(g.prompt_ids))
                         for r in range(world)}
    else:
        mine = list(range(n_prompts))
        groups, group_of_rank = None, {0: 0}
    eng = make_engine(tgt[mine].max())
    lanes = eng.n_slots

    def prompt_tokens(pid):
        return np.random.default_rng([args.seed, 1000 + pid]).integers(0, cfg.vocab, size=P, dtype=np.int32)

    prompts = sample_prompts(prompt_tokens, mine, S, cfg.vocab)
    keys = [pid * S + j for pid in mine for j in range(S)]
    targets = [int(tgt[pid, j]) for pid in mine for j in range(S)]
    reqs = [SeqRequest(key=k, prompt=prompts[i], target_len=t, slot=i) for i, (k, t) in enumerate(zip(keys, targets))]
    # length-aware admission: longest predicted (the prompt's last-epoch median) first
    order = sorted(range(len(reqs)), key=lambda i: (-med[mine[i // S]], i))
    queue = [reqs[i] for i in order]
    migrate = bool(args.migrate and world > 1)
    # last epoch's lengths: this epoch's targets over a per-rollout growth factor; stragglers that outgrow
    # beta x their group's longest history are the rollouts HistoPipe migrates (scheduler.py:304-330)
    hist_len = tgt_last
    policy = W.MigrationPolicy(alpha_pct=args.alpha_pct, beta=W.beta_from_history(list(growth)))
    run_no = [0]
    mig_log = {"evicted": 0, "received": 0}

    def run_epoch(idx_, spec_on):
        """One epoch of this rank's requests; with --migrate, stragglers move between ranks mid-epoch."""
        if not migrate:
            return eng.rollout_stream(queue, index=idx_, speculate=spec_on)
        run_no[0] += 1
        broker = W.MigrationBroker(dist.pg.distributed_c10d._get_default_store(), rank, world,
                                   tag="mig%d" % run_no[0])
        dist.barrier()
        g_me = group_of_rank[rank]
        max_hist = float(max(hist_len[p].max() for p in groups[g_me].prompt_ids))
        total = len(queue)
        done_keys = set()

        def on_check(live, gl, it, waiting):
            remaining = waiting + len(live)
            left = sum(max(0, queue_t[k] - int(gl[ln])) for ln, k in live.items())
            broker.publish_load(left)
            loads = broker.loads()
            act = {}
            for r, ld in loads.items():
                if r != rank and ld > 0:
                    act[group_of_rank[r]] = act.get(group_of_rank[r], 0.0) + ld
            out = []
            for ln, k in live.items():
                if k in moved_in:     # a rollout migrates at most once
                    continue
                kind, tg = W.migration_decision(g_me, max_hist, int(gl[ln]), total - remaining, total, policy,
                                                len(groups), act)
                if kind == "intra_step" and tg is not None:
                    dst = min((loads.get(r, 0.0), r) for r in range(world) if group_of_rank[r] == tg)[1]
                    out.append(ln)
                    dest[k] = dst
            return out

        def on_evict(req):
            mig_log["evicted"] += 1
            broker.post(dest.pop(req.key), req)

        def inbox():
            # a migrated-in rollout continues without drafts: its history slot indexes the source GPU's
            # GpuIndex (the receiving engine's graph holds this rank's index)
            got = [dataclasses.replace(r, slot=-1) for r in broker.poll()]
            for r in got:
                queue_t[r.key] = r.target_len
                moved_in.add(r.key)
            mig_log["received"] += len(got)
            return got

        dest = {}
        moved_in = set()
        res_ = eng.rollout_stream(queue, index=idx_, speculate=spec_on, on_check=on_check, on_evict=on_evict,
                                  inbox=inbox, keep_alive=broker.keep_alive, max_target=hi)
        dist.barrier()
        return res_

    queue_t = {r.key: r.target_len for r in reqs}
    # epoch 1: plain rollouts (the speculation-off baseline and the truth the speculative epochs reproduce)
    base = run_epoch(None, False)
    if migrate:   # rollouts that finished on another rank come home (host exchange of the few migrated ones)
        import torch.distributed as tdist
        gathered = [None] * world
        own = set(keys)
        tdist.all_gather_object(gathered, {k: v for k, v in base.tokens.items() if k not in own})
        for part in gathered:
            for k, v in part.items():
                if k in own:
                    base.tokens[k] = v
    n_tok = int(sum(targets))
    truth = np.concatenate([base.tokens[k] for k in keys]).astype(np.int32)
    resp_off = np.concatenate([[0], np.cumsum(targets)]).astype(np.int64)
    d_truth = torch.from_numpy(truth).to(dev)
    d_off = torch.from_numpy(resp_off).to(dev)
    h_resp_off = np.concatenate([[0], np.cumsum(np.repeat(targets, G))]).astype(np.int64)
    slot_resp_off = np.arange(len(reqs) + 1, dtype=np.int64) * G
    lib_hs = _lib.load()
    sweep = [float(x) for x in args.similarity_sweep.split(",")] if args.similarity_sweep else [args.similarity]
    stream = torch.cuda.current_stream(dev)
    rows = []
    head = None
    for si, sim in enumerate(sweep):
        # (D) history of every sequence from its own epoch-1 output, on the device
        hist = torch.empty(G * n_tok, dtype=torch.int32, device=dev)
        rfx = torch.empty(G * len(reqs), dtype=torch.int64, device=dev)
        _lib.check(lib_hs.hs_mutate_bursts(d_truth.data_ptr(), d_off.data_ptr(), len(reqs), G, sim, 4.0, cfg.vocab,
                                           args.seed * 7919 + si, hist.data_ptr(), rfx.data_ptr(), stream.cuda_stream))
        # hs_mutate_bursts lays member g of sequence i at G * off[i] + g * len[i]: slot-major, as K1 wants
        idx = GpuIndex.from_arrays(hist, h_resp_off, slot_resp_off, rfx.cpu().numpy())
        box = {}

        def step():
            box["res"] = run_epoch(idx, True)

        lc0, mc0, gl0 = lib_hs.hs_launch_count(), mlib().hm_launch_count(), eng.graph_launches
        e2e_ms, clocks = timed(step, args.steps, args.warmup if si == 0 else 1, dist, stream, dist.local)
        launches = ((lib_hs.hs_launch_count() - lc0) + (mlib().hm_launch_count() - mc0)
                    + (eng.graph_launches - gl0)) // (args.steps + (args.warmup if si == 0 else 1))
        res = box["res"]
        if migrate:   # every rollout finished somewhere: check it against its owner's epoch-1 output
            import hashlib
            import torch.distributed as tdist
            mine_h = {k: hashlib.sha1(np.ascontiguousarray(v, np.int32).tobytes()).hexdigest()
                      for k, v in res.tokens.items()}
            base_h = {k: hashlib.sha1(np.ascontiguousarray(base.tokens[k], np.int32).tobytes()).hexdigest()
                      for k in keys}
            ga, gb = [None] * world, [None] * world
            tdist.all_gather_object(ga, mine_h)
            tdist.all_gather_object(gb, base_h)
            fin = {k: h for part in ga for k, h in part.items()}
            ref = {k: h for part in gb for k, h in part.items()}
            exact = fin == ref
            st = np.sum(list(res.stats.values()), axis=0)
        else:
            exact = all(np.array_equal(res.tokens[k], base.tokens[k]) for k in keys)
            st = np.sum([res.stats[k] for k in keys], axis=0)
        value = dist.sum(n_tok) / (dist.max(e2e_ms) / 1e3)
        row = {"similarity": sim, "value": value, "ms_per_step": e2e_ms,
               "tokens_per_iteration": float(st[0] / max(st[3] + st[4], 1)),
               "mean_accepted_per_verify": float(st[2] / max(st[3], 1)),
               "occupancy": res.busy_lane_iters / max(1, res.iterations * lanes),
               "bit_exact_vs_greedy": bool(dist.sum(float(exact)) == world),
               "speedup_vs_nonspec": value / (dist.sum(n_tok) / dist.max(base.gpu_ms / 1e3))}
        rows.append(row)
        if head is None:
            head = (row, clocks, launches, res)
    # static waves on the same workload (no refill: a wave lasts as long as its longest rollout)
    waves_ms = 0.0
    if args.compare_waves:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for a in range(0, len(queue), lanes):
            chunk = queue[a:a + lanes]
            r = eng.rollout(np.stack([q.prompt for q in chunk]), [q.target_len for q in chunk],
                            slots=[q.slot for q in chunk], index=idx, speculate=True,
                            seq_keys=[q.key for q in chunk])
        e1.record(stream)
        torch.cuda.synchronize()
        waves_ms = e0.elapsed_time(e1)
    row, clocks, launches, res = head
    nonspec = dist.sum(n_tok) / dist.max(base.gpu_ms / 1e3)
    mine_stat = torch.tensor([float(n_tok), float(row["ms_per_step"]), float(lanes), float(row["occupancy"]),
                              float(len(reqs)), float(max(targets))], dtype=torch.float64, device=dev)
    if dist.pg is not None:
        allst = [torch.zeros_like(mine_stat) for _ in range(world)]
        dist.pg.all_gather(allst, mine_stat)
    else:
        allst = [mine_stat]
    ranks = [dict(zip(("tokens", "step_ms", "lanes", "occupancy", "sequences", "longest"), t.cpu().tolist()))
             for t in allst]
    line = {
        "metric": "rollout tokens/sec (greedy HistoSpec, long-tail lengths, continuous batching)",
        "value": row["value"], "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": row["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic prompts (sample-id token per sample), random-init weights (seed %d), (D) history per "
                "sequence (device burst mutation, G=%d)" % (args.seed, G),
        "config": {"workload": "configs[3]: %s, %d prompts x %d samples per GPU, lengths log-normal median %d "
                               "sigma %.2f clipped to [%d, %d] (%d tokens on rank 0), %d engine lanes" % (
                                   cfg.name, args.prompts, S, args.len_median, args.len_sigma, lo, hi, n_tok, lanes),
                   "lanes_per_rank": "KV budget %.0f GB / (longest assigned rollout x KV bytes per token), <= "
                                     "--batch %d" % (args.kv_gb, args.batch),
                   "step": "one speculative epoch of the rank's sequences through rollout_stream (admission "
                           "prefill + CUDA-graph iterations; value includes prefill)",
                   "parallelism": "dp%d, HistoPipe %s" % (world, "%s plan %s (d=%.3g s, t0=%.3g s)" % (
                       args.histopipe, plan.per_group_workers, plan.gradient_d, plan.t0)
                       if plan is not None and plan.feasible
                       else "single rank" if plan is None else "infeasible plan -> equal split"),
                   "l2": "KV cache (%.0f GB) streams far beyond the 126 MB L2" % (eng.cache.buf.numel() * 2 / 1e9)},
        "e2e": {"value": row["value"], "unit": "tokens/s", "h2d_bytes_per_step": int(len(reqs) * P * 4),
                "d2h_bytes_per_step": int(n_tok * 4 + len(reqs) * 40)},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "sweep": rows,
        "ranks": ranks,
        "migration": {"enabled": migrate, "alpha_pct": args.alpha_pct, "beta": policy.beta,
                      "evicted_rank0": mig_log["evicted"], "received_rank0": mig_log["received"],
                      "note": "intra-step straggler migration (scheduler.py:304-330) with KV recompute by prefill "
                              "on the receiving GPU; this epoch's lengths = last epoch's x exp(%.2f z) per "
                              "prompt, beta = beta_from_history(growth rates)" % g_sigma},
        "static_waves_value": (dist.sum(n_tok) / dist.max(waves_ms / 1e3)) if waves_ms else None,
        "occupancy": row["occupancy"],
        "nonspec_value": nonspec,
        "tokens_per_iteration": row["tokens_per_iteration"],
        "mean_accepted_per_verify": row["mean_accepted_per_verify"],
        "bit_exact_vs_greedy": row["bit_exact_vs_greedy"],
        "speedup_vs_nonspec": row["speedup_vs_nonspec"],
    }
    return line, {"cfg": cfg}


# ------------------------------------------------------------------ BASELINE.md section 4 CPU plan

def _ref_replay_shard(args):
    """One worker of the pool: the reference's build_tree + replay_response over a shard of prompts."""
    ref_path, items = args
    import sys as _sys
    if ref_path not in _sys.path:
        _sys.path.insert(0, ref_path)
    from rhymesim.history import Response, build_tree
    from rhymesim.spec_engine import SpecConfig, SpecStats, replay_response
    t_build = t_replay = 0.0
    st = SpecStats()
    tpis = []
    for pid, hist, truths in items:
        t0 = time.perf_counter()
        tree = build_tree(pid, 1, [Response(pid, 1, [int(x) for x in tok], float(r)) for tok, r in hist])
        t1 = time.perf_counter()
        for tr in truths:
            rr = replay_response([int(x) for x in tr], tree, SpecConfig(), stats=st)
            tpis.append(list(rr.tokens_per_iter))
        t_build += t1 - t0
        t_replay += time.perf_counter() - t1
    stats = np.array([st.tokens_total, st.tokens_speculated, st.tokens_accepted, st.verify_passes, st.decode_passes],
                     np.int64)
    return t_build, t_replay, stats, tpis


def run_cpu_plan(args, dist, pk):
    """(1) the reference's own HistoSpec bookkeeping (rhymesim build_tree +
    replay_response, from baseline/_ref) on the host cores, single process and a process pool, checked
    bit-exact against the GPU replay of the same inputs; (2) configs[0] end to end on CPU (tiny model, fp32
    torch on all threads, oracle drafting) beside the same workload on the GPU engine."""
    import multiprocessing as mproc
    import subprocess as sp
    import torch
    from paper_2508_18588_b200.engine import RolloutEngine
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.model import TINY, Weights
    from paper_2508_18588_b200.spec_engine import SpecConfig, replay_batch
    from paper_2508_18588_b200.workload import ReplayWorkload, history_lists
    cores = os.cpu_count() or 1
    try:
        model = [l.split(":", 1)[1].strip() for l in sp.run(["lscpu"], capture_output=True, text=True).stdout
                 .splitlines() if l.startswith("Model name")][0]
    except Exception:   # noqa: BLE001
        model = "unknown"
    out = {"impl": "cpu-plan", "host": {"cpu_count": cores, "lscpu_model": model}}
    # ---- (1) bookkeeping: configs[1]-shaped prompts (8 x 4096-token (D) histories at s, 8 truths each)
    ref = os.path.join(ROOT, "baseline", "_ref")
    data = ReplayWorkload(prompts=args.ref_prompts, samples=args.samples, length=args.length,
                          similarity=args.similarity, seed=args.seed).generate()
    hists = history_lists(data)
    S = args.samples
    items = [("p%d" % p, [(h, r) for h, r in hists[p]], [data["truths"][p * S + j] for j in range(S)])
             for p in range(len(hists))]
    n_tok = int(sum(len(t) for _, _, ts in items for t in ts))
    if os.path.isfile(os.path.join(ref, "rhymesim", "history.py")):
        t0 = time.perf_counter()
        tb, tr, st1, tpi1 = _ref_replay_shard((ref, items))
        single = time.perf_counter() - t0
        t0 = time.perf_counter()
        shards = [(ref, items[i::cores]) for i in range(min(cores, len(items)))]
        with mproc.get_context("spawn").Pool(len(shards)) as pool:
            parts = pool.map(_ref_replay_shard, shards)
        pooled = time.perf_counter() - t0
        # GPU replay of the same inputs: bit-exact tokens_per_iter and stats (the parity half of the plan)
        idx = GpuIndex([[(h, r) for h, r in hists[p]] for p in range(len(hists))])
        per, st_gpu = replay_batch(idx, [p for p in range(len(hists)) for _ in range(S)],
                                   [t for _, _, ts in items for t in ts], SpecConfig())
        out["bookkeeping"] = {
            "kind": "reference", "source": "rhymesim (baseline/_ref) build_tree + replay_response",
            "sample": "%d prompts x %d truths x %d tokens, G=8 (D) histories s=%.2f" % (
                len(items), S, args.length, args.similarity),
            "single_process_tokens_per_s": n_tok / single, "single_build_s": tb, "single_replay_s": tr,
            "pool_tokens_per_s": n_tok / pooled, "pool_workers": len(shards),
            "accepted_per_verify": float(st1[2] / max(st1[3], 1)),
            "gpu_bit_exact": bool(per == tpi1 and (st_gpu.sum(axis=0) == st1).all())}
    else:
        out["bookkeeping"] = {"unavailable": "baseline/_ref not installed (tools/install_reference.sh)"}
    # ---- (2) configs[0] end to end: tiny decoder, 64 prompts x 2 epochs (epoch 2 HistoSpec, (D) s = 0.7)
    from oracle import model_ref as R
    torch.set_num_threads(cores)
    n_p, P0, T0 = 64, 32, args.tiny_tokens
    prompts = np.random.default_rng([args.seed, 5]).integers(0, TINY.vocab, size=(n_p, P0), dtype=np.int32)
    Wc = R.weights_fp32(Weights(TINY, "cpu", seed=args.seed), "cpu")
    eng_c = R.CpuRollout(TINY, Wc, P0 + T0 + 40)
    base_c, pre0, dec0, _, _, _ = eng_c.rollout([list(p) for p in prompts], T0, None)
    rng = np.random.default_rng([args.seed, 6])
    toks, rew = derived_history(rng, np.asarray(base_c, dtype=np.int32), 0.7, 8, TINY.vocab)
    hc = [[(toks[p, g], float(rew[p, g])) for g in range(8)] for p in range(n_p)]
    out_c, pre1, dec1, it1, acc1, ver1 = eng_c.rollout([list(p) for p in prompts], T0, hc)
    n_gen = n_p * T0
    dev = torch.device("cuda", dist.local)
    wg = Weights(TINY, dev, seed=args.seed)
    eng = RolloutEngine(TINY, wg, n_slots=n_p, max_len=P0 + T0 + 8, device=dev)
    b0 = eng.rollout(prompts, [T0] * n_p, speculate=False)
    toks_g, rew_g = derived_history(np.random.default_rng([args.seed, 6]), b0.tokens, 0.7, 8, TINY.vocab)
    idx_g = GpuIndex([[(toks_g[p, g], float(rew_g[p, g])) for g in range(8)] for p in range(n_p)])
    b1 = eng.rollout(prompts, [T0] * n_p, slots=np.arange(n_p), index=idx_g, speculate=True)
    out["configs0"] = {
        "workload": "configs[0]: tiny 2-layer decoder (d 256, vocab 4096), %d prompts x 2 epochs, %d-token "
                    "greedy rollouts, epoch-2 HistoSpec with (D) s=0.7 G=8 history" % (n_p, T0),
        "cpu": {"kind": "port", "cores": cores, "epoch1_nonspec_tokens_per_s": n_gen / (pre0 + dec0),
                "epoch2_histospec_tokens_per_s": n_gen / (pre1 + dec1),
                "accepted_per_verify": acc1 / max(ver1, 1), "spec_equals_greedy": out_c == base_c,
                "note": "fp32 torch on all host threads, drafting by the C restatement of extract_draft "
                        "(pinned to the reference's golden vectors)"},
        "gpu": {"epoch1_nonspec_tokens_per_s": n_gen / (b0.gpu_ms / 1e3),
                "epoch2_histospec_tokens_per_s": n_gen / (b1.gpu_ms / 1e3),
                "spec_equals_greedy": bool(np.array_equal(b0.tokens, b1.tokens)),
                "note": "bf16 engine on one B200 (different arithmetic from the fp32 CPU model: outputs "
                        "are compared within each engine)"}}
    return out


# ------------------------------------------------------------------ lookup microbenchmark

def run_lookup(args, dist, pk):
    import ctypes
    import torch
    from paper_2508_18588_b200 import _lib
    from paper_2508_18588_b200.index import GpuIndex

    dev = torch.device("cuda", dist.local)
    torch.cuda.set_device(dev)
    wl, data = replay_setup(args, dist.rank)
    idx = GpuIndex.from_arrays(torch.from_numpy(data["hist_tokens"]).to(dev), data["resp_off"],
                               data["slot_resp_off"], data["reward_fx"])
    # one query per truth position (sliding 7-gram windows via gen_stride = 1)
    P, L = args.prompts, args.length
    truths = data["truths"][::args.samples]           # one row per prompt
    flat = torch.from_numpy(truths.reshape(-1).astype(np.int32)).to(dev)
    m = 7
    # query s = prefix flat[s : s+m] (gen_stride = 1 turns one buffer into n overlapping rows);
    # the m-1 windows per prompt that straddle a prompt boundary are ordinary misses/hits of slot s // L
    n = P * L - m
    slot = (torch.arange(n, device=dev) // L).to(torch.int32)
    gen_len = torch.full((n,), m, dtype=torch.int32, device=dev)
    prefix_len = torch.full((n,), m, dtype=torch.int32, device=dev)
    window = torch.full((n,), 32, dtype=torch.int32, device=dev)
    spec = torch.ones(n, dtype=torch.uint8, device=dev)
    out = torch.empty((n, 32), dtype=torch.int32, device=dev)
    dlen = torch.empty(n, dtype=torch.int32, device=dev)
    looked = torch.empty(n, dtype=torch.uint8, device=dev)
    found = torch.empty(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    lib = _lib.load()

    def launch():
        _lib.check(lib.hs_draft(ctypes.byref(idx.view), n, slot.data_ptr(), flat.data_ptr(), 1, gen_len.data_ptr(),
                                prefix_len.data_ptr(), window.data_ptr(), spec.data_ptr(), m, m, 32, out.data_ptr(),
                                32, dlen.data_ptr(), looked.data_ptr(), found.data_ptr(), stream.cuda_stream))

    ms, clocks = timed(launch, args.steps, args.warmup, dist, stream, dist.local)
    dl = int(dlen.sum().item())
    hits = int(found.sum().item())
    alg = n * (4 + 16 + 4 * m + 4 * 4 + 3) + hits * 0 + dl * 8
    achieved = alg / (ms / 1e3) / 1e9
    return {
        "metric": "draft lookups/sec (K2 hs_draft, every position of an epoch)", "value": dist.sum(n) / (ms / 1e3),
        "unit": "queries/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{n} queries (m=7, window 32) over {P} prompts x 8 x {L}-token (D) histories",
                   "l2": "index + outputs exceed L2"},
        "hit_rate": hits / n, "mean_draft_len": dl / n,
        "roofline": {"kernel": "k_draft", "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                     "traffic": measured_traffic("lookup:k_draft", (P, L) == (512, 4096))[0],
                     "traffic_source": measured_traffic("lookup:k_draft", (P, L) == (512, 4096))[1],
                     "bytes_per_query": alg / n},
        "gpu_launches": 1, "clocks": clocks,
    }, data


def cpu_similarity_sample(data, prompts, prefix_len):
    """The reference's algorithm (oracle restatement with its dict-of-grams index, tracegen.py:306-353)
    on one host core over the first `prompts` prompts of the same epoch pair."""
    from oracle import hs_oracle
    from paper_2508_18588_b200.workload import history_lists
    hl = history_lists(data)
    samples = data["truths"].shape[0] // len(hl)
    prev = {p: [t.tolist() for t, _ in hl[p]] for p in range(prompts)}
    cur = {p: [data["truths"][p * samples + i].tolist() for i in range(samples)] for p in range(prompts)}
    t0 = time.perf_counter()
    acc, total, _ = hs_oracle.token_similarity_replay_indexed(prev, cur, prefix_len)
    dt = time.perf_counter() - t0
    return {"value": total / dt, "accepted": acc,
            "sample": f"{prompts} prompts x {samples} responses (first prompts of the same epoch pair), "
                      f"dict-of-grams replay, 1 thread"}


def run_similarity(args, dist, pk):
    """token_similarity_replay (tracegen.py:306-353) of a configs[1]-sized epoch pair: every
    truth response replayed against its prompt's (D) history in one hs_similarity_replay launch."""
    import torch
    from paper_2508_18588_b200.index import GpuIndex
    from paper_2508_18588_b200.similarity import replay_against_index

    dev = torch.device("cuda", dist.local)
    torch.cuda.set_device(dev)
    wl, data = replay_setup(args, dist.rank)
    idx = GpuIndex.from_arrays(torch.from_numpy(data["hist_tokens"]).to(dev), data["resp_off"],
                               data["slot_resp_off"], data["reward_fx"])
    truths = data["truths"]
    n, L = truths.shape
    d_tok = torch.from_numpy(truths.reshape(-1).astype(np.int32)).to(dev)
    d_off = torch.arange(0, (n + 1) * L, L, dtype=torch.int64, device=dev)
    d_slot = torch.from_numpy(data["truth_slots"]).to(dev)
    plen = 3
    stream = torch.cuda.current_stream(dev)
    out = [None]

    def launch():
        out[0] = replay_against_index(idx, d_tok, d_off, d_slot, plen, stream=stream)

    ms, clocks = timed(launch, args.steps, args.warmup, dist, stream, dist.local)
    acc = int(out[0].sum().item())
    tokens = n * L
    # lower bound on search steps: every non-accepted position after the warm-up is one search
    steps = tokens - n * plen - acc
    depth = int(np.ceil(np.log2(max(2, idx.n_tokens // max(1, idx.n_slots)))))
    # response read once + the matched history continuation read once + an SA entry and a text chunk head
    # per probe
    alg = 4 * tokens + 4 * acc + steps * depth * 8
    achieved = alg / (ms / 1e3) / 1e9
    return {
        "metric": "similarity-replay tokens/sec (token_similarity_replay, prefix_len 3)",
        "value": dist.sum(tokens) / (ms / 1e3), "unit": "tokens/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{n} responses x {L} tokens vs {args.prompts} prompts x 8 (D) histories "
                               f"(s = {args.similarity})", "l2": "index + responses exceed L2"},
        "acceptance": acc / tokens, "acceptance_after_warmup": acc / max(1, tokens - n * plen),
        "roofline": {"kernel": "k_similarity_replay_isa", "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": None,
                     "note": "latency-bound dependent binary searches; bytes = 4 per response token + 4 per "
                             "accepted token + 8 per search probe (lower bound on probes)"},
        "gpu_launches": 1, "clocks": clocks,
    }, data


# ------------------------------------------------------------------ reference arm

def run_reference(args, dist):
    if dist.rank != 0:
        return None
    threads = os.cpu_count() or 1
    from paper_2508_18588_b200.workload import ReplayWorkload
    wl = ReplayWorkload(prompts=args.ref_prompts, samples=args.samples, length=args.length,
                        similarity=args.similarity, shard=0, seed=args.seed)
    data = wl.generate()
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_replay_sample(data, args.ref_prompts, threads)
        if i >= args.warmup:
            vals.append(r)
    tok = sum(r["tokens"] for r in vals)
    sec = sum(r["seconds"] for r in vals)
    value = tok / sec
    st = np.sum([r["stats"] for r in vals], axis=0)
    return {
        "impl": "reference", "metric": "rollout tokens/sec (HistoSpec replay path: ingest + draft + verify/accept, "
                                      "truth supplied)",
        "value": value, "unit": "tokens/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sec / len(vals), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic (D)-history s=%.2f, seeded" % args.similarity,
        "config": {"workload": "configs[1] shape, replay (reference algorithm on host cores)"},
        "mean_accepted_per_verify": float(st[2] / max(st[3], 1)),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------------ main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="rollout", choices=["rollout", "replay", "lookup", "similarity",
                                                                  "longtail", "cpu-plan"])
    ap.add_argument("--model", default="qwen2.5-1.5b-shape")
    ap.add_argument("--batch", type=int, default=1024, help="resident sequences per wave (rollout)")
    ap.add_argument("--prompt-len", type=int, default=256)
    ap.add_argument("--prompts", type=int, default=512)
    ap.add_argument("--samples", type=int, default=8)
    ap.add_argument("--length", type=int, default=4096)
    ap.add_argument("--similarity", type=float, default=0.7)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ref-prompts", type=int, default=96)
    ap.add_argument("--cpu-seqs", type=int, default=2)
    ap.add_argument("--cpu-tokens", type=int, default=48)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--waves", type=int, default=4, help="rollout: waves of --batch sequences per GPU (cycled)")
    ap.add_argument("--history", default="D", choices=["D", "T"], help="similarity definition (SURVEY 8(d))")
    ap.add_argument("--temperature", type=float, default=0.0, help="0: greedy verify; > 0: rejection sampling")
    ap.add_argument("--len-median", type=int, default=2048, help="longtail: median response length")
    ap.add_argument("--len-sigma", type=float, default=0.8, help="longtail: log-normal sigma of lengths")
    ap.add_argument("--similarity-sweep", default="", help="longtail: comma-separated similarities")
    ap.add_argument("--compare-waves", action="store_true", help="longtail: also time static waves")
    ap.add_argument("--kv-gb", type=float, default=120.0, help="longtail: KV-cache budget per GPU (GB)")
    ap.add_argument("--tp", type=int, default=1, choices=[1, 2], help="rollout: tensor-parallel GPUs per worker")
    ap.add_argument("--tiny-tokens", type=int, default=300, help="cpu-plan: configs[0] response length")
    ap.add_argument("--window-max", type=int, default=32, help="rollout: SpecConfig.window_max (reference default 32)")
    ap.add_argument("--migrate", action="store_true", help="longtail: intra-step straggler migration")
    ap.add_argument("--alpha-pct", type=float, default=10.0, help="longtail: migration alpha (percent)")
    ap.add_argument("--growth-sigma", type=float, default=0.25, help="longtail: epoch length-growth noise")
    ap.add_argument("--histopipe", default="makespan", choices=["makespan", "gradient"],
                    help="longtail: per-group GPU plan (gradient = the reference's plan_allocation)")
    ap.add_argument("--attention", default="tcgen05", choices=["tcgen05", "mma_sync"],
                    help="attention kernel family of the HistoSpec run (the baseline is measured with both)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        dist = Dist("gloo")
        if args.workload == "rollout":
            line = run_reference_rollout(args, dist)
        else:
            line = run_reference(args, dist)
        if line is not None:
            print(json.dumps(line), flush=True)
        dist.close()
        return

    dist = Dist("nccl")
    pk = peaks()
    if args.workload == "rollout":
        line, data = run_rollout(args, dist, pk)
    elif args.workload == "replay":
        line, data = run_replay(args, dist, pk)
    elif args.workload == "similarity":
        line, data = run_similarity(args, dist, pk)
    elif args.workload == "longtail":
        line, data = run_longtail(args, dist, pk)
    elif args.workload == "cpu-plan":
        print(json.dumps(run_cpu_plan(args, dist, pk)), flush=True)
        dist.close()
        return
    else:
        line, data = run_lookup(args, dist, pk)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        if args.workload == "replay":
            r = cpu_replay_sample(data, args.ref_prompts, threads)
            line["cpu_baseline"] = {"value": r["value"], "unit": "tokens/s", "cores": threads, "kind": "port",
                                    "sample": r["sample"]}
        elif args.workload == "similarity":
            r = cpu_similarity_sample(data, min(64, args.prompts), 3)
            line["cpu_baseline"] = {"value": r["value"], "unit": "tokens/s", "cores": 1, "kind": "port",
                                    "sample": r["sample"]}
        elif args.workload == "rollout":
            r, _ = cpu_rollout_sample(data["cfg"], args.seed, data["prompts"][:args.cpu_seqs * args.samples:
                                                                              args.samples],
                                      args.cpu_tokens, args.similarity, 8, threads)
            line["cpu_baseline"] = {"value": r["value"], "unit": "tokens/s", "cores": threads, "kind": "port",
                                    "sample": r["sample"], "nonspec_value": r["nonspec_value"],
                                    "accepted_per_verify": r["accepted_per_verify"]}
        print(json.dumps(line), flush=True)
    elif dist.rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()


def run_reference_rollout(args, dist):
    """Reference arm for the rollout metric: the CPU fp32 policy + oracle HistoSpec on the host cores."""
    if dist.rank != 0:
        return None
    from paper_2508_18588_b200.model import PRESETS
    threads = os.cpu_count() or 1
    cfg = PRESETS[args.model]
    rng = np.random.default_rng([args.seed, 1000])
    prompts = rng.integers(0, cfg.vocab, size=(args.cpu_seqs, args.prompt_len), dtype=np.int32)
    W = None
    vals = []
    for i in range(args.warmup + args.steps):
        r, W = cpu_rollout_sample(cfg, args.seed, prompts, args.cpu_tokens, args.similarity, 8, threads, W=W)
        if i >= args.warmup:
            vals.append(r)
    value = float(np.mean([r["value"] for r in vals]))
    return {
        "impl": "reference", "metric": "rollout tokens/sec (greedy HistoSpec: ingest + draft + verify forward + "
                                      "accept)",
        "value": value, "unit": "tokens/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean([r["decode_s"] for r in vals])), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic prompts, random-init weights (seed %d), (D) history s=%.2f" % (args.seed, args.similarity),
        "config": {"workload": "configs[1] %s on host cores (bounded sample)" % cfg.name},
        "mean_accepted_per_verify": float(np.mean([r["accepted_per_verify"] for r in vals])),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


if __name__ == "__main__":
    main()
