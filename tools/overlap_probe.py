"""Probe: can a KV-bound attention launch and a tensor-core-bound GEMM share the GPU by SM partition?

  python tools/overlap_probe.py [--ctx 2304] [--batch 1024]

Qwen2.5-1.5B shape, verify-block sizes from the round-1 T=4096 histogram.  For attention (layer 0,
half of the sequences) and the gate/up GEMM (half of the rows) it prints, per CTA cap, the time alone
and the time when the other kernel runs beside it on a second stream with the complementary cap.
Timing only (CUDA events); not a bench value.
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

QHIST = {1: 85016, 2: 272, 3: 351992, 4: 168, 5: 278288, 6: 64, 7: 177008, 8: 32, 9: 95296, 10: 16, 11: 42688,
         13: 15776, 15: 4952, 17: 1088, 19: 272, 21: 56, 23: 24, 25: 8, 27: 8, 29: 8, 31: 8, 33: 296}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=2304)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_2508_18588_b200.engine import RolloutEngine, profile_forward
    from paper_2508_18588_b200.model import EPI_SWIGLU, QWEN25_1P5B, Weights, check, lib
    torch.cuda.set_device(0)
    cfg = QWEN25_1P5B
    B = args.batch
    w = Weights(cfg, "cuda", seed=0)
    eng = RolloutEngine(cfg, w, n_slots=B, max_len=args.ctx + 64, device="cuda")
    vals = np.array(sorted(QHIST), dtype=np.int32)
    cnt = np.array([QHIST[v] for v in vals], dtype=np.float64)
    ql = np.random.default_rng(77).choice(vals, size=B, p=cnt / cnt.sum()).astype(np.int32)
    prof, M = profile_forward(eng, B, args.ctx, ql)
    print(json.dumps({"M": M, "full_forward_ms": {k: round(v[0], 3) for k, v in prof.items()}}), flush=True)
    L = lib()
    f = eng.fwd
    f.q.normal_(0, 1.0)
    f.h.normal_(0, 1.0)
    dev = torch.device("cuda", 0)
    i32 = dict(dtype=torch.int32, device=dev)
    # half-batch inputs: the first B/2 sequences
    Bh = B // 2
    qh = torch.as_tensor(ql[:Bh]).to(dev)
    q_off = torch.as_tensor(np.concatenate([[0], np.cumsum(ql[:Bh])[:-1]]).astype(np.int32)).to(dev)
    Mh = int(ql[:Bh].sum())
    pos0 = torch.full((Bh,), args.ctx, **i32)
    kv = torch.arange(Bh, **i32)
    work = torch.empty(int(L.hm_attention_work_size(Bh, int(ql.max()), cfg.n_heads, cfg.n_kv_heads)), **i32)
    st_a, st_g = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    check(L.hm_attention_plan(qh.data_ptr(), Bh, int(ql.max()), cfg.n_heads, cfg.n_kv_heads, work.data_ptr(),
                              st_a.cuda_stream))
    kc, vc = eng.cache.k(0).data_ptr(), eng.cache.v(0).data_ptr()
    kv_bytes = float((args.ctx + ql[:Bh]).sum()) * cfg.n_kv_heads * cfg.head_dim * 2 * 2

    def attn(s):
        check(L.hm_attention(f.q.data_ptr(), kc, vc, eng.cache.slot_stride, q_off.data_ptr(), qh.data_ptr(),
                             pos0.data_ptr(), kv.data_ptr(), Bh, int(ql.max()), cfg.n_heads, cfg.n_kv_heads,
                             cfg.head_dim, eng.cache.max_len, f.scale, f.attn.data_ptr(), work.data_ptr(), 1,
                             eng.cache.n_slots, f.max_rows, s.cuda_stream))

    gflop = 2.0 * Mh * 2 * cfg.ffn * cfg.d_model

    def gemm(s):
        check(L.hm_gemm(EPI_SWIGLU, f.h.data_ptr(), cfg.d_model, w.layers[0]["wgu"].data_ptr(), cfg.d_model, Mh,
                        2 * cfg.ffn, cfg.d_model, None, f.act.data_ptr(), cfg.ffn, None, 0, None, None, None,
                        s.cuda_stream))

    def run(jobs):
        """jobs: [(fn, stream, reps)] launched round-robin; returns per-job ms (from a common start)."""
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        ends = []
        for fn, s, n in jobs:
            s.wait_event(e0)
        for fn, s, n in jobs:
            for _ in range(n):
                fn(s)
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            ends.append(e)
        torch.cuda.synchronize()
        return [e0.elapsed_time(e) for e in ends]

    R = args.reps
    out = {"Mh": Mh, "attn_GBps": {}, "gemm_TFs": {}, "pairs": []}
    for cap in (0, 96, 74, 60, 48, 40, 32):
        check(L.hm_set_grid_caps(0, cap))
        run([(attn, st_a, 2)])
        t = run([(attn, st_a, R)])[0] / R
        out["attn_GBps"][cap] = round(kv_bytes / t / 1e6, 1)
    for cap in (0, 116, 108, 100, 88, 74):
        check(L.hm_set_grid_caps(cap, 0))
        run([(gemm, st_g, 2)])
        t = run([(gemm, st_g, R)])[0] / R
        out["gemm_TFs"][cap] = round(gflop / t / 1e9, 1)
    print(json.dumps(out), flush=True)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    for a_cap in (32, 40, 48, 60, 74):
        check(L.hm_set_grid_caps(n_sm - a_cap, a_cap))
        run([(attn, st_a, 2), (gemm, st_g, 2)])
        # attention timed while the GEMM stream stays busy for longer, and vice versa
        ta = run([(attn, st_a, R), (gemm, st_g, 4 * R)])[0] / R
        tg = run([(attn, st_a, 6 * R), (gemm, st_g, R)])[1] / R
        both = run([(attn, st_a, R), (gemm, st_g, R)])
        out["pairs"].append({"attn_cap": a_cap, "attn_GBps_shared": round(kv_bytes / ta / 1e6, 1),
                             "gemm_TFs_shared": round(gflop / tg / 1e9, 1),
                             "attn_ms": round(ta, 4), "gemm_ms": round(tg, 4),
                             "pair_ms_per_rep": round(max(both) / R, 4)})
        print(json.dumps(out["pairs"][-1]), flush=True)
    check(L.hm_set_grid_caps(0, 0))
    ta = run([(attn, st_a, R)])[0] / R
    tg = run([(gemm, st_g, R)])[0] / R
    print(json.dumps({"serial_ms_per_rep": round(ta + tg, 4), "attn_ms_full": round(ta, 4),
                      "gemm_ms_full": round(tg, 4)}), flush=True)


if __name__ == "__main__":
    main()
