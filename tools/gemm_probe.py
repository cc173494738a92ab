"""Probe: the verify-forward GEMMs of the Qwen2.5-1.5B shape alone, per M (CUDA events; not a bench value).

  python tools/gemm_probe.py [--m 1024,2560,5110] [--reps 20] [--once]

--once runs each GEMM a single time after one warm-up (for an ncu capture of exactly those launches).
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", default="1024,2560,5110")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--once", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2508_18588_b200.model import EPI_F32, EPI_SWIGLU, QWEN25_1P5B, check, lib
    torch.cuda.set_device(0)
    cfg = QWEN25_1P5B
    L = lib()
    dev = torch.device("cuda", 0)
    d, ffn, hd_all = cfg.d_model, cfg.ffn, cfg.n_heads * cfg.head_dim
    Mmax = max(int(m) for m in args.m.split(","))
    bf = dict(dtype=torch.bfloat16, device=dev)
    x = torch.randn(Mmax, max(d, ffn), **bf) * 0.5
    w_qkv = torch.randn(cfg.qkv_dim, d, **bf) * 0.02
    w_o = torch.randn(d, hd_all, **bf) * 0.02
    w_gu = torch.randn(2 * ffn, d, **bf) * 0.02
    w_d = torch.randn(d, ffn, **bf) * 0.02
    out_bf = torch.empty(Mmax, 2 * ffn, **bf)
    out_f = torch.empty(Mmax, d, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def qkv(M, st=st):
        check(L.hm_gemm(0, x.data_ptr(), x.shape[1], w_qkv.data_ptr(), d, M, cfg.qkv_dim, d, None,
                        out_bf.data_ptr(), cfg.qkv_dim, None, 0, None, None, None, st))

    def o(M, st=st):
        check(L.hm_gemm(EPI_F32, x.data_ptr(), x.shape[1], w_o.data_ptr(), hd_all, M, d, hd_all, None, None, 0,
                        out_f.data_ptr(), d, None, None, None, st))

    def gate_up(M, st=st):
        check(L.hm_gemm(EPI_SWIGLU, x.data_ptr(), x.shape[1], w_gu.data_ptr(), d, M, 2 * ffn, d, None,
                        out_bf.data_ptr(), ffn, None, 0, None, None, None, st))

    def down(M, st=st):
        check(L.hm_gemm(EPI_F32, x.data_ptr(), x.shape[1], w_d.data_ptr(), ffn, M, d, ffn, None, None, 0,
                        out_f.data_ptr(), d, None, None, None, st))

    shapes = {"qkv": (qkv, cfg.qkv_dim, d), "o": (o, d, hd_all), "gate_up": (gate_up, 2 * ffn, d),
              "down": (down, d, ffn)}
    for m in (int(v) for v in args.m.split(",")):
        row = {"M": m}
        for name, (fn, N, K) in shapes.items():
            fn(m)
            if args.once:
                torch.cuda.synchronize()
                fn(m)
                continue
            torch.cuda.synchronize()
            # the reps as one CUDA graph (as the engine runs them): host launch cost does not enter the time
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            with torch.cuda.stream(side):
                st_c = side.cuda_stream
                with torch.cuda.graph(graph, stream=side):
                    for _ in range(args.reps):
                        fn(m, st_c)
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            graph.replay()
            e1.record()
            torch.cuda.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / args.reps
            row[name] = {"us": round(us, 2), "tflops": round(2.0 * m * N * K / us / 1e6, 1)}
        torch.cuda.synchronize()
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
