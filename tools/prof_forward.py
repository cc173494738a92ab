"""Small driver for ncu captures: one Qwen2.5-1.5B-shape verify forward + one K2 lookup batch.

  python tools/prof_forward.py [--ctx 2048] [--q 5] [--batch 1024]

Prints the CUDA-event per-kernel profile (not a bench value).
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--q", type=int, default=5)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--skip-lookup", action="store_true")
    ap.add_argument("--launch-rows", type=int, default=None, help="engine-style launch rows (live count on device)")
    ap.add_argument("--launch-q", type=int, default=None, help="engine-style max rows per sequence")
    ap.add_argument("--qhist-json", default=None,
                    help="bench.py JSON line: sample per-sequence verify rows from its verify_rows_hist")
    args = ap.parse_args()
    import torch
    from paper_2508_18588_b200.engine import RolloutEngine, profile_forward
    from paper_2508_18588_b200.model import QWEN25_1P5B, Weights
    torch.cuda.set_device(0)
    w = Weights(QWEN25_1P5B, "cuda", seed=0)
    eng = RolloutEngine(QWEN25_1P5B, w, n_slots=args.batch, max_len=args.ctx + 64, device="cuda")
    q = args.q
    if args.qhist_json:
        h = json.load(open(args.qhist_json))["verify_rows_hist"]
        vals = np.array([int(k) for k in h], dtype=np.int32)
        cnt = np.array([h[k] for k in h], dtype=np.float64)
        q = np.random.default_rng(77).choice(vals, size=args.batch, p=cnt / cnt.sum())
    prof, M = profile_forward(eng, args.batch, args.ctx, q, launch_rows=args.launch_rows, launch_q=args.launch_q)
    print(json.dumps({"M": M, "ctx": args.ctx, "kernels": {k: v[0] for k, v in prof.items()}}))
    if not args.skip_lookup:
        import ctypes
        from paper_2508_18588_b200 import _lib
        from paper_2508_18588_b200.index import GpuIndex
        from paper_2508_18588_b200.workload import ReplayWorkload
        data = ReplayWorkload(prompts=128).generate()
        idx = GpuIndex.from_arrays(torch.from_numpy(data["hist_tokens"]).cuda(), data["resp_off"],
                                   data["slot_resp_off"], data["reward_fx"])
        flat = torch.from_numpy(data["truths"][::8].reshape(-1).astype(np.int32)).cuda()
        m, L = 7, 4096
        n = flat.numel() - m
        i32 = dict(dtype=torch.int32, device="cuda")
        slot = (torch.arange(n, device="cuda") // L).to(torch.int32)
        args_ = [torch.full((n,), m, **i32), torch.full((n,), m, **i32), torch.full((n,), 32, **i32),
                 torch.ones(n, dtype=torch.uint8, device="cuda")]
        out = torch.empty((n, 32), **i32)
        dl = torch.empty(n, **i32)
        lk = torch.empty(n, dtype=torch.uint8, device="cuda")
        fd = torch.empty(n, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            _lib.check(_lib.load().hs_draft(ctypes.byref(idx.view), n, slot.data_ptr(), flat.data_ptr(), 1,
                                            args_[0].data_ptr(), args_[1].data_ptr(), args_[2].data_ptr(),
                                            args_[3].data_ptr(), m, m, 32, out.data_ptr(), 32, dl.data_ptr(),
                                            lk.data_ptr(), fd.data_ptr(), torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        print(json.dumps({"lookup_queries": n, "hits": int(fd.sum())}))


if __name__ == "__main__":
    main()
