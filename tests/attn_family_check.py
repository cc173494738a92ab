"""Checks run in a fresh process per attention kernel family (the family is chosen once per process
from HM_ATTN_MMA / HM_ATTN_W8): varlen blocks vs an fp32 reference, one-row-at-a-time invariance,
many work items per persistent CTA, and greedy-with-speculation == greedy on the tiny model.
Used by tests/test_model_gpu.py::test_attention_family_subprocess."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18588_b200.model as Mo  # noqa: E402


def _kv_major(q, KVH):
    """[rows, H, hd] -> the kernels' kv-group-major [KVH][rows][G][hd] layout (hm_rope_kv_append's)."""
    M, H, hd = q.shape
    return q.view(M, KVH, H // KVH, hd).transpose(0, 1).contiguous()



def attn(q, kc, vc, seqs, H, KVH, hd, max_len, slots, work, M):
    i32 = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
    out = torch.zeros(M, H * hd, dtype=torch.bfloat16, device="cuda")
    meta = [i32([s[j] for s in seqs]) for j in range(4)]
    Mo.check(Mo.lib().hm_attention(_kv_major(q, KVH).data_ptr(), kc.data_ptr(), vc.data_ptr(), KVH * max_len * hd,
                                   meta[0].data_ptr(), meta[1].data_ptr(), meta[2].data_ptr(), meta[3].data_ptr(),
                                   len(seqs), max(s[1] for s in seqs), H, KVH, hd, max_len, 1.0 / np.sqrt(hd),
                                   out.data_ptr(), work.data_ptr(), 0, slots, M, 0))
    torch.cuda.synchronize()
    return out.view(M, H, hd)


def main():
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(7)
    for H, KVH, hd in ((12, 2, 128), (4, 4, 64)):
        rng = np.random.default_rng(H)
        n, max_len = 300, 700
        kc = torch.randn(n, KVH, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
        vc = torch.randn(n, KVH, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
        q_len = rng.integers(1, 34, size=n)
        q_off = np.concatenate([[0], np.cumsum(q_len)[:-1]])
        pos0 = rng.integers(0, max_len - 34, size=n)
        M = int(q_len.sum())
        q = torch.randn(M, H, hd, device="cuda", generator=g).to(torch.bfloat16)
        work = torch.empty(2 * M + 2, dtype=torch.int32, device="cuda")   # >= hm_attention_work_size
        seqs = [(int(q_off[s]), int(q_len[s]), int(pos0[s]), s) for s in range(n)]
        out = attn(q, kc, vc, seqs, H, KVH, hd, max_len, n, work, M)
        # fp32 reference on a sample of rows
        for s in range(0, n, 37):
            for i in range(int(q_len[s])):
                r, pos = int(q_off[s]) + i, int(pos0[s]) + i
                for h in range(H):
                    kh = h // (H // KVH)
                    sc = (kc[s, kh, :pos + 1].float() @ q[r, h].float()) / np.sqrt(hd)
                    ref = torch.softmax(sc, 0) @ vc[s, kh, :pos + 1].float()
                    assert torch.allclose(out[r, h].float(), ref, atol=2e-2, rtol=2e-2), (H, s, i, h)
        # every row again as its own decode query: bit-identical
        seq_of_row = np.repeat(np.arange(n), q_len)
        rows = [(r, 1, int(pos0[seq_of_row[r]] + r - q_off[seq_of_row[r]]), int(seq_of_row[r])) for r in range(M)]
        dec = attn(q, kc, vc, rows, H, KVH, hd, max_len, n, work, M)
        assert torch.equal(out, dec), (H, "decode rows differ from their verify blocks")
    from paper_2508_18588_b200.engine import smoke
    smoke()   # greedy with speculation == greedy, bit for bit
    print("OK")


if __name__ == "__main__":
    main()
