"""Per-stage pipeline timestamps of the tcgen05 attention kernel (CTA 0), decode or verify shape.
Needs libhsmodel.so built with -DHM_TC_TRACE (debugging aid)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_18588_b200.model as Mo


def _kv_major(q, KVH):
    """[rows, H, hd] -> the kernels' kv-group-major [KVH][rows][G][hd] layout (hm_rope_kv_append's)."""
    M, H, hd = q.shape
    return q.view(M, KVH, H // KVH, hd).transpose(0, 1).contiguous()

torch.cuda.set_device(0)
q_rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1
H, KVH, hd = 12, 2, 128
n, max_len, ctx = 1024, 2400, 2304
kc = torch.randn(n, KVH, max_len, hd, device="cuda").to(torch.bfloat16)
vc = torch.randn(n, KVH, max_len, hd, device="cuda").to(torch.bfloat16)
ql = np.full(n, q_rows, np.int32)
qo = (np.arange(n) * q_rows).astype(np.int32)
p0 = np.full(n, ctx, np.int32)
M = int(ql.sum())
q = torch.randn(M, H, hd, device="cuda").to(torch.bfloat16)
out = torch.empty(M, H * hd, dtype=torch.bfloat16, device="cuda")
work = torch.empty(3 * n + 2, dtype=torch.int32, device="cuda")
i32 = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int32)).cuda()
meta = [i32(qo), i32(ql), i32(p0), i32(np.arange(n))]
L = Mo.lib()
for _ in range(3):
    Mo.check(L.hm_attention(_kv_major(q, KVH).data_ptr(), kc.data_ptr(), vc.data_ptr(), KVH * max_len * hd, meta[0].data_ptr(),
                            meta[1].data_ptr(), meta[2].data_ptr(), meta[3].data_ptr(), n, q_rows, H, KVH, hd,
                            max_len, 1.0 / np.sqrt(hd), out.data_ptr(), work.data_ptr(), 0, n, M, 0))
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (16 * 512))()
f = L.hm_debug_attn_trace
f.argtypes = [ctypes.c_void_p]
print("rc", f(ctypes.addressof(buf)))
t = np.frombuffer(buf, dtype=np.int64).reshape(16, 512).astype(np.float64)
t0 = t[0, 0]
names = ["S issued", "p_full seen", "softmax S ready", "softmax P done", "K ready", "V ready"]
for gs in list(range(0, 6)) + list(range(34, 42)) + list(range(100, 106)):
    print(gs, " ".join("%s=%7.0f" % (names[e][:10], t[e, gs] - t0) for e in range(6)))
d = np.diff(t[3, 40:200])
print("softmax P-done period: median %.0f cycles" % np.median(d[d > 0]))
for e in range(6):
    x = np.diff(t[e, 40:200]); x = x[x > 0]
    print(names[e], "period median", np.median(x))
print("lag S-issued -> softmax ready (median)", np.median((t[2] - t[0])[40:200]))
print("lag softmax ready -> P done (median)", np.median((t[3] - t[2])[40:200]))
print("lag P done -> p_full seen by MMA (median)", np.median((t[1] - t[3])[40:200]))
print("lag p_full seen -> V ready (median)", np.median((t[5] - t[1])[40:200]))
ep0, ep1 = t[6, :16] - t0, t[7, :16] - t0
print("epilogue start/end per item:", " ".join("%.0f/%.0f" % (a, b) for a, b in zip(ep0, ep1)))
print("epilogue duration median", np.median((t[7] - t[6])[1:12]))
inames = {8: "s0 top", 9: "s0 info", 10: "s0 q_ready", 6: "s0 o_ready", 11: "s0 l_ready", 7: "s0 o_free",
          12: "s1 top", 13: "s1 stages done", 14: "K cursor enters", 15: "MMA q_full"}
for it in range(1, 5):
    print("item", it, " ".join("%s=%.0f" % (n, t[e, it] - t0) for e, n in sorted(inames.items(), key=lambda x: t[x[0], it])))
nst = int(sys.argv[2]) if len(sys.argv) > 2 else 19
for gs in range(nst - 2, 2 * nst + 3):
    print(gs, " ".join("%s=%7.0f" % (names[e][:10], t[e, gs] - t0) for e in range(6)))
