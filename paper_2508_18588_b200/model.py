"""Qwen2-style policy for the verify forward, running on the libhsmodel.so kernels.

The reference has no model; this is the "policy" whose greedy
argmax is the truth that HistoSpec drafts are verified against
(SURVEY.md 8(a) a15).  Shapes follow public Qwen2.5 configs; weights are
random-init (seeded) because there is no network for checkpoints.

Forward (M rows = all live sequences' verify rows):
  embed -> L x [RMSNorm -> QKV GEMM(+bias) -> RoPE + KV append -> attention
  -> O GEMM (+= residual) -> RMSNorm -> gate/up GEMM with SwiGLU epilogue
  -> down GEMM (+= residual)] -> RMSNorm -> LM head GEMM with argmax epilogue.
Residual stream bf16 (fp32 optional, Forward(residual=...)); GEMM operands bf16; accumulators fp32 (TMEM).
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib

LIB_PATH = os.path.join(_lib.PKG, "libhsmodel.so")
_P, _I32, _I64, _F32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
SIGNATURES = {
    "hm_last_error": None,
    "hm_launch_count": None,
    "hm_gemm": [_I32, _P, _I64, _P, _I64, _I32, _I32, _I32, _P, _P, _I64, _P, _I64, _P, _P, _P, _P],
    "hm_argmax_reduce": [_P, _P, _I32, _I32, _P, _P, _P],
    "hm_gemm_bn": [_I32],
    "hm_lm_head_sample": [_P, _I64, _P, _I64, _I32, _I32, _I32, _P, _P, ctypes.c_uint64, _F32, _P, _P, _P, _P],
    "hm_embed": [_P, _P, _I32, _I32, _P, _P, _P],
    "hm_rmsnorm": [_P, _P, _I32, _I32, _F32, _P, _P, _P],
    "hm_rmsnorm_residual": [_P, _P, _P, _I32, _I32, _F32, _P, _P, _P],
    "hm_rope_kv_append": [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _I64, _I32, _P, _P],
    "hm_gemm_qkv_rope": [_P, _I64, _P, _I64, _I32, _I32, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P,
                         _I64, _I32, _P, _P],
    "hm_attention": [_P, _P, _P, _I64, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _F32, _P, _P, _I32, _I32,
                     _I32, _P],
    "hm_attention_plan": [_P, _I32, _I32, _I32, _I32, _P, _P],
    "hm_attention_work_size": [_I32, _I32, _I32, _I32],
    "hm_set_attention_family": [_I32],
    "hm_set_grid_caps": [_I32, _I32],
    "hm_set_gemm_pair": [_I32],
    "hm_rmsnorm_residual2": [_P, _P, _P, _P, _I32, _I32, _F32, _P, _P, _P],
    "hm_tp_barrier": [_P, _P, _P, _P],
    "hm_rmsnorm_residual_bf16": [_P, _P, _P, _P, _I32, _I32, _F32, _P, _P, _P],
    "hm_embed_bf16": [_P, _P, _I32, _I32, _P, _P, _P],
    "hm_f32_gemm": [_P, _I64, _P, _I64, _I32, _I32, _I32, _P, _P, _I64, _I32, _P],
    "hm_f32_rmsnorm": [_P, _P, _I32, _I32, _F32, _P, _P],
    "hm_f32_rope_kv_append": [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _I64, _I32, _P],
    "hm_f32_attention": [_P, _P, _P, _I64, _P, _P, _I32, _I32, _I32, _I32, _I32, _F32, _P, _P],
    "hm_f32_swiglu": [_P, _I32, _I32, _I32, _P, _P],
    "hm_attention_family": [],
    "hm_build_verify_batch": [_I32, _P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                              _I32, _P, _P, _P],
}
EPI_STORE, EPI_SWIGLU, EPI_RESIDUAL, EPI_ARGMAX, EPI_F32 = 0, 1, 2, 3, 4

_lib_model = None
_lock = threading.Lock()


ATTENTION_FAMILIES = {"mma_sync": 0, "tcgen05": 1}


def set_attention_family(name: str):
    """Select the attention kernel family for the forwards that follow (process-wide; see hsmodel.h)."""
    check(lib().hm_set_attention_family(ATTENTION_FAMILIES[name]))


def attention_family() -> str:
    return {v: k for k, v in ATTENTION_FAMILIES.items()}[lib().hm_attention_family()]


def lib():
    global _lib_model
    with _lock:
        if _lib_model is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} missing: build with `python -m paper_2508_18588_b200.build_ext`")
            L = ctypes.CDLL(LIB_PATH)
            for name, argt in SIGNATURES.items():
                fn = getattr(L, name)
                if name == "hm_last_error":
                    fn.restype, fn.argtypes = ctypes.c_char_p, []
                elif name in ("hm_launch_count", "hm_attention_work_size"):
                    fn.restype, fn.argtypes = ctypes.c_int64, argt or []
                else:
                    fn.restype, fn.argtypes = ctypes.c_int, argt
            _lib_model = L
    return _lib_model


def check(rc):
    if rc != 0:
        msg = lib().hm_last_error().decode(errors="replace")
        raise (ValueError if rc == -1 else RuntimeError)(f"hsmodel error {rc}: {msg}")


@dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    tied: bool
    rope_theta: float = 1e6
    eps: float = 1e-6
    init_std: float = 0.02

    @property
    def qkv_dim(self):
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def kv_bytes_per_token(self):
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2

    def param_count(self):
        d, L = self.d_model, self.n_layers
        body = L * (self.qkv_dim * d + self.qkv_dim + d * self.n_heads * self.head_dim + 3 * d * self.ffn + 2 * d) + d
        emb = self.vocab * d * (1 if self.tied else 2)
        return body + emb

    def body_params(self):
        return self.param_count() - self.vocab * self.d_model * (1 if self.tied else 2)


TINY = ModelConfig("tiny-2L-d256", 2, 256, 4, 4, 64, 1024, 4096, True)
QWEN25_1P5B = ModelConfig("qwen2.5-1.5b-shape", 28, 1536, 12, 2, 128, 8960, 151936, True)
QWEN25_7B = ModelConfig("qwen2.5-7b-shape", 28, 3584, 28, 4, 128, 18944, 152064, False)
QWEN25_32B = ModelConfig("qwen2.5-32b-shape", 64, 5120, 40, 8, 128, 27648, 152064, False)
PRESETS = {c.name: c for c in (TINY, QWEN25_1P5B, QWEN25_7B, QWEN25_32B)}


def tp_local_config(cfg: ModelConfig, tp_size: int) -> ModelConfig:
    """One GPU's share of a tensor-parallel group: q / kv heads and FFN columns split evenly (Megatron-style
    column-parallel QKV and gate/up, row-parallel O and down); embeddings, norms and the LM head replicated."""
    if tp_size == 1:
        return cfg
    if cfg.n_heads % tp_size or cfg.n_kv_heads % tp_size or cfg.ffn % (tp_size * 128):
        raise ValueError(f"{cfg.name}: heads, kv heads and ffn/128 must divide by tp={tp_size}")
    import dataclasses
    return dataclasses.replace(cfg, name=f"{cfg.name}-tp{tp_size}", n_heads=cfg.n_heads // tp_size,
                               n_kv_heads=cfg.n_kv_heads // tp_size, ffn=cfg.ffn // tp_size)


def gemm_bn(n: int) -> int:
    """Mirror of hm_gemm_bn: GEMM tile width for an output width n (function of n only)."""
    return 256 if n >= 1536 else 128


def swiglu_half(ffn: int) -> int:
    """Gate/up interleave granularity of the fused SwiGLU GEMM (half its N tile)."""
    return gemm_bn(2 * ffn) // 2


def interleave_gate_up(gate, up, tile=None):
    """[ffn, d] x 2 -> [2*ffn, d] with gate/up halves of `tile` rows per GEMM N tile."""
    import torch
    f, d = gate.shape
    tile = swiglu_half(f) if tile is None else tile
    g = gate.view(f // tile, tile, d)
    u = up.view(f // tile, tile, d)
    return torch.stack([g, u], dim=1).reshape(2 * f, d).contiguous()


class Weights:
    """Random-init bf16 weights on `device` (seeded, generated on the device)."""

    def __init__(self, cfg: ModelConfig, device, seed: int = 0, keep_fp32_split: bool = False, tp_rank: int = 0,
                 tp_size: int = 1):
        """tp_size > 1: this GPU's shard of the same seeded weights (the full tensors are generated in the
        TP=1 order, one layer at a time, and sliced); `cfg` becomes the local shape, `global_cfg` the model."""
        import torch
        self.global_cfg = cfg
        self.tp_rank, self.tp_size = tp_rank, tp_size
        cfg_l = tp_local_config(cfg, tp_size)
        self.cfg = cfg_l
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        std = cfg.init_std

        def rnd(*shape):
            return (torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * std).to(torch.bfloat16)

        d, hd = cfg.d_model, cfg.head_dim
        self.embed = rnd(cfg.vocab, d)
        self.lm_head = self.embed if cfg.tied else rnd(cfg.vocab, d)
        self.layers = []
        t = tp_rank
        Hq, Hk, F = cfg_l.n_heads * hd, cfg_l.n_kv_heads * hd, cfg_l.ffn

        def qkv_rows(a):   # this rank's q heads, k heads, v heads (column-parallel QKV)
            if tp_size == 1:
                return a
            q0, k0, v0 = 0, cfg.n_heads * hd, (cfg.n_heads + cfg.n_kv_heads) * hd
            return torch.cat([a[q0 + t * Hq:q0 + (t + 1) * Hq], a[k0 + t * Hk:k0 + (t + 1) * Hk],
                              a[v0 + t * Hk:v0 + (t + 1) * Hk]]).contiguous()

        def cols(a, n):    # this rank's slice of the K dimension (row-parallel O / down)
            return a if tp_size == 1 else a[:, t * n:(t + 1) * n].contiguous()

        def rows(a, n):
            return a if tp_size == 1 else a[t * n:(t + 1) * n].contiguous()

        for _ in range(cfg.n_layers):
            gate, up = rnd(cfg.ffn, d), rnd(cfg.ffn, d)
            gate, up = rows(gate, F), rows(up, F)
            layer = {
                "ln1": torch.ones(d, dtype=torch.bfloat16, device=device),
                "wqkv": qkv_rows(rnd(cfg.qkv_dim, d)),
                "bqkv": qkv_rows(rnd(cfg.qkv_dim)),
                "wo": cols(rnd(d, cfg.n_heads * hd), Hq),
                "ln2": torch.ones(d, dtype=torch.bfloat16, device=device),
                "wgu": interleave_gate_up(gate, up),
                "wd": cols(rnd(d, cfg.ffn), F),
            }
            if keep_fp32_split:
                layer["gate"], layer["up"] = gate, up
            self.layers.append(layer)
        self.final_ln = torch.ones(d, dtype=torch.bfloat16, device=device)
        self._flatten()
        half = hd // 2
        inv = 1.0 / (cfg.rope_theta ** (np.arange(half, dtype=np.float64) * 2.0 / hd))
        self._inv_freq = inv

    def tensors(self):
        """Every weight tensor, in a fixed order (the tied LM head once)."""
        out = [self.embed] + ([] if self.cfg.tied else [self.lm_head]) + [self.final_ln]
        for layer in self.layers:
            out += [layer[k] for k in ("ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wd")]
        return out

    def _flatten(self):
        """Re-home every weight in one contiguous bf16 buffer (`self.flat`), each tensor a 256-byte-aligned view,
        so the epoch-boundary policy broadcast is one NCCL call (workers.broadcast_weights)."""
        import torch
        ts = self.tensors()
        offs, n = [], 0
        for t in ts:
            offs.append(n)
            n += (t.numel() + 127) // 128 * 128
        flat = torch.empty(n, dtype=torch.bfloat16, device=ts[0].device)
        views = []
        for t, o in zip(ts, offs):
            v = flat[o:o + t.numel()].view(t.shape)
            v.copy_(t)
            views.append(v)
        it = iter(views)
        self.embed = next(it)
        self.lm_head = self.embed if self.cfg.tied else next(it)
        self.final_ln = next(it)
        for layer in self.layers:
            for k in ("ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wd"):
                layer[k] = next(it)
        self.flat = flat

    def rope_tables(self, max_pos, device):
        """cos/sin [max_pos, hd/2] fp32, computed in float64 on the host (same table for every backend)."""
        import torch
        ang = np.arange(max_pos, dtype=np.float64)[:, None] * self._inv_freq[None, :]
        return (torch.from_numpy(np.cos(ang).astype(np.float32)).to(device),
                torch.from_numpy(np.sin(ang).astype(np.float32)).to(device))

    def nbytes(self):
        n = self.embed.numel() * 2 + (0 if self.cfg.tied else self.lm_head.numel() * 2)
        for L in self.layers:
            n += sum(t.numel() * 2 for k, t in L.items() if k not in ("gate", "up"))
        return n


class KVCache:
    """Slot-contiguous KV cache: [layers][k|v][slot][kv_head][pos][head_dim] bf16 (zero-initialized)."""

    def __init__(self, cfg: ModelConfig, n_slots: int, max_len: int, device):
        import torch
        self.cfg, self.n_slots, self.max_len = cfg, n_slots, max_len
        self.buf = torch.zeros((cfg.n_layers, 2, n_slots, cfg.n_kv_heads, max_len, cfg.head_dim),
                               dtype=torch.bfloat16, device=device)
        self.slot_stride = cfg.n_kv_heads * max_len * cfg.head_dim

    def k(self, layer):
        return self.buf[layer, 0]

    def v(self, layer):
        return self.buf[layer, 1]


class Forward:
    """Preallocated activations for up to max_rows verify rows; runs the forward."""

    def __init__(self, w: Weights, cache: KVCache, max_rows: int, device, residual: str | None = None):
        """residual: "bf16" (default; HM_RESIDUAL=fp32 in the environment changes it) keeps the residual stream
        x and the O / down projection outputs y in bf16, the precision bf16 inference keeps them in; "fp32"
        keeps both in fp32 (round 1's layout: 2x the bytes through every norm)."""
        import torch
        cfg = w.cfg
        self.w, self.cache, self.cfg, self.max_rows, self.device = w, cache, cfg, max_rows, device
        M, d = max_rows, cfg.d_model
        bf = dict(dtype=torch.bfloat16, device=device)
        self.residual = residual or os.environ.get("HM_RESIDUAL", "bf16")
        if self.residual not in ("bf16", "fp32"):
            raise ValueError(f"residual must be 'bf16' or 'fp32', got {self.residual!r}")
        rdt = torch.bfloat16 if self.residual == "bf16" else torch.float32
        self.x = torch.empty((M, d), dtype=rdt, device=device)
        self.y = torch.empty((M, d), dtype=rdt, device=device)   # O/down-proj output, added in the norm
        self.h = torch.empty((M, d), **bf)
        self.qkv = torch.empty((M, cfg.qkv_dim), **bf)
        self.q = torch.empty((M, cfg.n_heads, cfg.head_dim), **bf)   # used as [KVH][rows][G][hd] (hm_rope_kv_append)
        self.attn = torch.empty((M, cfg.n_heads * cfg.head_dim), **bf)
        self.act = torch.empty((M, cfg.ffn), **bf)
        self.n_tiles = cfg.vocab // 128
        self.amax_val = torch.empty((M, self.n_tiles), dtype=torch.float32, device=device)
        self.amax_idx = torch.empty((M, self.n_tiles), dtype=torch.int32, device=device)
        self.argmax = torch.empty(M, dtype=torch.int32, device=device)
        # attention work list (tile prefix + tile -> sequence map), grown on demand outside graph capture
        self.attn_work = torch.empty(2 * M + 2, dtype=torch.int32, device=device)
        self.cos, self.sin = w.rope_tables(cache.max_len + 64, device)
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        self.temperature = 0.0   # 0 = greedy argmax; > 0 = Gumbel-max sampling (hm_lm_head_sample)
        self.fused_qkv_rope = True   # False: hm_gemm + hm_rope_kv_append (tests compare the two)
        # True: the O and down projections add into the residual stream in their epilogues (HM_EPI_RESIDUAL)
        # and the norms that follow read x alone; False: they store fp32 and the next norm adds (same bits)
        self.residual_in_gemm = os.environ.get("HM_RESIDUAL_IN_GEMM", "0") == "1"
        self.seed = 0
        self.tp = None   # tp.TensorParallel: O / down partials all-reduced over peer memory (set by the engine)

    def run(self, M, tokens, pos, row_slot, q_off, q_len, pos0, kv_slot, n_seq, max_q_len, stream=None, m_dev=None,
            logits_out=None, prof=None, row_key=None):
        """Full forward over M rows; returns self.argmax[:M] (int32 next-token ids).

        `logits_out` (bf16 [M, V], optional, tests only) also receives the LM-head logits.
        `row_key` (int32 [M], optional): per-row sampling key (default: the row's KV slot).
        """
        import torch
        if M > self.max_rows:
            raise ValueError(f"{M} rows > max_rows {self.max_rows}")
        L = lib()
        cfg, w = self.cfg, self.w
        need = L.hm_attention_work_size(n_seq, max_q_len, cfg.n_heads, cfg.n_kv_heads)
        if need > self.attn_work.numel():
            if torch.cuda.is_current_stream_capturing():
                raise ValueError(f"attention work list needs {need} entries: run once before capturing")
            self.attn_work = torch.empty(need, dtype=torch.int32, device=self.device)
        s_obj = stream or torch.cuda.current_stream(self.device)
        st = s_obj.cuda_stream
        mp = m_dev.data_ptr() if m_dev is not None else None
        d = cfg.d_model

        def k(label, rc_fn):
            # prof: list collecting (label, start, end) CUDA events around each launch
            if prof is None:
                check(rc_fn())
                return
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s_obj)
            check(rc_fn())
            e1.record(s_obj)
            prof.append((label, e0, e1))

        r16 = self.residual == "bf16"
        if r16 and self.residual_in_gemm:
            raise ValueError("residual_in_gemm is an fp32-residual option")
        if r16:
            k("embed", lambda: L.hm_embed_bf16(tokens.data_ptr(), w.embed.data_ptr(), M, d, self.x.data_ptr(), mp, st))
        else:
            k("embed", lambda: L.hm_embed(tokens.data_ptr(), w.embed.data_ptr(), M, d, self.x.data_ptr(), mp, st))
        hd_all = cfg.n_heads * cfg.head_dim
        y = self.y.data_ptr()
        k("attn_plan", lambda: L.hm_attention_plan(q_len.data_ptr(), n_seq, max_q_len, cfg.n_heads, cfg.n_kv_heads,
                                                   self.attn_work.data_ptr(), st))
        tp = self.tp
        if tp is not None and self.residual_in_gemm:
            raise ValueError("tensor parallelism needs the O / down partials in fp32 buffers (residual_in_gemm off)")

        def norm(yb, wt):
            # x += y (the previous O / down projection; with TP, y = both GPUs' partials), h = rmsnorm(x)
            if r16:
                if tp is None:
                    loc, peer = yb, None
                else:
                    loc, peer = (None, None) if yb is None else (tp.y[yb].data_ptr(), tp.y_peer[yb].data_ptr())
                k("rmsnorm", lambda: L.hm_rmsnorm_residual_bf16(self.x.data_ptr(), loc, peer, wt, M, d, cfg.eps,
                                                                self.h.data_ptr(), mp, st))
            elif tp is None:   # (hm_rmsnorm_residual2 without a second partial: the d <= 4096 kernel or any-d one)
                k("rmsnorm", lambda: L.hm_rmsnorm_residual2(self.x.data_ptr(), yb, None, wt, M, d, cfg.eps,
                                                            self.h.data_ptr(), mp, st))
            else:
                loc, peer = (None, None) if yb is None else (tp.y[yb].data_ptr(), tp.y_peer[yb].data_ptr())
                k("rmsnorm", lambda: L.hm_rmsnorm_residual2(self.x.data_ptr(), loc, peer, wt, M, d, cfg.eps,
                                                            self.h.data_ptr(), mp, st))

        def y_out(b):   # where the O (b = 0) / down (b = 1) projection writes its fp32 (partial) output
            return y if tp is None else tp.y[b].data_ptr()

        def allreduce_sync():
            if tp is not None:
                k("tp_barrier", lambda: tp.barrier(s_obj) or 0)

        for li, layer in enumerate(w.layers):
            kc, vc = self.cache.k(li).data_ptr(), self.cache.v(li).data_ptr()
            if li == 0 or self.residual_in_gemm:
                norm(None, layer["ln1"].data_ptr())
            else:
                norm(y if tp is None else 1, layer["ln1"].data_ptr())
            if self.fused_qkv_rope:   # QKV projection, RoPE and the KV append in one kernel (same bits)
                k("gemm_qkv", lambda: L.hm_gemm_qkv_rope(
                    self.h.data_ptr(), d, layer["wqkv"].data_ptr(), d, M, d, layer["bqkv"].data_ptr(), cfg.n_heads,
                    cfg.n_kv_heads, cfg.head_dim, pos.data_ptr(), row_slot.data_ptr(), self.cos.data_ptr(),
                    self.sin.data_ptr(), self.q.data_ptr(), M, kc, vc, self.cache.slot_stride, self.cache.max_len,
                    mp, st))
            else:
                k("gemm_qkv", lambda: L.hm_gemm(EPI_STORE, self.h.data_ptr(), d, layer["wqkv"].data_ptr(), d, M,
                                                cfg.qkv_dim, d, layer["bqkv"].data_ptr(), self.qkv.data_ptr(),
                                                cfg.qkv_dim, None, 0, None, None, mp, st))
                k("rope_kv", lambda: L.hm_rope_kv_append(self.qkv.data_ptr(), pos.data_ptr(), row_slot.data_ptr(),
                                                         self.cos.data_ptr(), self.sin.data_ptr(), M, cfg.n_heads,
                                                         cfg.n_kv_heads, cfg.head_dim, self.q.data_ptr(), kc, vc,
                                                         self.cache.slot_stride, self.cache.max_len, mp, st))
            k("attention", lambda: L.hm_attention(self.q.data_ptr(), kc, vc, self.cache.slot_stride,
                                                  q_off.data_ptr(), q_len.data_ptr(), pos0.data_ptr(),
                                                  kv_slot.data_ptr(), n_seq, max_q_len, cfg.n_heads,
                                                  cfg.n_kv_heads, cfg.head_dim, self.cache.max_len, self.scale,
                                                  self.attn.data_ptr(), self.attn_work.data_ptr(), 1,
                                                  self.cache.n_slots, M, st))
            epi_r = EPI_RESIDUAL if self.residual_in_gemm else EPI_F32
            y_o = self.x.data_ptr() if self.residual_in_gemm else y_out(0)
            if r16:   # the projection stored in bf16 (EPI_STORE) for the bf16 residual add in the norm
                k("gemm_o", lambda: L.hm_gemm(EPI_STORE, self.attn.data_ptr(), hd_all, layer["wo"].data_ptr(), hd_all,
                                              M, d, hd_all, None, y_o, d, None, 0, None, None, mp, st))
            else:
                k("gemm_o", lambda: L.hm_gemm(epi_r, self.attn.data_ptr(), hd_all, layer["wo"].data_ptr(), hd_all,
                                              M, d, hd_all, None, None, 0, y_o, d, None, None, mp, st))
            allreduce_sync()
            norm(None if self.residual_in_gemm else (y if tp is None else 0), layer["ln2"].data_ptr())
            k("gemm_gate_up", lambda: L.hm_gemm(EPI_SWIGLU, self.h.data_ptr(), d, layer["wgu"].data_ptr(), d, M,
                                                2 * cfg.ffn, d, None, self.act.data_ptr(), cfg.ffn, None, 0, None,
                                                None, mp, st))
            y_d = self.x.data_ptr() if self.residual_in_gemm else y_out(1)
            if r16:
                k("gemm_down", lambda: L.hm_gemm(EPI_STORE, self.act.data_ptr(), cfg.ffn, layer["wd"].data_ptr(),
                                                 cfg.ffn, M, d, cfg.ffn, None, y_d, d, None, 0, None, None, mp, st))
            else:
                k("gemm_down", lambda: L.hm_gemm(epi_r, self.act.data_ptr(), cfg.ffn, layer["wd"].data_ptr(),
                                                 cfg.ffn, M, d, cfg.ffn, None, None, 0, y_d, d, None, None, mp, st))
            allreduce_sync()
        norm(None if self.residual_in_gemm else (y if tp is None else 1), w.final_ln.data_ptr())
        if logits_out is not None:
            check(L.hm_gemm(EPI_STORE, self.h.data_ptr(), d, w.lm_head.data_ptr(), d, M, cfg.vocab, d, None,
                            logits_out.data_ptr(), cfg.vocab, None, 0, None, None, mp, st))
        if self.temperature > 0.0:
            # rejection-sampling verify: Gumbel-max sample keyed by (seed, kv slot, position)
            k("gemm_lm_head_argmax", lambda: L.hm_lm_head_sample(
                self.h.data_ptr(), d, w.lm_head.data_ptr(), d, M, cfg.vocab, d,
                (row_key if row_key is not None else row_slot).data_ptr(), pos.data_ptr(),
                self.seed, self.temperature, self.amax_val.data_ptr(), self.amax_idx.data_ptr(), mp, st))
        else:
            k("gemm_lm_head_argmax", lambda: L.hm_gemm(EPI_ARGMAX, self.h.data_ptr(), d, w.lm_head.data_ptr(), d, M,
                                                       cfg.vocab, d, None, None, 0, None, 0,
                                                       self.amax_val.data_ptr(), self.amax_idx.data_ptr(), mp, st))
        k("argmax_reduce", lambda: L.hm_argmax_reduce(self.amax_val.data_ptr(), self.amax_idx.data_ptr(), M,
                                                      self.n_tiles, mp, self.argmax.data_ptr(), st))
        return self.argmax[:M]

    def gemm_shapes(self):
        """(label, N, K) of every GEMM in one forward (per layer ones repeated n_layers times)."""
        cfg = self.cfg
        d, hd_all = cfg.d_model, cfg.n_heads * cfg.head_dim
        return {"gemm_qkv": (cfg.qkv_dim, d), "gemm_o": (d, hd_all), "gemm_gate_up": (2 * cfg.ffn, d),
                "gemm_down": (d, cfg.ffn), "gemm_lm_head_argmax": (cfg.vocab, d)}

    def flops(self, q_rows, ctx_rows):
        """Algorithmic flops of one forward: 2*(P_body+V*d)*M + 4*L*H*hd*sum q*(ctx+(q+1)/2)."""
        cfg = self.cfg
        lin = 2 * (cfg.body_params() + cfg.vocab * cfg.d_model) * q_rows
        return lin + 4 * cfg.n_layers * cfg.n_heads * cfg.head_dim * ctx_rows


class Fp32Forward:
    """The verify forward in fp32 (tests only): fp32 operands, accumulation and KV cache.

    SURVEY.md 8(c) item 4 holds GPU logits to 1e-3 relative of an fp32
    restatement; the bf16 tcgen05 path can only meet a documented bf16 bound,
    so this twin runs the same layer sequence on the hm_f32_* SIMT kernels
    (weights: the same bf16 tensors, widened exactly).  Not on the rollout path.
    """

    def __init__(self, w: Weights, n_slots: int, max_len: int, max_rows: int, device):
        import torch
        cfg = w.cfg
        self.w, self.cfg, self.max_rows, self.max_len, self.device = w, cfg, max_rows, max_len, device
        f32 = dict(dtype=torch.float32, device=device)
        self.kv = torch.zeros((cfg.n_layers, 2, n_slots, cfg.n_kv_heads, max_len, cfg.head_dim), **f32)
        self.slot_stride = cfg.n_kv_heads * max_len * cfg.head_dim
        M, d = max_rows, cfg.d_model
        self.x = torch.empty((M, d), **f32)
        self.h = torch.empty((M, d), **f32)
        self.qkv = torch.empty((M, cfg.qkv_dim), **f32)
        self.q = torch.empty((M, cfg.n_heads * cfg.head_dim), **f32)
        self.attn = torch.empty((M, cfg.n_heads * cfg.head_dim), **f32)
        self.gu = torch.empty((M, 2 * cfg.ffn), **f32)
        self.act = torch.empty((M, cfg.ffn), **f32)
        self.cos, self.sin = w.rope_tables(max_len + 64, device)
        self.scale = 1.0 / math.sqrt(cfg.head_dim)

    def run(self, M, tokens, pos, row_slot, stream=None):
        """Rows (token, position, slot) in causal order per slot; returns fp32 logits [M, V]."""
        import torch
        if M > self.max_rows:
            raise ValueError(f"{M} rows > max_rows {self.max_rows}")
        L, cfg, w = lib(), self.cfg, self.w
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        d, hd_all = cfg.d_model, cfg.n_heads * cfg.head_dim
        check(L.hm_embed(tokens.data_ptr(), w.embed.data_ptr(), M, d, self.x.data_ptr(), None, st))
        for li, layer in enumerate(w.layers):
            kc, vc = self.kv[li, 0].data_ptr(), self.kv[li, 1].data_ptr()
            check(L.hm_f32_rmsnorm(self.x.data_ptr(), layer["ln1"].data_ptr(), M, d, cfg.eps, self.h.data_ptr(), st))
            check(L.hm_f32_gemm(self.h.data_ptr(), d, layer["wqkv"].data_ptr(), d, M, cfg.qkv_dim, d,
                                layer["bqkv"].data_ptr(), self.qkv.data_ptr(), cfg.qkv_dim, 0, st))
            check(L.hm_f32_rope_kv_append(self.qkv.data_ptr(), pos.data_ptr(), row_slot.data_ptr(),
                                          self.cos.data_ptr(), self.sin.data_ptr(), M, cfg.n_heads, cfg.n_kv_heads,
                                          cfg.head_dim, self.q.data_ptr(), kc, vc, self.slot_stride, self.max_len, st))
            check(L.hm_f32_attention(self.q.data_ptr(), kc, vc, self.slot_stride, pos.data_ptr(), row_slot.data_ptr(),
                                     M, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, self.max_len, self.scale,
                                     self.attn.data_ptr(), st))
            check(L.hm_f32_gemm(self.attn.data_ptr(), hd_all, layer["wo"].data_ptr(), hd_all, M, d, hd_all, None,
                                self.x.data_ptr(), d, 1, st))
            check(L.hm_f32_rmsnorm(self.x.data_ptr(), layer["ln2"].data_ptr(), M, d, cfg.eps, self.h.data_ptr(), st))
            check(L.hm_f32_gemm(self.h.data_ptr(), d, layer["wgu"].data_ptr(), d, M, 2 * cfg.ffn, d, None,
                                self.gu.data_ptr(), 2 * cfg.ffn, 0, st))
            check(L.hm_f32_swiglu(self.gu.data_ptr(), M, cfg.ffn, swiglu_half(cfg.ffn), self.act.data_ptr(), st))
            check(L.hm_f32_gemm(self.act.data_ptr(), cfg.ffn, layer["wd"].data_ptr(), cfg.ffn, M, d, cfg.ffn, None,
                                self.x.data_ptr(), d, 1, st))
        check(L.hm_f32_rmsnorm(self.x.data_ptr(), w.final_ln.data_ptr(), M, d, cfg.eps, self.h.data_ptr(), st))
        logits = torch.empty((M, cfg.vocab), dtype=torch.float32, device=self.device)
        check(L.hm_f32_gemm(self.h.data_ptr(), d, w.lm_head.data_ptr(), d, M, cfg.vocab, d, None, logits.data_ptr(),
                            cfg.vocab, 0, st))
        return logits
