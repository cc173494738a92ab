"""Plain-PyTorch restatement of the verify-forward policy (TEST INFRASTRUCTURE ONLY).

The reference has no model, so this part is "parity unpinned"
by the reference: it restates the public Qwen2 architecture that
paper_2508_18588_b200/model.py runs on the sm_100a kernels -- RMSNorm (eps
1e-6, weight * x * rsqrt(mean(x^2)+eps)), QKV with bias, rotate-half RoPE
(theta 1e6, host float64 tables), GQA causal softmax attention, SwiGLU MLP,
tied LM head.  `emulate_bf16=True` rounds activations to bf16 at exactly the
points where the GPU path stores bf16 (normed inputs, qkv, rotated q/k, v,
attention output, SwiGLU output) so the comparison isolates accumulation
order; `emulate_bf16=False` is the plain fp32 reference.
"""

from __future__ import annotations

import math

import numpy as np
import torch


def _r(x, on):
    return x.to(torch.bfloat16).to(torch.float32) if on else x


def weights_fp32(w, device="cpu"):
    """Copy a model.Weights (bf16, any device) to fp32 tensors with split gate/up."""
    cfg = w.cfg
    out = {"embed": w.embed.float().to(device), "lm_head": w.lm_head.float().to(device),
           "final_ln": w.final_ln.float().to(device), "layers": []}
    for L in w.layers:
        wgu = L["wgu"].float().to(device)
        f = cfg.ffn
        t = wgu.view(f // 64, 2, 64, cfg.d_model)
        out["layers"].append({
            "ln1": L["ln1"].float().to(device), "wqkv": L["wqkv"].float().to(device),
            "bqkv": L["bqkv"].float().to(device), "wo": L["wo"].float().to(device),
            "ln2": L["ln2"].float().to(device), "gate": t[:, 0].reshape(f, cfg.d_model),
            "up": t[:, 1].reshape(f, cfg.d_model), "wd": L["wd"].float().to(device)})
    return out


def rope_tables(cfg, max_pos):
    half = cfg.head_dim // 2
    inv = 1.0 / (cfg.rope_theta ** (np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


def rmsnorm(x, w, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def rope(x, cos, sin):
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)


def forward_logits(cfg, W, tokens, emulate_bf16=True):
    """Causal forward over one full sequence; returns fp32 logits [T, V]."""
    dev = W["embed"].device
    tok = torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=dev)
    T = tok.numel()
    H, KVH, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    cos, sin = rope_tables(cfg, T)
    cos, sin = cos.to(dev), sin.to(dev)
    x = W["embed"][tok]
    mask = torch.full((T, T), float("-inf"), device=dev).triu(1)
    for L in W["layers"]:
        h = _r(rmsnorm(x, L["ln1"], cfg.eps), emulate_bf16)
        qkv = _r(h @ L["wqkv"].T + L["bqkv"], emulate_bf16)
        q = qkv[:, :H * hd].view(T, H, hd)
        k = qkv[:, H * hd:(H + KVH) * hd].view(T, KVH, hd)
        v = qkv[:, (H + KVH) * hd:].view(T, KVH, hd)
        q = _r(rope(q, cos[:, None, :], sin[:, None, :]), emulate_bf16)
        k = _r(rope(k, cos[:, None, :], sin[:, None, :]), emulate_bf16)
        g = H // KVH
        kk = k.repeat_interleave(g, dim=1)
        vv = v.repeat_interleave(g, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, kk) / math.sqrt(hd) + mask
        p = torch.softmax(s, dim=-1)
        o = _r(torch.einsum("hqk,khd->qhd", p, vv).reshape(T, H * hd), emulate_bf16)
        x = x + o @ L["wo"].T
        h = _r(rmsnorm(x, L["ln2"], cfg.eps), emulate_bf16)
        a = _r(torch.nn.functional.silu(h @ L["gate"].T) * (h @ L["up"].T), emulate_bf16)
        x = x + a @ L["wd"].T
    h = _r(rmsnorm(x, W["final_ln"], cfg.eps), emulate_bf16)
    return h @ W["lm_head"].T


def greedy(cfg, W, prompt, n_new, emulate_bf16=True):
    """Greedy continuation by full recomputation (slow; tiny model only)."""
    seq = list(int(t) for t in prompt)
    out = []
    for _ in range(n_new):
        logits = forward_logits(cfg, W, seq, emulate_bf16)
        nxt = int(torch.argmax(logits[-1]).item())
        out.append(nxt)
        seq.append(nxt)
    return out
