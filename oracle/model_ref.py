"""Plain-PyTorch restatement of the verify-forward policy (TEST INFRASTRUCTURE ONLY).

The reference has no model, so this part is "parity unpinned"
by the reference: it restates the public Qwen2 architecture that
paper_2508_18588_b200/model.py runs on the sm_100a kernels -- RMSNorm (eps
1e-6, weight * x * rsqrt(mean(x^2)+eps)), QKV with bias, rotate-half RoPE
(theta 1e6, host float64 tables), GQA causal softmax attention, SwiGLU MLP,
tied LM head.  `emulate_bf16=True` rounds activations to bf16 at exactly the
points where the GPU path stores bf16 (residual stream and projection outputs, normed inputs, qkv, rotated q/k, v,
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
    from paper_2508_18588_b200.model import swiglu_half
    cfg = w.cfg
    out = {"embed": w.embed.float().to(device), "lm_head": w.lm_head.float().to(device),
           "final_ln": w.final_ln.float().to(device), "layers": []}
    half = swiglu_half(cfg.ffn)
    for L in w.layers:
        wgu = L["wgu"].float().to(device)
        f = cfg.ffn
        t = wgu.view(f // half, 2, half, cfg.d_model)
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
        # the GPU path's default bf16 residual stream: projection rounded to bf16, sum rounded to bf16
        x = _r(x + _r(o @ L["wo"].T, emulate_bf16), emulate_bf16)
        h = _r(rmsnorm(x, L["ln2"], cfg.eps), emulate_bf16)
        a = _r(torch.nn.functional.silu(h @ L["gate"].T) * (h @ L["up"].T), emulate_bf16)
        x = _r(x + _r(a @ L["wd"].T, emulate_bf16), emulate_bf16)
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


class CpuRollout:
    """fp32 CPU rollout of the same policy with HistoSpec drafting (the CPU baseline / reference arm).

    KV-cached incremental forward (all host threads via torch), drafts from
    the C oracle (`hs_oracle_c.draft`, brute-force scan of the prompt's
    history = history.py:302-333 semantics), accept = spec_engine.py:217-240.
    """

    def __init__(self, cfg, W, max_len):
        self.cfg, self.W, self.max_len = cfg, W, max_len
        self.cos, self.sin = rope_tables(cfg, max_len + 64)

    def _forward(self, caches, blocks):
        """blocks: list of (seq, tokens, start_pos); returns argmax per row, per block."""
        cfg, W = self.cfg, self.W
        H, KVH, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        toks = torch.as_tensor(np.concatenate([np.asarray(t, dtype=np.int64) for _, t, _ in blocks]))
        pos = np.concatenate([np.arange(p0, p0 + len(t)) for _, t, p0 in blocks])
        cos, sin = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        x = W["embed"][toks]
        n = x.shape[0]
        for li, L in enumerate(W["layers"]):
            h = rmsnorm(x, L["ln1"], cfg.eps)
            qkv = h @ L["wqkv"].T + L["bqkv"]
            q = rope(qkv[:, :H * hd].view(n, H, hd), cos, sin)
            k = rope(qkv[:, H * hd:(H + KVH) * hd].view(n, KVH, hd), cos, sin)
            v = qkv[:, (H + KVH) * hd:].view(n, KVH, hd)
            outs, r = [], 0
            for s, t, p0 in blocks:
                m = len(t)
                K, V = caches[s][li]
                K[:, p0:p0 + m] = k[r:r + m].transpose(0, 1)
                V[:, p0:p0 + m] = v[r:r + m].transpose(0, 1)
                kk = K[:, :p0 + m].repeat_interleave(H // KVH, 0)
                vv = V[:, :p0 + m].repeat_interleave(H // KVH, 0)
                sc = torch.einsum("qhd,hkd->hqk", q[r:r + m], kk) / math.sqrt(hd)
                mask = torch.arange(p0 + m)[None, :] > torch.arange(p0, p0 + m)[:, None]
                sc = sc.masked_fill(mask[None], float("-inf"))
                outs.append(torch.einsum("hqk,hkd->qhd", torch.softmax(sc, -1), vv).reshape(m, H * hd))
                r += m
            x = x + torch.cat(outs) @ L["wo"].T
            h = rmsnorm(x, L["ln2"], cfg.eps)
            x = x + (torch.nn.functional.silu(h @ L["gate"].T) * (h @ L["up"].T)) @ L["wd"].T
        am = (rmsnorm(x, W["final_ln"], cfg.eps) @ W["lm_head"].T).argmax(-1).numpy()
        out, r = [], 0
        for _, t, _ in blocks:
            out.append(am[r:r + len(t)])
            r += len(t)
        return out

    def rollout(self, prompts, target, histories, spec_cfg=(2, 2, 32, 7, 3)):
        """Greedy HistoSpec rollout; returns (tokens per seq, prefill_s, decode_s, iterations, accepted, verifies)."""
        import time
        from oracle import hs_oracle_c as C
        cfg = self.cfg
        B = len(prompts)
        caches = [[(torch.zeros(cfg.n_kv_heads, self.max_len, cfg.head_dim),
                    torch.zeros(cfg.n_kv_heads, self.max_len, cfg.head_dim)) for _ in range(cfg.n_layers)]
                  for _ in range(B)]
        wi, wa, wm, pi, pm = spec_cfg
        t0 = time.perf_counter()
        first = self._forward(caches, [(b, prompts[b], 0) for b in range(B)])
        t1 = time.perf_counter()
        gen = [[int(first[b][-1])] for b in range(B)]
        win, cur = [wi] * B, [pi] * B
        iters = acc_tot = ver = 0
        P = [len(p) for p in prompts]
        while any(len(g) < target for g in gen):
            blocks, drafts = [], {}
            for b in range(B):
                g = gen[b]
                if len(g) >= target:
                    continue
                d, found = [], False
                looked = histories is not None and len(g) >= cur[b]
                if looked:
                    d, found, _ = C.draft(histories[b], g[len(g) - cur[b]:], win[b])
                drafts[b] = (d, looked, found)
                blocks.append((b, [g[-1]] + d, P[b] + len(g) - 1))
            am = self._forward(caches, blocks)
            for (b, _t, _p), row in zip(blocks, am):
                d, looked, found = drafts[b]
                g = gen[b]
                rest = target - len(g)
                if not d:
                    g.append(int(row[0]))
                    if looked:
                        cur[b] = pi if found else max(cur[b] - 1, pm)
                    continue
                a = 0
                while a < len(d) and a < rest and d[a] == int(row[a]):
                    a += 1
                g.extend(d[:min(a, rest)])
                if len(g) < target:
                    g.append(int(row[min(a, rest)]))
                win[b] = min(win[b] + wa, wm) if a == len(d) else wi
                cur[b] = pi
                acc_tot += min(a, rest)
                ver += 1
            iters += 1
        t2 = time.perf_counter()
        return gen, t1 - t0, t2 - t1, iters, acc_tot, ver
