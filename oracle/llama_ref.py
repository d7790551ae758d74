"""torch-CPU fp32 Llama forward with a slot-addressed KV cache and explicit attention masks.

Test oracle only.  The reference has no model arithmetic; this restates the
standard Llama block in plain fp32 torch ops with the exact conventions the device path uses:
RMSNorm (x * rsqrt(mean(x^2) + eps) * g), rotate-half RoPE with inv_freq = 1/theta^(2i/hd),
GQA attention with scale 1/sqrt(hd), SwiGLU, and weight layouts documented in
paper_2512_23858_b200/model.py.
"""

from __future__ import annotations

import math

import torch


class RefCache:
    def __init__(self, cfg, S: int):
        self.k = torch.zeros(cfg.n_layers, cfg.n_kv_heads, S, cfg.head_dim)
        self.v = torch.zeros(cfg.n_layers, cfg.n_kv_heads, S, cfg.head_dim)

    def move(self, src: list, dst: list, layers=None) -> None:
        """Copy slots src -> dst (all sources read before any write)."""
        if not src:
            return
        s = torch.tensor(src)
        d = torch.tensor(dst)
        self.k[:, :, d] = self.k[:, :, s].clone()
        self.v[:, :, d] = self.v[:, :, s].clone()


def rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    """x [M, H, hd]; rotate-half convention."""
    hd = x.shape[-1]
    half = hd // 2
    inv_freq = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float32) / hd))
    ang = pos.to(torch.float32)[:, None] * inv_freq[None, :]
    cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def rmsnorm(x: torch.Tensor, g: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * g


class RefLlama:
    def __init__(self, cfg, weights: dict):
        self.cfg = cfg
        f = lambda t: t.detach().to("cpu", torch.float32)  # noqa: E731
        self.layers = [{k: f(v) for k, v in lw.items()} for lw in weights["layers"]]
        self.embed = f(weights["embed"])
        self.head = f(weights["lm_head"])
        self.final_norm = f(weights["final_norm"])

    @torch.no_grad()
    def forward(self, cache: RefCache, tokens, pos, slots, visible: torch.Tensor) -> torch.Tensor:
        """tokens/pos/slots: [M]; visible: bool [M, S] over cache slots (after this pass's
        K/V writes).  Returns f32 logits [M, V]."""
        c = self.cfg
        tokens = torch.as_tensor(tokens, dtype=torch.long)
        pos = torch.as_tensor(pos, dtype=torch.long)
        slots = torch.as_tensor(slots, dtype=torch.long)
        M = tokens.numel()
        h = self.embed[tokens].clone()
        Hq, Hkv, hd = c.n_heads, c.n_kv_heads, c.head_dim
        G = Hq // Hkv
        scale = 1.0 / math.sqrt(hd)
        neg = torch.full((M, visible.shape[1]), -math.inf)
        bias = torch.where(visible, torch.zeros(()), neg)
        for li, lw in enumerate(self.layers):
            x = rmsnorm(h, lw["attn_norm"], c.norm_eps)
            qkv = x @ lw["wqkv"].T
            q = qkv[:, : Hq * hd].view(M, Hq, hd)
            k = qkv[:, Hq * hd : (Hq + Hkv) * hd].view(M, Hkv, hd)
            v = qkv[:, (Hq + Hkv) * hd :].view(M, Hkv, hd)
            q = rope(q, pos, c.rope_theta)
            k = rope(k, pos, c.rope_theta)
            cache.k[li][:, slots] = k.transpose(0, 1)
            cache.v[li][:, slots] = v.transpose(0, 1)
            K = cache.k[li].repeat_interleave(G, dim=0)  # [Hq, S, hd]
            V = cache.v[li].repeat_interleave(G, dim=0)
            sc = torch.einsum("mhd,hsd->hms", q, K) * scale + bias[None]
            p = torch.softmax(sc, dim=-1)
            p = torch.nan_to_num(p, nan=0.0)
            o = torch.einsum("hms,hsd->mhd", p, V).reshape(M, Hq * hd)
            h = h + o @ lw["wo"].T
            x = rmsnorm(h, lw["mlp_norm"], c.norm_eps)
            gu = x @ lw["wgu"].T
            g_, u_ = gu[:, : c.ffn], gu[:, c.ffn :]
            h = h + (torch.nn.functional.silu(g_) * u_) @ lw["wdown"].T
        x = rmsnorm(h, self.final_norm, c.norm_eps)
        return x @ self.head.T


def causal_visible(P0: int, S: int) -> torch.Tensor:
    v = torch.zeros(P0, S, dtype=torch.bool)
    for i in range(P0):
        v[i, : i + 1] = True
    return v


def greedy_ar(model: RefLlama, prompt: list, n_tokens: int, S: int) -> list:
    """Plain greedy autoregressive decoding (the draft-independent oracle)."""
    cache = RefCache(model.cfg, S)
    P0 = len(prompt)
    logits = model.forward(cache, prompt, list(range(P0)), list(range(P0)), causal_visible(P0, S))
    out = [int(torch.argmax(logits[-1]))]
    P = P0
    while len(out) < n_tokens:
        vis = torch.zeros(1, S, dtype=torch.bool)
        vis[0, : P + 1] = True
        logits = model.forward(cache, [out[-1]], [P], [P], vis)
        out.append(int(torch.argmax(logits[0])))
        P += 1
    return out
