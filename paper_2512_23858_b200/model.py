"""Llama-shaped target / draft model definitions and seeded synthetic weights.

The reference has no model arithmetic at all: its verifier and drafter are priced by
``latency_at(profile, width)`` (pkg/src/specsim/simulator.py:202-214) and the draft
distribution is a plugin (``DrafterDistribution``, egt.py:52-62).  These shapes make the
forwards real; SURVEY.md §8(d) fixes the shapes and the synthetic-weight recipe.

Weight layout (row-major, rows = output features, which is the K-major operand layout the
swap-AB tcgen05 GEMM streams):
  wqkv [(Hq + 2 Hkv) hd, d]  (q rows, then k rows, then v rows)
  wo   [d, Hq hd]
  wgu  [2 F, d]              (gate rows, then up rows)
  wdown[d, F]
  embed / lm_head [V, d]

Coupled synthetic weights.  Independent random target and draft agree on almost nothing
(AAL ~ 1).  ``coupling`` builds both models around one shared synthetic
"language": a random permutation pi of the vocabulary and a shared semantic table Phi
[V, r] (r = the smaller model width).  Both embeddings carry Phi in their first r
dimensions and both LM heads score token v by Phi[pi^-1(v)], so each model's preferred
continuation of x is pi(x) unless its own (independent) random layers and head noise
perturb it; the noise scales set how often target and draft disagree, i.e. the AAL.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import torch


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
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    tied: bool = False

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def q_dim(self) -> int:
        return self.n_heads * self.head_dim

    def matmul_params(self) -> int:
        """Parameters streamed by one forward (all matmuls incl. the LM head)."""
        per_layer = self.qkv_dim * self.d_model + self.d_model * self.q_dim + 3 * self.ffn * self.d_model
        return self.n_layers * per_layer + self.vocab * self.d_model

    def kv_bytes_per_token(self, elem_bytes: int = 2) -> int:
        return self.n_layers * 2 * self.n_kv_heads * self.head_dim * elem_bytes


PRESETS: dict[str, ModelConfig] = {
    # cfg1 (BASELINE.json configs[0]): tiny target + 1-layer draft.
    "tiny-target": ModelConfig("tiny-target", 4, 256, 4, 2, 64, 768, 32000, rope_theta=10000.0),
    "tiny-draft": ModelConfig("tiny-draft", 1, 256, 4, 2, 64, 768, 32000, rope_theta=10000.0),
    # Llama-3-8B / Llama-3.2-1B / Llama-3-70B shapes.
    "llama3-8b": ModelConfig("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256),
    "llama3.2-1b": ModelConfig("llama3.2-1b", 16, 2048, 32, 8, 64, 8192, 128256, tied=True),
    "llama3-70b": ModelConfig("llama3-70b", 80, 8192, 64, 8, 128, 28672, 128256),
}


def preset(name: str, **overrides) -> ModelConfig:
    cfg = PRESETS[name]
    return replace(cfg, **overrides) if overrides else cfg


@dataclass(frozen=True)
class Coupling:
    """Shared synthetic language for a (target, draft) pair (see module docstring)."""

    seed: int = 1234
    rank: int = 256            # width of the shared semantic table Phi
    logit_scale: float = 1.0   # head scale (sharpness of the next-token distribution)
    head_noise: float = 0.0    # per-model head noise relative to Phi
    layer_gain: float = 1.0    # scale of the residual-branch output projections


def _randn(shape, gen, device, std=1.0):
    t = torch.randn(*shape, generator=gen, device=device, dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    return t


def _shared_language(vocab: int, rank: int, seed: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    phi = _randn((vocab, rank), g, device)
    perm = torch.randperm(vocab, generator=g, device=device)
    return phi, perm


def init_weights(
    cfg: ModelConfig,
    seed: int,
    dtype: torch.dtype = torch.bfloat16,
    device: str | torch.device = "cpu",
    coupling: Coupling | None = None,
) -> dict:
    """Seeded random-init weights (``torch.manual_seed``-style generator on ``device``).

    Generation happens in f32 on ``device`` tensor by tensor and is then cast, so the same
    (cfg, seed, device) always yields identical values; the CPU oracle and the GPU engine
    compare on weights generated on the CPU and copied.
    """
    device = torch.device(device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    d, L = cfg.d_model, cfg.n_layers
    gain = coupling.layer_gain if coupling else 1.0
    out_std = gain / math.sqrt(2.0 * L)
    layers = []
    for _ in range(L):
        layers.append(
            {
                "wqkv": _randn((cfg.qkv_dim, d), g, device, 1.0 / math.sqrt(d)).to(dtype),
                "wo": _randn((d, cfg.q_dim), g, device, out_std / math.sqrt(cfg.q_dim)).to(dtype),
                "wgu": _randn((2 * cfg.ffn, d), g, device, 1.0 / math.sqrt(d)).to(dtype),
                "wdown": _randn((d, cfg.ffn), g, device, out_std / math.sqrt(cfg.ffn)).to(dtype),
                "attn_norm": torch.ones(d, device=device, dtype=dtype),
                "mlp_norm": torch.ones(d, device=device, dtype=dtype),
            }
        )
    if coupling is None:
        embed = _randn((cfg.vocab, d), g, device)
        head = embed if cfg.tied else _randn((cfg.vocab, d), g, device, 4.0 / math.sqrt(d))
    else:
        r = min(coupling.rank, d)
        phi, perm = _shared_language(cfg.vocab, coupling.rank, coupling.seed, device)
        phi = phi[:, :r]
        embed = torch.zeros(cfg.vocab, d, device=device)
        embed[:, :r] = phi
        if d > r:
            embed[:, r:] = _randn((cfg.vocab, d - r), g, device, 0.05)
        inv = torch.empty_like(perm)
        inv[perm] = torch.arange(cfg.vocab, device=device)
        # head row v scores Phi[pi^-1(v)]: the preferred continuation of x is pi(x).
        head = torch.zeros(cfg.vocab, d, device=device)
        head[:, :r] = phi[inv]
        if coupling.head_noise > 0:
            head[:, :r] += _randn((cfg.vocab, r), g, device, coupling.head_noise)
        head.mul_(coupling.logit_scale / math.sqrt(r))
    w = {
        "layers": layers,
        "embed": embed.to(dtype),
        "final_norm": torch.ones(d, device=device, dtype=dtype),
    }
    # A coupled model always carries its own head (see module docstring); an uncoupled tied
    # model reuses the embedding table exactly like Llama-3.2-1B.
    w["lm_head"] = w["embed"] if (cfg.tied and coupling is None) else head.to(dtype)
    return w


def weights_to(w: dict, device, dtype: torch.dtype | None = None) -> dict:
    def mv(t):
        return t.to(device=device, dtype=dtype or t.dtype).contiguous()

    out = {
        "layers": [{k: mv(v) for k, v in lw.items()} for lw in w["layers"]],
        "embed": mv(w["embed"]),
        "final_norm": mv(w["final_norm"]),
    }
    out["lm_head"] = out["embed"] if w["lm_head"] is w["embed"] else mv(w["lm_head"])
    return out


def qkv_row_permutation(cfg: ModelConfig) -> torch.Tensor:
    """Row order of the fused-path QKV weight: inside every head, RoPE pairs (i, i + hd/2) become
    adjacent rows (new row 2i <- i, 2i+1 <- i + hd/2) so one warp-lane pair holds a rotation pair."""
    hd, half = cfg.head_dim, cfg.head_dim // 2
    heads = cfg.n_heads + 2 * cfg.n_kv_heads
    within = torch.stack([torch.arange(half), torch.arange(half) + half], 1).reshape(-1)
    return (torch.arange(heads)[:, None] * hd + within[None, :]).reshape(-1)


def gate_up_interleave(cfg: ModelConfig) -> torch.Tensor:
    """Row order of the fused-path gate|up weight: row 2j <- gate j, row 2j+1 <- up j."""
    F = cfg.ffn
    return torch.stack([torch.arange(F), torch.arange(F) + F], 1).reshape(-1)


def prepare_fused_(w: dict, cfg: ModelConfig) -> dict:
    """In-place conversion to the fused bf16 layout (idempotent): RMSNorm gains folded into the
    following matmul (wqkv, wgu, lm_head columns), QKV rows RoPE-pair-interleaved, gate/up rows
    interleaved.  The per-token rstd is applied by the consumer GEMM's epilogue."""
    if w.get("_layout") == "fused":
        return w
    dev = w["embed"].device
    qperm = qkv_row_permutation(cfg).to(dev)
    gperm = gate_up_interleave(cfg).to(dev)
    for lw in w["layers"]:
        an = lw["attn_norm"].float()
        mn = lw["mlp_norm"].float()
        lw["wqkv"] = (lw["wqkv"].float() * an[None, :]).to(lw["wqkv"].dtype)[qperm].contiguous()
        lw["wgu"] = (lw["wgu"].float() * mn[None, :]).to(lw["wgu"].dtype)[gperm].contiguous()
        lw["attn_norm"] = torch.ones_like(lw["attn_norm"])
        lw["mlp_norm"] = torch.ones_like(lw["mlp_norm"])
    fn = w["final_norm"].float()
    if not bool(torch.all(fn == 1)):
        w["lm_head"] = (w["lm_head"].float() * fn[None, :]).to(w["lm_head"].dtype)
    w["final_norm"] = torch.ones_like(w["final_norm"])
    w["_layout"] = "fused"
    return w


def rope_table(cfg: ModelConfig, positions: int, device) -> torch.Tensor:
    """[positions, hd/2, 2] (cos, sin) of the RoPE angle for the fused QKV epilogue.

    The angle is formed exactly like the fp32 reference (inv_freq = 1/theta^(2i/hd) in f32, angle =
    f32(pos) * inv_freq rounded to f32); cos/sin are then evaluated in f64 and rounded once, so the
    table is within half an ulp of the exact cosine of the reference's f32 angle."""
    hd = cfg.head_dim
    inv_freq = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float32) / hd))
    ang = torch.arange(positions, dtype=torch.float32)[:, None] * inv_freq[None, :]
    ang64 = ang.double()
    return torch.stack([torch.cos(ang64), torch.sin(ang64)], -1).float().contiguous().to(device)
