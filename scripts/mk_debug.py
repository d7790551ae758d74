"""Debug: run the persistent forward truncated after k phases (YGG_MK_STOP) and compare layer-0
intermediates with torch references.  1-layer tiny-draft config."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.llama_ref import rope  # noqa: E402
from paper_2512_23858_b200.forward import Forward, new_cache  # noqa: E402
from paper_2512_23858_b200.model import init_weights, preset, weights_to  # noqa: E402

cuda = torch.device("cuda")
cfg = preset(sys.argv[1] if len(sys.argv) > 1 else "tiny-draft")
B, R, P = 1, 8, 40
w = weights_to(init_weights(cfg, 0, torch.float32, "cpu"), cuda, torch.bfloat16)
cache0 = new_cache(cfg, B, P + R + 64, torch.bfloat16, cuda)
g = torch.Generator(device="cuda").manual_seed(1)
cache0.copy_((torch.randn(cache0.shape, device=cuda, generator=g) * 0.5).to(torch.bfloat16))
tokens = torch.randint(0, cfg.vocab, (R,), device=cuda, generator=g, dtype=torch.int32)
pos = P + torch.arange(R, device=cuda, dtype=torch.int32)
lw = w["layers"][0]
d, hd, Hq, Hkv = cfg.d_model, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads


def run(stop):
    os.environ["YGG_MK_STOP"] = str(stop)
    cache = cache0.clone()
    f = Forward(cfg, w, cache, B, R, 0, torch.bfloat16, persistent=True)
    f.tokens.copy_(tokens); f.pos.copy_(pos); f.slot.copy_(pos); f.req.zero_()
    f.blk_start.fill_(P); f.blk_len.fill_(R)
    f.run(); torch.cuda.synchronize()
    return f, cache


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / max(b.abs().max(), 1e-30))


f, cache = run(1)
emb = w["embed"][tokens.long()].double()
print("embed resid", rel(f.resid, emb), "hb", rel(f.xn, emb))
ss_ref = (f.resid.double() ** 2).view(R, d // 128, 128).sum(-1).T
print("ss0", rel(f.ss[0], ss_ref))
f, cache = run(2)
h = emb
rstd = torch.rsqrt((h * h).mean(-1) + cfg.norm_eps)
y = (f.xn.double() @ lw["wqkv"].double().T) * rstd[:, None]
q_ref = rope(y[:, : Hq * hd].view(R, Hq, hd).float().cpu(), pos.cpu(), cfg.rope_theta)
k_ref = rope(y[:, Hq * hd:(Hq + Hkv) * hd].view(R, Hkv, hd).float().cpu(), pos.cpu(), cfg.rope_theta)
v_ref = y[:, (Hq + Hkv) * hd:].view(R, Hkv, hd).float().cpu()
print("q", rel(f.q.view(R, Hq, hd).cpu(), q_ref))
kc = cache[0, 0, 0].float().cpu()  # [Hkv, S, hd]
print("k", rel(kc[:, P:P + R, :].permute(1, 0, 2), k_ref))
vt = cache[0, 0, 1].float().cpu().reshape(Hkv, hd, -1)
print("v", rel(vt[:, :, P:P + R].permute(2, 0, 1), v_ref))
f, cache = run(4)
# attention reference over prefix keys [0,P) + causal block
K = cache[0, 0, 0].double().cpu()  # [Hkv,S,hd]
Vt = cache[0, 0, 1].double().cpu().reshape(Hkv, hd, -1)
qd = f.q.view(R, Hq, hd).double().cpu()
out = torch.zeros(R, Hq, hd, dtype=torch.float64)
G = Hq // Hkv
for i in range(R):
    n = P + i + 1
    for hh in range(Hq):
        kv = hh // G
        s = (K[kv, :n] @ qd[i, hh]) / math.sqrt(hd)
        p = torch.softmax(s, 0)
        out[i, hh] = Vt[kv, :, :n] @ p
print("attn", rel(f.attn.view(R, Hq, hd).cpu(), out))
f, cache = run(5)
o = f.attn.double() @ lw["wo"].double().T
h1 = emb + o
print("resid1", rel(f.resid, h1), "ss1", rel(f.ss[1], (f.resid.double() ** 2).view(R, d // 128, 128).sum(-1).T))
f, cache = run(6)
r1 = torch.rsqrt((h1 * h1).mean(-1) + cfg.norm_eps)
gu = (f.xn.double() @ lw["wgu"].double().T) * r1[:, None]
act = torch.nn.functional.silu(gu[:, :cfg.ffn]) * gu[:, cfg.ffn:]
print("mlp", rel(f.mlp, act))
f, cache = run(7)
h2 = h1 + f.mlp.double() @ lw["wdown"].double().T
print("resid2", rel(f.resid, h2))
f, cache = run(8)
r2 = torch.rsqrt((h2 * h2).mean(-1) + cfg.norm_eps)
lg = (f.xn.double() @ w["lm_head"].double().T) * r2[:, None]
print("logits", rel(f.logits, lg))
f, cache = run(6)
print("resid after down gemm (should be h1)", rel(f.resid, h1))
f, cache = run(7)
dd = (f.resid.double() - h2).abs()
print("err by row", dd.max(1).values.tolist())
print("err by 128-col tile", dd.view(R, -1, 128).amax((0, 2)).tolist())
print("err by col%128 (first 16)", dd.amax(0).view(-1, 128).amax(0)[:16].tolist())
f2, _ = run(7)
print("rerun diff", float((f2.resid - f.resid).abs().max()))
