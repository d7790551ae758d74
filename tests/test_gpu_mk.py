"""Persistent forward (csrc/mk.cu, one launch per pass) vs the per-kernel bf16 forward.

Both paths run the same bf16 weights over the same rows (tokens, positions, KV slots, tree
masks) against identical KV caches.  Tolerance: 2e-2 relative to the logit scale (north_star's
bf16 bound; the two paths round the GEMM inputs differently — folded RMSNorm vs normalised
input), and the KV rows appended by the pass must agree to bf16 rounding.  A second launch of
the same plan must reproduce the logits bit-for-bit (fixed-order stream-K reduction, grid
counter reset by the last CTA).
"""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

MID = dict(n_layers=2, d_model=1024, n_heads=8, n_kv_heads=2, head_dim=128, ffn=2048, vocab=4096)


def _setup(cfg, B, R, mask_words, P, cuda, seed=0):
    from paper_2512_23858_b200.forward import new_cache
    from paper_2512_23858_b200.model import init_weights, weights_to

    w = weights_to(init_weights(cfg, seed, torch.float32, "cpu"), cuda, torch.bfloat16)
    S = P + R + 64
    cache = new_cache(cfg, B, S, torch.bfloat16, cuda)
    g = torch.Generator(device="cuda").manual_seed(seed + 1)
    cache.copy_((torch.randn(cache.shape, device=cuda, generator=g) * 0.5).to(torch.bfloat16))
    M = B * R
    tokens = torch.randint(0, cfg.vocab, (M,), device=cuda, generator=g, dtype=torch.int32)
    r = torch.arange(M, device=cuda, dtype=torch.int32) % R
    if mask_words:
        # random tree: parent[i] < i, mask row = parent row | self
        n = R
        par = [-1] + [int(torch.randint(0, i, (1,), generator=torch.Generator().manual_seed(seed * 97 + i))) for i in
                      range(1, n)]
        rows = []
        for i in range(n):
            bits = 0 if par[i] < 0 else rows[par[i]]
            rows.append(bits | (1 << i))
        depth = [0] * n
        for i in range(1, n):
            depth[i] = depth[par[i]] + 1
        qm = torch.zeros(M, mask_words, dtype=torch.int64)
        for b in range(B):
            for i in range(n):
                for wdx in range(mask_words):
                    qm[b * R + i, wdx] = (rows[i] >> (32 * wdx)) & 0xFFFFFFFF
        qmask = qm.to(torch.int32).to(cuda)
        pos = (P + torch.tensor(depth * B, dtype=torch.int32)).to(cuda)
    else:
        qmask = None
        pos = P + r
    slot = P + r
    req = torch.arange(M, device=cuda, dtype=torch.int32) // R
    return w, cache, tokens, pos, slot, req, qmask


def _forward(cfg, w, cache, B, R, mask_words, persistent, inputs, P):
    from paper_2512_23858_b200.forward import Forward

    tokens, pos, slot, req, qmask = inputs
    f = Forward(cfg, w, cache, B, R, mask_words, torch.bfloat16, persistent=persistent, gemv=False)
    assert f.mk == persistent
    f.tokens.copy_(tokens)
    f.pos.copy_(pos)
    f.slot.copy_(slot)
    f.req.copy_(req)
    if qmask is not None:
        f.qmask.copy_(qmask)
    f.blk_start.fill_(P)
    f.blk_len.fill_(R)
    return f


@pytest.mark.parametrize(
    "name,B,R,mask_words,P",
    [
        ("tiny", 1, 8, 1, 40),
        ("tiny", 2, 17, 1, 100),
        ("tiny", 1, 1, 0, 77),
        ("mid", 1, 50, 2, 300),
        ("mid", 2, 8, 1, 130),
        ("mid", 1, 33, 0, 64),
    ],
)
def test_persistent_matches_per_kernel(name, B, R, mask_words, P, cuda):
    from paper_2512_23858_b200.model import ModelConfig, preset

    cfg = preset("tiny-target") if name == "tiny" else ModelConfig("mid", **MID)
    w, cache, *inp = _setup(cfg, B, R, mask_words, P, cuda)
    c_ref, c_mk = cache.clone(), cache.clone()
    ref = _forward(cfg, w, c_ref, B, R, mask_words, False, inp, P)
    mk = _forward(cfg, w, c_mk, B, R, mask_words, True, inp, P)
    ref.run()
    mk.run()
    torch.cuda.synchronize()
    scale = float(ref.logits.abs().max())
    err = float((mk.logits - ref.logits).abs().max())
    assert err <= 2e-2 * scale, (err, scale)
    # the appended KV rows (and nothing else) match
    assert (c_mk.float() - c_ref.float()).abs().max() <= 2e-2 * float(c_ref.float().abs().max())
    # determinism: a relaunch of the same plan is bit-identical
    first = mk.logits.clone()
    mk.logits.zero_()
    mk.run()
    torch.cuda.synchronize()
    assert torch.equal(mk.logits, first)


def test_persistent_graph_replay(cuda):
    """Captured in a CUDA graph and replayed back to back (the grid counter resets itself)."""
    from paper_2512_23858_b200.model import preset

    cfg = preset("tiny-target")
    B, R, P = 1, 8, 60
    w, cache, *inp = _setup(cfg, B, R, 1, P, cuda, seed=3)
    mk = _forward(cfg, w, cache, B, R, 1, True, inp, P)
    mk.run()
    torch.cuda.synchronize()
    first = mk.logits.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        mk.run(s)
        mk.run(s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(mk.logits, first)
    assert math.isfinite(float(first.abs().max()))
