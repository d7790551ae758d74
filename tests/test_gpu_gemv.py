"""Row-block GEMV forward (csrc/gemv.cu, decode passes of <= 16 rows) vs the per-kernel bf16 forward.

Same bf16 weights (separate copies: the GEMV path converts its dict to the fused layout), same rows,
identical KV caches.  Tolerance 2e-2 relative to the logit scale (north_star's bf16 bound; the two
paths round the GEMM inputs differently — folded vs applied RMSNorm — and accumulate in different
orders); appended KV rows must agree to bf16 rounding.  Relaunches are bit-identical.
"""

import copy

import numpy as np

import pytest
import torch

pytestmark = pytest.mark.gpu

MID = dict(n_layers=2, d_model=1024, n_heads=8, n_kv_heads=2, head_dim=128, ffn=2048, vocab=4096)


def _inputs(cfg, B, R, mask_words, P, cuda, seed=0):
    from paper_2512_23858_b200.forward import new_cache

    S = P + R + 64
    cache = new_cache(cfg, B, S, torch.bfloat16, cuda)
    g = torch.Generator(device="cuda").manual_seed(seed + 1)
    cache.copy_((torch.randn(cache.shape, device=cuda, generator=g) * 0.5).to(torch.bfloat16))
    M = B * R
    tokens = torch.randint(0, cfg.vocab, (M,), device=cuda, generator=g, dtype=torch.int32)
    r = torch.arange(M, device=cuda, dtype=torch.int32) % R
    qmask = None
    pos = P + r
    if mask_words:
        rows, depth = [], []
        for i in range(R):
            par = -1 if i == 0 else (i - 1) // 2  # binary-ish tree
            rows.append((rows[par] if par >= 0 else 0) | (1 << i))
            depth.append(0 if par < 0 else depth[par] + 1)
        qm = torch.tensor([[(rows[i] >> (32 * w)) & 0xFFFFFFFF for w in range(mask_words)] for i in range(R)] * B,
                          dtype=torch.int64)
        qmask = qm.to(torch.int32).to(cuda)
        pos = (P + torch.tensor(depth * B, dtype=torch.int32)).to(cuda)
    return cache, (tokens, pos, P + r, torch.arange(M, device=cuda, dtype=torch.int32) // R, qmask)


def _fwd(cfg, w, cache, B, R, mask_words, gemv, inp, P):
    from paper_2512_23858_b200.forward import Forward

    tokens, pos, slot, req, qmask = inp
    f = Forward(cfg, w, cache, B, R, mask_words, torch.bfloat16, gemv=gemv)
    assert f.gemv == gemv
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
    [("tiny", 1, 8, 1, 40), ("tiny", 2, 8, 1, 100), ("tiny", 1, 1, 1, 77), ("mid", 1, 8, 1, 300),
     ("mid", 2, 4, 1, 130), ("mid", 1, 16, 1, 64), ("mid", 1, 3, 0, 50)],
)
def test_gemv_matches_per_kernel(name, B, R, mask_words, P, cuda):
    from paper_2512_23858_b200.model import ModelConfig, init_weights, preset, weights_to

    cfg = preset("tiny-target") if name == "tiny" else ModelConfig("mid", **MID)
    w0 = weights_to(init_weights(cfg, 0, torch.float32, "cpu"), cuda, torch.bfloat16)
    w_ref, w_gv = copy.deepcopy(w0), copy.deepcopy(w0)
    cache, inp = _inputs(cfg, B, R, mask_words, P, cuda)
    c_ref, c_gv = cache.clone(), cache.clone()
    ref = _fwd(cfg, w_ref, c_ref, B, R, mask_words, False, inp, P)
    gv = _fwd(cfg, w_gv, c_gv, B, R, mask_words, True, inp, P)
    ref.run()
    gv.run()
    torch.cuda.synchronize()
    scale = float(ref.logits.abs().max())
    err = float((gv.logits - ref.logits).abs().max())
    assert err <= 2e-2 * scale, (err, scale)
    assert (c_gv.float() - c_ref.float()).abs().max() <= 2e-2 * float(c_ref.float().abs().max())
    first = gv.logits.clone()
    gv.logits.zero_()
    gv.run()
    torch.cuda.synchronize()
    assert torch.equal(gv.logits, first)


@pytest.mark.parametrize("M,V,k,temp", [(8, 128256, 8, 1.0), (5, 32000, 8, 0.7), (1, 4096, 3, 1.0), (8, 1008, 8, 1.3)])
def test_gemv_fused_topk_matches_topk_softmax(M, V, k, temp, cuda):
    """STORE_TOPK (LM-head GEMV epilogue partials + ygg_topk_merge) == ygg_topk_softmax over the
    logits the same launch stored: identical tokens, probabilities to 1e-12 (f64 sums in another
    order), and the oracle's topk_softmax on those logits."""
    import ctypes as C

    import numpy as np

    from oracle import tree_ref as T
    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    K = 256
    g = torch.Generator(device="cuda").manual_seed(V + M)
    W = (torch.randn(V, K, device=cuda, generator=g) * 0.2).to(torch.bfloat16)
    X = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    W[V // 3] = W[V // 2]  # an exact logit tie (token order decides)
    mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
    L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), M, V, K, 0))
    grid = int(lib.ygg_gemv_grid(mem))
    part = torch.empty(int(lib.ygg_topk_partial_bytes(M, grid)), dtype=torch.uint8, device=cuda)
    logits = torch.zeros(M, V, dtype=torch.float32, device=cuda)
    e = L.YggGemvEpilogue()
    e.kind = L.YGG_GEMV_STORE_TOPK
    e.out = logits.data_ptr()
    e.ld = V
    e.topk_part = part.data_ptr()
    e.topk_k = k
    e.inv_temp = 1.0 / temp
    L.check(lib.ygg_gemv_run(mem, C.byref(e), L.stream_ptr()))
    tok = torch.zeros(M, k, dtype=torch.int32, device=cuda)
    prob = torch.zeros(M, k, dtype=torch.float64, device=cuda)
    L.check(lib.ygg_topk_merge(part.data_ptr(), M, grid, k, tok.data_ptr(), prob.data_ptr(), None, L.stream_ptr()))
    ws = torch.empty(int(lib.ygg_topk_workspace(M, V, k)), dtype=torch.uint8, device=cuda)
    tok2 = torch.zeros_like(tok)
    prob2 = torch.zeros_like(prob)
    L.check(lib.ygg_topk_softmax(logits.data_ptr(), L.YGG_F32, M, V, V, k, temp, tok2.data_ptr(), prob2.data_ptr(),
                                 None, ws.data_ptr(), ws.numel(), L.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(tok, tok2)
    np.testing.assert_allclose(prob.cpu().numpy(), prob2.cpu().numpy(), rtol=1e-12)
    if temp != 1.0:  # the oracle divides by the temperature, the kernels multiply by its inverse
        return
    lg = logits.cpu().numpy()
    for r in range(M):
        ref = T.topk_softmax(lg[r], k, temp)
        assert tok[r].cpu().tolist() == [t for t, _ in ref]
        np.testing.assert_allclose(prob[r].cpu().numpy(), [p for _, p in ref], rtol=1e-12)


def test_gemv_fused_topk_rejects_wide_rows(cuda):
    import ctypes as C

    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    W = torch.zeros(256, 128, dtype=torch.bfloat16, device=cuda)
    X = torch.zeros(12, 128, dtype=torch.bfloat16, device=cuda)
    mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
    L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), 12, 256, 128, 0))
    out = torch.zeros(12, 256, dtype=torch.float32, device=cuda)
    part = torch.empty(1 << 20, dtype=torch.uint8, device=cuda)
    e = L.YggGemvEpilogue()
    e.kind = L.YGG_GEMV_STORE_TOPK
    e.out = out.data_ptr()
    e.ld = 256
    e.topk_part = part.data_ptr()
    e.topk_k = 4
    e.inv_temp = 1.0
    with pytest.raises(ValueError):
        L.check(lib.ygg_gemv_run(mem, C.byref(e), L.stream_ptr()))


def test_gemv_plan_rejects_bad_shapes(cuda):
    import ctypes as C

    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
    W = torch.zeros(64, 128, dtype=torch.bfloat16, device=cuda)
    X = torch.zeros(17, 128, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ValueError):
        L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), 17, 64, 128, 0))
    with pytest.raises(ValueError):
        L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), 8, 60, 128, 0))


@pytest.mark.parametrize("hd,Hq,Hkv,B,T,P,mw", [(64, 32, 8, 1, 8, 300, 1), (128, 32, 8, 2, 16, 130, 1),
                                                (64, 8, 2, 1, 1, 77, 0), (128, 8, 2, 1, 5, 64, 0),
                                                (128, 32, 8, 1, 50, 512, 2), (64, 32, 8, 2, 33, 90, 2),
                                                (128, 32, 8, 1, 40, 64, 0)])
@pytest.mark.parametrize("kvsplit", ["1", "2", "3", "8"])
def test_decode_attention_vs_fp32(hd, Hq, Hkv, B, T, P, mw, kvsplit, cuda):
    """ygg_attn_dec_run vs a float64 softmax(QK^T/sqrt(hd)) V over the visible keys (prefix + tree /
    causal block), with the key chunks split over 1..8 CTAs of a cluster.  bf16 operands; tolerance
    2e-2 of the output scale (bf16 P and output rounding); repeated launches are bit-identical."""
    import ctypes as C
    import math

    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    S = ((P + T + 63) // 64) * 64
    g = torch.Generator(device="cuda").manual_seed(hd + T)
    M = B * T
    q = torch.randn(M, Hq, hd, device=cuda, generator=g).to(torch.bfloat16)
    cache = torch.randn(B, 2, Hkv, S, hd, device=cuda, generator=g).to(torch.bfloat16)  # kv=1 holds V^T rows
    par = [-1] + [(i - 1) // 2 for i in range(1, T)]
    rows = []
    for i in range(T):
        rows.append((rows[par[i]] if par[i] >= 0 else 0) | (1 << i))
    nwords = max(mw, 1)
    qmask = torch.tensor([[(rows[i] >> (32 * w)) & 0xFFFFFFFF for w in range(nwords)] for i in range(T)] * B,
                         dtype=torch.int64).to(torch.int32).to(cuda)
    bs = torch.full((B,), P, dtype=torch.int32, device=cuda)
    bl = torch.full((B,), T, dtype=torch.int32, device=cuda)
    out = torch.zeros(M, Hq, hd, dtype=torch.bfloat16, device=cuda)
    mem = C.create_string_buffer(int(lib.ygg_attn_dec_plan_size()))
    L.check(lib.ygg_attn_dec_plan_init(mem, q.data_ptr(), cache.data_ptr(), B, T, Hq, Hkv, hd, S, int(kvsplit), 0, 0))
    scale = 1.0 / math.sqrt(hd)
    ws = torch.zeros(int(lib.ygg_attn_dec_workspace_size(mem)) // 4 + 64, dtype=torch.float32, device=cuda)
    outs = []
    for _ in range(2):  # twice: the merge order is fixed, so the results must be bit-identical
        L.check(lib.ygg_attn_dec_run(mem, bs.data_ptr(), bl.data_ptr(), qmask.data_ptr() if mw else None, mw, scale,
                                     out.data_ptr(), ws.data_ptr(), L.stream_ptr()))
        outs.append(out.clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    K = cache[:, 0].double().cpu()                         # [B, Hkv, S, hd]
    Vt = cache[:, 1].double().cpu().reshape(B, Hkv, hd, S)  # V^T rows
    qd = q.double().cpu()
    ref = torch.zeros(M, Hq, hd, dtype=torch.float64)
    G = Hq // Hkv
    for b in range(B):
        for t in range(T):
            vis = list(range(P))
            for j in range(T):
                if (mw and (rows[t] >> j) & 1) or (not mw and j <= t):
                    vis.append(P + j)
            vis = torch.tensor(vis)
            for h in range(Hq):
                kv = h // G
                s = K[b, kv, vis] @ qd[b * T + t, h] * scale
                p = torch.softmax(s, 0)
                ref[b * T + t, h] = Vt[b, kv][:, vis] @ p
    err = (out.double().cpu() - ref).abs().max()
    assert err <= 2e-2 * ref.abs().max(), float(err)


def test_l2_prefetch_regions_leave_results_unchanged(cuda):
    """The optional L2 prefetch regions of the GEMV / decode attention / top-k merge only move data
    into L2: every output is bit-identical with and without them; bad regions are rejected."""
    import ctypes as C

    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    g = torch.Generator(device="cuda").manual_seed(7)
    V, K, M, k = 4096, 256, 8, 8
    W = (torch.randn(V, K, device=cuda, generator=g) * 0.2).to(torch.bfloat16)
    X = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    other = torch.randn(1 << 20, device=cuda, generator=g)  # 4 MB "next weights"
    mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
    L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), M, V, K, 0))
    grid = int(lib.ygg_gemv_grid(mem))
    part = torch.empty(int(lib.ygg_topk_partial_bytes(M, grid)), dtype=torch.uint8, device=cuda)
    outs = []
    for pf in (0, other.numel() * 4):
        L.check(lib.ygg_gemv_set_l2_prefetch(mem, 0, other.data_ptr() if pf else None, pf))
        L.check(lib.ygg_gemv_set_l2_prefetch(mem, 1, other.data_ptr() if pf else None, pf // 2))
        logits = torch.zeros(M, V, dtype=torch.float32, device=cuda)
        e = L.YggGemvEpilogue()
        e.kind, e.out, e.ld = L.YGG_GEMV_STORE_TOPK, logits.data_ptr(), V
        e.topk_part, e.topk_k, e.inv_temp = part.data_ptr(), k, 1.0
        L.check(lib.ygg_gemv_run(mem, C.byref(e), L.stream_ptr()))
        tok = torch.zeros(M, k, dtype=torch.int32, device=cuda)
        prob = torch.zeros(M, k, dtype=torch.float64, device=cuda)
        regs = (L.YggL2Region * 4)(L.YggL2Region(other.data_ptr(), pf)) if pf else None
        L.check(lib.ygg_topk_merge_l2(part.data_ptr(), M, grid, k, tok.data_ptr(), prob.data_ptr(), None, regs,
                                      1 if pf else 0, L.stream_ptr()))
        torch.cuda.synchronize()
        outs.append((logits.clone(), tok.clone(), prob.clone()))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    with pytest.raises(ValueError):  # misaligned region
        L.check(lib.ygg_gemv_set_l2_prefetch(mem, 0, other.data_ptr() + 4, 1024))
    with pytest.raises(ValueError):  # too many regions
        L.check(lib.ygg_topk_merge_l2(part.data_ptr(), M, grid, k, tok.data_ptr(), prob.data_ptr(), None,
                                      (L.YggL2Region * 5)(), 5, L.stream_ptr()))
    # decode attention: same output with both prefetch regions set
    Hq, Hkv, hd, T, P = 32, 8, 64, 8, 300
    S = ((P + T + 63) // 64) * 64
    q = torch.randn(T, Hq, hd, device=cuda, generator=g).to(torch.bfloat16)
    cache = torch.randn(1, 2, Hkv, S, hd, device=cuda, generator=g).to(torch.bfloat16)
    bs = torch.full((1,), P, dtype=torch.int32, device=cuda)
    bl = torch.full((1,), T, dtype=torch.int32, device=cuda)
    att = C.create_string_buffer(int(lib.ygg_attn_dec_plan_size()))
    L.check(lib.ygg_attn_dec_plan_init(att, q.data_ptr(), cache.data_ptr(), 1, T, Hq, Hkv, hd, S, 0, 0, 0))
    res = []
    for pf in (0, 1 << 20):
        for rg in (0, 1):
            L.check(lib.ygg_attn_dec_set_l2_prefetch(att, rg, other.data_ptr() if pf else None, pf))
        out = torch.zeros(T, Hq, hd, dtype=torch.bfloat16, device=cuda)
        L.check(lib.ygg_attn_dec_run(att, bs.data_ptr(), bl.data_ptr(), None, 0, 0.125, out.data_ptr(), None,
                                     L.stream_ptr()))
        torch.cuda.synchronize()
        res.append(out.clone())
    assert torch.equal(res[0], res[1])
    with pytest.raises(ValueError):
        L.check(lib.ygg_attn_dec_set_l2_prefetch(att, 2, other.data_ptr(), 1024))


def test_kernel_timeline_trace_slots(cuda):
    """ygg_trace_arm: a traced launch fills its slot with start <= release <= end (globaltimer ns)."""
    import ctypes as C

    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    W = torch.randn(2048, 512, device=cuda).to(torch.bfloat16)
    X = torch.randn(8, 512, device=cuda).to(torch.bfloat16)
    out = torch.zeros(8, 2048, dtype=torch.float32, device=cuda)
    mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
    L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), 8, 2048, 512, 0))
    buf = torch.zeros(4, 8, dtype=torch.int64, device=cuda)
    buf[:, :2] = -1
    L.check(lib.ygg_trace_arm(buf.data_ptr(), 4))
    e = L.YggGemvEpilogue()
    e.kind, e.out, e.ld = L.YGG_GEMV_STORE, out.data_ptr(), 2048
    L.check(lib.ygg_gemv_run(mem, C.byref(e), L.stream_ptr()))
    ids = (C.c_int * 4)()
    n = lib.ygg_trace_used(ids, 4)
    L.check(lib.ygg_trace_arm(None, 0))
    torch.cuda.synchronize()
    assert n == 1 and ids[0] == 1
    s, r, t = [int(x) for x in buf[0, :3].cpu()]
    assert 0 < s <= r <= t, (s, r, t)
    torch.testing.assert_close(out, (X.float() @ W.float().T), rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("hd,Hq,Hkv", [(128, 32, 8), (64, 32, 8)])
def test_decode_attention_wide_tree_mask(hd, Hq, Hkv, cuda):
    """cfg5-shaped draft level: 16 query rows (the newest level of a D8 W16 tree) over a 129-key
    tree block (5 mask words) after a 300-token prefix; vs float64 attention over the visible keys."""
    import ctypes as C
    import math

    from oracle import tree_ref as T
    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    rng = np.random.default_rng(hd)
    t = T.Tree.root(0, 0.9)
    for _ in range(8):
        cands = {}
        for f in t.levels()[-1]:
            ps = np.sort(rng.dirichlet(np.ones(17))[:16])[::-1]
            cands[f] = [(int(x), float(p)) for x, p in zip(rng.choice(10**5, 16, replace=False), ps)]
        T.grow_step(t, lambda tr, n, kk: cands[n], 16, 16)
    N = len(t)
    assert N == 129
    B, R, P, mw = 2, 16, 300, 5
    rows_nodes = t.levels()[-1]
    masks = []
    for i in rows_nodes:
        m = 0
        for a in t.path(i):
            m |= 1 << a
        masks.append(m)
    S = ((P + N + 63) // 64) * 64
    g = torch.Generator(device="cuda").manual_seed(hd)
    M = B * R
    q = torch.randn(M, Hq, hd, device=cuda, generator=g).to(torch.bfloat16)
    cache = torch.randn(B, 2, Hkv, S, hd, device=cuda, generator=g).to(torch.bfloat16)
    qmask = torch.tensor([[(m >> (32 * w)) & 0xFFFFFFFF for w in range(mw)] for m in masks] * B,
                         dtype=torch.int64).to(torch.int32).to(cuda)
    bs = torch.full((B,), P, dtype=torch.int32, device=cuda)
    bl = torch.full((B,), N, dtype=torch.int32, device=cuda)
    out = torch.zeros(M, Hq, hd, dtype=torch.bfloat16, device=cuda)
    mem = C.create_string_buffer(int(lib.ygg_attn_dec_plan_size()))
    L.check(lib.ygg_attn_dec_plan_init(mem, q.data_ptr(), cache.data_ptr(), B, R, Hq, Hkv, hd, S, 0, 0, 0))
    ws = torch.zeros(int(lib.ygg_attn_dec_workspace_size(mem)) // 4 + 64, dtype=torch.float32, device=cuda)
    scale = 1.0 / math.sqrt(hd)
    L.check(lib.ygg_attn_dec_run(mem, bs.data_ptr(), bl.data_ptr(), qmask.data_ptr(), mw, scale, out.data_ptr(),
                                 ws.data_ptr(), L.stream_ptr()))
    torch.cuda.synchronize()
    K = cache[:, 0].double().cpu()
    Vt = cache[:, 1].double().cpu().reshape(B, Hkv, hd, S)
    qd = q.double().cpu()
    ref = torch.zeros(M, Hq, hd, dtype=torch.float64)
    G = Hq // Hkv
    for b in range(B):
        for r, m in enumerate(masks):
            vis = torch.tensor(list(range(P)) + [P + j for j in range(N) if (m >> j) & 1])
            for h in range(Hq):
                s = K[b, h // G, vis] @ qd[b * R + r, h] * scale
                ref[b * R + r, h] = Vt[b, h // G][:, vis] @ torch.softmax(s, 0)
    err = (out.double().cpu() - ref).abs().max()
    assert err <= 2e-2 * ref.abs().max(), float(err)
