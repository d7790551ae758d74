"""GPU parity of each kernel against the CPU oracle (trees) or a torch fp32 reference (dense ops).

Tolerances: tree kernels are bit-exact (f64 compared with ==); GEMM/attention compare against
fp32 references of the same bf16/f32 inputs with the bound written in each test.
"""

import math

import numpy as np
import pytest
import torch

from oracle import tree_ref as T

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2512_23858_b200 import _lib as L

    return L


# ---------------------------------------------------------------------------
# K3 GEMM
# ---------------------------------------------------------------------------
def _gemm(M, N, K, dtype, num_ctas, cuda):
    from paper_2512_23858_b200.forward import GemmPlan

    L = _lib()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    X = torch.randn(M, K, device=cuda, generator=g).to(dtype)
    W = (torch.randn(N, K, device=cuda, generator=g) / math.sqrt(K)).to(dtype)
    plan = GemmPlan(W, X, M, num_ctas)
    ws = torch.zeros(max(plan.ws_bytes // 4, 1), device=cuda)
    out = torch.zeros(M, N, device=cuda)
    L.check(L.lib().ygg_gemm_run(plan.handle, ws.data_ptr(), L.stream_ptr()))
    L.check(L.lib().ygg_epi_store(plan.handle, ws.data_ptr(), out.data_ptr(), L.YGG_F32, N, L.stream_ptr()))
    torch.cuda.synchronize()
    ref = X.double() @ W.double().T
    return out.double(), ref


@pytest.mark.parametrize(
    "M,N,K,ctas",
    [(1, 128, 64, 0), (8, 512, 256, 0), (16, 1024, 512, 7), (50, 6144, 4096, 0), (65, 4096, 1024, 0),
     (65, 2048, 4096, 37), (130, 768, 256, 0), (300, 1024, 512, 0), (33, 32000, 256, 0)],
)
def test_gemm_bf16_tcgen05(M, N, K, ctas, cuda):
    out, ref = _gemm(M, N, K, torch.bfloat16, ctas, cuda)
    # bf16 operands are exact in f32; only the f32 summation order differs from the f64 reference.
    err = (out - ref).abs().max().item()
    assert err <= 2e-4 * math.sqrt(K) * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (18, 512, 256), (32, 768, 256), (70, 256, 768)])
def test_gemm_f32_simt(M, N, K, cuda):
    out, ref = _gemm(M, N, K, torch.float32, 0, cuda)
    assert torch.allclose(out, ref, rtol=1e-5, atol=1e-5 * math.sqrt(K))


# ---------------------------------------------------------------------------
# K2 attention (bitmask / causal) vs a torch fp32 reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("path", ["simt_f32", "simt_bf16", "tc_bf16"])
@pytest.mark.parametrize("hd,Hq,Hkv", [(64, 4, 2), (128, 32, 8), (64, 32, 8)])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("T", [19, 50])
def test_attention(path, hd, Hq, Hkv, causal, T, cuda):
    """Cache layout: kv=0 half K [Hkv][S][hd], kv=1 half V^T [Hkv][hd][S]."""
    from paper_2512_23858_b200.forward import AttnPlan
    from paper_2512_23858_b200.model import preset

    L = _lib()
    dtype = torch.float32 if path == "simt_f32" else torch.bfloat16
    B, S = 2, 320
    g = torch.Generator(device="cuda").manual_seed(hd + Hq + T)
    q = torch.randn(B * T, Hq, hd, device=cuda, generator=g).to(dtype)
    cache = torch.randn(B, 2, Hkv, S, hd, device=cuda, generator=g).to(dtype)
    blk_start = torch.tensor([37, 190], dtype=torch.int32, device=cuda)
    blk_len = torch.tensor([T, T], dtype=torch.int32, device=cuda)
    mw = (T + 31) // 32
    rng = np.random.default_rng(3)
    masks = torch.zeros(B * T, mw, dtype=torch.int64)
    vis = torch.zeros(B * T, S, dtype=torch.bool)
    for b in range(B):
        for i in range(T):
            bits = 1 << i
            if not causal:
                for j in range(i):
                    if rng.random() < 0.4:
                        bits |= 1 << j
            else:
                bits = (1 << (i + 1)) - 1
            for w in range(mw):
                masks[b * T + i, w] = (bits >> (32 * w)) & 0xFFFFFFFF
            vis[b * T + i, : int(blk_start[b])] = True
            for j in range(T):
                if (bits >> j) & 1:
                    vis[b * T + i, int(blk_start[b]) + j] = True
    masks_d = torch.from_numpy(masks.numpy().astype(np.uint32).view(np.int32)).to(cuda)
    out = torch.zeros(B * T, Hq * hd, device=cuda, dtype=dtype)
    scale = 1.0 / math.sqrt(hd)
    qm = None if causal else masks_d.data_ptr()
    nw = 0 if causal else mw
    if path == "tc_bf16":
        cfg = preset("tiny-target", n_heads=Hq, n_kv_heads=Hkv, head_dim=hd)
        plan = AttnPlan(q, cache.data_ptr(), B, B * T, cfg, S)
        part = torch.empty(plan.partial_bytes // 4 + 1, device=cuda)
        L.check(L.lib().ygg_attention_tc(plan.handle, blk_start.data_ptr(), blk_len.data_ptr(), qm, nw, scale,
                                         part.data_ptr(), out.data_ptr(), L.stream_ptr()))
    else:
        L.check(L.lib().ygg_attention(q.data_ptr(), cache.data_ptr(), L.dtype_code(dtype), B * T, B, Hq, Hkv, hd, S,
                                      blk_start.data_ptr(), blk_len.data_ptr(), qm, nw, scale, out.data_ptr(),
                                      L.stream_ptr()))
    torch.cuda.synchronize()
    G = Hq // Hkv
    ref = torch.zeros(B * T, Hq, hd, dtype=torch.float64)
    qc, cc = q.double().cpu(), cache.double().cpu()
    for b in range(B):
        K = cc[b, 0].repeat_interleave(G, 0)
        V = cc[b, 1].reshape(Hkv, hd, S).transpose(1, 2).repeat_interleave(G, 0)
        rows = slice(b * T, (b + 1) * T)
        sc = torch.einsum("thd,hsd->hts", qc[rows], K) * scale
        sc = sc.masked_fill(~vis[rows][None], -math.inf)
        p = torch.softmax(sc, -1)
        ref[rows] = torch.einsum("hts,hsd->thd", p, V)
    # bf16: P is rounded to bf16 before P.V on the tensor-core path (|O| <~ 4 here)
    tol = 2e-5 if dtype == torch.float32 else 3e-2
    got = out.double().cpu().view(B * T, Hq, hd)
    assert torch.allclose(got, ref, atol=tol, rtol=tol), (got - ref).abs().max().item()


# ---------------------------------------------------------------------------
# K1a top-k softmax vs oracle
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("V,k", [(32000, 8), (128256, 8), (128256, 16), (5000, 32)])
def test_topk_softmax(V, k, cuda):
    L = _lib()
    rows = 6
    g = torch.Generator(device="cuda").manual_seed(V + k)
    x = torch.randn(rows, V, device=cuda, generator=g) * 3
    x[0, 17] = x[0, 99] = 50.0  # exact tie -> token order
    tok = torch.zeros(rows, k, dtype=torch.int32, device=cuda)
    prob = torch.zeros(rows, k, dtype=torch.float64, device=cuda)
    ws = torch.empty(int(L.lib().ygg_topk_workspace(rows, V, k)), dtype=torch.uint8, device=cuda)
    L.check(L.lib().ygg_topk_softmax(x.data_ptr(), L.YGG_F32, rows, V, V, k, 1.0, tok.data_ptr(), prob.data_ptr(),
                                     None, ws.data_ptr(), ws.numel(), L.stream_ptr()))
    torch.cuda.synchronize()
    xc = x.cpu().numpy()
    for r in range(rows):
        ref = T.topk_softmax(xc[r], k)
        assert tok[r].cpu().tolist() == [t for t, _ in ref]
        np.testing.assert_allclose(prob[r].cpu().numpy(), [p for _, p in ref], rtol=1e-12)
        assert float(prob[r].sum()) <= 1.0 + 1e-9
    assert tok[0, 0].item() == 17 and tok[0, 1].item() == 99


# ---------------------------------------------------------------------------
# K1b grow_level, K7 build_mask vs the oracle (bit-exact)
# ---------------------------------------------------------------------------
def _random_cands(rng, n, k, vocab=1000):
    out = []
    for _ in range(n):
        cnt = int(rng.integers(0, k + 1))
        ps = np.sort(rng.dirichlet(np.ones(cnt + 1))[:cnt])[::-1] if cnt else []
        # a few exact ties to exercise the (score, parent, rank) order
        if cnt >= 2 and rng.random() < 0.3:
            ps = ps * 0.5
            ps[1] = ps[0]
        toks = rng.choice(vocab, size=cnt, replace=False)
        out.append([(int(t), float(p)) for t, p in zip(toks, ps)])
    return out


@pytest.mark.parametrize("seed", range(8))
def test_grow_levels_match_oracle(seed, cuda):
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    rng = np.random.default_rng(seed)
    B, D, W, k = 3, 5, int(rng.integers(1, 9)), 8
    cap = 1 + D * W
    dt = DeviceTrees(B, cap, cuda)
    refs = [T.Tree.root(int(rng.integers(0, 99)), float(rng.uniform(0.2, 1.0))) for _ in range(B)]
    dt.load_host([r.to_dict() for r in refs])
    stopped = [False] * B
    for _ in range(D):
        Fmax = max(len(r.levels()[-1]) for r in refs)
        ctok = torch.zeros(B, Fmax, k, dtype=torch.int32)
        cprob = torch.zeros(B, Fmax, k, dtype=torch.float64)
        cn = torch.zeros(B, Fmax, dtype=torch.int32)
        per = []
        for b, r in enumerate(refs):
            fr = r.levels()[-1]
            cands = _random_cands(rng, len(fr), k)
            per.append(dict(zip(fr, cands)))
            for f, cl in enumerate(cands):
                cn[b, f] = len(cl)
                for j, (t, p) in enumerate(cl):
                    ctok[b, f, j], cprob[b, f, j] = t, p
        ctok_d, cprob_d, cn_d = ctok.cuda(), cprob.cuda(), cn.cuda()  # keep alive across the async launch
        L.check(L.lib().ygg_egt_grow_level(dt.struct, Fmax, k, W, ctok_d.data_ptr(), cprob_d.data_ptr(),
                                           cn_d.data_ptr(), L.stream_ptr()))
        torch.cuda.synchronize()
        for b, r in enumerate(refs):
            if not stopped[b]:  # grow_egt stops after a level that added nothing (egt.py:145-146)
                stopped[b] = not T.grow_step(r, lambda tr, node, kk, b=b: per[b][node], W, k)
    torch.cuda.synchronize()
    got = dt.to_dicts()
    for b, r in enumerate(refs):
        assert got[b] == r.to_dict()
        np.testing.assert_array_equal(dt.masks_bool(b).numpy(), T.build_mask(r))


@pytest.mark.parametrize("seed", range(3))
def test_grow_wide_levels_match_oracle(seed, cuda):
    """cfg5 shape: D8 W16 k16 -> 129-node trees (5 mask words), candidate lists mostly full."""
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    rng = np.random.default_rng(50 + seed)
    B, D, W, k = 2, 8, 16, 16
    cap = 1 + D * W
    dt = DeviceTrees(B, cap, cuda)
    refs = [T.Tree.root(int(rng.integers(0, 99)), float(rng.uniform(0.2, 1.0))) for _ in range(B)]
    dt.load_host([r.to_dict() for r in refs])
    for _ in range(D):
        Fmax = max(len(r.levels()[-1]) for r in refs)
        ctok = torch.zeros(B, Fmax, k, dtype=torch.int32)
        cprob = torch.zeros(B, Fmax, k, dtype=torch.float64)
        cn = torch.zeros(B, Fmax, dtype=torch.int32)
        per = []
        for b, r in enumerate(refs):
            fr = r.levels()[-1]
            cands = []
            for _f in fr:
                ps = np.sort(rng.dirichlet(np.ones(k + 1))[:k])[::-1]
                if rng.random() < 0.3:  # exact score ties across parents / ranks
                    ps = ps * 0.5
                    ps[1] = ps[0]
                toks = rng.choice(128256, size=k, replace=False)
                cands.append([(int(t), float(p)) for t, p in zip(toks, ps)])
            per.append(dict(zip(fr, cands)))
            for f, cl in enumerate(cands):
                cn[b, f] = len(cl)
                for j, (t, p) in enumerate(cl):
                    ctok[b, f, j], cprob[b, f, j] = t, p
        ctok_d, cprob_d, cn_d = ctok.cuda(), cprob.cuda(), cn.cuda()
        L.check(L.lib().ygg_egt_grow_level(dt.struct, Fmax, k, W, ctok_d.data_ptr(), cprob_d.data_ptr(),
                                           cn_d.data_ptr(), L.stream_ptr()))
        torch.cuda.synchronize()
        for b, r in enumerate(refs):
            T.grow_step(r, lambda tr, node, kk, b=b: per[b][node], W, k)
    got = dt.to_dicts()
    for b, r in enumerate(refs):
        assert len(r) == cap
        assert got[b] == r.to_dict()
        np.testing.assert_array_equal(dt.masks_bool(b).numpy(), T.build_mask(r))


def test_grow_rejects_contract_violations(cuda):
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    dt = DeviceTrees(1, 8, cuda)
    dt.load_host([T.Tree.root(1, 1.0).to_dict()])
    ctok = torch.tensor([[[1, 2]]], dtype=torch.int32, device=cuda)
    cprob = torch.tensor([[[0.2, 0.5]]], dtype=torch.float64, device=cuda)  # not descending
    L.check(L.lib().ygg_egt_grow_level(dt.struct, 1, 2, 1, ctok.data_ptr(), cprob.data_ptr(), None, L.stream_ptr()))
    assert int(dt.flags[0]) & L.FLAG_CONTRACT
    assert int(dt.size[0]) == 1


# ---------------------------------------------------------------------------
# K6 knapsack + prune vs the oracle (bit-exact keep sets, w_verify, f64 aal/speedup)
# ---------------------------------------------------------------------------
def _random_tree(rng, n_max=40):
    t = T.Tree.root(0, float(rng.uniform(0.1, 1.0)))
    for i in range(int(rng.integers(0, n_max))):
        p = int(rng.integers(0, len(t)))
        room = 1.0 - sum(t.prob[c] for c in t.children(p))
        if room <= 0.02:
            continue
        t.add(p, i + 1, float(rng.uniform(0.01, 0.9)) * room)
    return t


def _profiles(rng):
    def prof():
        n = int(rng.integers(2, 5))
        ws = sorted(set(int(x) for x in rng.integers(1, 128, size=n)))
        if len(ws) < 2:
            ws = [1, 64]
        lat = np.cumsum(rng.uniform(0, 50, size=len(ws))) + rng.uniform(1, 50)
        return tuple((w, float(l)) for w, l in zip(ws, lat))

    return prof(), prof()


@pytest.mark.parametrize("seed", range(12))
def test_knapsack_prune_matches_oracle(seed, cuda):
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    rng = np.random.default_rng(100 + seed)
    B = 4
    trees = [_random_tree(rng, 60 if seed % 2 else 12) for _ in range(B)]
    dprof, vprof = _profiles(rng)
    max_verify = int(rng.integers(1, 40))
    d_draft, w_draft = 8, 8
    cap = 64
    dt = DeviceTrees(B, cap, cuda)
    dt.load_host([t.to_dict() for t in trees])
    probs = torch.zeros(B, cap, dtype=torch.float64)
    for b, t in enumerate(trees):
        probs[b, : len(t)] = torch.tensor(t.prob, dtype=torch.float64) * 0.97
    pp = torch.frombuffer(bytearray(L.profile_pair_bytes(dprof, vprof)), dtype=torch.uint8).cuda()
    i32 = dict(dtype=torch.int32, device=cuda)
    keep = torch.zeros(B, cap, **i32)
    new = torch.zeros(B, cap, **i32)
    wv = torch.zeros(B, **i32)
    aal = torch.zeros(B, dtype=torch.float64, device=cuda)
    sp = torch.zeros_like(aal)
    aal_cap = torch.zeros_like(aal)
    sp_cap = torch.zeros_like(aal)
    args = L.YggPruneArgs(max_verify, d_draft, w_draft, 0)
    probs_d = probs.cuda()
    L.check(L.lib().ygg_knapsack_prune(dt.struct, probs_d.data_ptr(), pp.data_ptr(), args, keep.data_ptr(),
                                       new.data_ptr(), wv.data_ptr(), aal.data_ptr(), sp.data_ptr(),
                                       aal_cap.data_ptr(), sp_cap.data_ptr(), None, None, L.stream_ptr()))
    torch.cuda.synchronize()
    for b, t in enumerate(trees):
        pr = T.prune_verify(t, probs[b, : len(t)].tolist(), dprof, vprof, d_draft, w_draft, max_verify)
        kept = [i for i in keep[b].tolist() if i >= 0]
        assert tuple(kept) == pr.kept
        assert int(wv[b]) == pr.w_verify
        assert float(aal[b]) == pr.expected_aal
        assert float(sp[b]) == pr.speedup
        dp = T.Knapsack(t, T.path_products(t, probs[b, : len(t)].tolist()), max_verify)
        assert float(aal_cap[b]) == 1.0 + dp.best[0][dp.cap]


@pytest.mark.parametrize("seed", range(4))
def test_knapsack_prune_129_nodes_cap_64(seed, cuda):
    """cfg3 / cfg5 shape: EGT trees of 129 nodes (D8 W16 / D16 W8), max_verify 64, surrogate gains."""
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    rng = np.random.default_rng(300 + seed)
    B = 3
    D, W = (8, 16) if seed % 2 == 0 else (16, 8)
    trees = []
    for _ in range(B):
        t = T.Tree.root(0, float(rng.uniform(0.5, 1.0)))
        for _lvl in range(D):
            cands = {}
            for f in t.levels()[-1]:
                ps = np.sort(rng.dirichlet(np.ones(17))[:16])[::-1]
                cands[f] = [(int(x), float(p)) for x, p in zip(rng.choice(10**6, 16, replace=False), ps)]
            T.grow_step(t, lambda tr, n, kk: cands[n], W, 16)
        assert len(t) == 129
        trees.append(t)
    cap = 129
    dprof = ((1, 400.0), (16, 410.0), (64, 430.0), (128, 470.0))
    vprof = ((1, 2400.0), (17, 2430.0), (65, 2600.0), (129, 3100.0))
    dt = DeviceTrees(B, cap, cuda)
    dt.load_host([t.to_dict() for t in trees])
    pp = torch.frombuffer(bytearray(L.profile_pair_bytes(dprof, vprof)), dtype=torch.uint8).cuda()
    i32 = dict(dtype=torch.int32, device=cuda)
    keep, new = torch.zeros(B, cap, **i32), torch.zeros(B, cap, **i32)
    wv = torch.zeros(B, **i32)
    aal = torch.zeros(B, dtype=torch.float64, device=cuda)
    sp = torch.zeros_like(aal)
    args = L.YggPruneArgs(64, D, W, 0)
    L.check(L.lib().ygg_knapsack_prune(dt.struct, None, pp.data_ptr(), args, keep.data_ptr(), new.data_ptr(),
                                       wv.data_ptr(), aal.data_ptr(), sp.data_ptr(), None, None, None, None,
                                       L.stream_ptr()))
    torch.cuda.synchronize()
    for b, t in enumerate(trees):
        pr = T.prune_verify(t, t.prob, dprof, vprof, D, W, 64)
        assert tuple(i for i in keep[b].tolist() if i >= 0) == pr.kept
        assert int(wv[b]) == pr.w_verify
        assert float(aal[b]) == pr.expected_aal
        assert float(sp[b]) == pr.speedup
        m = {old: i for i, old in enumerate(pr.kept)}
        assert [m.get(i, -1) for i in range(cap)] == new[b].tolist()


# ---------------------------------------------------------------------------
# K5 acceptance walk vs the oracle
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(6))
def test_accept_probs_matches_oracle(seed, cuda):
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    rng = np.random.default_rng(7 + seed)
    B, cap, nu = 5, 48, 12
    trees = [_random_tree(rng, 45) for _ in range(B)]
    dt = DeviceTrees(B, cap, cuda)
    dt.load_host([t.to_dict() for t in trees])
    probs = torch.zeros(B, cap, dtype=torch.float64)
    for b, t in enumerate(trees):
        probs[b, : len(t)] = torch.tensor(t.prob, dtype=torch.float64)
    uni = torch.from_numpy(rng.random((B, nu)))
    i32 = dict(dtype=torch.int32, device=cuda)
    path = torch.zeros(B, cap, **i32)
    plen = torch.zeros(B, **i32)
    alen = torch.zeros(B, **i32)
    nd = torch.zeros(B, **i32)
    probs_d, uni_d = probs.cuda(), uni.cuda()
    L.check(L.lib().ygg_accept(dt.struct, L.YGG_ACCEPT_PROBS, probs_d.data_ptr(), uni_d.data_ptr(), nu,
                               None, None, 0, 0, 0, None, 1.0, path.data_ptr(), plen.data_ptr(), alen.data_ptr(),
                               None, nd.data_ptr(), L.stream_ptr()))
    torch.cuda.synchronize()
    for b, t in enumerate(trees):
        rp, rl, used = T.sample_with_probs(t, probs[b, : len(t)].tolist(), iter(uni[b].tolist()))
        assert path[b, : int(plen[b])].tolist() == rp
        assert int(alen[b]) == rl
        assert int(nd[b]) == used


def _sample_oracle(t, lg, inv_t, uni):
    """SAMPLE acceptance in f64 (acceptance.py:208-241 with p = softmax(logits / T) of the parent's
    verify row): the walk, then the residual bonus by inverse CDF over the stop row with the rejected
    group's tokens removed."""
    x = lg.astype(np.float64) * inv_t
    lse = x.max(1) + np.log(np.exp(x - x.max(1, keepdims=True)).sum(1))
    path, cursor, used, excl = [], None, 0, []
    while True:
        group = [0] if cursor is None else t.children(cursor)
        if not group:
            excl = []
            break
        row = 0 if cursor is None else 1 + cursor
        u = uni[used]
        used += 1
        acc, chosen, excl = 0.0, None, []
        for c in group:
            excl.append(t.token[c])
            acc += float(np.exp(x[row, t.token[c]] - lse[row]))
            if u < acc:
                chosen = c
                break
        if chosen is None:
            break
        path.append(chosen)
        cursor = chosen
    stop = 0 if cursor is None else 1 + cursor
    p = np.exp(x[stop] - lse[stop])
    p[excl] = 0.0
    cum = np.cumsum(p)
    bonus = int(np.searchsorted(cum, uni[-1] * cum[-1], side="right"))
    return path, used, bonus


@pytest.mark.parametrize("with_stats", [False, True])
def test_accept_sample_vs_oracle(with_stats, cuda):
    """SAMPLE acceptance (tree walk with softmax(target / T) child probabilities + residual bonus) vs an
    f64 restatement, with the per-row log-sum-exp computed by the accept kernel itself (the engine's
    path) or passed in from ygg_row_stats.  The walk must match exactly; the residual draw inverts an
    f32-exponential CDF, so a draw within ~1e-6 of a token boundary may land on the neighbour (<= 1 of
    64 requests)."""
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    rng = np.random.default_rng(11 + with_stats)
    B, cap, V, nu, temp = 64, 48, 3000, 16, 0.7
    trees = [_random_tree(rng, 45) for _ in range(B)]
    dt = DeviceTrees(B, cap, cuda)
    dt.load_host([t.to_dict() for t in trees])
    rows = cap + 1
    lg = rng.standard_normal((B, rows, V)).astype(np.float32) * 2.0
    for b, t in enumerate(trees):  # make the walks go deep: each row favours one child of its node
        lg[b, 0, t.token[0]] += 9.0
        for n in range(len(t)):
            ch = t.children(n)
            if ch:
                lg[b, 1 + n, t.token[ch[int(rng.integers(0, len(ch)))]]] += float(rng.uniform(6.0, 10.0))
    uni = rng.random((B, nu))
    logits = torch.from_numpy(lg.reshape(B * rows, V)).to(cuda)
    uni_d = torch.from_numpy(uni).to(cuda)
    i32 = dict(dtype=torch.int32, device=cuda)
    path, plen, alen, bonus, nd = (torch.zeros(B, cap, **i32), torch.zeros(B, **i32), torch.zeros(B, **i32),
                                   torch.zeros(B, **i32), torch.zeros(B, **i32))
    stats = None
    if with_stats:
        stats = torch.zeros(B * rows, 2, device=cuda)
        am = torch.zeros(B * rows, **i32)
        L.check(L.lib().ygg_row_stats(logits.data_ptr(), L.YGG_F32, B * rows, V, V, temp, am.data_ptr(),
                                      stats.data_ptr(), L.stream_ptr()))
    L.check(L.lib().ygg_accept(dt.struct, L.YGG_ACCEPT_SAMPLE, None, uni_d.data_ptr(), nu, None, logits.data_ptr(),
                               L.YGG_F32, V, V, None if stats is None else stats.data_ptr(), temp, path.data_ptr(),
                               plen.data_ptr(), alen.data_ptr(), bonus.data_ptr(), nd.data_ptr(), L.stream_ptr()))
    torch.cuda.synchronize()
    miss = 0
    deep = 0
    for b, t in enumerate(trees):
        rp, used, rb = _sample_oracle(t, lg[b], 1.0 / temp, uni[b])
        assert path[b, : int(plen[b])].tolist() == rp, b
        assert int(alen[b]) == len(rp) + 1 and int(nd[b]) == used
        deep += len(rp) >= 2
        miss += int(bonus[b]) != rb
    assert miss <= 1
    assert deep >= B // 4  # the planted preferences make many walks accept several nodes


def test_accept_greedy_and_kv_compact(cuda):
    from paper_2512_23858_b200.device_tree import DeviceTrees

    L = _lib()
    rng = np.random.default_rng(5)
    B, cap = 3, 40
    trees = []
    for _ in range(B):
        t = T.Tree.root(int(rng.integers(0, 50)), 0.5)
        for _ in range(30):
            p = int(rng.integers(0, len(t)))
            used = {t.token[c] for c in t.children(p)}
            tok = int(rng.integers(0, 50))
            if tok in used:
                continue
            t.add(p, tok, 0.0)
        trees.append(t)
    dt = DeviceTrees(B, cap, cuda)
    dt.load_host([t.to_dict() for t in trees])
    T_rows = cap + 1
    argmax = torch.from_numpy(rng.integers(0, 50, size=(B, T_rows)).astype(np.int32))
    # plant a long accepted path in tree 0
    t0 = trees[0]
    node = 0
    argmax[0, 0] = t0.token[0]
    while t0.children(node):
        c = t0.children(node)[-1]
        argmax[0, 1 + node] = t0.token[c]
        node = c
    i32 = dict(dtype=torch.int32, device=cuda)
    path = torch.zeros(B, cap, **i32)
    plen = torch.zeros(B, **i32)
    alen = torch.zeros(B, **i32)
    bonus = torch.zeros(B, **i32)
    argmax_d = argmax.cuda()
    L.check(L.lib().ygg_accept(dt.struct, L.YGG_ACCEPT_GREEDY, None, None, 0, argmax_d.data_ptr(), None, 0, 0, 0,
                               None, 1.0, path.data_ptr(), plen.data_ptr(), alen.data_ptr(), bonus.data_ptr(), None,
                               L.stream_ptr()))
    torch.cuda.synchronize()
    for b, t in enumerate(trees):
        rp, rb = T.greedy_walk(t, argmax[b].tolist())
        assert path[b, : int(plen[b])].tolist() == rp
        assert int(bonus[b]) == rb
    assert int(plen[0]) >= 2
    # KV compaction of the accepted paths (2 layers, bf16)
    Ly, Hkv, S, hd = 2, 2, 128, 64
    cache = torch.randn(Ly, B, 2, Hkv, S, hd, device=cuda).to(torch.bfloat16)
    before = cache.clone()
    base = torch.tensor([10, 20, 30], **i32)
    L.check(L.lib().ygg_kv_compact(cache.data_ptr(), L.YGG_BF16, Ly, B, Hkv, S, hd, cache.stride(0), base.data_ptr(),
                                   path.data_ptr(), plen.data_ptr(), cap, None, 0, None, 0, 0, L.stream_ptr()))
    torch.cuda.synchronize()
    exp = before.clone()
    kx, vx = exp[:, :, 0], exp[:, :, 1].view(Ly, B, Hkv, hd, S)  # K [S][hd]; V^T [hd][S]
    kb, vb = before[:, :, 0], before[:, :, 1].view(Ly, B, Hkv, hd, S)
    for b in range(B):
        p = path[b, : int(plen[b])].tolist()
        src = [int(base[b]) + 1 + n for n in p]
        dst = [int(base[b]) + 1 + i for i in range(len(p))]
        if src:
            kx[:, b, :, dst] = kb[:, b, :, src]
            vx[:, b, :, :, dst] = vb[:, b, :, :, src]
    assert torch.equal(cache, exp)
