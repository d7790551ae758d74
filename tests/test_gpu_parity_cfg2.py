"""Production-path parity at the headline dimensions (cfg2: Llama-3-8B target / Llama-3.2-1B draft).

Models keep every cfg2 dimension (d, heads, kv heads, head_dim, ffn, V = 128256) but only 2 layers
each, so the fp32 CPU oracle (oracle/llama_ref.py, oracle/spec_ref.py) finishes in seconds.  Weights
are the cfg2 coupled synthetic weights generated on the CPU; the bf16 kernels get them rounded to
bf16 and the oracle gets the same rounded values in fp32, so only the kernels' arithmetic differs.

(a) the bf16 draft pass on the production kernels — row-block GEMV with the fused weight layout
    (folded RMSNorm, RoPE-pair-interleaved QKV, interleaved gate|up) and its fused epilogues (RoPE +
    KV append, residual + sums of squares, SwiGLU, LM head with the fused top-k partials + merge):
    logits within 2e-2 of the logit scale (north_star bf16 bound), appended KV within 2e-2, and the
    candidate lists equal to tree_ref.topk_softmax of the oracle logits wherever the top-(k+1) logit
    gaps exceed twice the measured logit error;
(b) the bf16 verify pass at T = 50 rows with a real EGT (D6 W8 k8) ancestor mask on the tcgen05
    GEMM + epilogues + decode-attention path: logits within 2e-2, argmax equal where the margin allows;
(c) the fp32 speculative step over 5 steps vs RefSpecDecoder: grown trees, kept sets, accepted paths
    and bonus tokens bit-exact; drafted probabilities within 5e-3 relative (f32 logits of magnitude
    ~50 summed over K = 4096 in another order differ by ~1e-5 relative, i.e. ~5e-4 in the logit).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

COUPLING = dict(rank=2048, logit_scale=16.0, head_noise=6.0, layer_gain=2.0)  # bench.py cfg2
DRAFT_PROF = ((1, 400.0), (64, 420.0), (128, 460.0))
VERIFY_PROF = ((1, 2400.0), (64, 2450.0), (128, 2600.0))
P0 = 256


@pytest.fixture(scope="module")
def pair():
    from paper_2512_23858_b200.model import Coupling, init_weights, preset, weights_to

    tc, dc = preset("llama3-8b", n_layers=2), preset("llama3.2-1b", n_layers=2)
    cp = Coupling(**COUPLING)
    tw = init_weights(tc, 0, torch.float32, "cpu", cp)
    dw = init_weights(dc, 1, torch.float32, "cpu", cp)
    # bf16-rounded values, held in fp32 for the oracle
    tw16 = weights_to(weights_to(tw, "cpu", torch.bfloat16), "cpu", torch.float32)
    dw16 = weights_to(weights_to(dw, "cpu", torch.bfloat16), "cpu", torch.float32)
    prompt = torch.randint(0, tc.vocab, (P0,), generator=torch.Generator().manual_seed(1000))
    return dict(tc=tc, dc=dc, tw=tw, dw=dw, tw16=tw16, dw16=dw16, prompt=prompt)


def _egt_tree(rng, D, W, k, vocab):
    """A real EGT shape: D grow steps (reference grow_step, egt.py:83-114) over random candidates."""
    from oracle import tree_ref as T

    t = T.Tree.root(int(rng.integers(vocab)), float(rng.uniform(0.3, 0.9)))
    for _ in range(D):
        cands = {}
        for f in t.levels()[-1]:
            ps = np.sort(rng.dirichlet(np.ones(k + 1))[:k])[::-1]
            cands[f] = [(int(x), float(p)) for x, p in zip(rng.choice(vocab, k, replace=False), ps)]
        T.grow_step(t, lambda tr, n, kk: cands[n], W, k)
    return t


def _rel_err(a, b):
    return float((a - b).abs().max() / b.abs().max())


def _oracle_prefill(model, cfg, S, prompt):
    from oracle.llama_ref import RefCache, causal_visible

    cache = RefCache(cfg, S)
    pos = list(range(len(prompt)))
    model.forward(cache, prompt.tolist(), pos, pos, causal_visible(len(prompt), S))
    return cache


def test_cfg2_draft_gemv_pass_vs_oracle(pair, cuda):
    import ctypes as C

    from oracle import tree_ref as T
    from oracle.llama_ref import RefLlama
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.forward import Forward, new_cache, prefill_causal
    from paper_2512_23858_b200.model import weights_to

    dc = pair["dc"]
    rng = np.random.default_rng(3)
    tree = _egt_tree(rng, 2, 8, 8, dc.vocab)  # root + 2 levels of 8 = 17 nodes
    n = len(tree)
    S = 512
    prompt = pair["prompt"]
    # ---- GPU: prefill (per-kernel path), then pass A (root + level 1, 9 rows) and pass B (level 2, 8
    # rows, fused top-k) on the row-block GEMV
    w = weights_to(pair["dw16"], cuda, torch.bfloat16)
    cache = new_cache(dc, 1, S, torch.bfloat16, cuda)
    prefill_causal(dc, w, cache, prompt[None].to(cuda, torch.int32), torch.bfloat16, False)
    lv = tree.levels()
    rows_a, rows_b = lv[0] + lv[1], lv[2]
    k = 8

    def run(rows, fuse):
        f = Forward(dc, w, cache, 1, len(rows), 1, torch.bfloat16)
        assert f.gemv
        f.tokens.copy_(torch.tensor([tree.token[i] for i in rows], dtype=torch.int32))
        f.pos.copy_(torch.tensor([P0 + 1 + tree.depth[i] for i in rows], dtype=torch.int32))
        f.slot.copy_(torch.tensor([P0 + 1 + i for i in rows], dtype=torch.int32))
        masks = []
        for i in rows:
            m = 0
            for a in tree.path(i):
                m |= 1 << a
            masks.append(m)
        f.qmask.copy_(torch.tensor([[m] for m in masks], dtype=torch.int64).to(torch.int32))
        f.blk_start.fill_(P0 + 1)
        f.blk_len.fill_(n)
        cand = None
        if fuse:
            assert f.fuse_topk(k)
        f.run()
        if fuse:
            tok = torch.zeros(len(rows), k, dtype=torch.int32, device=cuda)
            prob = torch.zeros(len(rows), k, dtype=torch.float64, device=cuda)
            L.check(L.lib().ygg_topk_merge(f.topk_part.data_ptr(), len(rows), f.topk_chunks, k, tok.data_ptr(),
                                           prob.data_ptr(), None, L.stream_ptr()))
            cand = (tok, prob)
        torch.cuda.synchronize()
        return f.logits.cpu().clone(), cand

    la, _ = run(rows_a, False)
    lb, (ctok, cprob) = run(rows_b, True)
    # ---- oracle: same rows, same slots and visibility, fp32
    ref = RefLlama(dc, pair["dw16"])
    rc = _oracle_prefill(ref, dc, S, prompt)

    def ref_pass(rows):
        vis = torch.zeros(len(rows), S, dtype=torch.bool)
        vis[:, : P0 + 1] = True
        for r, i in enumerate(rows):
            for a in tree.path(i):
                vis[r, P0 + 1 + a] = True
        return ref.forward(rc, [tree.token[i] for i in rows], [P0 + 1 + tree.depth[i] for i in rows],
                           [P0 + 1 + i for i in rows], vis)

    ra, rb = ref_pass(rows_a), ref_pass(rows_b)
    ea, eb = _rel_err(la, ra), _rel_err(lb, rb)
    assert ea <= 2e-2 and eb <= 2e-2, (ea, eb)
    # appended KV of the tree slots (K rows and V^T columns) vs the oracle cache
    for li in range(dc.n_layers):
        kg = cache[li, 0, 0].float().cpu()[:, P0 + 1 : P0 + 1 + n, :]
        vt = cache[li, 0, 1].float().cpu().reshape(dc.n_kv_heads, dc.head_dim, S)  # V^T rows [hd][S]
        vg = vt[:, :, P0 + 1 : P0 + 1 + n].transpose(1, 2)
        assert _rel_err(kg, rc.k[li][:, P0 + 1 : P0 + 1 + n]) <= 2e-2
        assert _rel_err(vg, rc.v[li][:, P0 + 1 : P0 + 1 + n]) <= 2e-2
    # fused top-k: exactly the oracle's softmax top-k of the GPU logits; against the oracle's own
    # logits, every rank whose separation from its neighbours exceeds twice this row's logit error
    # must hold the same token, and every token clearly inside the oracle's top-k must be drafted
    checked = 0
    for r in range(len(rows_b)):
        mine = T.topk_softmax(lb[r].numpy(), k)
        assert ctok[r].tolist() == [t for t, _ in mine]
        np.testing.assert_allclose(cprob[r].cpu().numpy(), [p for _, p in mine], rtol=1e-9, atol=1e-12)
        err = float((lb[r] - rb[r]).abs().max())
        ref_vals, ref_idx = torch.sort(rb[r], descending=True)
        vals, idx = ref_vals[: k + 1].numpy(), ref_idx[: k + 1].tolist()
        for j in range(k):
            below = vals[j] - vals[j + 1]
            above = vals[j - 1] - vals[j] if j > 0 else np.inf
            if min(below, above) > 2 * err:
                assert ctok[r, j].item() == idx[j], (r, j)
                checked += 1
            if vals[j] - vals[k] > 2 * err:
                assert idx[j] in ctok[r].tolist(), (r, j)
    assert checked >= len(rows_b)  # at least one separated rank per row on average (top-1 is)


def test_cfg2_verify_pass_vs_oracle(pair, cuda):
    from oracle.llama_ref import RefLlama
    from paper_2512_23858_b200.forward import Forward, new_cache, prefill_causal
    from paper_2512_23858_b200.model import weights_to

    tc = pair["tc"]
    rng = np.random.default_rng(5)
    tree = _egt_tree(rng, 6, 8, 8, tc.vocab)  # D6 W8: 49 nodes
    assert len(tree) == 49
    T_rows = len(tree) + 1
    S = 512
    prompt = pair["prompt"]
    w = weights_to(pair["tw16"], cuda, torch.bfloat16)
    cache = new_cache(tc, 1, S, torch.bfloat16, cuda)
    prefill_causal(tc, w, cache, prompt[None].to(cuda, torch.int32), torch.bfloat16, False)
    bonus = int(rng.integers(tc.vocab))
    tokens = [bonus] + tree.token
    pos = [P0] + [P0 + 1 + d for d in tree.depth]
    slots = [P0 + i for i in range(T_rows)]
    masks = [1]
    for i in range(len(tree)):
        m = 1
        for a in tree.path(i):
            m |= 1 << (1 + a)
        masks.append(m)
    f = Forward(tc, w, cache, 1, T_rows, 2, torch.bfloat16)
    assert not f.gemv
    f.tokens.copy_(torch.tensor(tokens, dtype=torch.int32))
    f.pos.copy_(torch.tensor(pos, dtype=torch.int32))
    f.slot.copy_(torch.tensor(slots, dtype=torch.int32))
    f.qmask.copy_(torch.tensor([[m & 0xFFFFFFFF, m >> 32] for m in masks], dtype=torch.int64).to(torch.int32))
    f.blk_start.fill_(P0)
    f.blk_len.fill_(T_rows)
    f.run()
    torch.cuda.synchronize()
    got = f.logits.cpu()
    ref = RefLlama(tc, pair["tw16"])
    rc = _oracle_prefill(ref, tc, S, prompt)
    vis = torch.zeros(T_rows, S, dtype=torch.bool)
    vis[:, :P0] = True
    for r, m in enumerate(masks):
        for j in range(T_rows):
            if (m >> j) & 1:
                vis[r, P0 + j] = True
    want = ref.forward(rc, tokens, pos, slots, vis)
    err = _rel_err(got, want)
    assert err <= 2e-2, err
    row_err = (got - want).abs().max(1).values
    top2 = want.topk(2, dim=1).values
    clear = (top2[:, 0] - top2[:, 1]) > 2 * row_err
    assert int(clear.sum()) >= T_rows // 2
    assert torch.equal(got.argmax(1)[clear], want.argmax(1)[clear])


def test_cfg2_fp32_step_trace_vs_oracle(pair, cuda):
    from oracle.llama_ref import RefLlama
    from oracle.spec_ref import RefSpecDecoder
    from oracle.tree_ref import Profile
    from paper_2512_23858_b200.engine import SpecDecoder, StepShape
    from paper_2512_23858_b200.model import weights_to

    tc, dc = pair["tc"], pair["dc"]
    prompt = pair["prompt"][:128]
    n_steps = 5
    S = 512

    class PP:
        drafter = Profile(DRAFT_PROF)
        verifier = Profile(VERIFY_PROF)

    ref = RefSpecDecoder(RefLlama(tc, pair["tw"]), RefLlama(dc, pair["dw"]), 6, 8, 8, 64, PP.drafter, PP.verifier, S)
    ref.prefill(prompt.tolist())
    for _ in range(n_steps):
        ref.step()
    sd = SpecDecoder(tc, weights_to(pair["tw"], cuda), dc, weights_to(pair["dw"], cuda), StepShape(6, 8, 8, 64),
                     batch=1, max_seq=S, act_dtype=torch.float32, profiles=PP)
    sd.prefill_len = len(prompt)
    sd.prefill(prompt[None])
    for i, rec in enumerate(ref.trace):
        sd.step(use_graph=False)
        torch.cuda.synchronize()
        grown = sd.grown.to_dicts()[0]
        assert [x["token"] for x in grown["nodes"]] == [x["token"] for x in rec["tree"]["nodes"]], f"step {i}"
        assert [x["parent"] for x in grown["nodes"]] == [x["parent"] for x in rec["tree"]["nodes"]], f"step {i}"
        for a, b in zip(grown["nodes"], rec["tree"]["nodes"]):
            assert abs(a["prob"] - b["prob"]) <= 5e-3 * max(b["prob"], 1e-6), f"step {i}"
        assert [x for x in sd.keep_idx[0].tolist() if x >= 0] == rec["kept"], f"step {i}"
        assert sd.path[0, : int(sd.path_len[0])].tolist() == rec["path"], f"step {i}"
        assert int(sd.bonus[0]) == rec["bonus"], f"step {i}"
    n = len(ref.hist) - len(prompt)
    assert sd.generated(0)[:n] == ref.hist[len(prompt):]


def test_cfg2_verify_pass_cluster_fused_vs_oracle(pair, cuda):
    """The verify forward with the fused weight layout and cluster split-K GEMMs (QKV / O / down:
    DSMEM-reduced partials, RoPE + KV append / residual + sums of squares applied by the cluster
    leader; gate|up and the LM head stream-K fused): logits within 2e-2 of the fp32 oracle on the same
    T = 50 EGT verify rows as the per-kernel path."""
    from oracle.llama_ref import RefLlama
    from paper_2512_23858_b200.forward import Forward, new_cache, prefill_causal
    from paper_2512_23858_b200.model import weights_to
    from paper_2512_23858_b200.plan import ForwardPlan

    tc = pair["tc"]
    rng = np.random.default_rng(5)
    tree = _egt_tree(rng, 6, 8, 8, tc.vocab)
    T_rows = len(tree) + 1
    S = 512
    prompt = pair["prompt"]
    w = weights_to(pair["tw16"], cuda, torch.bfloat16)
    cache = new_cache(tc, 1, S, torch.bfloat16, cuda)
    prefill_causal(tc, w, cache, prompt[None].to(cuda, torch.int32), torch.bfloat16, False)
    bonus = int(rng.integers(tc.vocab))
    tokens = [bonus] + tree.token
    pos = [P0] + [P0 + 1 + d for d in tree.depth]
    slots = [P0 + i for i in range(T_rows)]
    masks = [1]
    for i in range(len(tree)):
        m = 1
        for a in tree.path(i):
            m |= 1 << (1 + a)
        masks.append(m)
    f = Forward(tc, w, cache, 1, T_rows, 2, torch.bfloat16, plan=ForwardPlan(fused_epilogues=True))
    assert f.fused and [p["qkv"].cluster for p in f.plans] == [2, 2] and f.plans[0]["o"].cluster == 4
    assert f.plans[0]["down"].cluster == 4
    f.tokens.copy_(torch.tensor(tokens, dtype=torch.int32))
    f.pos.copy_(torch.tensor(pos, dtype=torch.int32))
    f.slot.copy_(torch.tensor(slots, dtype=torch.int32))
    f.qmask.copy_(torch.tensor([[m & 0xFFFFFFFF, m >> 32] for m in masks], dtype=torch.int64).to(torch.int32))
    f.blk_start.fill_(P0)
    f.blk_len.fill_(T_rows)
    f.run()
    torch.cuda.synchronize()
    got = f.logits.cpu().clone()
    f.run()  # relaunch: bit-identical (fixed reduction order)
    torch.cuda.synchronize()
    assert torch.equal(f.logits.cpu(), got)
    ref = RefLlama(tc, pair["tw16"])
    rc = _oracle_prefill(ref, tc, S, prompt)
    vis = torch.zeros(T_rows, S, dtype=torch.bool)
    vis[:, :P0] = True
    for r, m in enumerate(masks):
        for j in range(T_rows):
            if (m >> j) & 1:
                vis[r, P0 + j] = True
    want = ref.forward(rc, tokens, pos, slots, vis)
    err = _rel_err(got, want)
    assert err <= 2e-2, err


@pytest.mark.parametrize("fused_gemm", [False, True])
def test_cfg2_draft_prefill_fused_layout_vs_oracle(pair, cuda, fused_gemm):
    """Causal prefill of the 1B-dims draft on fused-layout weights (RoPE-pair-interleaved QKV rows,
    interleaved gate|up rows, folded norms) — the path every draft prefill takes: stream-K GEMMs with
    the layout-aware QKV / SwiGLU epilogue kernels (ygg_gemm_plan_set_layout), causal tree attention and
    the last-row LM head (default), or the fused-epilogue GEMMs (fused_layout_gemm).  The last row's
    logits within 2e-2 of the fp32 oracle, the whole prompt's K / V within 2e-2."""
    from oracle.llama_ref import RefLlama
    from paper_2512_23858_b200.forward import new_cache, prefill_causal
    from paper_2512_23858_b200.model import prepare_fused_, weights_to
    from paper_2512_23858_b200.plan import ForwardPlan

    dc = pair["dc"]
    S, n = 512, P0
    prompt = pair["prompt"]
    w = prepare_fused_(weights_to(pair["dw16"], cuda, torch.bfloat16), dc)
    cache = new_cache(dc, 1, S, torch.bfloat16, cuda)
    fwd = {}
    last = prefill_causal(dc, w, cache, prompt[None].to(cuda, torch.int32), torch.bfloat16, True, fwd,
                          plan=ForwardPlan(fused_layout_gemm=fused_gemm))
    f = next(iter(fwd.values()))
    assert f.layout_fused and f.fused == fused_gemm and f.last_logits and f.at_plans is not None
    got = last.cpu()
    assert got.shape == (1, dc.vocab)
    ref = RefLlama(dc, pair["dw16"])
    from oracle.llama_ref import RefCache, causal_visible

    rc = RefCache(dc, S)
    pos = list(range(n))
    want = ref.forward(rc, prompt.tolist(), pos, pos, causal_visible(n, S))[-1:]
    err = _rel_err(got, want)
    assert err <= 2e-2, err
    for li in range(dc.n_layers):
        kg = cache[li, 0, 0].float().cpu()[:, :n, :]
        vg = cache[li, 0, 1].float().cpu().reshape(dc.n_kv_heads, dc.head_dim, S)[:, :, :n].transpose(1, 2)
        assert _rel_err(kg, rc.k[li][:, :n]) <= 2e-2
        assert _rel_err(vg, rc.v[li][:, :n]) <= 2e-2


def test_cfg5_dims_batched_verify_vs_oracle(cuda):
    """The batched verify at the cfg5 target's dimensions (Llama-3-70B: d 8192, 64 query / 8 kv heads,
    ffn 28672, V 128256; 2 layers): two requests, each verifying 65 rows (the bonus + the first 64
    nodes of a D8 W16 k16 EGT: 3 mask words, 8 query heads per kv head on the tree attention's
    single-CTA long-context path) against the fp32 oracle within 2e-2; argmax equal where the margin
    allows."""
    from oracle.llama_ref import RefCache, RefLlama, causal_visible
    from paper_2512_23858_b200.forward import Forward, new_cache, prefill_causal
    from paper_2512_23858_b200.model import Coupling, init_weights, preset, weights_to

    tc = preset("llama3-70b", n_layers=2)
    w32 = init_weights(tc, 7, torch.float32, "cpu", Coupling(**COUPLING))
    w16 = weights_to(weights_to(w32, "cpu", torch.bfloat16), "cpu", torch.float32)
    del w32
    B, P = 2, 192
    S = 512
    rng = np.random.default_rng(11)
    prompts = torch.randint(0, tc.vocab, (B, P), generator=torch.Generator().manual_seed(77))
    trees = []
    for b in range(B):
        full = _egt_tree(rng, 8, 16, 16, tc.vocab)  # 129 nodes; nodes are added level by level,
        trees.append(full)                          # so the first 64 form a connected subtree
    n_nodes = 64
    T_rows = n_nodes + 1
    mw = (T_rows + 31) // 32
    w = weights_to(w16, cuda, torch.bfloat16)
    cache = new_cache(tc, B, S, torch.bfloat16, cuda)
    prefill_causal(tc, w, cache, prompts.to(cuda, torch.int32), torch.bfloat16, False)
    f = Forward(tc, w, cache, B, T_rows, mw, torch.bfloat16)
    assert not f.gemv and f.at_plans is not None
    tokens, pos, slots, masks, bonuses = [], [], [], [], []
    for b, tree in enumerate(trees):
        bonus = int(rng.integers(tc.vocab))
        bonuses.append(bonus)
        tokens += [bonus] + tree.token[:n_nodes]
        pos += [P] + [P + 1 + d for d in tree.depth[:n_nodes]]
        slots += [P + i for i in range(T_rows)]
        masks.append(1)
        for i in range(n_nodes):
            m = 1
            for a in tree.path(i):
                m |= 1 << (1 + a)
            masks.append(m)
    f.tokens.copy_(torch.tensor(tokens, dtype=torch.int32))
    f.pos.copy_(torch.tensor(pos, dtype=torch.int32))
    f.slot.copy_(torch.tensor(slots, dtype=torch.int32))
    words = [[(m >> (32 * k)) & 0xFFFFFFFF for k in range(mw)] for m in masks]
    f.qmask.copy_(torch.tensor(words, dtype=torch.int64).to(torch.int32))
    f.blk_start.fill_(P)
    f.blk_len.fill_(T_rows)
    f.run()
    torch.cuda.synchronize()
    got = f.logits.cpu().view(B, T_rows, -1)
    ref = RefLlama(tc, w16)
    for b in range(B):
        rc = RefCache(tc, S)
        pp = list(range(P))
        ref.forward(rc, prompts[b].tolist(), pp, pp, causal_visible(P, S))
        vis = torch.zeros(T_rows, S, dtype=torch.bool)
        vis[:, :P] = True
        for r, m in enumerate(masks[b * T_rows:(b + 1) * T_rows]):
            for j in range(T_rows):
                if (m >> j) & 1:
                    vis[r, P + j] = True
        want = ref.forward(rc, tokens[b * T_rows:(b + 1) * T_rows], pos[b * T_rows:(b + 1) * T_rows],
                           slots[b * T_rows:(b + 1) * T_rows], vis)
        err = _rel_err(got[b], want)
        assert err <= 2e-2, (b, err)
        row_err = (got[b] - want).abs().max(1).values
        top2 = want.topk(2, dim=1).values
        clear = (top2[:, 0] - top2[:, 1]) > 2 * row_err
        assert int(clear.sum()) >= T_rows // 2
        assert torch.equal(got[b].argmax(1)[clear], want.argmax(1)[clear])
