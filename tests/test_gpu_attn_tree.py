"""tcgen05 tree attention (csrc/attn_tree.cu) vs float64 attention over the visible keys, vs the
mma.sync decode attention, and the row-independence the lossless-greedy identity relies on.

Visible keys of a query token t of request b: the committed prefix [0, blk_start) plus the tree-block
keys its ancestor mask selects (causal without a mask) — token_tree.py:205-218 applied to the cache.
bf16 operands (Q, K, V, P) with f32 accumulation: tolerance 2e-2 of the output scale (north_star's
bf16 bound).  The merge order is fixed, so relaunches are bit-identical.
"""

import ctypes as C
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _tree_rows(T, kind="binary"):
    rows = []
    for i in range(T):
        par = -1 if i == 0 else ((i - 1) // 2 if kind == "binary" else i - 1)
        rows.append((rows[par] if par >= 0 else 0) | (1 << i))
    return rows


def _case(hd, Hq, Hkv, B, T, P, mw, cuda, seed=0):
    S = ((P + T + 63) // 64) * 64
    g = torch.Generator(device="cuda").manual_seed(1000 * hd + T + seed)
    q = torch.randn(B * T, Hq, hd, device=cuda, generator=g).to(torch.bfloat16)
    cache = torch.randn(B, 2, Hkv, S, hd, device=cuda, generator=g).to(torch.bfloat16)  # kv=1: V^T rows
    rows = _tree_rows(T)
    nwords = max(mw, 1)
    qmask = torch.tensor([[(rows[i] >> (32 * w)) & 0xFFFFFFFF for w in range(nwords)] for i in range(T)] * B,
                         dtype=torch.int64).to(torch.int32).to(cuda)
    return S, q, cache, rows, qmask


def _reference(q, cache, rows, B, T, P, mw, Hq, Hkv, hd, S):
    """float64 softmax(Q K^T / sqrt(hd)) V over each row's visible keys (vectorised over heads)."""
    G = Hq // Hkv
    K = cache[:, 0].double().cpu()                         # [B, Hkv, S, hd]
    V = cache[:, 1].double().cpu().reshape(B, Hkv, hd, S).transpose(2, 3)  # [B, Hkv, S, hd]
    qd = q.double().cpu().reshape(B, T, Hq, hd)
    vis = torch.zeros(T, S, dtype=torch.bool)
    vis[:, :P] = True
    for t in range(T):
        for j in range(T):
            if (mw and (rows[t] >> j) & 1) or (not mw and j <= t):
                vis[t, P + j] = True
    Kh = K.repeat_interleave(G, dim=1)                     # [B, Hq, S, hd]
    Vh = V.repeat_interleave(G, dim=1)
    s = torch.einsum("bthd,bhsd->bths", qd, Kh) / math.sqrt(hd)
    s = s.masked_fill(~vis[None, :, None, :], float("-inf"))
    return torch.einsum("bths,bhsd->bthd", torch.softmax(s, -1), Vh).reshape(B * T, Hq, hd)


def _tree_plan(lib, q, cache, B, T, Hq, Hkv, hd, S, csplit=0, row_tiles=0):
    from paper_2512_23858_b200 import _lib as L

    mem = C.create_string_buffer(int(lib.ygg_attn_tree_plan_size()))
    L.check(lib.ygg_attn_tree_plan_init(mem, q.data_ptr(), cache.data_ptr(), B, T, Hq, Hkv, hd, S, csplit, row_tiles))
    return mem


def _run_tree(lib, mem, bs, bl, qmask, mw, scale, out):
    from paper_2512_23858_b200 import _lib as L

    L.check(lib.ygg_attn_tree_run(mem, bs.data_ptr(), bl.data_ptr(), qmask.data_ptr() if mw else None, mw, scale,
                                  out.data_ptr(), L.stream_ptr()))


@pytest.mark.parametrize("hd,Hq,Hkv,B,T,P,mw", [
    (128, 32, 8, 1, 50, 512, 2),   # cfg2 verify
    (64, 32, 8, 1, 8, 300, 1),     # cfg2 draft level
    (128, 32, 8, 2, 16, 130, 1),
    (64, 8, 2, 1, 1, 77, 0),
    (128, 8, 2, 1, 5, 64, 0),
    (64, 32, 8, 2, 33, 90, 2),
    (128, 32, 8, 1, 40, 64, 0),
    (128, 32, 8, 1, 65, 700, 3),   # cfg3 widest verify (3 row tiles)
    (128, 32, 8, 1, 50, 2000, 2),  # several rounds per CTA
])
@pytest.mark.parametrize("csplit", [0, 1, 2, 4])
def test_tree_attention_vs_fp64(hd, Hq, Hkv, B, T, P, mw, csplit, cuda):
    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    S, q, cache, rows, qmask = _case(hd, Hq, Hkv, B, T, P, mw, cuda)
    bs = torch.full((B,), P, dtype=torch.int32, device=cuda)
    bl = torch.full((B,), T, dtype=torch.int32, device=cuda)
    out = torch.zeros(B * T, Hq, hd, dtype=torch.bfloat16, device=cuda)
    mem = _tree_plan(lib, q, cache, B, T, Hq, Hkv, hd, S, csplit)
    scale = 1.0 / math.sqrt(hd)
    outs = []
    for _ in range(2):
        _run_tree(lib, mem, bs, bl, qmask, mw, scale, out)
        outs.append(out.clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    ref = _reference(q, cache, rows, B, T, P, mw, Hq, Hkv, hd, S)
    err = (out.double().cpu() - ref).abs().max()
    assert err <= 2e-2 * ref.abs().max(), float(err)


@pytest.mark.parametrize("hd,T,P,mw", [(128, 50, 512, 2), (64, 8, 300, 1)])
def test_tree_attention_matches_decode_attention(hd, T, P, mw, cuda):
    """Same inputs through the tcgen05 tree kernel and the mma.sync decode kernel: equal to bf16
    rounding of P and the output (different reduction orders)."""
    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    Hq, Hkv, B = 32, 8, 1
    S, q, cache, rows, qmask = _case(hd, Hq, Hkv, B, T, P, mw, cuda, seed=5)
    bs = torch.full((B,), P, dtype=torch.int32, device=cuda)
    bl = torch.full((B,), T, dtype=torch.int32, device=cuda)
    scale = 1.0 / math.sqrt(hd)
    a = torch.zeros(B * T, Hq, hd, dtype=torch.bfloat16, device=cuda)
    b = torch.zeros_like(a)
    _run_tree(lib, _tree_plan(lib, q, cache, B, T, Hq, Hkv, hd, S), bs, bl, qmask, mw, scale, a)
    mem = C.create_string_buffer(int(lib.ygg_attn_dec_plan_size()))
    L.check(lib.ygg_attn_dec_plan_init(mem, q.data_ptr(), cache.data_ptr(), B, T, Hq, Hkv, hd, S, 0, 0, 0))
    L.check(lib.ygg_attn_dec_run(mem, bs.data_ptr(), bl.data_ptr(), qmask.data_ptr(), mw, scale, b.data_ptr(), None,
                                 L.stream_ptr()))
    torch.cuda.synchronize()
    scale_out = b.float().abs().max()
    assert (a.float() - b.float()).abs().max() <= 2e-2 * scale_out


@pytest.mark.parametrize("hd,T,P", [(128, 50, 530), (64, 8, 300)])
def test_tree_attention_rows_independent_of_pass_shape(hd, T, P, cuda):
    """A causal T-row pass and T separate 1-row passes (row t with the keys before it committed) give
    bit-identical rows: the key chunks are absolute, each row's scores / softmax / P V depend only on
    its own keys, and the merge order is fixed — the property the lossless spec == AR identity uses."""
    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    Hq, Hkv, B = 32, 8, 1
    S, q, cache, _, _ = _case(hd, Hq, Hkv, B, T, P, 0, cuda, seed=9)
    scale = 1.0 / math.sqrt(hd)
    full = torch.zeros(T, Hq, hd, dtype=torch.bfloat16, device=cuda)
    bs = torch.full((1,), P, dtype=torch.int32, device=cuda)
    bl = torch.full((1,), T, dtype=torch.int32, device=cuda)
    _run_tree(lib, _tree_plan(lib, q, cache, B, T, Hq, Hkv, hd, S, csplit=4), bs, bl, bs, 0, scale, full)
    q1 = torch.zeros(1, Hq, hd, dtype=torch.bfloat16, device=cuda)
    one = torch.zeros(1, Hq, hd, dtype=torch.bfloat16, device=cuda)
    mem1 = _tree_plan(lib, q1, cache, 1, 1, Hq, Hkv, hd, S, csplit=4)
    for t in (0, 1, T // 2, T - 1):
        q1.copy_(q[t:t + 1])
        bs.fill_(P + t)
        bl.fill_(1)
        _run_tree(lib, mem1, bs, bl, bs, 0, scale, one)
        torch.cuda.synchronize()
        assert torch.equal(one[0], full[t]), t


def test_tree_attention_wide_mask_129_nodes(cuda):
    """cfg5-shaped draft level: 16 rows of the newest level of a D8 W16 tree over a 129-key block
    (5 mask words) after a 300-token prefix, B = 2, vs float64."""
    from oracle import tree_ref as TR
    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    rng = np.random.default_rng(3)
    t = TR.Tree.root(0, 0.9)
    for _ in range(8):
        cands = {}
        for f in t.levels()[-1]:
            ps = np.sort(rng.dirichlet(np.ones(17))[:16])[::-1]
            cands[f] = [(int(x), float(p)) for x, p in zip(rng.choice(10**5, 16, replace=False), ps)]
        TR.grow_step(t, lambda tr, n, kk: cands[n], 16, 16)
    N = len(t)
    assert N == 129
    hd, Hq, Hkv, B, R, P, mw = 128, 32, 8, 2, 16, 300, 5
    masks = []
    for i in t.levels()[-1]:
        m = 0
        for a in t.path(i):
            m |= 1 << a
        masks.append(m)
    S = ((P + N + 63) // 64) * 64
    g = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn(B * R, Hq, hd, device=cuda, generator=g).to(torch.bfloat16)
    cache = torch.randn(B, 2, Hkv, S, hd, device=cuda, generator=g).to(torch.bfloat16)
    qmask = torch.tensor([[(m >> (32 * w)) & 0xFFFFFFFF for w in range(mw)] for m in masks] * B,
                         dtype=torch.int64).to(torch.int32).to(cuda)
    bs = torch.full((B,), P, dtype=torch.int32, device=cuda)
    bl = torch.full((B,), N, dtype=torch.int32, device=cuda)
    out = torch.zeros(B * R, Hq, hd, dtype=torch.bfloat16, device=cuda)
    scale = 1.0 / math.sqrt(hd)
    _run_tree(lib, _tree_plan(lib, q, cache, B, R, Hq, Hkv, hd, S), bs, bl, qmask, mw, scale, out)
    torch.cuda.synchronize()
    K = cache[:, 0].double().cpu()
    Vt = cache[:, 1].double().cpu().reshape(B, Hkv, hd, S)
    qd = q.double().cpu()
    ref = torch.zeros(B * R, Hq, hd, dtype=torch.float64)
    G = Hq // Hkv
    for b in range(B):
        for r, m in enumerate(masks):
            vis = torch.tensor(list(range(P)) + [P + j for j in range(N) if (m >> j) & 1])
            for h in range(Hq):
                s = K[b, h // G, vis] @ qd[b * R + r, h] * scale
                ref[b * R + r, h] = Vt[b, h // G][:, vis] @ torch.softmax(s, 0)
    err = (out.double().cpu() - ref).abs().max()
    assert err <= 2e-2 * ref.abs().max(), float(err)


def test_tree_attention_plan_rejects_bad_args(cuda):
    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    q = torch.zeros(8, 32, 128, dtype=torch.bfloat16, device=cuda)
    cache = torch.zeros(1, 2, 8, 128, 128, dtype=torch.bfloat16, device=cuda)
    mem = C.create_string_buffer(int(lib.ygg_attn_tree_plan_size()))
    with pytest.raises(ValueError):  # head dim
        L.check(lib.ygg_attn_tree_plan_init(mem, q.data_ptr(), cache.data_ptr(), 1, 8, 32, 8, 96, 128, 0, 0))
    for cs in (3, 8):  # cluster size
        with pytest.raises(ValueError):
            L.check(lib.ygg_attn_tree_plan_init(mem, q.data_ptr(), cache.data_ptr(), 1, 8, 32, 8, 128, 128, cs, 0))
    with pytest.raises(ValueError):  # S not a multiple of 64
        L.check(lib.ygg_attn_tree_plan_init(mem, q.data_ptr(), cache.data_ptr(), 1, 8, 32, 8, 128, 100, 0, 0))
    with pytest.raises(ValueError):  # 50 tokens x 4 heads do not fit one tile
        L.check(lib.ygg_attn_tree_plan_init(mem, q.data_ptr(), cache.data_ptr(), 1, 50, 32, 8, 128, 128, 0, 1))
