"""Fused tcgen05 GEMM epilogues vs torch fp64 references of the same bf16 operands.

Covers single-segment tiles (finished from TMEM), multi-segment stream-K tiles (last-arrival
reduction), via different CTA counts, and cluster split-K plans ("cN": N CTAs per tile, partials
reduced through DSMEM in the cluster's leader).  Tolerance: 2e-3 relative to the output scale (bf16
operands are exact; f32 accumulation order differs), and bf16 rounding of stored outputs.
"""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _plan(W, X, M, ctas):
    """ctas: stream-K CTA count (0 = default), or "cN" = cluster split-K with N CTAs per tile."""
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.forward import GemmPlan

    if isinstance(ctas, str):
        p = GemmPlan(W, X, M, 0)
        rc = L.lib().ygg_gemm_plan_set_cluster(p.handle, int(ctas[1:]))
        if rc == L.YGG_ERR_UNSUPPORTED:  # more tiles than co-resident clusters (wide token counts)
            pytest.skip("cluster shape does not fit one wave")
        L.check(rc)
        assert L.lib().ygg_gemm_plan_cluster(p.handle) == int(ctas[1:])
        return p
    return GemmPlan(W, X, M, ctas)


def _run(plan, epi, cuda):
    from paper_2512_23858_b200 import _lib as L
    import ctypes as C

    ws = torch.zeros(plan.ws_bytes // 4 + 16, device=cuda)
    L.check(L.lib().ygg_gemm_fused(plan.handle, ws.data_ptr(), C.byref(epi), L.stream_ptr()))
    torch.cuda.synchronize()


def _epi(kind, counters, **kw):
    from paper_2512_23858_b200 import _lib as L

    e = L.YggEpilogue()
    e.kind = kind
    e.counters = counters.data_ptr()
    for k, v in kw.items():
        setattr(e, k, v)
    return e


@pytest.mark.parametrize("ctas", [0, 5, 37, "c1", "c2", "c3", "c4"])
@pytest.mark.parametrize("M", [8, 50, 300, 800])
def test_store_f32_with_rstd(ctas, M, cuda):
    from paper_2512_23858_b200 import _lib as L

    N, K = 1024, 512
    g = torch.Generator(device="cuda").manual_seed(M + len(str(ctas)))
    X = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device=cuda, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    ss = torch.rand(4, M, device=cuda, generator=g) * 100
    out = torch.zeros(M, N, device=cuda)
    try:
        plan = _plan(W, X, M, ctas)
    except ValueError as exc:  # wide token tiles: the cluster's receive slots may leave no room for a ring
        assert ctas in ("c3", "c4") and M > 256 and "ring" in str(exc)
        return
    cnt = torch.zeros(plan.tiles, dtype=torch.int32, device=cuda)
    _run(plan, _epi(L.YGG_EPI_STORE_F32, cnt, ss_in=ss.data_ptr(), ss_tiles=4, norm_dim=512, eps=1e-5,
                    out=out.data_ptr(), ld=N), cuda)
    rstd = torch.rsqrt(ss.double().sum(0) / 512 + 1e-5)
    ref = (X.double() @ W.double().T) * rstd[:, None]
    assert (out.double() - ref).abs().max() <= 2e-3 * ref.abs().max()
    # epoch counters: a second launch of the same plan reproduces the result bit-for-bit
    first = out.clone()
    out.zero_()
    _run(plan, _epi(L.YGG_EPI_STORE_F32, cnt, ss_in=ss.data_ptr(), ss_tiles=4, norm_dim=512, eps=1e-5,
                    out=out.data_ptr(), ld=N), cuda)
    assert torch.equal(out, first)


@pytest.mark.parametrize("M", [40, 800])
@pytest.mark.parametrize("ctas", [0, 11, "c2", "c4"])
def test_resid_and_swiglu(ctas, M, cuda):
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.model import gate_up_interleave, preset

    d, F = 512, 768
    g = torch.Generator(device="cuda").manual_seed(len(str(ctas)) + 3)
    # RESID: resid += X W^T, hb = bf16(resid), ss per 128-feature tile
    X = torch.randn(M, F, device=cuda, generator=g).to(torch.bfloat16)
    W = (torch.randn(d, F, device=cuda, generator=g) / math.sqrt(F)).to(torch.bfloat16)
    resid = torch.randn(M, d, device=cuda, generator=g)
    r0 = resid.clone()
    hb = torch.zeros(M, d, dtype=torch.bfloat16, device=cuda)
    ss = torch.zeros(d // 128, M, device=cuda)
    plan = _plan(W, X, M, ctas)
    cnt = torch.zeros(plan.tiles, dtype=torch.int32, device=cuda)
    _run(plan, _epi(L.YGG_EPI_RESID, cnt, resid=resid.data_ptr(), hb=hb.data_ptr(), ss_out=ss.data_ptr()), cuda)
    ref = r0.double() + X.double() @ W.double().T
    assert (resid.double() - ref).abs().max() <= 2e-3 * ref.abs().max()
    assert torch.equal(hb, resid.to(torch.bfloat16))
    ref_ss = (resid.double() ** 2).view(M, d // 128, 128).sum(-1).T
    assert torch.allclose(ss.double(), ref_ss, rtol=1e-5)
    # SWIGLU with interleaved gate/up rows
    cfg = preset("tiny-target", ffn=F, d_model=d)
    Xs = torch.randn(M, d, device=cuda, generator=g).to(torch.bfloat16)
    Wgu = (torch.randn(2 * F, d, device=cuda, generator=g) / math.sqrt(d)).to(torch.bfloat16)
    Wp = Wgu[gate_up_interleave(cfg).to(cuda)].contiguous()
    act = torch.zeros(M, F, dtype=torch.bfloat16, device=cuda)
    plan2 = _plan(Wp, Xs, M, ctas)
    cnt2 = torch.zeros(plan2.tiles, dtype=torch.int32, device=cuda)
    _run(plan2, _epi(L.YGG_EPI_SWIGLU, cnt2, act_out=act.data_ptr()), cuda)
    gu = Xs.double() @ Wgu.double().T
    ref2 = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    assert (act.double() - ref2).abs().max() <= 1e-2 * ref2.abs().max()


@pytest.mark.parametrize("M", [12, 800])
@pytest.mark.parametrize("hd,Hq,Hkv", [(64, 4, 2), (128, 8, 2)])
@pytest.mark.parametrize("ctas", [0, 9, "c3", "c4"])
def test_qkv_rope_kv_append(hd, Hq, Hkv, ctas, M, cuda):
    from oracle.llama_ref import rope
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.model import preset, qkv_row_permutation, rope_table

    d, B = 256, 2
    S = 64 if M < 100 else 512
    cfg = preset("tiny-target", d_model=d, n_heads=Hq, n_kv_heads=Hkv, head_dim=hd)
    g = torch.Generator(device="cuda").manual_seed(hd + len(str(ctas)))
    X = torch.randn(M, d, device=cuda, generator=g).to(torch.bfloat16)
    W = (torch.randn(cfg.qkv_dim, d, device=cuda, generator=g) / math.sqrt(d)).to(torch.bfloat16)
    Wp = W[qkv_row_permutation(cfg).to(cuda)].contiguous()
    # token metadata as views whose tails are poisoned: a load past row M - 1 (the token tile's rows
    # beyond M) would index the RoPE table / cache far out of bounds and fault
    pos = torch.full((M + 64,), 1 << 30, device=cuda, dtype=torch.int32)[:M]
    pos.copy_(torch.randint(0, 1000, (M,), device=cuda, dtype=torch.int32))
    slot = torch.full((M + 64,), 1 << 30, device=cuda, dtype=torch.int32)[:M]
    slot.copy_(torch.arange(M, device=cuda, dtype=torch.int32) % (M // B) + 5)
    req = torch.full((M + 64,), 1 << 20, device=cuda, dtype=torch.int32)[:M]
    req.copy_(torch.arange(M, device=cuda, dtype=torch.int32) // (M // B))
    rope_cs = rope_table(cfg, 1000, cuda) if M >= 100 else None  # the table path (Forward's) and sincos
    q = torch.zeros(M, Hq, hd, dtype=torch.bfloat16, device=cuda)
    cache = torch.zeros(B, 2, Hkv, S, hd, dtype=torch.bfloat16, device=cuda)
    plan = _plan(Wp, X, M, ctas)
    cnt = torch.zeros(plan.tiles, dtype=torch.int32, device=cuda)
    _run(plan, _epi(L.YGG_EPI_QKV_ROPE, cnt, q_out=q.data_ptr(), cache=cache.data_ptr(), S=S, Hq=Hq, Hkv=Hkv,
                    hd=hd, rope_theta=cfg.rope_theta, pos=pos.data_ptr(), slot=slot.data_ptr(),
                    req=req.data_ptr(), rope_cs=0 if rope_cs is None else rope_cs.data_ptr()), cuda)
    y = (X.double() @ W.double().T).float().cpu()
    qr = rope(y[:, : Hq * hd].view(M, Hq, hd), pos.cpu(), cfg.rope_theta)
    kr = rope(y[:, Hq * hd : (Hq + Hkv) * hd].view(M, Hkv, hd), pos.cpu(), cfg.rope_theta)
    v = y[:, (Hq + Hkv) * hd :].view(M, Hkv, hd)
    tol = 2e-2 * float(y.abs().max())
    assert (q.float().cpu() - qr).abs().max() <= tol
    c = cache.float().cpu()
    for m in range(M):
        b, s = int(req[m]), int(slot[m])
        assert (c[b, 0, :, s, :] - kr[m]).abs().max() <= tol
        vt = c[b, 1].reshape(Hkv, hd, S)[:, :, s]  # V^T [hd][S]
        assert (vt - v[m]).abs().max() <= tol


@pytest.mark.parametrize("ctas", [0, 7, 37])
@pytest.mark.parametrize("M", [1, 50, 130])
def test_argmax_epilogue_equals_argmax_of_stored_logits(ctas, M, cuda):
    """YGG_EPI_ARGMAX (greedy LM head: per-tile first-maximum keys, no logits) + ygg_argmax_reduce ==
    the first argmax of the STORE_F32 logits of the same plan, including exact ties (duplicated
    weight rows) across and inside tiles, split and whole stream-K tiles."""
    from paper_2512_23858_b200 import _lib as L

    N, K = 4096, 512
    g = torch.Generator(device="cuda").manual_seed(M + ctas)
    X = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device=cuda, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    W[3000] = W[77]   # a tie across tiles: the lower index must win
    W[78] = W[77]     # and inside a tile
    out = torch.zeros(M, N, device=cuda)
    plan = _plan(W, X, M, ctas)
    cnt = torch.zeros(plan.tiles, dtype=torch.int32, device=cuda)
    _run(plan, _epi(L.YGG_EPI_STORE_F32, cnt, out=out.data_ptr(), ld=N), cuda)
    keys = torch.zeros(N // 128, M, dtype=torch.int64, device=cuda)
    cnt2 = torch.zeros(plan.tiles, dtype=torch.int32, device=cuda)
    _run(plan, _epi(L.YGG_EPI_ARGMAX, cnt2, out=keys.data_ptr(), ld=N), cuda)
    am = torch.zeros(M, dtype=torch.int32, device=cuda)
    L.check(L.lib().ygg_argmax_reduce(keys.data_ptr(), N // 128, M, am.data_ptr(), L.stream_ptr()))
    torch.cuda.synchronize()
    want = torch.tensor([int(torch.nonzero(r == r.max())[0]) for r in out.cpu()], dtype=torch.int32)
    assert torch.equal(am.cpu(), want)
    assert not (am.cpu() == 78).any() and not (am.cpu() == 3000).any()
