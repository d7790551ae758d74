"""Prologue epilogues (ygg_gemm_plan_set_prologue): the previous GEMM's f32 partials finished into this
GEMM's X by the epilogue warps of all its CTAs, published through an epoch arrival counter.

Checked against fp64 torch references of the same bf16 operands (2e-3 of the output scale): RESID
(X = bf16(resid += prev), per-block sums of squares), SWIGLU (X = bf16(silu(g r) (u r)) with the rstd
from sums of squares), over several stream-K CTA counts and three consecutive launches (the epochs must
advance without any reset), plus the argument checks.
"""

import ctypes as C
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _pro(kind, prev, pws, **kw):
    from paper_2512_23858_b200 import _lib as L

    q = L.YggPrologue()
    q.kind = kind
    q.prev_plan = C.addressof(prev.handle)
    q.prev_ws = pws.data_ptr()
    for k, v in kw.items():
        setattr(q, k, v)
    return q


def _run(plan, ws):
    from paper_2512_23858_b200 import _lib as L

    L.check(L.lib().ygg_gemm_run(plan.handle, ws.data_ptr(), L.stream_ptr()))


def _store(plan, ws, M, N, cuda):
    from paper_2512_23858_b200 import _lib as L

    out = torch.zeros(M, N, device=cuda)
    L.check(L.lib().ygg_epi_store(plan.handle, ws.data_ptr(), out.data_ptr(), L.YGG_F32, N, L.stream_ptr()))
    return out


@pytest.mark.parametrize("ctas", [0, 7, 64])
@pytest.mark.parametrize("M", [1, 50, 130])
def test_resid_prologue(ctas, M, cuda):
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.forward import GemmPlan

    K0, D, N1 = 512, 1024, 384  # prev: [M, K0] x [D, K0]^T -> D features; next: [M, D] x [N1, D]^T
    g = torch.Generator(device="cuda").manual_seed(M * 7 + ctas)
    X0 = torch.randn(M, K0, device=cuda, generator=g).to(torch.bfloat16)
    W0 = (torch.randn(D, K0, device=cuda, generator=g) / math.sqrt(K0)).to(torch.bfloat16)
    W1 = (torch.randn(N1, D, device=cuda, generator=g) / math.sqrt(D)).to(torch.bfloat16)
    X1 = torch.zeros(M, D, dtype=torch.bfloat16, device=cuda)
    resid0 = torch.randn(M, D, device=cuda, generator=g)
    resid = resid0.clone()
    ss = torch.zeros(D // 64, M, device=cuda)
    state = torch.zeros(D // 64 + 148, dtype=torch.int32, device=cuda)
    p0, p1 = GemmPlan(W0, X0, M, ctas), GemmPlan(W1, X1, M, ctas)
    ws0 = torch.zeros(p0.ws_bytes // 4 + 16, device=cuda)
    ws1 = torch.zeros(p1.ws_bytes // 4 + 16, device=cuda)
    q = _pro(L.YGG_PRO_RESID, p0, ws0, resid=resid.data_ptr(), ss_out=ss.data_ptr(),
             flags=state.data_ptr(), launches=state.data_ptr() + 4 * (D // 64))
    L.check(L.lib().ygg_gemm_plan_set_prologue(p1.handle, C.byref(q)))
    prev = (X0.double() @ W0.double().T)
    want_resid = resid0.double()
    outs = []
    for launch in range(3):  # epochs advance launch after launch; resid accumulates prev each time
        _run(p0, ws0)
        _run(p1, ws1)
        outs.append(_store(p1, ws1, M, N1, cuda))
        torch.cuda.synchronize()
        want_resid = want_resid + prev
        x_ref = want_resid.float().to(torch.bfloat16)
        assert (resid.double() - want_resid).abs().max() <= 2e-3 * want_resid.abs().max(), launch
        assert torch.equal(X1, resid.to(torch.bfloat16)), launch
        y_ref = x_ref.double() @ W1.double().T
        assert (outs[-1].double() - y_ref).abs().max() <= 2e-3 * y_ref.abs().max(), launch
        ss_ref = (resid.double() ** 2).reshape(M, D // 64, 64).sum(-1).T
        assert (ss.double() - ss_ref).abs().max() <= 1e-4 * ss_ref.abs().max(), launch
    launches = state[D // 64:]
    grid = int((launches > 0).sum())
    assert int(launches.max()) == 3 and int(launches.min()) == 0 and int(state[0]) == 3 * grid


@pytest.mark.parametrize("ctas", [0, 9])
@pytest.mark.parametrize("M", [8, 50])
def test_swiglu_prologue(ctas, M, cuda):
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.forward import GemmPlan

    K0, F, N1 = 256, 640, 256  # prev: gate|up [2F, K0]; next: [N1, F]
    g = torch.Generator(device="cuda").manual_seed(M + 31 * ctas)
    X0 = torch.randn(M, K0, device=cuda, generator=g).to(torch.bfloat16)
    W0 = (torch.randn(2 * F, K0, device=cuda, generator=g) / math.sqrt(K0)).to(torch.bfloat16)
    W1 = (torch.randn(N1, F, device=cuda, generator=g) / math.sqrt(F)).to(torch.bfloat16)
    X1 = torch.zeros(M, F, dtype=torch.bfloat16, device=cuda)
    ss_in = torch.rand(6, M, device=cuda, generator=g) * 50 + 1
    state = torch.zeros(F // 64 + 148, dtype=torch.int32, device=cuda)
    p0, p1 = GemmPlan(W0, X0, M, ctas), GemmPlan(W1, X1, M, ctas)
    ws0 = torch.zeros(p0.ws_bytes // 4 + 16, device=cuda)
    ws1 = torch.zeros(p1.ws_bytes // 4 + 16, device=cuda)
    q = _pro(L.YGG_PRO_SWIGLU, p0, ws0, ss_in=ss_in.data_ptr(), ss_tiles=6, norm_dim=384, eps=1e-5,
             flags=state.data_ptr(), launches=state.data_ptr() + 4 * (F // 64))
    L.check(L.lib().ygg_gemm_plan_set_prologue(p1.handle, C.byref(q)))
    gu = X0.double() @ W0.double().T
    r = torch.rsqrt(ss_in.double().sum(0) / 384 + 1e-5)[:, None]
    gate, up = gu[:, :F] * r, gu[:, F:] * r
    act = (gate / (1 + torch.exp(-gate)) * up)
    for launch in range(2):
        _run(p0, ws0)
        _run(p1, ws1)
        out = _store(p1, ws1, M, N1, cuda)
        torch.cuda.synchronize()
        assert (X1.double() - act).abs().max() <= 1e-2 * act.abs().max(), launch
        y_ref = X1.double() @ W1.double().T  # the kernel's own bf16 X
        assert (out.double() - y_ref).abs().max() <= 2e-3 * y_ref.abs().max(), launch


def test_prologue_argument_checks(cuda):
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.forward import GemmPlan

    M = 16
    X0 = torch.zeros(M, 256, dtype=torch.bfloat16, device=cuda)
    W0 = torch.zeros(512, 256, dtype=torch.bfloat16, device=cuda)
    X1 = torch.zeros(M, 512, dtype=torch.bfloat16, device=cuda)
    W1 = torch.zeros(256, 512, dtype=torch.bfloat16, device=cuda)
    p0, p1 = GemmPlan(W0, X0, M), GemmPlan(W1, X1, M)
    ws0 = torch.zeros(p0.ws_bytes // 4 + 16, device=cuda)
    st = torch.zeros(512, dtype=torch.int32, device=cuda)
    resid = torch.zeros(M, 512, device=cuda)
    ss = torch.zeros(8, M, device=cuda)
    lib = L.lib()
    # SWIGLU needs previous N == 2K (512 != 1024)
    q = _pro(L.YGG_PRO_SWIGLU, p0, ws0, ss_in=ss.data_ptr(), ss_tiles=8, norm_dim=512, eps=1e-5,
             flags=st.data_ptr(), launches=st.data_ptr() + 64)
    assert lib.ygg_gemm_plan_set_prologue(p1.handle, C.byref(q)) == L.YGG_ERR_VALUE
    # RESID without flags
    q = _pro(L.YGG_PRO_RESID, p0, ws0, resid=resid.data_ptr(), ss_out=ss.data_ptr())
    assert lib.ygg_gemm_plan_set_prologue(p1.handle, C.byref(q)) == L.YGG_ERR_VALUE
    # a prologue plan must not write the partials it reads
    q = _pro(L.YGG_PRO_RESID, p0, ws0, resid=resid.data_ptr(), ss_out=ss.data_ptr(), flags=st.data_ptr(),
             launches=st.data_ptr() + 64)
    L.check(lib.ygg_gemm_plan_set_prologue(p1.handle, C.byref(q)))
    assert lib.ygg_gemm_run(p1.handle, ws0.data_ptr(), L.stream_ptr()) == L.YGG_ERR_VALUE
    L.check(lib.ygg_gemm_plan_set_prologue(p1.handle, None))
