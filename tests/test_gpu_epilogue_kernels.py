"""The separate epilogue kernels of the stream-K GEMM (csrc/gemm.cu epi_*_kernel) vs torch fp64
references of the same bf16 operands, at decode, cfg5-verify and cfg4-verify row counts (the wide
passes take several tokens per thread), in both weight row layouts (ygg_gemm_plan_set_layout), with
single-segment and multi-segment (stream-K split) tiles.  Tolerance as test_gpu_fused.py: 1e-2 of the
output scale after the bf16 store."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ctas", [0, 37])
@pytest.mark.parametrize("il", [0, 1])
@pytest.mark.parametrize("M", [50, 300, 800])
def test_swiglu_epilogue_kernel(M, il, ctas, cuda):
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.forward import GemmPlan
    from paper_2512_23858_b200.model import gate_up_interleave, preset

    lib = L.lib()
    F, d = 1024, 512
    cfg = preset("tiny-target", ffn=F, d_model=d)
    g = torch.Generator(device="cuda").manual_seed(M + 10 * il + ctas)
    X = torch.randn(M, d, device=cuda, generator=g).to(torch.bfloat16)
    Wgu = (torch.randn(2 * F, d, device=cuda, generator=g) / math.sqrt(d)).to(torch.bfloat16)
    W = Wgu[gate_up_interleave(cfg).to(cuda)].contiguous() if il else Wgu
    plan = GemmPlan(W, X, M, ctas)
    if il:
        L.check(lib.ygg_gemm_plan_set_layout(plan.handle, 1))
    ws = torch.zeros(plan.ws_bytes // 4 + 16, device=cuda)
    act = torch.zeros(M + 4, F, dtype=torch.bfloat16, device=cuda)  # rows past M must stay untouched
    L.check(lib.ygg_gemm_run(plan.handle, ws.data_ptr(), L.stream_ptr()))
    L.check(lib.ygg_epi_swiglu(plan.handle, ws.data_ptr(), act.data_ptr(), L.dtype_code(torch.bfloat16), L.stream_ptr()))
    torch.cuda.synchronize()
    gu = X.double() @ Wgu.double().T
    ref = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    assert (act[:M].double() - ref).abs().max() <= 1e-2 * ref.abs().max()
    assert not act[M:].any()
