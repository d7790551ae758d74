"""Structured-input diagnostic of the tcgen05 GEMM (one tile): reveals operand/accumulator layout."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2512_23858_b200 import _lib as L
from paper_2512_23858_b200.forward import GemmPlan
L.require_device(); lib = L.lib()
out = {}
for name, shift in (("k0", 0), ("k16", 16), ("k48", 48)):
    M, N, K = 16, 128, 64
    X = torch.zeros(M, K)
    for m in range(M):
        X[m, (m + shift) % K] = 1.0
    W = torch.zeros(N, K)
    for n in range(N):
        for k in range(K):
            W[n, k] = float((n % 16) * 16 + (k % 16)) + 256 * (k // 16) * 0  # exact in bf16
    Wb, Xb = W.cuda().to(torch.bfloat16), X.cuda().to(torch.bfloat16)
    plan = GemmPlan(Wb, Xb, M, 1)
    ws = torch.zeros(plan.ws_bytes // 4 + 16, device="cuda")
    L.check(lib.ygg_gemm_run(plan.handle, ws.data_ptr(), L.stream_ptr()))
    y = torch.zeros(M, N, device="cuda")
    L.check(lib.ygg_epi_store(plan.handle, ws.data_ptr(), y.data_ptr(), L.YGG_F32, N, L.stream_ptr()))
    torch.cuda.synchronize()
    ref = Xb.float() @ Wb.float().T
    out[name] = {"y": y.cpu().tolist(), "ref": ref.cpu().tolist(), "ws": ws[: 16 * 128].view(16, 128).cpu().tolist()}
    print(name, "maxerr", (y - ref).abs().max().item())
# random K=64 single tile, and K=128 two k-blocks
for K in (64, 128, 256):
    torch.manual_seed(0)
    M, N = 16, 128
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16); W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    plan = GemmPlan(W, X, M, 1)
    ws = torch.zeros(plan.ws_bytes // 4 + 16, device="cuda")
    L.check(lib.ygg_gemm_run(plan.handle, ws.data_ptr(), L.stream_ptr()))
    y = torch.zeros(M, N, device="cuda")
    L.check(lib.ygg_epi_store(plan.handle, ws.data_ptr(), y.data_ptr(), L.YGG_F32, N, L.stream_ptr()))
    torch.cuda.synchronize()
    ref = X.float() @ W.float().T
    print("rand K", K, "maxerr", (y - ref).abs().max().item(), "refmax", ref.abs().max().item())
json.dump(out, open("gpurun_out/gemm_diag.json", "w"))
