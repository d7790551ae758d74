"""Per-launch overhead inside CUDA graphs: trivial kernels and small GEMMs (1 / 148 CTAs)."""
import ctypes as C, json, math, sys
import torch
sys.path.insert(0, ".")
from paper_2512_23858_b200 import _lib as L
from paper_2512_23858_b200.forward import GemmPlan
L.require_device(); lib = L.lib()

def graph_time(fn, n=100, reps=10):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (reps * n)

res = {}
slot = torch.zeros(4, dtype=torch.int64, device="cuda")
res["stamp_us"] = graph_time(lambda: L.check(lib.ygg_stamp(slot.data_ptr(), L.stream_ptr())))
for name, (N, K, M, ctas) in {"gemm_1cta": (128, 64, 8, 1), "gemm_148cta_tiny": (128 * 148, 64, 8, 148),
                              "gemm_148cta_1MB": (128 * 148, 256, 8, 148), "gemm_64cta_1b_o": (2048, 2048, 8, 64),
                              "gemm_1b_o_default": (2048, 2048, 8, 0), "gemm_1b_gu_default": (16384, 2048, 8, 0)}.items():
    W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    plan = GemmPlan(W, X, M, ctas)
    ws = torch.zeros(plan.ws_bytes // 4 + 16, device="cuda")
    res[name + "_us"] = graph_time(lambda: L.check(lib.ygg_gemm_run(plan.handle, ws.data_ptr(), L.stream_ptr())), n=50)
    # fused STORE epilogue
    out = torch.zeros(M, N, device="cuda")
    cnt = torch.zeros(plan.tiles, dtype=torch.int32, device="cuda")
    e = L.YggEpilogue(); e.kind = L.YGG_EPI_STORE_F32; e.counters = cnt.data_ptr(); e.out = out.data_ptr(); e.ld = N
    res[name + "_fused_us"] = graph_time(lambda: L.check(lib.ygg_gemm_fused(plan.handle, ws.data_ptr(), C.byref(e), L.stream_ptr())), n=50)
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
