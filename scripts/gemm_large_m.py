"""Compute-bound GEMM timing (TFLOP/s) of the stream-K tcgen05 GEMM at prefill / batched-verify row
counts.   python scripts/gemm_large_m.py [name ...]"""
import json
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23858_b200 import _lib as L  # noqa: E402
from paper_2512_23858_b200.forward import GemmPlan  # noqa: E402

L.require_device()
lib = L.lib()
cases = {  # name: (M, N, K)
    "8b.gu.512": (512, 28672, 4096), "8b.down.512": (512, 4096, 14336), "8b.gu.800": (800, 28672, 4096),
    "70b.gu.520": (520, 57344, 8192), "70b.qkv.520": (520, 10240, 8192), "70b.down.520": (520, 8192, 28672),
}
names = sys.argv[1:] or list(cases)
res = []
for name in names:
    M, N, K = cases[name]
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16) / math.sqrt(K)
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    p = GemmPlan(W, X, M)
    ws = torch.empty(p.ws_bytes // 4 + 1, device="cuda")
    s = L.stream_ptr()
    for _ in range(3):
        L.check(lib.ygg_gemm_run(p.handle, ws.data_ptr(), s))
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.check(lib.ygg_gemm_run(p.handle, ws.data_ptr(), s))
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        torch.matmul(X, W.T)
    b.record()
    torch.cuda.synchronize()
    cub = a.elapsed_time(b) * 1e3 / reps
    fl = 2 * M * N * K
    res.append({"case": name, "us": round(us, 2), "tflops": round(fl / us / 1e6, 1), "cublas_us": round(cub, 2),
                "cublas_tflops": round(fl / cub / 1e6, 1), "segments": p.segments, "tiles": p.tiles})
    del W, X, p, ws
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
