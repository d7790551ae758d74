"""Kernel-level timing of the weight-streaming GEMM on Llama-3-8B / 3.2-1B shapes.

Weights are rotated over >L2 (126 MB) worth of copies so every launch streams from HBM.
Prints achieved GB/s (algorithmic weight bytes / CUDA-event time) per shape."""
import json
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23858_b200 import _lib as L  # noqa: E402
from paper_2512_23858_b200.forward import GemmPlan  # noqa: E402

L.require_device()
lib = L.lib()
shapes = {
    "8b.qkv": (6144, 4096), "8b.o": (4096, 4096), "8b.gu": (28672, 4096), "8b.down": (4096, 14336),
    "8b.lm_head": (128256, 4096), "1b.qkv": (3072, 2048), "1b.gu": (16384, 2048), "1b.down": (2048, 8192),
    "1b.lm_head": (128256, 2048),
}
Ms = [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["16", "50", "65"])]
res = []
for name, (N, K) in shapes.items():
    nbytes = N * K * 2
    copies = max(2, math.ceil(400e6 / nbytes))
    Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) / math.sqrt(K) for _ in range(copies)]
    for M in Ms:
        X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        plans = [GemmPlan(W, X, M) for W in Ws]
        ws = torch.empty(max(p.ws_bytes for p in plans) // 4 + 1, device="cuda")
        s = L.stream_ptr()
        for i in range(3 * copies):
            L.check(lib.ygg_gemm_run(plans[i % copies].handle, ws.data_ptr(), s))
        torch.cuda.synchronize()
        reps = 10 * copies
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            L.check(lib.ygg_gemm_run(plans[i % copies].handle, ws.data_ptr(), s))
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        L.check(lib.ygg_gemm_run(plans[0].handle, ws.data_ptr(), s))
        out = torch.zeros(M, N, device="cuda")
        L.check(lib.ygg_epi_store(plans[0].handle, ws.data_ptr(), out.data_ptr(), L.YGG_F32, N, s))
        ref = X.float() @ Ws[0].float().T
        err = ((out - ref).abs().max() / ref.abs().max()).item()
        r = {"shape": name, "M": M, "N": N, "K": K, "us": round(us, 2), "GBps": round(nbytes / us / 1e3, 1),
             "rel_err": err, "segments": plans[0].segments}
        print(json.dumps(r), flush=True)
        res.append(r)
        del plans
    del Ws
    torch.cuda.empty_cache()
