"""Standalone timing of ygg_topk_merge (fused draft top-k partials) vs ygg_topk_softmax (profiling)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_23858_b200 import _lib as L  # noqa: E402

L.require_device()
lib = L.lib()
dev = torch.device("cuda")
M, V, K, k = 8, 128256, 2048, 8
W = (torch.randn(V, K, device=dev) * 0.05).to(torch.bfloat16)
X = torch.randn(M, K, device=dev).to(torch.bfloat16)
mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), M, V, K, 0))
grid = int(lib.ygg_gemv_grid(mem))
part = torch.empty(int(lib.ygg_topk_partial_bytes(M, grid)), dtype=torch.uint8, device=dev)
logits = torch.zeros(M, V, device=dev)
e = L.YggGemvEpilogue()
e.kind = L.YGG_GEMV_STORE_TOPK
e.out = logits.data_ptr()
e.ld = V
e.topk_part = part.data_ptr()
e.topk_k = k
e.inv_temp = 1.0
e_store = L.YggGemvEpilogue()
e_store.kind = L.YGG_GEMV_STORE
e_store.out = logits.data_ptr()
e_store.ld = V
tok = torch.zeros(M, k, dtype=torch.int32, device=dev)
prob = torch.zeros(M, k, dtype=torch.float64, device=dev)
ws = torch.empty(int(lib.ygg_topk_workspace(M, V, k)), dtype=torch.uint8, device=dev)
s = L.stream_ptr()


def t(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n * 1000, 2)


res = {
    "gemv_store_topk_us": t(lambda: L.check(lib.ygg_gemv_run(mem, C.byref(e), s))),
    "merge_us": t(lambda: L.check(lib.ygg_topk_merge(part.data_ptr(), M, grid, k, tok.data_ptr(), prob.data_ptr(),
                                                      None, s))),
    "topk_softmax_us": t(lambda: L.check(lib.ygg_topk_softmax(logits.data_ptr(), L.YGG_F32, M, V, V, k, 1.0,
                                                               tok.data_ptr(), prob.data_ptr(), None, ws.data_ptr(),
                                                               ws.numel(), s))),
    "grid": grid,
}
print(res)


def pair():
    L.check(lib.ygg_gemv_run(mem, C.byref(e), s))
    L.check(lib.ygg_topk_merge(part.data_ptr(), M, grid, k, tok.data_ptr(), prob.data_ptr(), None, s))


def pair_old():
    L.check(lib.ygg_gemv_run(mem, C.byref(e_store), s))
    L.check(lib.ygg_topk_softmax(logits.data_ptr(), L.YGG_F32, M, V, V, k, 1.0, tok.data_ptr(), prob.data_ptr(),
                                 None, ws.data_ptr(), ws.numel(), s))

print({"gemv_topk_then_merge_us": t(pair), "gemv_store_then_topk_softmax_us": t(pair_old),
       "gemv_store_us": t(lambda: L.check(lib.ygg_gemv_run(mem, C.byref(e_store), s)))})
