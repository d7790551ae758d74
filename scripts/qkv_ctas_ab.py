"""Same-box A/B: the draft QKV GEMV on fewer CTAs (premise check for a QKV + attention fusion that
would run the QKV projection on one cluster per kv head).   python scripts/qkv_ctas_ab.py"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.draft
lib = L.lib()
orig = [ops[0][0] for ops in f.gv]
res = {}
graphs = {}
for n in (0, 128, 96, 64):
    mems = []
    for li, lw in enumerate(f.w["layers"]):
        if n == 0:
            f.gv[li][0] = (orig[li], f.gv[li][0][1])
            continue
        mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
        N, K = lw["wqkv"].shape
        L.check(lib.ygg_gemv_plan_init(mem, lw["wqkv"].data_ptr(), f.xn.data_ptr(), f.M, N, K, n))
        mems.append(mem)
        f.gv[li][0] = (mem, f.gv[li][0][1])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    graphs[n] = (g, mems)
for li in range(len(f.gv)):
    f.gv[li][0] = (orig[li], f.gv[li][0][1])
torch.cuda.synchronize()
out = {k: [] for k in graphs}
for _ in range(3):
    for n, (g, _) in graphs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        out[n].append(round(a.elapsed_time(b) / 50, 4))
print(json.dumps({f"qkv_ctas_{k or 'default'}": {"ms": v, "min": min(v)} for k, v in out.items()}), flush=True)
