"""Same-box A/B: one draft GEMV matrix (GV_IDX: 0 qkv, 1 o, 2 gate|up, 3 down) on GV_CTAS CTAs (0 = the
plan's default) with GV_STAGES ring stages (0 = default), in the graph-replayed cfg2 draft pass.
    GV_IDX=1 GV_CTAS=0,116,112 GV_STAGES=9 python scripts/gemv_ctas_ab.py"""
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
IDX = int(os.environ.get("GV_IDX", "1"))
orig = [ops[IDX][0] for ops in f.gv]
res = {}
graphs = {}
for n in [int(x) for x in os.environ.get("GV_CTAS", "0,116,112,100").split(",")]:
    mems = []
    for li, lw in enumerate(f.w["layers"]):
        if n == 0:
            f.gv[li][IDX] = (orig[li], f.gv[li][IDX][1])
            continue
        mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
        wname = ("wqkv", "wo", "wgu", "wdown")[IDX]
        N, K = lw[wname].shape
        L.check(lib.ygg_gemv_plan_init(mem, lw[wname].data_ptr(), (f.xn, f.attn, f.xn, f.mlp)[IDX].data_ptr(), f.M, N, K, n))
        if int(os.environ.get("GV_STAGES", "0")):
            L.check(lib.ygg_gemv_plan_set_stages(mem, int(os.environ["GV_STAGES"])))
        mems.append(mem)
        f.gv[li][IDX] = (mem, f.gv[li][IDX][1])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    graphs[n] = (g, mems)
for li in range(len(f.gv)):
    f.gv[li][IDX] = (orig[li], f.gv[li][IDX][1])
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
print(json.dumps({f"gv_ctas_{k or 'default'}": {"ms": v, "min": min(v)} for k, v in out.items()}), flush=True)
