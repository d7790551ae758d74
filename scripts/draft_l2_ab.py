"""Same-box A/B: L2 prefetch of the NEXT layer's QKV / O weights from this layer's gate|up or down GEMV
(issued by each CTA after its own weight stream), in the graph-replayed cfg2 draft pass.
  python scripts/draft_l2_ab.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

# variant: list of (source matrix index in the layer's gv list: 2 = gate|up, 3 = down, region, target, fraction)
VARIANTS = {
    "base": [],
    "down>qkv1.0": [(3, 0, "wqkv", 1.0)],
    "down>qkv0.5": [(3, 0, "wqkv", 0.5)],
    "gu>qkv0.5": [(2, 0, "wqkv", 0.5)],
    "down>qkv1.0+o1.0": [(3, 0, "wqkv", 1.0), (3, 1, "wo", 1.0)],
    "gu>qkv1.0": [(2, 0, "wqkv", 1.0)],
}
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.draft
lib = L.lib()
layers = f.w["layers"]
graphs = {}
for name, regs in VARIANTS.items():
    for li in range(len(f.gv)):
        for src in (2, 3):
            for rg in (0, 1):
                L.check(lib.ygg_gemv_set_l2_prefetch(f.gv[li][src][0], rg, None, 0))
        if li + 1 >= len(f.gv):
            continue
        for src, rg, tgt, frac in regs:
            W = layers[li + 1][tgt]
            n = int(W.numel() * W.element_size() * frac) & ~255
            L.check(lib.ygg_gemv_set_l2_prefetch(f.gv[li][src][0], rg, W.data_ptr(), n))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    graphs[name] = g
torch.cuda.synchronize()
res = {k: [] for k in graphs}
for _ in range(3):
    for name, g in graphs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        res[name].append(round(a.elapsed_time(b) / 50, 4))
print(json.dumps({k: {"ms": v, "min": min(v)} for k, v in res.items()}), flush=True)
