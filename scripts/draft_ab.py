"""Same-box A/B of the GEMV ring depth per matrix in the graph-replayed cfg2 draft pass (interleaved
repeats).  Variants: {matrix: stages} overrides via ygg_gemv_plan_set_stages (0 = plan default).

  python scripts/draft_ab.py [--reps 50] [--rounds 3]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

VARIANTS = {
    "default": {},           # plan defaults (o: 224 KB solo ring = 9 stages)
    "o4": {"o": 4},          # o ring = its 4 chunks (co-resident with the attention CTAs): slower
    "down6": {"down": 6},
    "down4": {"down": 4},
    "qkv2_gu2": {"qkv": 2, "gu": 2},
}
IDX = {"qkv": 0, "o": 1, "gu": 2, "down": 3}

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--variants", default=",".join(VARIANTS))
args = ap.parse_args()
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.draft
lib = L.lib()
info = (L.C.c_int(), L.C.c_int(), L.C.c_int())
wmap = L.C.create_string_buffer(128)
defaults = {}
for name, i in IDX.items():
    pl = f.gv[0][i][0]
    L.check(lib.ygg_gemv_stream_info(pl, wmap, L.C.byref(info[0]), L.C.byref(info[1]), L.C.byref(info[2])))
    defaults[name] = info[2].value
graphs = {}
for v in args.variants.split(","):
    over = VARIANTS[v]
    for ops in f.gv:
        for name, i in IDX.items():
            L.check(lib.ygg_gemv_plan_set_stages(ops[i][0], over.get(name, defaults[name])))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    graphs[v] = g
for ops in f.gv:  # restore
    for name, i in IDX.items():
        L.check(lib.ygg_gemv_plan_set_stages(ops[i][0], defaults[name]))
torch.cuda.synchronize()
res = {k: [] for k in graphs}
for _ in range(args.rounds):
    for v, g in graphs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        res[v].append(round(a.elapsed_time(b) / args.reps, 4))
print(json.dumps({"defaults": defaults, **{k: {"ms": v, "min": min(v)} for k, v in res.items()}}), flush=True)
