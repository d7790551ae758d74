"""Same-box A/B: overlap of the verify O-projection GEMM's weight fill with the tree attention.
The attention triggers its dependents early or late (ygg_attn_tree_set_trigger); the O GEMM runs on
fewer CTAs than SMs so that it can land on the SMs the attention leaves free.

  python scripts/o_overlap_ab.py [--reps 20] [--rounds 3]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402
from paper_2512_23858_b200.forward import GemmPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--rounds", type=int, default=3)
args = ap.parse_args()
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.verify
lib = L.lib()
assert f.at_plans is not None
orig_o = [p["o"] for p in f.plans]
alt = {}
for n in (116, 100):
    alt[n] = [GemmPlan(p["o"].W, p["o"].X, p["o"].M, n) for p in f.plans]
    need = max(q.ws_bytes for q in alt[n]) // 4 + 1
    assert need <= f.ws.numel(), (need, f.ws.numel())
variants = [("late_148", 1, None), ("early_148", 0, None), ("early_116", 0, 116), ("early_100", 0, 100),
            ("late_116", 1, 116)]
graphs = {}
for name, late, n in variants:
    for pl in f.at_plans:
        L.check(lib.ygg_attn_tree_set_trigger(pl, late))
    for li, p in enumerate(f.plans):
        p["o"] = orig_o[li] if n is None else alt[n][li]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    graphs[name] = g
for pl in f.at_plans:
    L.check(lib.ygg_attn_tree_set_trigger(pl, 1))
for li, p in enumerate(f.plans):
    p["o"] = orig_o[li]
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
print(json.dumps({k: {"ms": v, "min": min(v)} for k, v in res.items()}), flush=True)
