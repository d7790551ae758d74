"""Same-box A/B of verify-forward plans (graph-replayed cfg2 verify, interleaved repeats); the forwards
share the decoder's weights (plans that change the weight layout are not supported here).

  python scripts/verify_plan_ab.py [--reps 20] [--rounds 3]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200.forward import Forward  # noqa: E402
from paper_2512_23858_b200.plan import ForwardPlan, L2Prefetch  # noqa: E402

VARIANTS = {
    "default": ForwardPlan(),
    "csplit2": ForwardPlan(tree_csplit=2),
    "csplit1": ForwardPlan(tree_csplit=1),
    "rowtiles4": ForwardPlan(tree_row_tiles=4),
    "rowtiles4_cs2": ForwardPlan(tree_row_tiles=4, tree_csplit=2),
    "attn_gu_0.1_o": ForwardPlan(verify_attn_l2=(L2Prefetch("wgu", 0.1), L2Prefetch("wo", 0.25))),
}

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
graphs = {}
for name, plan in VARIANTS.items():
    g = Forward(f.cfg, f.w, f.cache, f.B, f.R, f.mask_words, f.act_dtype, plan=plan, lm_argmax=f.lm_argmax)
    for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
        getattr(g, t).copy_(getattr(f, t))
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg):
        g.run()
    for _ in range(3):
        cg.replay()
    graphs[name] = (g, cg)
torch.cuda.synchronize()
res = {k: [] for k in graphs}
for _ in range(args.rounds):
    for name, (g, cg) in graphs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            cg.replay()
        b.record()
        torch.cuda.synchronize()
        res[name].append(round(a.elapsed_time(b) / args.reps, 4))
print(json.dumps({k: {"ms": v, "min": min(v)} for k, v in res.items()}), flush=True)
