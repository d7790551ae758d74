"""Same-box A/B of verify-forward plans (graph-replayed cfg2 verify, interleaved repeats).

  python scripts/verify_ab.py [--reps 20] [--rounds 3]
Each plan gets its own copy of the target weights (the hybrid folds its copy in place)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200.forward import Forward  # noqa: E402
from paper_2512_23858_b200.model import weights_to  # noqa: E402
from paper_2512_23858_b200.plan import ForwardPlan  # noqa: E402

PLANS = {
    "plain": ForwardPlan(hybrid=False),
    "plain_early": ForwardPlan(hybrid=False, epi_early_trigger=True),
    "hybrid": ForwardPlan(hybrid=True),
    "hybrid_early": ForwardPlan(hybrid=True, epi_early_trigger=True),
}

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--plans", default=",".join(PLANS))
args = ap.parse_args()
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"), plan=ForwardPlan(hybrid=False))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.verify
graphs = {}
for name in args.plans.split(","):
    w = weights_to(sd.tw, f.cache.device)
    g = Forward(f.cfg, w, f.cache, f.B, f.R, f.mask_words, f.act_dtype, plan=PLANS[name], lm_argmax=f.lm_argmax)
    for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
        getattr(g, t).copy_(getattr(f, t))
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg):
        g.run()
    for _ in range(3):
        cg.replay()
    graphs[name] = (g, cg, w)
torch.cuda.synchronize()
res = {k: [] for k in graphs}
for _ in range(args.rounds):
    for name, (g, cg, _) in graphs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            cg.replay()
        b.record()
        torch.cuda.synchronize()
        res[name].append(round(a.elapsed_time(b) / args.reps, 4))
print(json.dumps({k: {"ms": v, "min": min(v)} for k, v in res.items()}), flush=True)
