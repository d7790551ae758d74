"""Same-box A/B of L2-prefetch plans for the cfg2 verify forward (graph-replayed, interleaved rounds):
which later weight streams the separate epilogue kernels and the attention pull into L2.

  python scripts/epi_l2_ab.py [--reps 20] [--rounds 3]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200.forward import Forward  # noqa: E402
from paper_2512_23858_b200.plan import ForwardPlan, L2Prefetch as P  # noqa: E402

GU0 = (P("wgu", 0.1),)
PLANS = {
    "base": ForwardPlan(),
    "all": ForwardPlan(verify_epi_l2=(("qkv", P("wo", 0.5)), ("o", P("wgu", 0.1, 0.1)), ("gu", P("wdown", 0.2)),
                                      ("down", P("wqkv", 0.4, next_layer=True)))),
    "all_big": ForwardPlan(verify_epi_l2=(("qkv", P("wo", 0.8)), ("o", P("wgu", 0.13, 0.1)), ("gu", P("wdown", 0.26)),
                                          ("down", P("wqkv", 0.6, next_layer=True)))),
    "qkv_wo": ForwardPlan(verify_epi_l2=(("qkv", P("wo", 0.5)),)),
    "o_gu": ForwardPlan(verify_epi_l2=(("o", P("wgu", 0.1, 0.1)),)),
    "gu_down": ForwardPlan(verify_epi_l2=(("gu", P("wdown", 0.2)),)),
    "down_qkv": ForwardPlan(verify_epi_l2=(("down", P("wqkv", 0.4, next_layer=True)),)),
    "attn_wo": ForwardPlan(verify_attn_l2=(P("wo", 0.5, 0.5), P("wgu", 0.1)),
                           verify_epi_l2=(("qkv", P("wo", 0.5)),)),
    "tree": ForwardPlan(tree_attn=True),
    "tree_c4r4": ForwardPlan(tree_attn=True, tree_csplit=4, tree_row_tiles=4),
    "tree_c4r2": ForwardPlan(tree_attn=True, tree_csplit=4),
    "tree_c2": ForwardPlan(tree_attn=True, tree_csplit=2),
    "tree_nopf": ForwardPlan(tree_attn=True, verify_attn_l2=(), draft_attn_l2=()),
    "tree_wo": ForwardPlan(tree_attn=True, verify_attn_l2=(P("wo", 0.5),)),
    "tree_wo_gu": ForwardPlan(tree_attn=True, verify_attn_l2=(P("wo", 0.4), P("wgu", 0.05))),
    "tree_gu15": ForwardPlan(tree_attn=True, verify_attn_l2=(P("wgu", 0.15),), draft_attn_l2=(P("wdown", 0.5),)),
    # *_late: the tree attention triggers its dependent launch only at the end (ygg_attn_tree_set_trigger)
    "tree_late": ForwardPlan(tree_attn=True),
    "tree_wo9_late": ForwardPlan(tree_attn=True, verify_attn_l2=(P("wo", 0.9),)),
    "tree_wo5gu_late": ForwardPlan(tree_attn=True, verify_attn_l2=(P("wo", 0.5), P("wgu", 0.1))),
    "tree_gu2_late": ForwardPlan(tree_attn=True, verify_attn_l2=(P("wgu", 0.2),)),
    "tree_wo9gu_late": ForwardPlan(tree_attn=True, verify_attn_l2=(P("wo", 0.9), P("wgu", 0.1))),
}


def graph_of(f):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    return g


def timeit(g, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--only", default="")
ap.add_argument("--which", default="verify")
args = ap.parse_args()
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.verify if args.which == "verify" else sd.draft
names = [n for n in PLANS if not args.only or n in args.only.split(",") or n == "base"]
fwds, graphs = {}, {}
for n in names:
    g = Forward(f.cfg, f.w, f.cache, f.B, f.R, f.mask_words, f.act_dtype, plan=PLANS[n], lm_argmax=f.lm_argmax)
    for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
        getattr(g, t).copy_(getattr(f, t))
    if n.endswith("_late") and g.at_plans:
        from paper_2512_23858_b200 import _lib as LL
        for pl in g.at_plans:
            LL.check(LL.lib().ygg_attn_tree_set_trigger(pl, 1))
    fwds[n] = g
    graphs[n] = graph_of(g)
res = {n: [] for n in names}
for _ in range(args.rounds):
    for n in names:
        res[n].append(timeit(graphs[n], args.reps))
out = {n: round(min(v), 4) for n, v in res.items()}
out["spread"] = {n: round(max(v) - min(v), 4) for n, v in res.items()}
print(json.dumps(out), flush=True)
