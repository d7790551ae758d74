"""Same-box A/B of forward plans for one pass of a bench workload (graph-replayed, interleaved repeats;
all variants share the decoder's weights).

  python scripts/cfg_plan_ab.py cfg4 verify 'tree_attn=1' 'tree_attn=0,decode_attn_wide=1'
  (an empty variant string = ForwardPlan())"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200.forward import Forward  # noqa: E402

wl_name, which = sys.argv[1], sys.argv[2]
variants = sys.argv[3:] or [""]
wl = dict(bench.WORKLOADS[wl_name])
wl.setdefault("batch", wl.get("global_batch", 1))
sd, tc, dc = bench.build_decoder(wl, wl_name, torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.verify if which == "verify" else sd.draft
graphs = {}
for v in variants:
    items = [x for x in v.split(",") if x]
    ctas = [int(x.split("=")[1]) for x in items if x.startswith("ctas=")]  # GEMM CTA count override
    plan = bench.plan_from_args([x for x in items if not x.startswith("ctas=")])
    g = Forward(f.cfg, f.w, f.cache, f.B, f.R, f.mask_words, f.act_dtype, plan=plan,
                lm_argmax=getattr(f, "lm_argmax", False), num_ctas=ctas[0] if ctas else 0)
    for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
        getattr(g, t).copy_(getattr(f, t))
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg):
        g.run()
    for _ in range(3):
        cg.replay()
    graphs[v or "default"] = (g, cg, {"fused": g.fused, "gemv": g.gemv, "tree": g.at_plans is not None,
                                      "dec": g.ad_plans is not None})
torch.cuda.synchronize()
res = {k: [] for k in graphs}
for _ in range(3):
    for name, (g, cg, _) in graphs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            cg.replay()
        b.record()
        torch.cuda.synchronize()
        res[name].append(round(a.elapsed_time(b) / 10, 4))
print(json.dumps({k: {"ms": v, "min": min(v), "kinds": graphs[k][2]} for k, v in res.items()}), flush=True)
