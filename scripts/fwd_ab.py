"""Same-box A/B of the cfg2 verify forward (graph-replayed): per-kernel epilogues (plain layout) vs
the fused layout with cluster split-K (QKV / O / down) vs the fused layout with stream-K fixups.

  python scripts/fwd_ab.py [--reps 20]
"""
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


def timeit(f, n):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n, 4)


ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.verify
res = {"verify_plain_ms": timeit(f, args.reps)}
wf = weights_to(sd.tw, f.cache.device)  # separate copy: the fused layout is applied in place
for tag, plan in (("fused_cluster", ForwardPlan(fused_epilogues=True)),
                  ("fused_streamk", ForwardPlan(fused_epilogues=True, cluster_split_k=False))):
    g = Forward(f.cfg, wf, f.cache, f.B, f.R, f.mask_words, f.act_dtype, plan=plan)
    for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
        getattr(g, t).copy_(getattr(f, t))
    res[f"verify_{tag}_ms"] = timeit(g, args.reps)
    res[f"{tag}_clusters"] = [g.plans[0][k].cluster for k in ("qkv", "o", "gu", "down")]
    del g
print(json.dumps(res), flush=True)
