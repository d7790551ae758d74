"""Same-box A/B of the decode attention configuration (cluster key splits x ring stages) inside the
graph-replayed cfg2 verify and draft forwards.  python scripts/attn_ab.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200.forward import Forward  # noqa: E402
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


wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
res = {}
DRAFT = [(0, 0, 0)]
for name, f, variants in (("draft", sd.draft, DRAFT),):
    for kv, st, ksp in variants:  # (kvsplit, stages, in-CTA key-split groups); 0 = automatic
        g = Forward(f.cfg, f.w, f.cache, f.B, f.R, f.mask_words, f.act_dtype, gemv=f.gemv,
                    plan=ForwardPlan(attn_kvsplit=kv, attn_stages=st, attn_ksplit=ksp, tree_attn=False))
        for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
            getattr(g, t).copy_(getattr(f, t))
        res[f"{name}_kv{kv}_st{st}_ks{ksp}_ms"] = timeit(g, 20)
        del g
print(json.dumps(res), flush=True)
