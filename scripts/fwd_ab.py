"""Same-box A/B: graph-replayed cfg2 draft / verify forward, per-kernel path vs persistent forward."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200.forward import Forward  # noqa: E402


def timeit(f, n=20):
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
variants = {"draft": (("kern", dict(gemv=False, persistent=False)), ("gemv", dict(gemv=True))),
            "verify": (("kern", dict(persistent=False)), ("mk", dict(persistent=True)))}
for name, f in (("draft", sd.draft), ("verify", sd.verify)):
    for tag, kw in variants[name]:
        g = Forward(f.cfg, f.w, f.cache, f.B, f.R, f.mask_words, f.act_dtype, **kw)
        for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
            getattr(g, t).copy_(getattr(f, t))
        res[f"{name}_{tag}_ms"] = timeit(g)
        del g
print(json.dumps(res), flush=True)
