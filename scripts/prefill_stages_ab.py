"""Same-box A/B of the GEMM ring depth of the cfg2 target prefill forward (512 rows, graph-replayed).
  python scripts/prefill_stages_ab.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
torch.cuda.synchronize()
lib = L.lib()
res = {}
for f in list(sd._prefill_fwd.values()):
    plans = [q for p in f.plans for q in p.values()]  # (the 1-row LM head keeps its ring)
    for st in (3, 4, 2, 3):
        for q in plans:
            L.check(lib.ygg_gemm_plan_set_stages(q.handle, st))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f.run()
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        res.setdefault(f.cfg.name, {}).setdefault(f"stages{st}", []).append(round(a.elapsed_time(b) / 5, 3))
        del g
print(json.dumps(res), flush=True)
