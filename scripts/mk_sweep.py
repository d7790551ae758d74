"""A/B sweep of persistent-forward knobs (L2 look-ahead depth) on cfg2 draft / verify forwards."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
prompts = bench.prompts_for(wl, tc.vocab, 0)
sd.prefill(prompts)
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()


def timeit(f, n=10):
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


res = {}
for look in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,8,16,32,64").split(",")]:
    for name, f in (("draft", sd.draft), ("verify", sd.verify)):
        f._mk_desc.lookahead = look
        L.check(L.lib().ygg_mk_plan_init(f._mk_plan, C.byref(f._mk_desc), f.mk_table.data_ptr(), f.mk_table.numel()))
        res[f"{name}_look{look}"] = timeit(f)
print(json.dumps(res))
