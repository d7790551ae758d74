"""In-graph kernel timeline of the cfg2 prefill forwards (512-token prompt), target and draft, from the
kernels' own %globaltimer stamps (ygg_trace_arm).  Profiling only.   python scripts/prefill_timeline.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

NAMES = {1: "gemv", 2: "attn_dec", 3: "gemm", 4: "epi_store", 5: "epi_resid", 6: "epi_swiglu", 7: "epi_qkv",
         8: "attn_tc", 9: "attn_combine", 10: "topk_merge", 11: "grow", 13: "level_inputs", 14: "embed", 15: "attn_tree"}
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
torch.cuda.synchronize()
lib = L.lib()
CAP = 1024
buf = torch.zeros(CAP, 8, dtype=torch.int64, device="cuda")
out = {}
for f in list(sd._prefill_fwd.values()):
    name = f.cfg.name
    graph = torch.cuda.CUDAGraph()
    L.check(lib.ygg_trace_arm(buf.data_ptr(), CAP))
    with torch.cuda.graph(graph):
        f.run()
    ids = (L.C.c_int * CAP)()
    n = lib.ygg_trace_used(ids, CAP)
    L.check(lib.ygg_trace_arm(None, 0))
    for _ in range(3):
        graph.replay()
    buf[:, 0] = -1
    buf[:, 1] = -1
    buf[:, 2:] = 0
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    t = buf[:n].cpu().tolist()
    t0 = t[0][0]
    tot, cnt, gaps = {}, {}, 0.0
    prev = None
    gemm_i = 0
    for i in range(n):
        k = NAMES.get(ids[i], ids[i])
        if k == "gemm":
            k = f"gemm#{gemm_i % 4 if i < n - 1 or not f.lm_plan else 'lm'}"
            gemm_i += 1
        s, w, e = t[i][0], t[i][1], t[i][2]
        tot[k] = tot.get(k, 0.0) + (e - w) / 1e3
        cnt[k] = cnt.get(k, 0) + 1
        if prev is not None:
            gaps += (w - prev) / 1e3
        prev = e
    out[name] = {"M": f.M, "fused": f.fused, "total_us": round((t[n - 1][2] - t0) / 1e3, 1), "launches": n,
                 "gaps_us": round(gaps, 1),
                 "per_kernel_us": {k: [round(v / cnt[k], 2), cnt[k]] for k, v in tot.items()}}
print(json.dumps(out, indent=1), flush=True)
