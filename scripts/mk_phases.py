"""Per-phase timeline of the persistent forward (cfg2 draft and verify), from per-CTA
%globaltimer stamps at each phase end.  Also graph-replayed forward timings."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

NAMES = ["qkv_gemm", "qkv_epi", "attn", "combine", "o_gemm", "o_resid", "gu_gemm", "swiglu", "down_gemm",
         "down_resid"]
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
prompts = bench.prompts_for(wl, tc.vocab, 0)
sd.prefill(prompts)
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
out = {}
for name, f in (("draft", sd.draft), ("verify", sd.verify)):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    out[name + "_ms"] = round(a.elapsed_time(b) / 20, 4)
    st = f.mk_phase_stamps(True)
    for _ in range(3):
        f.run()
    torch.cuda.synchronize()
    t = st.cpu().double()
    ends = t.max(0).values  # phase end = last CTA to finish it
    starts_min = t.min(0).values
    L = f.cfg.n_layers
    dur = (ends[1:] - ends[:-1]) / 1000.0
    agg = {"embed": float((ends[0] - starts_min[0]) / 1000.0)}
    for i in range(L):
        for j, nm in enumerate(NAMES):
            agg.setdefault(nm, []).append(float(dur[i * 10 + j]))
    agg["lm_gemm"] = float(dur[L * 10])
    agg["lm_store"] = float(dur[L * 10 + 1])
    summ = {k: (round(sum(v) / len(v), 2) if isinstance(v, list) else round(v, 2)) for k, v in agg.items()}
    spread = ((t.max(0).values - t.min(0).values) / 1000.0)
    summ["total_us"] = round(float((ends[-1] - ends[0]) / 1000.0), 1)
    summ["avg_cta_spread_us"] = round(float(spread.mean()), 2)
    out[name] = summ
    f.mk_phase_stamps(False)
print(json.dumps(out))
