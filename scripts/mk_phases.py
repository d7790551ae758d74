"""Per-phase timeline of the persistent forward (cfg2 draft and verify), from per-CTA
%globaltimer stamps at each phase end.  Also graph-replayed forward timings."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

NAMES = ["qkv", "attn", "combine", "o", "gu", "down"]
wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
prompts = bench.prompts_for(wl, tc.vocab, 0)
sd.prefill(prompts)
for _ in range(0 if (os.environ.get("YGG_MK_NOATTN") or os.environ.get("YGG_MK_XFLAGS")) else 2):
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
    G = st.shape[0] // 8
    t3 = st.cpu().double()
    t, tdrain, tw, tgrp, twork, tfence, fxcyc, fxitems = (t3[i * G:(i + 1) * G] for i in range(8))
    ends = t.max(0).values  # phase end = last CTA to finish it
    # within-phase breakdown for GEMM phases: W issue end (max over CTAs), TMEM drain end (max), phase end
    brk = {}
    L_ = f.cfg.n_layers
    for j, nm in enumerate(NAMES):
        if nm in ("attn", "combine"):
            continue
        rows = []
        for i in range(L_):
            ph = 1 + i * 6 + j
            st0 = ends[ph - 1]
            wmax = tw[:, ph][tw[:, ph] > 0].max() if (tw[:, ph] > 0).any() else st0
            dmax = tdrain[:, ph][tdrain[:, ph] > 0].max() if (tdrain[:, ph] > 0).any() else st0
            gmax = tgrp[:, ph][tgrp[:, ph] > 0].max() if (tgrp[:, ph] > 0).any() else st0
            rows.append([float(wmax - st0) / 1e3, float(dmax - st0) / 1e3, float(gmax - st0) / 1e3,
                         float(twork[:, ph].max() - st0) / 1e3, float(tfence[:, ph].max() - st0) / 1e3,
                         float(ends[ph] - st0) / 1e3])
        brk[nm] = [round(sum(r[k] for r in rows) / len(rows), 2) for k in range(6)]
    out[name + "_breakdown(w_issued,drained,groups_done,work_done,fenced,end)"] = brk
    fx = {}
    for j, nm in enumerate(NAMES):
        if nm in ("attn", "combine"):
            continue
        ph = 1 + 2 * 6 + j  # layer 2
        cyc = fxcyc[:, ph]
        it = fxitems[:, ph]
        k = int(cyc.argmax())
        fx[nm] = {"max_cyc": int(cyc.max()), "mean_cyc": int(cyc.mean()), "items_at_max": int(it[k] // 1000),
                  "groups_at_max": int(it[k] % 1000), "mean_items": float((it // 1000).mean())}
    out[name + "_fixup"] = fx
    starts_min = t.min(0).values
    L = f.cfg.n_layers
    dur = (ends[1:] - ends[:-1]) / 1000.0
    agg = {"embed": float((ends[0] - starts_min[0]) / 1000.0)}
    for i in range(L):
        for j, nm in enumerate(NAMES):
            agg.setdefault(nm, []).append(float(dur[i * 6 + j]))
    agg["lm"] = float(dur[L * 6])
    summ = {k: (round(sum(v) / len(v), 2) if isinstance(v, list) else round(v, 2)) for k, v in agg.items()}
    spread = ((t.max(0).values - t.min(0).values) / 1000.0)
    summ["total_us"] = round(float((ends[-1] - ends[0]) / 1000.0), 1)
    summ["avg_cta_spread_us"] = round(float(spread.mean()), 2)
    out[name] = summ
    f.mk_phase_stamps(False)
print(json.dumps(out))
