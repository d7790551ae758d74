"""In-graph kernel timeline of one cfg2 draft forward (GEMV path), from the kernels' own
%globaltimer stamps (ygg_trace_arm): per launch, when its first CTA started, when its grid
dependency released (previous kernel done), and when its last CTA finished.  Profiling only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402
from paper_2512_23858_b200.forward import Forward  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "draft"
WL = os.environ.get("YGG_WORKLOAD", "cfg2")  # tooling: which bench workload to trace
wl = dict(bench.WORKLOADS[WL])
wl.setdefault("batch", wl.get("global_batch", 1))
sd, tc, dc = bench.build_decoder(wl, WL, torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
f = sd.verify if which.startswith("verify") else sd.draft
if which == "verify_fused":  # fused layout + cluster split-K on a separate weight copy
    from paper_2512_23858_b200.model import weights_to
    from paper_2512_23858_b200.plan import ForwardPlan

    g = Forward(f.cfg, weights_to(sd.tw, f.cache.device), f.cache, f.B, f.R, f.mask_words, f.act_dtype,
                plan=ForwardPlan(fused_epilogues=True, cluster_split_k="nocluster" not in sys.argv))
else:
    from paper_2512_23858_b200.plan import ForwardPlan

    kw, late = {}, False
    for a in sys.argv[2:]:  # plan overrides, e.g. tree_attn=1 tree_csplit=4 (late_trigger=1, nopf=1)
        k, v = a.split("=")
        if k == "late_trigger":
            late = bool(int(v))
        elif k == "nopf":
            kw["verify_attn_l2"] = ()
            kw["draft_attn_l2"] = ()
        else:
            kw[k] = int(v) if k != "tree_attn" else bool(int(v))
    g = Forward(f.cfg, f.w, f.cache, f.B, f.R, f.mask_words, f.act_dtype, plan=ForwardPlan(**kw))
    if late and g.at_plans:
        for pl in g.at_plans:
            L.check(L.lib().ygg_attn_tree_set_trigger(pl, 1))
for t in ("tokens", "pos", "slot", "req", "qmask", "blk_start", "blk_len"):
    getattr(g, t).copy_(getattr(f, t))
lib = L.lib()
dbg = None
if getattr(g, "at_plans", None):  # per-CTA checkpoints of layer 10's tree attention
    dbg = torch.zeros(1024, 16, dtype=torch.int64, device="cuda")
    L.check(lib.ygg_attn_tree_set_debug(g.at_plans[10], dbg.data_ptr()))
CAP = 2048
buf = torch.zeros(CAP, 8, dtype=torch.int64, device="cuda")


def reset():
    buf[:, 0] = -1  # ~0 as u64 (atomicMin fields)
    buf[:, 1] = -1
    buf[:, 2:] = 0


def level(stream=None):
    """One EGT draft level exactly as the step enqueues it (engine.SpecDecoder._launch_step)."""
    sh = sd.shape
    s = L.stream_ptr(stream)
    dr, gr = sd.draft, sd.grown
    L.check(lib.ygg_level_inputs(gr.struct, sd.seq.struct, sd.R, sh.expansion_k, dr.tokens.data_ptr(),
                                 dr.pos.data_ptr(), dr.slot.data_ptr(), dr.req.data_ptr(), dr.qmask.data_ptr(),
                                 dr.mask_words, dr.blk_start.data_ptr(), dr.blk_len.data_ptr(),
                                 sd.cand_n.data_ptr(), s))
    dr.run(stream)
    sd._draft_topk(sd.B * sd.R, sh.expansion_k, s)
    L.check(lib.ygg_egt_grow_level(gr.struct, sd.R, sh.expansion_k, sh.width, sd.cand_tok.data_ptr(),
                                   sd.cand_prob.data_ptr(), sd.cand_n.data_ptr(), s))


if which == "level":  # start from a fresh tree (pass 0 + roots), as the step does
    sh0 = sd.shape
    dr0, gr0 = sd.draft, sd.grown
    L.check(lib.ygg_pass0_inputs(sd.seq.struct, sd.R, sd.tree_cap, dr0.tokens.data_ptr(), dr0.pos.data_ptr(),
                                 dr0.slot.data_ptr(), dr0.req.data_ptr(), dr0.qmask.data_ptr(), dr0.mask_words,
                                 dr0.blk_start.data_ptr(), dr0.blk_len.data_ptr(), L.stream_ptr()))
    dr0.run()
    sd._draft_topk(sd.B * sd.R, sh0.expansion_k, L.stream_ptr())
    L.check(lib.ygg_init_roots(gr0.struct, sd.cand_tok.data_ptr(), sd.cand_prob.data_ptr(), sh0.expansion_k, sd.R, 1,
                               L.stream_ptr()))
    torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
L.check(lib.ygg_trace_arm(buf.data_ptr(), CAP))
with torch.cuda.graph(graph):
    if which == "level":
        level()
    else:
        g.run()
ids = (L.C.c_int * CAP)()
n = lib.ygg_trace_used(ids, CAP)
L.check(lib.ygg_trace_arm(None, 0))
tree_state = [x.clone() for x in (sd.grown.token, sd.grown.parent, sd.grown.depth, sd.grown.prob, sd.grown.cum,
                                   sd.grown.mask, sd.grown.size, sd.grown.frontier, sd.grown.frontier_n,
                                   sd.grown.flags)]


def restore():
    for dst, src in zip((sd.grown.token, sd.grown.parent, sd.grown.depth, sd.grown.prob, sd.grown.cum, sd.grown.mask,
                         sd.grown.size, sd.grown.frontier, sd.grown.frontier_n, sd.grown.flags), tree_state):
        dst.copy_(src)


for _ in range(5):
    restore()
    graph.replay()
restore()
reset()
torch.cuda.synchronize()
graph.replay()
torch.cuda.synchronize()
t = buf[:n].cpu().tolist()
names = {1: "gemv", 2: "attn_dec", 3: "gemm", 4: "epi_store", 5: "epi_resid", 6: "epi_swiglu", 7: "epi_qkv",
         8: "attn_tc", 9: "attn_combine", 10: "topk_merge", 11: "grow", 13: "level_inputs", 14: "embed", 15: "attn_tree"}
t0 = t[0][0]
rows = []
prev_end = None
for i in range(n):
    s, w, e = (t[i][0] - t0) / 1e3, (t[i][1] - t0) / 1e3, (t[i][2] - t0) / 1e3
    gap = None if prev_end is None else round(w - prev_end, 2)
    marks = [round((t[i][j] - t0) / 1e3 - w, 2) for j in range(3, 8) if t[i][j]]
    rows.append({"i": i, "k": names.get(ids[i], ids[i]), "start": round(s, 2), "released": round(w, 2),
                 "end": round(e, 2), "after_release": round(e - w, 2), "release_gap": gap, "marks": marks})
    prev_end = e
for r in rows:
    print(json.dumps(r))
tot, gaps, seen = {}, {}, {}
for r in rows:
    k = r["k"]
    seen[k] = seen.get(k, 0) + 1
    per_layer = {"gemv": 5, "gemm": 4, "epi_resid": 2, "attn_dec": 1, "attn_tree": 1}.get(k)  # gemv: qkv/attn/o/gu/down slots by index
    if k == "gemv":
        key = f"gemv#{r['i'] % 5 if r['i'] < n - 1 else 'lm'}"
    elif per_layer:
        key = f"{k}#{(seen[k] - 1) % per_layer}"
    else:
        key = k
    tot.setdefault(key, []).append(r["after_release"])
    if r["release_gap"] is not None:
        gaps.setdefault(key, []).append(r["release_gap"])
print(json.dumps({k: [round(sum(v) / len(v), 2), len(v)] for k, v in tot.items()}))
print(json.dumps({"gap_" + k: round(sum(v) / len(v), 2) for k, v in gaps.items()}))
print(json.dumps({"sum_after_release": round(sum(sum(v) for v in tot.values()), 1),
                  "sum_gaps": round(sum(sum(v) for v in gaps.values()), 1)}))
print(json.dumps({"total_us": round((t[n - 1][2] - t0) / 1e3, 2), "launches": n}))
if dbg is not None:
    NAMES = ["entry", "cluster_sync", "released", "q", "kv0", "kv_last_r0", "p_r0", "o_done", "pushed", "recv",
             "end", "rounds", "s_r0"]
    d = dbg.cpu()
    d = d[: int((d[:, 2] > 0).sum())].double()
    t0 = d[:, 2].min()
    st = {}
    for k, nm in enumerate(NAMES):
        col = d[:, k]
        v = col[col > 0]
        if nm != "rounds" and len(v):
            st[nm] = [round(float((v.median() - t0) / 1e3), 2), round(float((v.max() - t0) / 1e3), 2)]
    print(json.dumps({"attn_tree_stamps": st}))
