"""Isolated per-launch time of the tree-attention kernels at cfg2 shapes (graph of back-to-back
launches over 32 layers' caches, CUDA events): mma.sync decode attention vs the tcgen05 tree kernel
in several (csplit, row_tiles) plans.  Profiling aid; prints one JSON line.

  python scripts/attn_tree_bench.py [--which verify|draft] [--reps 20]
"""
import argparse
import ctypes as C
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_23858_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="verify")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--P", type=int, default=560)
ap.add_argument("--plans", default="0:0,4:4,4:0,8:0,2:0")
args = ap.parse_args()
L.require_device()
lib = L.lib()
cuda = torch.device("cuda")
if args.which == "verify":
    hd, Hq, Hkv, T, mw, layers = 128, 32, 8, 50, 2, 32
else:
    hd, Hq, Hkv, T, mw, layers = 64, 32, 8, 8, 1, 16
P, B = args.P, 1
S = ((P + T + 63) // 64 + 1) * 64
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(B * T, Hq, hd, device=cuda, generator=g).to(torch.bfloat16)
cache = torch.randn(layers, B, 2, Hkv, S, hd, device=cuda, generator=g).to(torch.bfloat16)
rows = []
for i in range(T):
    par = -1 if i == 0 else (i - 1) // 2
    rows.append((rows[par] if par >= 0 else 0) | (1 << i))
qmask = torch.tensor([[(rows[i] >> (32 * w)) & 0xFFFFFFFF for w in range(mw)] for i in range(T)] * B,
                     dtype=torch.int64).to(torch.int32).to(cuda)
bs = torch.full((B,), P, dtype=torch.int32, device=cuda)
bl = torch.full((B,), T, dtype=torch.int32, device=cuda)
out = torch.zeros(B * T, Hq, hd, dtype=torch.bfloat16, device=cuda)
scale = 1.0 / math.sqrt(hd)
es = cache.element_size()


def layer_ptr(li):
    return cache.data_ptr() + li * cache.stride(0) * es


def timed(launch):
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for li in range(layers):
            launch(li)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) * 1e3 / args.reps / layers, 2)


res = {}
ad = []
for li in range(layers):
    mem = C.create_string_buffer(int(lib.ygg_attn_dec_plan_size()))
    L.check(lib.ygg_attn_dec_plan_init(mem, q.data_ptr(), layer_ptr(li), B, T, Hq, Hkv, hd, S, 0, 0, 0))
    ad.append(mem)
res["attn_dec_us"] = timed(lambda li: L.check(lib.ygg_attn_dec_run(ad[li], bs.data_ptr(), bl.data_ptr(), qmask.data_ptr(),
                                                                   mw, scale, out.data_ptr(), None, L.stream_ptr())))
ref = out.clone()
for spec in args.plans.split(","):
    cs, rt = (int(x) for x in spec.split(":"))
    at = []
    for li in range(layers):
        mem = C.create_string_buffer(int(lib.ygg_attn_tree_plan_size()))
        L.check(lib.ygg_attn_tree_plan_init(mem, q.data_ptr(), layer_ptr(li), B, T, Hq, Hkv, hd, S, cs, rt))
        at.append(mem)
    info = [C.c_int(), C.c_int(), C.c_int()]
    L.check(lib.ygg_attn_tree_info(at[0], *[C.byref(x) for x in info]))
    key = f"tree_c{info[0].value}_rt{info[1].value}_us"
    res[key] = timed(lambda li: L.check(lib.ygg_attn_tree_run(at[li], bs.data_ptr(), bl.data_ptr(), qmask.data_ptr(), mw,
                                                              scale, out.data_ptr(), L.stream_ptr())))
    res[key.replace("_us", "_maxdiff")] = round(float((out.float() - ref.float()).abs().max()), 4)
print(json.dumps(res), flush=True)

# Per-CTA checkpoints of one launch (layer 10) of each tree plan: median / max over CTAs of each stamp
# relative to the earliest dependency release (stamp 2), in microseconds.
NAMES = ["entry", "cluster_sync", "released", "q", "kv0", "kv_last_r0", "p_r0", "o_done", "pushed", "recv",
         "end", "rounds", "s_r0"]
stamps = {}
for spec in args.plans.split(","):
    cs, rt = (int(x) for x in spec.split(":"))
    at = []
    for li in range(layers):
        mem = C.create_string_buffer(int(lib.ygg_attn_tree_plan_size()))
        L.check(lib.ygg_attn_tree_plan_init(mem, q.data_ptr(), layer_ptr(li), B, T, Hq, Hkv, hd, S, cs, rt))
        at.append(mem)
    dbg = torch.zeros(1024, 16, dtype=torch.int64, device=cuda)
    L.check(lib.ygg_attn_tree_set_debug(at[10], dbg.data_ptr()))
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for li in range(layers):
            L.check(lib.ygg_attn_tree_run(at[li], bs.data_ptr(), bl.data_ptr(), qmask.data_ptr(), mw, scale,
                                          out.data_ptr(), L.stream_ptr()))
    gr.replay()
    gr.replay()
    torch.cuda.synchronize()
    d = dbg.cpu()
    ncta = int((d[:, 2] > 0).sum())
    d = d[:ncta].double()
    t0 = d[:, 2].min()
    st = {}
    for k, nm in enumerate(NAMES):
        col = d[:, k]
        if nm == "rounds":
            st[nm] = [int(col.min()), int(col.max())]
            continue
        v = col[col > 0]
        if len(v):
            st[nm] = [round(float((v.median() - t0) / 1e3), 2), round(float((v.max() - t0) / 1e3), 2)]
    stamps[spec] = st
print(json.dumps(stamps), flush=True)
