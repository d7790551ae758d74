"""Prefill cost of the cfg2 decoder (512-token prompt): host wall time vs device time, per model.
  python scripts/prefill_time.py"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200.forward import prefill_causal  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
prompts = bench.prompts_for(wl, tc.vocab, 0)
res = {}
for it in range(4):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    sd.prefill(prompts)
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res[f"prefill_{it}"] = {"host_enqueue_ms": round((t1 - t0) * 1e3, 3), "wall_ms": round((t2 - t0) * 1e3, 3),
                            "device_ms": round(a.elapsed_time(b), 3)}
pd = prompts.to("cuda", torch.int32)
for name, cfg, w, cache, logits in (("target", tc, sd.tw, sd.tcache, True), ("draft", dc, sd.dw, sd.dcache, False)):
    for it in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        prefill_causal(cfg, w, cache, pd, torch.bfloat16, logits, sd._prefill_fwd)
        b.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res[f"{name}_{it}"] = {"wall_ms": round((t2 - t0) * 1e3, 3), "device_ms": round(a.elapsed_time(b), 3)}
    # graph-replayed forward of the same chunk: the device floor without host launch overhead
    f = [v for k, v in sd._prefill_fwd.items() if k[0] == cfg.name][0]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.run()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    res[f"{name}_graph_ms"] = round(a.elapsed_time(b) / 5, 3)
    res[f"{name}_flops_T"] = round(2 * cfg.matmul_params() * pd.numel() / 1e12, 3)
print(json.dumps(res), flush=True)
