"""Graph-replayed timing of one draft forward and one verify forward (cfg2 shapes)."""
import json, os, sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
prompts = bench.prompts_for(wl, tc.vocab, 0)
sd.prefill_len = prompts.shape[1]
sd.prefill(prompts)
for _ in range(2):
    sd.step(use_graph=False)
torch.cuda.synchronize()
res = {k: os.environ.get(k) for k in ("YGG_NO_PDL", "YGG_GEMM_SMEM_KB", "YGG_GEMM_MIN_UNITS")}
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
    res[name + "_ms"] = round(a.elapsed_time(b) / 20, 4)
print(json.dumps(res), flush=True)
