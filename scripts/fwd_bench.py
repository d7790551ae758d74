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

# In-graph per-kernel timeline (stamp kernels between launches; perturbs PDL overlap slightly).
for name, f in (("draft", sd.draft), ("verify", sd.verify)):
    st = torch.zeros(6 * f.cfg.n_layers + 8, dtype=torch.int64, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        (f._run_fused if f.fused else f._run_unfused)(None, st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    t = st.cpu().tolist()
    if f.fused:
        n = 2 + 5 * f.cfg.n_layers + 1
        names = ["embed"] + ["qkv", "attn", "o", "gu", "down"] * f.cfg.n_layers + ["lm_head"]
    else:
        n = 1 + 5 * f.cfg.n_layers + 1
        names = ["qkv(+embed,norm)"] + ["attn", "o+resnorm", "gu+swiglu", "down+resnorm", "qkv+rope"] * f.cfg.n_layers
        names = names[: n - 2] + ["lm_head"]
    d = [(t[i + 1] - t[i]) / 1000 for i in range(n - 1)]
    agg = {}
    for nm, v in zip(names, d):
        agg.setdefault(nm, []).append(v)
    print(name, "total_us", round((t[n - 1] - t[0]) / 1000, 1),
          json.dumps({k: [round(sum(v) / len(v), 2), round(max(v), 2)] for k, v in agg.items()}), flush=True)
