"""Run a cfg2 speculative step eagerly (for ncu launch lists) or time kernels in isolation."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

wl = dict(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"])
wl.setdefault("batch", wl.get("global_batch", 1))
n_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sd, tc, dc = bench.build_decoder(wl, sys.argv[1] if len(sys.argv) > 1 else "cfg2", torch.device("cuda"))
prompts = bench.prompts_for(wl, tc.vocab, 0)
sd.prefill_len = prompts.shape[1]
sd.prefill(prompts)
torch.cuda.synchronize()
sd.step(use_graph=False)  # warm (first-use allocations, plan uploads)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("steps")
for _ in range(n_steps):
    sd.step(use_graph=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("aal", float(sd.seq.n_gen.sum()) / n_steps)
