"""Run the cfg2 draft forward a few times (for ncu launch lists of the draft pass)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
sd.step(use_graph=False)
torch.cuda.synchronize()
which = sys.argv[1] if len(sys.argv) > 1 else "draft"
f = sd.draft if which == "draft" else sd.verify
torch.cuda.nvtx.range_push("fwd")
for _ in range(2):
    f.run()
torch.cuda.synchronize()
print("done")
