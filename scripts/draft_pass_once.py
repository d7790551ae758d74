"""One cfg2 step (eager) then one more draft pass on its own — the launch sequence ncu filters:
prefill (no GEMV), 1 step = 7 draft passes x 65 GEMV launches, then the measured pass (65 launches).

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemv_kernel \\
      --launch-skip 455 --launch-count 65 --csv python scripts/draft_pass_once.py
"""
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
sd.draft.run()
torch.cuda.synchronize()
mats = [m for lw in sd.draft.w["layers"] for m in (lw["wqkv"], lw["wo"], lw["wgu"], lw["wdown"])] + [sd.draft.w["lm_head"]]
print("GEMV_WEIGHT_BYTES", [m.numel() * m.element_size() for m in mats])
