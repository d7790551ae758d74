"""Where does the e2e loop lose time vs the device-timed loop?  CPU cost of one replay, and the
e2e loop at several step counts (fixed vs per-step overhead)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
prompts = bench.prompts_for(wl, tc.vocab, 0)
sd.prefill_len = prompts.shape[1]
sd.prefill(prompts)
sd.capture()
for _ in range(4):
    sd.step()
torch.cuda.synchronize()

cpu = []
for _ in range(8):
    t0 = time.perf_counter()
    sd.step()
    cpu.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print("replay cpu ms", [round(x * 1e3, 3) for x in cpu])

ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for n in (8, 32, 96):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record()
    for _ in range(n):
        sd.step()
    ev[1].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev = ev[0].elapsed_time(ev[1]) * 1e-3
    r = bench.e2e_run(sd, n, torch.device("cuda"))
    print(f"n={n} back-to-back wall {wall / n * 1e3:.3f} ms dev {dev / n * 1e3:.3f} ms | e2e "
          f"{r['seconds'] / n * 1e3:.3f} ms/step")
