"""Sweep the synthetic-coupling knobs for the 8B/1B pair and report the greedy AAL."""
import json, sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
for noise in [float(x) for x in sys.argv[1].split(",")]:
    for gain in [float(x) for x in sys.argv[2].split(",")]:
        bench.COUPLING["cfg2"] = dict(rank=2048, logit_scale=16.0, head_noise=noise, layer_gain=gain)
        sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
        prompts = bench.prompts_for(wl, tc.vocab, 0)
        sd.prefill_len = prompts.shape[1]
        sd.prefill(prompts)
        sd.capture()
        n0 = int(sd.seq.n_gen.sum())
        for _ in range(24):
            sd.step()
        torch.cuda.synchronize()
        print(json.dumps({"noise": noise, "gain": gain, "aal": (int(sd.seq.n_gen.sum()) - n0) / 24}), flush=True)
        del sd
        torch.cuda.empty_cache()
