#!/usr/bin/env python
"""Benchmark of the B200 speculative-decoding step (BASELINE.json metric: accepted tokens/s and
p50 step latency per B200; % HBM roofline).

Default workload (N=1): BASELINE.json configs[1] = cfg2 — Llama-3-8B-shaped target + Llama-3.2-
1B-shaped draft (bf16, coupled synthetic random-init weights, random 512-token prompt), EGT
depth 6 width 8, expansion_k 8, max_verify 64, greedy, one request per GPU.  With --gpus N each
rank serves its own request (request sharding, weak scaling, no collective on the data path;
one NCCL all-gather of the generated ids at the end).

Timing: W warm-up graph replays, then K timed replays bracketed by barrier + synchronize, CUDA
events on the launching stream, max over ranks.  Every step streams ~17.5 GB of weights, far
more than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "cfg2": dict(target="llama3-8b", draft="llama3.2-1b", depth=6, width=8, k=8, max_verify=64, batch=1,
                 prompt=512, desc="cfg2: Llama-3-8B target + Llama-3.2-1B draft (bf16), EGT D6 W8 k8, "
                                  "max_verify 64, greedy, 1 request/GPU, 512-token prompt"),
    "cfg1": dict(target="tiny-target", draft="tiny-draft", depth=4, width=4, k=8, max_verify=64, batch=1,
                 prompt=32, desc="cfg1: tiny 4L d256 target + 1L draft, EGT D4 W4 k8, greedy, batch 1"),
    # cfg3: the cfg2 pair, latency-aware choice over 12 EGT shapes from an on-device profiled table.
    "cfg3": dict(target="llama3-8b", draft="llama3.2-1b", depth=6, width=8, k=8, max_verify=64, batch=1,
                 prompt=512, sweep=[(d, w, v) for d in (4, 8, 16) for w in (4, 8) for v in (16, 64)],
                 desc="cfg3: Llama-3-8B target + Llama-3.2-1B draft (bf16), latency-aware objective choosing "
                      "(depth, width, verify-size) from an on-device profiled latency table, sweep of 12 EGT "
                      "shapes, greedy, 1 request/GPU, 512-token prompt"),
    # cfg4: 16 requests sharded over the GPUs (16 / world per GPU), rejection sampling at T = 0.8.
    "cfg4": dict(target="llama3-8b", draft="llama3.2-1b", depth=6, width=8, k=8, max_verify=64, global_batch=16,
                 prompt=2048, gen=1024, mode="sample", temperature=0.8,
                 desc="cfg4: Llama-3-8B target + Llama-3.2-1B draft (bf16), EGT D6 W8 k8, rejection sampling "
                      "T=0.8, 16 requests sharded over the GPUs, 2048-token prompts"),
    # cfg5: the per-GPU slice of 64 requests over 8 GPUs (8 per GPU), 70B target + 8B draft.
    "cfg5": dict(target="llama3-70b", draft="llama3-8b", depth=8, width=16, k=16, max_verify=64, batch=8,
                 prompt=2048, gen=512,
                 desc="cfg5: Llama-3-70B target + Llama-3-8B draft (bf16), EGT D8 W16 k16, greedy, 8 requests "
                      "per GPU (64 over 8 GPUs), 2048-token prompts"),
}
# Coupled synthetic weights (paper_2512_23858_b200/model.py): shared semantic table + permutation.
COUPLING = {
    "cfg2": dict(rank=2048, logit_scale=16.0, head_noise=6.0, layer_gain=2.0),
    "cfg1": dict(rank=256, logit_scale=8.0, head_noise=2.0, layer_gain=2.0),
    "cfg3": dict(rank=2048, logit_scale=16.0, head_noise=6.0, layer_gain=2.0),
    "cfg4": dict(rank=2048, logit_scale=16.0, head_noise=6.0, layer_gain=2.0),
    "cfg5": dict(rank=2048, logit_scale=16.0, head_noise=6.0, layer_gain=2.0),
}
DRAFT_PROF = ((1, 400.0), (64, 420.0), (128, 460.0))    # placeholder Eq.3 table (us); refreshed by K8
VERIFY_PROF = ((1, 2400.0), (64, 2450.0), (128, 2600.0))


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured", d
    return 6650.0, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        try:
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[4 + i] and "Not" not in r[4 + i]})
        load = [s for s in sm if s > 0.5 * (max(sm) if sm else 0)]
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def plan_from_args(items):
    """ForwardPlan from ``key=value`` overrides (ints / bools / None); the default plan when empty."""
    if not items:
        return None
    from paper_2512_23858_b200.plan import ForwardPlan

    kw = {}
    for it in items:
        k, v = it.split("=", 1)
        kw[k] = None if v == "None" else int(v) if v.lstrip("-").isdigit() else v
        if k in ("gemv", "decode_attn", "tree_attn", "fused_epilogues", "fused_layout_gemm", "cluster_split_k",
                 "lm_store_fused", "topk_fused", "prefill_tree_attn") and kw[k] is not None:
            kw[k] = bool(kw[k])
    return ForwardPlan(**kw)


def build_decoder(wl: dict, name: str, device, seed_offset: int = 0, weights=None, profiles=None,
                  overlap_compaction: bool = False, plan=None):
    import torch

    from paper_2512_23858_b200.engine import SpecDecoder, StepShape
    from paper_2512_23858_b200.model import Coupling, init_weights, preset, weights_to

    tc, dc = preset(wl["target"]), preset(wl["draft"])
    if weights is None:
        # generated by CPU generators (like the reference arm, oracle/ref_arm.py), so both arms decode
        # with identical synthetic weights; tensors move to the GPU as bf16 one at a time
        # (a 70B target does not fit host RAM in fp32: cfg5 generates on the device)
        cp = Coupling(**COUPLING[name])
        gen = "cpu" if tc.matmul_params() * 4 < 64e9 else device
        gdt = torch.float32 if gen == "cpu" else torch.bfloat16  # (a 70B fp32 copy does not fit the GPU either)
        tw = weights_to(init_weights(tc, 0, gdt, gen, cp), device, torch.bfloat16)
        dw = weights_to(init_weights(dc, 1, gdt, gen, cp), device, torch.bfloat16)
    else:
        tw, dw = weights

    class PP:
        class drafter:
            breakpoints = DRAFT_PROF

        class verifier:
            breakpoints = VERIFY_PROF

    from paper_2512_23858_b200.engine import GREEDY

    shape = StepShape(wl["depth"], wl["width"], wl["k"], wl["max_verify"])
    max_seq = wl["prompt"] + wl.get("gen", 2048)  # room for the timed steps of up to D+2 tokens
    sd = SpecDecoder(tc, tw, dc, dw, shape, batch=wl["batch"], max_seq=max_seq, act_dtype=torch.bfloat16,
                     profiles=profiles if profiles is not None else PP, device=device, mode=wl.get("mode", GREEDY),
                     temperature=wl.get("temperature", 1.0), overlap_compaction=overlap_compaction, plan=plan)
    if weights is not None:
        return sd, tc, dc
    sd._bench_weights = (tw, dw)
    return sd, tc, dc


def profile_latency(sd, draft_widths=(1, 2, 4, 8, 16), verify_widths=(1, 17, 33, 49, 65), reps=10):
    """K8 on real models: graph-replayed forward latency of the draft at each width (rows of one EGT
    level) and of the target at each verify width, as reference LatencyProfile breakpoints
    (latency.py:34-82, width -> us).  Uses the decoder's weights and caches (contents irrelevant)."""
    import torch

    from paper_2512_23858_b200.forward import Forward

    def time_fwd(cfg, w, cache, rows, gemv=None):
        mw = max(1, (rows + 31) // 32)
        # the target always runs its verify families (never the draft's GEMV, which would also rewrite
        # the shared target weights into the fused layout)
        f = Forward(cfg, w, cache, 1, rows, mw, torch.bfloat16, gemv=gemv)
        f.blk_start.fill_(int(sd.seq.P[0]))
        f.blk_len.fill_(rows)
        f.pos.copy_(f.blk_start[0] + torch.arange(rows, dtype=torch.int32, device=cache.device))
        f.slot.copy_(f.pos)
        f.qmask.fill_(-1)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f.run()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        del g, f
        return a.elapsed_time(b) * 1e3 / reps

    def monotone(pts):  # the reference requires non-decreasing latencies (latency.py:34-65): running max
        out, hi = [], 0.0
        for w, us in pts:
            hi = max(hi, us)
            out.append((w, round(hi, 2)))
        return tuple(out)

    dbp = monotone([(w, time_fwd(sd.dc, sd.dw, sd.dcache, max(w, 2))) for w in draft_widths])
    vbp = monotone([(w, time_fwd(sd.tc, sd.tw, sd.tcache, w, gemv=False)) for w in verify_widths])
    return dbp, vbp


def cfg3_study(base, prompts, steps: int, warmup: int, learn_steps: int = 128, export: str | None = None) -> dict:  # noqa: C901
    """cfg3: the latency-aware objective over 12 EGT shapes D in {4, 8, 16} x W in
    {4, 8} x max_verify in {16, 64} on the cfg2 models.

    1. K8 profiles the draft forward at each level width and the verify at each verify width on the
       device (LatencyProfile breakpoints) and loads them into the table the prune objective reads.
    2. Every shape runs alone (one runtime.AdaptiveDecoder holds all 12 step graphs over one decoding
       state) with the calibrated Eq.3 (per-position acceptance measured on the device during its
       warm-up): measured tokens/s, realized AAL, and the objective's calibrated expected AAL -> its
       predicted tokens/s = E[AAL] / (profiled step latency).  The objective's choice is the shape with
       the best prediction; the measured best is the shape with the best measurement.
    3. The runtime policy (bandit on measured accepted tokens per device-second) learns over
       ``learn_steps`` steps, then decodes ``steps`` timed steps from a fresh prefill."""
    import numpy as np
    import torch

    from paper_2512_23858_b200.engine import StepShape
    from paper_2512_23858_b200.latency import LatencyProfile, latency_at
    from paper_2512_23858_b200.runtime import AdaptiveDecoder

    grid = [(d, w, v) for d in (4, 8, 16) for w in (4, 8) for v in (16, 64)]
    dbp, vbp = profile_latency(base)

    class PP:
        drafter = LatencyProfile(dbp, "drafter")
        verifier = LatencyProfile(vbp, "verifier")

    if export:
        from paper_2512_23858_b200.profiler import write_profile_csv

        Path(export).mkdir(parents=True, exist_ok=True)
        write_profile_csv(list(dbp), Path(export) / "draft_profile.csv")
        write_profile_csv(list(vbp), Path(export) / "verify_profile.csv")
    shapes = [StepShape(d, w, 8, v) for d, w, v in grid]
    ad = AdaptiveDecoder(base.tc, base.tw, base.dc, base.dw, shapes, batch=base.B,
                         max_seq=prompts.shape[1] + (max(learn_steps, 64) + max(steps, 40) + max(warmup, 24)) * 18 + 64,
                         profiles=PP, device=base.dev, calibrate=True, explore_steps=6, explore_share=0.05, seed=0,
                         proj_dim=8)
    ad.prefill(prompts)
    ad.capture()

    def timed(fn, n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        g0 = ad.seq.n_gen.clone()
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return float((ad.seq.n_gen - g0).sum()), a.elapsed_time(b) * 1e-3

    rows = []
    n_shape = max(steps, 40)  # per-shape window: accepted lengths vary 1..D+2 step to step
    for i, (d, w, v) in enumerate(grid):
        dec = ad.decs[i]
        ad.prefill(prompts)
        for j in range(max(warmup, 24)):  # warm-up doubles as the calibration window of this shape
            dec.step()
            if j % 4 == 3:
                dec.set_node_table(dec.node_rates())
        ad.prefill(prompts)
        exp = []

        def one():
            dec.step()
            exp.append(dec.exp_aal.clone())

        tokens, secs = timed(one, n_shape)
        exp_aal = float(torch.stack(exp).mean())
        wv = int(dec.w_verify[0])
        step_us = d * latency_at(PP.drafter, max(w, 2)) + latency_at(PP.drafter, 2) + latency_at(PP.verifier, wv + 1)
        rows.append({"depth": d, "width": w, "max_verify": v, "tokens_per_s": round(tokens / secs, 2),
                     "ms_per_step": round(secs * 1e3 / n_shape, 3), "aal": round(tokens / n_shape / base.B, 3),
                     "calibrated_expected_aal": round(exp_aal, 3), "w_verify_last": wv,
                     "predicted_tokens_per_s": round(exp_aal * base.B / (step_us * 1e-6), 2)})
    chosen = max(rows, key=lambda r: r["predicted_tokens_per_s"])
    best = max(rows, key=lambda r: r["tokens_per_s"])
    # acceptance of the deepest shape as the reference's DepthDecayAcceptance, for the offline bridge
    from paper_2512_23858_b200.runtime import fit_depth_decay

    deep = grid.index((16, 8, 64))
    p0, gamma = fit_depth_decay(ad.decs[deep].accept_counts.cpu().numpy(), 16, 8)
    if export:
        from paper_2512_23858_b200.profiler import write_stage_csv

        st = stage_profile(base)
        D = base.shape.depth
        write_stage_csv([("Verify", "base", round(st["Verify"], 2)), ("Accept", "base", round(st["Accept"], 2)),
                         ("BonusSample", "base", 0.0), ("TailDraft", "base", 0.0),
                         ("HeadDraft", "base", round(st["HeadDraft"], 2)),
                         ("DraftStep", "base", round(st["DraftLevels"] / D, 2)),
                         ("PrepareVerify", "base", round(st["Prune"], 2))], Path(export) / "stages.csv")
        cfg = {"seed": 0, "iterations": 512, "acceptance": {"variant": "depth_decay", "p0": round(p0, 6),
                                                              "gamma": round(gamma, 6)},
               "workload": {"variant": "stationary", "drafter": {"variant": "geometric", "top_mass": 0.9,
                                                                 "decay": 0.9}},
               "profiles": {"draft": "draft_profile.csv", "verify": "verify_profile.csv"}, "stages": "stages.csv",
               "policy": {"variant": "egt", "candidate_widths": [1, 2, 4, 8], "max_depth": 16, "max_verify": 64,
                          "expansion_k": 8, "fallback_depth": 8, "predictor": {"variant": "ema", "window": 4,
                                                                               "alpha": 0.4}},
               "plan_search": True}
        (Path(export) / "config.json").write_text(json.dumps(cfg, indent=2) + "\n")
    # runtime policy: learn, then a timed window from a fresh prefill
    ad.prefill(prompts)
    for _ in range(learn_steps):
        ad.step()
        if ad.seq.P.max() > ad.seq.p_limit - 64:
            ad.drain()
            ad.prefill(prompts)
    ad.drain()
    ad.prefill(prompts)
    tokens, secs = timed(ad.step, steps)
    ad.drain()
    counts = np.bincount(np.asarray(ad.trace.chosen[-steps:], dtype=np.int64), minlength=len(grid))
    top = int(counts.argmax())
    bandit = {"tokens_per_s": round(tokens / secs, 2), "ms_per_step": round(secs * 1e3 / steps, 3)}
    # depth predictor (§8 f3): profile (features, realized length) on the deepest shape, train the
    # reference's perceptron on them, then let it choose the depth per step (width: best measured)
    from paper_2512_23858_b200.depth_predictor import TrainConfig, train_predictor

    ad.prefill(prompts)
    samples = ad.collect_depth_samples(deep, 96)
    trained = train_predictor(samples, TrainConfig(max_depth=16, epochs=100))
    ad.policy, ad.predictor = "predictor", trained.predictor
    ad.prefill(prompts)
    n0 = len(ad.trace.chosen)
    ptok, psecs = timed(ad.step, steps)
    ad.drain()
    pdepth = np.bincount([grid[i][0] for i in ad.trace.chosen[n0:]], minlength=17)
    predictor = {"tokens_per_s": round(ptok / psecs, 2), "ms_per_step": round(psecs * 1e3 / steps, 3),
                 "samples": len(samples), "features": ad.features.dim,
                 "train_loss": [round(trained.initial_loss, 4), round(trained.final_loss, 4)],
                 "depth_histogram": {str(d): int(pdepth[d]) for d in (4, 8, 16)},
                 "vs_best": round((ptok / psecs) / best["tokens_per_s"], 4)}
    res = {"profile": {"drafter": dbp, "verifier": vbp}, "sweep": rows,
           "depth_decay_fit": {"p0": round(p0, 4), "gamma": round(gamma, 4), "shape": "D16 W8 V64"},
           "objective_choice": {k: chosen[k] for k in ("depth", "width", "max_verify", "tokens_per_s")},
           "measured_best": {k: best[k] for k in ("depth", "width", "max_verify", "tokens_per_s")},
           "objective_vs_best": round(chosen["tokens_per_s"] / best["tokens_per_s"], 4),
           "adaptive": {**bandit, "policy": "bandit", "learn_steps": learn_steps,
                        "most_used": dict(zip(("depth", "width", "max_verify"), grid[top])),
                        "most_used_share": round(float(counts[top]) / steps, 3),
                        "vs_best": round(bandit["tokens_per_s"] / best["tokens_per_s"], 4)},
           "predictor": predictor}
    del ad
    torch.cuda.empty_cache()
    return res


def run_cfg3(args, device):
    """--workload cfg3: the cfg3 study as its own JSON line (value = the runtime policy's tokens/s)."""
    wl = dict(WORKLOADS["cfg3"])
    base, tc, dc = build_decoder(wl, "cfg3", device)
    prompts = prompts_for(wl, tc.vocab, 0)
    base.prefill(prompts)
    res = cfg3_study(base, prompts, args.steps, args.warmup, export=args.export_profiles)
    line = {"metric": "accepted tokens/s", "value": res["adaptive"]["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["adaptive"]["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (coupled random-init weights, random prompts)",
            "config": {"workload": wl["desc"]}, "cfg3": res}
    print(json.dumps(line), flush=True)


def prompts_for(wl, vocab, rank):
    import torch

    rows = []
    for b in range(wl["batch"]):
        g = torch.Generator().manual_seed(1000 + rank * wl["batch"] + b)
        rows.append(torch.randint(0, vocab, (wl["prompt"],), generator=g))
    return torch.stack(rows)


def _ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per GEMM launch from the committed ncu capture."""
    p = ROOT / "profiles" / "gemm_traffic.json"
    if not p.exists():
        return {"traffic": None}
    t = json.loads(p.read_text())
    return {"traffic": t["dram_bytes_per_launch"], "traffic_algorithmic": t["algorithmic_bytes_per_launch"],
            "traffic_source": t["source"]}


def gemm_roofline(sd, peak_gbs):
    """Per-launch CUDA-event timing of every GEMM of one verify forward (the dominant kernel),
    each launch streaming a different layer's weights from HBM."""
    import torch

    from paper_2512_23858_b200 import _lib as L

    lib = L.lib()
    vf = sd.verify
    plans = vf.gemm_calls()
    s = torch.cuda.current_stream()
    sp = L.stream_ptr()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in plans]
    for _ in range(2):
        for p in plans:
            vf.launch_gemm(p, sp)
    torch.cuda.synchronize()
    for p, (a, b) in zip(plans, ev):
        a.record(s)
        vf.launch_gemm(p, sp)
        b.record(s)
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) * 1e-3 for a, b in ev]
    nbytes = [p.W.numel() * p.W.element_size() for p in plans]
    flops = [2.0 * p.M * p.N * p.K for p in plans]
    achieved = sum(nbytes) / sum(times) / 1e9
    _, _, pk = _peaks()
    tc_peak = float(pk.get("bf16_tflops", 1630.0))
    ridge = tc_peak * 1e12 / (peak_gbs * 1e9)  # FLOP per byte where the two roofs cross
    if vf.M > ridge:  # weight-streaming intensity is M FLOP/B: at cfg4 / cfg5 batch the tensor pipe bounds
        tf = sum(flops) / sum(times) / 1e12
        return {"bound": "tensor", "achieved": round(tf, 1), "peak": tc_peak, "unit": "TFLOP/s",
                "frac": round(tf / tc_peak, 4), "traffic": None,
                "kernel": "gemm_bf16_tc_kernel (swap-AB tcgen05 stream-K)", "launches_timed": len(plans),
                "flops_per_launch_avg": int(sum(flops) / len(plans)), "rows": vf.M,
                "avg_launch_us": round(sum(times) / len(times) * 1e6, 2), "hbm_gbs": round(achieved, 1)}
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak_gbs, "unit": "GB/s",
            "frac": round(achieved / peak_gbs, 4), **_ncu_traffic(),
            "kernel": "gemm_bf16_tc_kernel (swap-AB tcgen05 stream-K weight streaming)",
            "launches_timed": len(plans), "bytes_per_launch_avg": int(sum(nbytes) / len(plans)),
            "avg_launch_us": round(sum(times) / len(times) * 1e6, 2)}


def gemv_roofline(sd, peak_gbs):
    """The dominant kernel (row-block GEMV, 4 per draft layer + the LM head) measured IN the graph of
    one draft pass (profiler.kernel_timeline): each launch's incremental cost to the pass (its end minus
    the previous kernel's end, so dependency gaps are charged to it); achieved = weight bytes of the
    pass's GEMVs / the sum of those costs.  The isolated per-launch event timing (launch overhead
    included) is kept beside it."""
    import ctypes as C

    import torch

    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.profiler import kernel_timeline

    lib = L.lib()
    f = sd.draft
    if not getattr(f, "gemv", False):
        return None
    mats = [m for lw in f.w["layers"] for m in (lw["wqkv"], lw["wo"], lw["wgu"], lw["wdown"])] + [f.w["lm_head"]]
    nbytes = [m.numel() * m.element_size() for m in mats]
    rows = [r for r in kernel_timeline(f.run) if r["kernel"] == "gemv"]
    assert len(rows) == len(mats), (len(rows), len(mats))
    inc = [r["incremental"] * 1e-6 for r in rows]
    own = [(r["end"] - r["released"]) * 1e-6 for r in rows]
    achieved = sum(nbytes) / sum(inc) / 1e9
    # isolated launches (events around each), for comparison with round 1
    calls = [op for layer in f.gv for op in layer] + [f.gv_lm]
    s = torch.cuda.current_stream()
    sp = L.stream_ptr()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in calls]
    for (pl, ep), (a, b) in zip(calls, ev):
        a.record(s)
        L.check(lib.ygg_gemv_run(pl, C.byref(ep), sp))
        b.record(s)
    torch.cuda.synchronize()
    iso = [a.elapsed_time(b) * 1e-3 for a, b in ev]
    out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak_gbs, "unit": "GB/s",
           "frac": round(achieved / peak_gbs, 4), "traffic": None,
           "kernel": "gemv_kernel (row-block GEMV, mma.sync from a 128B-swizzled TMA ring, fused epilogues)",
           "timing": "in-graph, one draft pass, per-launch incremental cost (end - previous end)",
           "launches_timed": len(rows), "bytes_per_launch_avg": int(sum(nbytes) / len(rows)),
           "avg_launch_us": round(sum(inc) / len(inc) * 1e6, 2),
           "achieved_release_to_end": round(sum(nbytes) / sum(own) / 1e9, 1),
           "lm_head_gbs": round(nbytes[-1] / inc[-1] / 1e9, 1),
           "isolated_events": {"achieved": round(sum(nbytes) / sum(iso) / 1e9, 1),
                               "avg_launch_us": round(sum(iso) / len(iso) * 1e6, 2)}}
    p = ROOT / "profiles" / "gemv_traffic.json"
    if p.exists():
        t = json.loads(p.read_text())
        out.update({"traffic": t["dram_bytes_per_launch"], "traffic_algorithmic": t["algorithmic_bytes_per_launch"],
                    "traffic_source": t["source"]})
    return out


def verify_roofline(sd, peak_gbs, reps=10):
    """Whole verify forward (graph-captured) vs its algorithmic HBM bytes (weights + KV read)."""
    import torch

    vf = sd.verify
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        vf.run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) * 1e-3 / reps
    P = int(sd.seq.P.max())
    kv = sd.B * (P + sd.T) * sd.tc.kv_bytes_per_token(2)
    nbytes = vf.weight_bytes() + kv
    return {"verify_ms": round(t * 1e3, 3), "bytes": nbytes, "achieved_gbs": round(nbytes / t / 1e9, 1),
            "frac": round(nbytes / t / 1e9 / peak_gbs, 4)}


def stage_profile(sd, steps=4):
    """K8: on-device globaltimer stamps around each stage of one step (separate graph)."""
    import torch

    from paper_2512_23858_b200 import profiler

    prof = profiler.StageProfiler(sd)
    return prof.measure(steps)


def host_steps(wl_name: str, steps: int, warmup: int) -> dict:
    """The speculative step on the host CPU (oracle/ref_arm.py): the reference's own specsim tree
    logic from baseline/_ref + the fp32 torch-CPU model port, every host thread, full workload
    (same model shapes, tree shape and prompt length), ``warmup`` untimed then ``steps`` timed steps."""
    from oracle import ref_arm

    wl = WORKLOADS[wl_name]
    res = ref_arm.run_host_steps(wl, COUPLING[wl_name], steps, warmup, DRAFT_PROF, VERIFY_PROF)
    res.update(ref_arm.host_info())
    return res


def _host_sample(res: dict, steps: int, warmup: int) -> str:
    return (f"{steps} timed speculative steps (+{warmup} untimed) of the full workload on the host: "
            f"{res['target_layers']}-layer target + {res['draft_layers']}-layer draft in fp32 torch-CPU "
            f"({res['threads']} threads, {res['cpu_model']}), tree logic = {res['tree_impl']} "
            f"({res['tree_logic_ms_per_step']:.2f} ms/step), measured AAL {res['aal']:.3f}")


def run_reference(args, rank, world):
    """Reference arm: the step on the host CPU (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    res = host_steps(args.workload, args.steps, args.warmup)
    kind = "reference" if res["tree_impl"] == "specsim" else "port"
    v = round(res["tokens_per_s"], 4)
    line = {"impl": "reference", "metric": "accepted tokens/s", "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(res["ms_per_step"], 2), "p50_step_ms": round(res["p50_step_ms"], 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (coupled random-init weights from CPU generators, random prompt)",
            "config": {"workload": wl["desc"], "aal": round(res["aal"], 4)},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": res["threads"], "kind": kind,
                             "sample": _host_sample(res, args.steps, args.warmup)},
            "host": {"cpu_model": res["cpu_model"], "cpu_count": res["cpu_count"], "init_s": res["init_s"],
                     "prefill_s": res["prefill_s"], "tree_impl": res["tree_impl"],
                     "tree_logic_ms_per_step": round(res["tree_logic_ms_per_step"], 3)},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2512_23858_b200 import _lib as L

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    wl = dict(WORKLOADS[args.workload])
    if "global_batch" in wl:
        wl["batch"] = max(1, wl["global_batch"] // world)
    peak, peak_kind, _ = _peaks()
    sd, tc, dc = build_decoder(wl, args.workload, device, overlap_compaction=args.overlap_compaction,
                               plan=plan_from_args(args.plan))
    prompts = prompts_for(wl, tc.vocab, rank)
    sd.prefill_len = prompts.shape[1]
    sd.prefill(prompts)
    n0 = L.launches["count"]
    sd.capture()
    launches_per_step = L.launches["count"] - n0
    sample = sd.mode != "greedy"
    for i in range(args.warmup):
        if sample:
            sd.set_uniforms(i, rank)
        sd.step()
    # The timed window is the first K steps after a fresh prefill of the same prompts, so that the
    # end-to-end run below (prefill + the same K steps through the public API) decodes exactly the
    # same steps: greedy (and seeded SAMPLE) decoding is deterministic.
    sd.prefill(prompts)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    gen0 = sd.seq.n_gen.clone()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize()
    evs[0].record()
    for i in range(args.steps):
        if sample:  # host-pregenerated acceptance uniforms, default_rng([seed, step]) (simulator.py:306)
            sd.set_uniforms(i, rank)
        sd.step()
        evs[i + 1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_s = evs[0].elapsed_time(evs[-1]) * 1e-3
    tokens = int((sd.seq.n_gen - gen0).sum())
    t = torch.tensor([total_s, float(tokens)], dtype=torch.float64, device=device)
    if world > 1:
        tmax = t[0:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t[1:2].clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        total_s, tokens_all = float(tmax), float(tsum)
    else:
        tokens_all = float(tokens)
    aal = tokens / (args.steps * sd.B)

    # ---- e2e through the public API: pinned H2D of the step inputs, replay, D2H of the emitted tokens
    e2e = e2e_run(sd, prompts, args.steps, device, rank)
    e2e_tokens = torch.tensor([e2e["tokens"]], dtype=torch.float64, device=device)
    e2e_t = torch.tensor([e2e["seconds"]], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(e2e_tokens, op=dist.ReduceOp.SUM)
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)

    gemm = gemm_roofline(sd, peak)
    gv = gemv_roofline(sd, peak)
    ver = verify_roofline(sd, peak)
    try:
        stages = stage_profile(sd)
    except Exception as exc:  # profiler is diagnostic only
        stages = {"error": str(exc)}
    ar = ar_baseline(sd, prompts) if not args.no_ar_baseline else None
    # Acceptance over a longer decode (untimed; after every other measurement, which all run at the
    # timed window's context length): the K-step window's AAL is a property of the synthetic weights and
    # of where the greedy text happens to go, so the line also reports the AAL of the first K + extra
    # steps after a fresh prefill and the token rate it implies at the timed step time.
    long_steps = 0 if sample else args.aal_steps
    aal_long, frozen = None, False
    if long_steps:
        sd.prefill(prompts)
        g_long = sd.seq.n_gen.clone()
        for _ in range(long_steps + args.steps):
            sd.step()
        torch.cuda.synchronize()
        frozen = bool((sd.seq.status != 0).any())
        aal_long = float((sd.seq.n_gen - g_long).sum()) / ((long_steps + args.steps) * sd.B)
    # final result gather of every request's generated ids (the only collective)
    from paper_2512_23858_b200.dist import gather_generated

    mine = {rank * sd.B + b: sd.generated(b) for b in range(sd.B)}
    merged = gather_generated(mine, world)
    gathered = {"ranks": world, "requests": len(merged), "tokens": sum(len(v) for v in merged.values())}
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        res = host_steps(args.workload, 2, 1)
        cpu = {"value": round(res["tokens_per_s"], 4), "unit": "tokens/s", "cores": res["threads"],
               "kind": "reference" if res["tree_impl"] == "specsim" else "port",
               "sample": _host_sample(res, 2, 1)}
    line = {
        "metric": "accepted tokens/s", "value": round(tokens_all / total_s, 2), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_s * 1e3 / args.steps, 4), "p50_step_ms": round(statistics.median(step_ms), 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (coupled random-init weights, random prompts)",
        "config": {"workload": wl["desc"], "aal": round(aal, 4), "requests_per_gpu": sd.B,
                   "parallelism": f"request sharding x{world} (replicas, no collective in the step)",
                   "l2": "inputs > L2: ~17.5 GB of weights streamed per step (126 MB L2)",
                   "coupling": COUPLING[args.workload]},
        "roofline": gv if gv is not None else gemm, "verify_gemm_roofline": gemm, "verify_roofline": ver,
        "stage_us": stages,
        "e2e": {"value": round(float(e2e_tokens) / float(e2e_t), 2), "unit": "tokens/s",
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "ms_per_step": round(float(e2e_t) * 1e3 / args.steps, 4),
                "aal": round(e2e["tokens"] / (args.steps * sd.B), 4),
                "note": "prompt H2D + prefill + the same K steps as the timed window (fresh prefill of "
                        "the same prompt; deterministic decoding) with streamed per-step readback, all timed"},
        "aal_long": None if not long_steps else {
            "steps": long_steps + args.steps, "aal": round(aal_long, 4), "frozen": frozen,
            "tokens_per_s_at_step_time": round(aal_long * sd.B * world / (total_s / args.steps), 2),
            "note": "greedy AAL over the first K + extra steps after a fresh prefill (untimed, after every other "
                    "measurement); the value above uses the timed window's own AAL"},
        "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
        "clocks": clk, "cpu_baseline": cpu, "peak_kind": peak_kind, "gathered": gathered, "ar_baseline": ar,
        "speculative_speedup_vs_ar": round((tokens_all / total_s) / (world * ar["tokens_per_s"]), 3) if ar else None,
    }
    print(json.dumps(line), flush=True)


def e2e_run(sd, prompts, steps, device, rank=0):
    """End to end through the public API, as a user serving one batch: the prompts go host -> device
    from pinned memory, the decoder prefills them, then every step (SAMPLE: after the H2D of its
    acceptance uniforms from a pinned double buffer) replays the step graph and its emitted tokens come
    back to pinned host memory.  The readback is double-buffered: the host consumes step i-1's tokens
    (event wait) while step i runs, as a server streaming tokens would.  Everything from the prompt
    upload to the last token on the host is inside the timed region."""
    import torch

    B = sd.B
    sample = sd.mode != "greedy"
    n_emit = sd.emit.shape[1]
    host_out = [torch.zeros(B, n_emit, dtype=torch.int32).pin_memory() for _ in range(2)]
    host_prompts = prompts.to(torch.int32).pin_memory()
    h2d = host_prompts.numel() * host_prompts.element_size()
    if sample:
        h2d += steps * sd.uniforms.numel() * sd.uniforms.element_size()
    d2h = steps * host_out[0].numel() * host_out[0].element_size()
    done = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    streamed = 0
    t0 = time.perf_counter()
    sd.prefill(host_prompts.to(device, non_blocking=True))
    gen0 = sd.seq.n_gen.clone()
    for i in range(steps):
        if sample:  # pinned double-buffered H2D of this step's uniforms, enqueued before the replay
            sd.set_uniforms(i, rank)
        sd.step()
        sd.read_emitted(host_out[i % 2])
        done[i % 2].record()
        if i > 0:
            done[(i - 1) % 2].synchronize()
            streamed += int(host_out[(i - 1) % 2][:, 0].sum())
    done[(steps - 1) % 2].synchronize()
    streamed += int(host_out[(steps - 1) % 2][:, 0].sum())
    dt = time.perf_counter() - t0
    tokens = int((sd.seq.n_gen - gen0).sum())
    if streamed != tokens:
        raise RuntimeError(f"e2e: host received {streamed} tokens, device generated {tokens}")
    return {"tokens": tokens, "seconds": dt, "h2d": h2d // steps, "d2h": d2h // steps}


def ar_baseline(sd, prompts, n_tokens: int = 32) -> dict:
    """Plain greedy autoregressive decoding of the target alone (engine.ARDecoder: graph-replayed
    single-row forwards through the verify kernel families), for the speculative speed-up."""
    import torch

    from paper_2512_23858_b200.engine import ARDecoder

    ar = ARDecoder(sd.tc, sd.tw, batch=sd.B, max_seq=prompts.shape[1] + n_tokens + 8, device=sd.dev)
    ar.generate(prompts, 4)  # builds the prefill plans and captures the token graph
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n_tokens):
        ar.graph.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n_tokens
    del ar
    torch.cuda.empty_cache()
    return {"tokens_per_s": round(1e3 * sd.B / ms, 2), "ms_per_token": round(ms, 4),
            "kernels": "verify families at 1 row (tcgen05 stream-K GEMM + epilogues, decode attention)"}


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ar-baseline", action="store_true")
    ap.add_argument("--plan", action="append", default=[],
                    help="ForwardPlan override key=value (A/B runs), e.g. --plan fused_layout_gemm=1")
    ap.add_argument("--aal-steps", type=int, default=180,
                    help="untimed extra greedy steps after the e2e run for the long-window AAL (0 = off)")
    ap.add_argument("--overlap-compaction", action="store_true",
                    help="two-lane step: target KV compaction on a side stream under the next draft phase")
    ap.add_argument("--export-profiles", default=None,
                    help="cfg3: write the K8-measured draft / verify latency profiles (reference CSV format) here")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-run this script under torch.distributed.run with N ranks
        from paper_2512_23858_b200.dist import launch

        sys.exit(launch(args.gpus, str(Path(__file__).resolve()), sys.argv[1:]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.workload == "cfg3":
            if rank == 0:
                import torch

                run_cfg3(args, torch.device("cuda", local_rank))
            return
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
