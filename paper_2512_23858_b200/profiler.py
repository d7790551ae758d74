"""K8: on-device stage profiler feeding the latency-aware objective.

A profiling copy of the step graph carries ``ygg_stamp`` kernels (one thread reading
%globaltimer) at the stage boundaries of ``SpecDecoder._launch_step``; replays are read back
once at the end, so the measured step runs without host synchronisation.  The per-stage
durations become the reference's on-disk formats: ``stage,variant,duration_us`` rows
(StageProfiles, pkg/src/specsim/scheduler.py:82-103) and ``width,latency_us`` breakpoints
(LatencyProfile, latency.py:164-190), and can refresh the device latency table that K6's Eq.3
objective reads (``SpecDecoder.set_profiles``).
"""

from __future__ import annotations

import statistics

import torch

from . import _lib as L

STAGES = ("HeadDraft", "DraftLevels", "Prune", "Verify", "Accept")


class StageProfiler:
    def __init__(self, decoder):
        self.sd = decoder
        self.stamps = torch.zeros(6, dtype=torch.int64, device=decoder.dev)
        self.graph = None

    def _capture(self):
        lib = L.lib()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.sd._launch_step(stamp=lambda i: L.check(lib.ygg_stamp(self.stamps[i:].data_ptr(), L.stream_ptr())))
        self.graph = g

    def measure(self, steps: int = 4) -> dict:
        """Replay ``steps`` profiled steps; return median per-stage microseconds."""
        if self.graph is None:
            self._capture()
        per = {s: [] for s in STAGES}
        for _ in range(steps):
            self.graph.replay()
            t = self.stamps.cpu().tolist()  # one readback per profiled step (diagnostic path only)
            for i, s in enumerate(STAGES):
                per[s].append((t[i + 1] - t[i]) / 1e3)
        out = {s: round(statistics.median(v), 2) for s, v in per.items()}
        out["step"] = round(sum(out[s] for s in STAGES), 2)
        return out

    def stage_rows(self, med: dict, depth: int) -> list[tuple[str, str, float]]:
        """Reference StageProfiles rows: HeadDraft = pass 0 + first level pass, DraftStep = mean
        of the remaining level passes, Verify, Accept (scheduler.py:37-38, 219-221)."""
        per_level = med["DraftLevels"] / max(depth, 1)
        return [
            ("Verify", "base", med["Verify"] + med["Prune"]),
            ("Accept", "base", med["Accept"]),
            ("HeadDraft", "base", med["HeadDraft"] + per_level),
            ("DraftStep", "base", per_level),
        ]


def write_stage_csv(rows, path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write("stage,variant,duration_us\n")
        for stage, variant, us in rows:
            f.write(f"{stage},{variant},{us!r}\n")


def write_profile_csv(breakpoints, path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write("width,latency_us\n")
        for w, us in breakpoints:
            f.write(f"{int(w)},{float(us)!r}\n")


KERNEL_NAMES = {1: "gemv", 2: "attn_dec", 3: "gemm", 4: "epi_store", 5: "epi_resid", 6: "epi_swiglu", 7: "epi_qkv",
                8: "attn_tc", 9: "attn_combine", 10: "topk_merge", 11: "grow", 13: "level_inputs", 14: "embed"}


def kernel_timeline(run, cap: int = 1024, replays: int = 5, before=None) -> list[dict]:
    """In-graph kernel timeline (profiling only): capture ``run()`` as a graph with the library's
    timeline tracing armed (ygg_trace_arm), replay it, and return per traced launch its kernel name,
    first-CTA start, grid-dependency release and last-CTA end (us, relative to the first start).
    ``before()`` (optional) restores state before each replay.  Launches are PDL-chained, so a kernel's
    incremental cost to the pass is end - previous end."""
    lib = L.lib()
    buf = torch.zeros(cap, 8, dtype=torch.int64, device="cuda")
    g = torch.cuda.CUDAGraph()
    L.check(lib.ygg_trace_arm(buf.data_ptr(), cap))
    try:
        with torch.cuda.graph(g):
            run()
        ids = (L.C.c_int * cap)()
        n = lib.ygg_trace_used(ids, cap)
    finally:
        L.check(lib.ygg_trace_arm(None, 0))
    for _ in range(replays):
        if before:
            before()
        g.replay()
    if before:
        before()
    buf[:, 0] = -1  # ~0 as u64: atomicMin fields
    buf[:, 1] = -1
    buf[:, 2:] = 0
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    t = buf[:n].cpu().tolist()
    t0 = t[0][0]
    rows, prev = [], None
    for i in range(n):
        s, w, e = ((x - t0) / 1e3 for x in t[i][:3])
        rows.append({"kernel": KERNEL_NAMES.get(ids[i], str(ids[i])), "start": s, "released": w, "end": e,
                     "incremental": e - (prev if prev is not None else w)})
        prev = e
    del g
    return rows
