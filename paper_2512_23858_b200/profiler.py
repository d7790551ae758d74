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
