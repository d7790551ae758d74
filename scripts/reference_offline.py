"""Profile -> objective -> simulator bridge: run the reference's OWN offline drivers
(specsim installed unmodified in baseline/_ref) on the latency / stage profiles measured on the B200
by `bench.py --workload cfg3 --export-profiles DIR` (K8 profiler, reference CSV formats):
simulator.run, sweep_grid (simulator.py:516-550), breakdown (:629-709) and compare (:359-387).

  python scripts/reference_offline.py profiles/b200_cfg2 [out.json]
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

from specsim import simulator  # noqa: E402
from specsim.config import load_config  # noqa: E402


def stats(s):
    return {"aal": s.aal, "step_latency_us": s.step_latency_us, "tpot_us": s.tpot_us, "speedup": s.speedup}


def main(bundle: str, out: str | None = None) -> dict:
    cfg_path = Path(bundle) / "config.json"
    cfg = load_config(str(cfg_path))
    res = {"bundle": str(bundle), "run": stats(simulator.run(cfg))}
    grid = simulator.sweep_grid(cfg, ["draft_depth", "verify_width"], [[2, 4, 6, 8, 12, 16], [8, 16, 32, 64]])
    res["sweep_grid"] = [[r.value, r.aal, r.step_us, r.tpot_us, r.speedup] for r in grid]
    res["breakdown"] = [{k: getattr(r, k) for k in r.__dataclass_fields__} for r in simulator.breakdown(cfg)]
    # compare: EGT with the measured profiles vs the same run with plan search off
    import dataclasses

    other = dataclasses.replace(cfg, plan_search=False)
    rows = simulator.compare([cfg, other], ["egt_plan_search", "egt_serial"])
    res["compare"] = [{"label": r.label, "relative_speedup": r.relative_speedup, **stats(r.stats)} for r in rows]
    text = json.dumps(res, indent=1, default=str)
    if out:
        Path(out).write_text(text + "\n")
    return res


if __name__ == "__main__":
    r = main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
    print(json.dumps(r["run"]))
