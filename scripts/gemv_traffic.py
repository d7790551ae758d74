"""Summarise scripts/gpu/gemv_traffic.sh (ncu DRAM bytes of the 65 GEMV launches of one cfg2 draft
pass) into profiles/gemv_traffic.json, which bench.py reports as roofline.traffic (per launch, like
roofline.achieved)."""
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
src = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "gemv_traffic_ncu.csv")
rows = list(csv.reader(src.open()))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
ix = {k: hdr.index(k) for k in ("ID", "Metric Name", "Metric Unit", "Metric Value")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3, "nsecond": 1}
per: dict = {}
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1)
    per.setdefault(int(r[ix["ID"]]), {})[r[ix["Metric Name"]]] = v
launches = [per[k] for k in sorted(per)]
traffic = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in launches]
log = (src.parent / "gemv_traffic_stdout.log").read_text()
weights = json.loads(re.search(r"GEMV_WEIGHT_BYTES (\[.*?\])", log).group(1))
out = {"source": "ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum over the 65 gemv_kernel "
                 "launches of one cfg2 draft pass (scripts/gpu/gemv_traffic.sh)",
       "launches": len(traffic), "dram_bytes_per_launch": int(sum(traffic) / len(traffic)),
       "algorithmic_bytes_per_launch": int(sum(weights) / len(weights)),
       "per_launch_dram_bytes": [int(t) for t in traffic],
       "note": "algorithmic = weight bytes; the QKV / O GEMVs also pull the next 2 x 16 MB of the layer's gate|up "
               "into L2 (counted where it is read from DRAM)"}
(ROOT / "profiles" / "gemv_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(out["dram_bytes_per_launch"], out["algorithmic_bytes_per_launch"])
