"""ncu target: one verify forward's GEMM launches inside a cudaProfilerStart/Stop window.

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/gemm_traffic.csv python scripts/gemm_traffic.py
    python scripts/gemm_traffic.py --summarise gpurun_out/gemm_traffic.csv   # -> profiles/gemm_traffic.json

Algorithmic bytes per launch = weights (bf16) + activations in (bf16) + f32 output; the bench's
``achieved`` counts the weight bytes only.
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
ALG = ROOT / "gpurun_out" / "gemm_alg.json"


def capture():
    import torch

    import bench
    from paper_2512_23858_b200 import _lib as L

    wl = bench.WORKLOADS["cfg2"]
    sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
    prompts = bench.prompts_for(wl, tc.vocab, 0)
    sd.prefill_len = prompts.shape[1]
    sd.prefill(prompts)
    vf = sd.verify
    plans = vf.gemm_calls()
    sp = L.stream_ptr()
    for p in plans:
        vf.launch_gemm(p, sp)
    torch.cuda.synchronize()
    alg = [p.W.numel() * 2 + p.M * p.K * 2 + p.M * p.N * 4 for p in plans]
    wb = [p.W.numel() * 2 for p in plans]
    ALG.parent.mkdir(exist_ok=True)
    ALG.write_text(json.dumps({"algorithmic": alg, "weights": wb}))
    torch.cuda.profiler.start()
    for p in plans:
        vf.launch_gemm(p, sp)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    per = {}
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        per.setdefault(int(d["ID"]), {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")),
                                                              d["Metric Unit"])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = [sum(v[m][0] * scale[v[m][1]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            for _, v in sorted(per.items())]
    alg = json.loads(ALG.read_text())
    n = len(dram)
    assert n == len(alg["algorithmic"]), (n, len(alg["algorithmic"]))
    out = {"dram_bytes_per_launch": int(sum(dram) / n),
           "algorithmic_bytes_per_launch": int(sum(alg["algorithmic"]) / n),
           "weight_bytes_per_launch": int(sum(alg["weights"]) / n),
           "launches": n,
           "source": "ncu dram__bytes_read.sum+dram__bytes_write.sum over the 129 GEMM launches of one cfg2 "
                     "verify forward (scripts/gemm_traffic.py)"}
    (ROOT / "profiles" / "gemm_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarise":
        summarise(sys.argv[2])
    else:
        capture()
