"""Summarise ncu artefacts into profiles/: per-kernel launch-list shares and key metrics of full captures.

    python scripts/ncu_summary.py <launches.csv> <out.md> [report.ncu-rep ...]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:60]
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"Launches profiled: {len(data)}; summed kernel time {tot / 1e3:.3f} ms (ncu: serialised, cold L2 — "
           "compare shares, not absolutes)\n", "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / v[0]:.2f} | {100 * v[1] / tot:.1f}% |")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"**{d.get('Kernel Name', '?')[:90]}**\n")
        out.append("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in d:
                out.append(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
        out.append("")
    return "\n".join(out)


def main():
    launches, dst = sys.argv[1], sys.argv[2]
    parts = ["## Launch list (one speculative step, eager)\n", launch_table(launches), ""]
    for rep in sys.argv[3:]:
        parts += [f"## Full capture: `{rep.split('/')[-1]}`\n", report(rep)]
    open(dst, "w").write("\n".join(parts) + "\n")


if __name__ == "__main__":
    main()
