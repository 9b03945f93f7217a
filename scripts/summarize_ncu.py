"""Summarize ncu outputs into small text files for profiles/ (the .ncu-rep files stay in gpurun_out/).

    python scripts/summarize_ncu.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --out profiles/r01_c2.txt
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def rep_summary(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"(no data in {path})\n"
    h, units = rows[0], rows[1]
    out = [f"ncu --set full: {path}"]
    for r in rows[2:]:
        out.append(f"kernel: {r[h.index('Kernel Name')]}")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"  {m:70s} {r[i]:>18s} {units[i]}")
    return "\n".join(out) + "\n"


def launches_summary(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki][:90]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = [f"ncu launch list (gpu__time_duration.sum, cold-cache serialised): {path}",
           f"{'launches':>8s} {'avg us':>10s} {'share':>7s}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{len(v):8d} {sum(v) / len(v) / 1000:10.1f} {100 * sum(v) / tot:6.1f}%  {k}")
    return "\n".join(out) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-out", help="write {kernel: dram read + write bytes per launch} (bench.py roofline)")
    a = ap.parse_args()
    parts = [launches_summary(p) for p in a.launches] + [rep_summary(p) for p in a.rep]
    if a.traffic_out:
        import json
        tr = {}
        for p in a.rep:
            raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rows = list(csv.reader(io.StringIO(raw)))
            h, units = rows[0], rows[1]
            for r in rows[2:]:
                name = r[h.index("Kernel Name")].replace("void ", "").split("<")[0].split("(")[0].strip()
                b = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v = float(r[h.index(m)].replace(",", ""))
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[h.index(m)], 1)
                    b += v * scale
                tr.setdefault(name, int(b))
        tr["source"] = "ncu --set full (cold caches): dram__bytes_read.sum + dram__bytes_write.sum per launch, " + ", ".join(a.rep)
        with open(a.traffic_out, "w") as f:
            json.dump(tr, f, indent=1)
    with open(a.out, "w") as f:
        f.write("\n".join(parts))
    print(open(a.out).read())


if __name__ == "__main__":
    main()
