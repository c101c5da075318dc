"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py <name> <report.ncu-rep> [<launches.csv>]
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    name, rep = sys.argv[1], sys.argv[2]
    h, units, rows = raw(rep)
    lines = [f"# ncu --set full summary: {name}", f"source report: {os.path.basename(rep)}", ""]
    summary = []
    for r in rows:
        kn = r[h.index("Kernel Name")]
        d = {"kernel": kn}
        lines.append(f"## {kn}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"- {k}: {r[i]} {units[i]}")
                d[k] = r[i] + (" " + units[i] if units[i] else "")
        stalls = []
        for i, k in enumerate(h):
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), k.split("stalled_")[-1]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:5]
        lines.append("- top stall reasons (pc sampling share): " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in top))
        rb = to_bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
        wb = to_bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
        d["dram_bytes"] = rb + wb
        lines.append(f"- DRAM bytes per launch (read+write): {rb + wb:.4e}")
        lines.append("")
        summary.append(d)
    if len(sys.argv) > 3:
        lines.append("## launch list (gpu__time_duration.sum, --clock-control none, serialised)")
        with open(sys.argv[3]) as f:
            for r in csv.reader(f):
                if len(r) > 10 and r[0].isdigit():
                    lines.append(f"- {r[0]} {r[4]} grid{r[8]} {int(r[-1]) / 1e6:.3f} ms")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{name}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(PROF, f"{name}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
