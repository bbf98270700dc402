"""Summarise an ncu --set full report and a launch list into profiles/.

    python tools/ncu_summary.py <report.ncu-rep> <launches.csv> <tag>

Writes profiles/<tag>_kernel.json (key metrics of the profiled launch),
profiles/<tag>_launches.csv (the launch list: kernel, duration) and updates
profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_op_imma.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__inst_executed.sum",
]


def raw_metrics(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        d[h] = (v, u)
    return d


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    d = raw_metrics(rep)
    summary = {"report": os.path.basename(rep), "kernel": d.get("Kernel Name", ("?",))[0]}
    for k in KEYS:
        if k in d:
            v, u = d[k]
            try:
                v = float(v.replace(",", ""))
            except ValueError:
                pass
            summary[k] = {"value": v, "unit": u}
    rb = summary.get("dram__bytes_read.sum", {}).get("value", 0.0)
    wb = summary.get("dram__bytes_write.sum", {}).get("value", 0.0)
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rb *= mult.get(summary.get("dram__bytes_read.sum", {}).get("unit", "byte"), 1)
    wb *= mult.get(summary.get("dram__bytes_write.sum", {}).get("unit", "byte"), 1)
    summary["dram_bytes_per_launch"] = rb + wb
    with open(os.path.join(prof, f"{tag}_kernel.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    # launch list -> shares
    text = open(launches).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    per = {}
    lines = ["kernel,launches,total_ns,share"]
    tot = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        ns = float(r["Metric Value"].replace(",", ""))
        c, t = per.get(name, (0, 0.0))
        per[name] = (c + 1, t + ns)
        tot += ns
    for name, (c, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        lines.append(f"{name},{c},{t:.0f},{t / tot:.4f}")
    with open(os.path.join(prof, f"{tag}_launch_shares.csv"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(prof, "ncu_summary.json"), "w") as fh:
        json.dump({"tag": tag, "kernel": summary["kernel"],
                   "dram_bytes_per_launch": summary["dram_bytes_per_launch"]}, fh, indent=1)
    import shutil
    shutil.copy(launches, os.path.join(prof, f"{tag}_launches.csv"))
    print(json.dumps(summary, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
