"""Summarise ncu --set full reports into profiles/ncu_summary.json.

usage: python tools/ncu_summary.py <round-tag> name=path.ncu-rep ...
Per kernel: duration, DRAM bytes per launch (dram__bytes_read.sum +
dram__bytes_write.sum), achieved occupancy, warp execution efficiency,
registers, issue-slot utilisation and the top stall reasons.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1.0}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def num(d, k, scale=True):
    u, v = d[k]
    x = float(v.replace(",", ""))
    return x * UNITS.get(u, 1.0) if scale else x


def main():
    tag = sys.argv[1]
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        d = raw(rep)
        stalls = sorted(((num(d, k, False), k.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", "")) for k in d if k.startswith("smsp__average_warps_issue_stalled_")
            and k.endswith("_per_issue_active.ratio")), reverse=True)[:5]
        summary[name] = {
            "round": tag,
            "report": os.path.relpath(rep, ROOT),
            "duration_s": num(d, "gpu__time_duration.sum"),
            "dram_bytes_per_launch": num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum"),
            "dram_throughput_pct": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", False),
            "registers_per_thread": num(d, "launch__registers_per_thread", False),
            "achieved_occupancy_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active", False),
            "warp_execution_efficiency_threads": num(d, "smsp__thread_inst_executed_per_inst_executed.ratio", False),
            "issue_slots_busy_pct": num(d, "sm__inst_issued.avg.pct_of_peak_sustained_active", False),
            "instructions_executed": num(d, "smsp__inst_executed.sum", False),
            "top_stalls_per_issue": {k: round(v, 3) for v, k in stalls},
        }
    json.dump(summary, open(path, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
