"""Executed instructions of the event-loop kernel per engine_core.cuh function.

usage: python tools/sass_phases.py gpurun_out/prof_sim_vN.ncu-rep [events]
Joins the ncu SASS source page (instructions executed per address) with the
inline-aware line table of the built library's sim_kernel<2,false> (nvdisasm
-gi) and charges each instruction to the innermost engine_core.cuh member
function it comes from (development aid; the .so must be the profiled build).
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2512_16099_b200", "csrc", "engine_core.cuh")
LIB = os.path.join(ROOT, "paper_2512_16099_b200", "libmigsched_b200.so")
KERNEL = os.environ.get("SIM_KERNEL", "_ZN4msgk10sim_kernelILi2ELb0ELb0ELb1EEEvNS_7SimArgsE")


def main():
    rep = sys.argv[1]
    events = float(sys.argv[2]) if len(sys.argv) > 2 else 1638400.0
    funcs = []
    for i, l in enumerate(open(SRC).read().split("\n"), 1):
        m = re.match(r"\s+MSG_DI (?:static )?[\w:<>]+ (\w+)\(", l)
        if m and i >= 150:
            funcs.append((i, m.group(1)))

    def fn(line):
        name = "pre"
        for l0, n in funcs:
            if line >= l0:
                name = n
        return name

    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "engine_kernels.sm_100a.cubin", LIB], cwd=d, check=True,
                       capture_output=True)
        sass = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, "engine_kernels.sm_100a.cubin")],
                              capture_output=True, text=True, check=True).stdout.split("\n")
    start = next(i for i, l in enumerate(sass) if l.startswith(KERNEL))
    chain, a2p, pending = [], {}, False
    for l in sass[start + 1:]:
        if l.startswith("//-----"):
            break
        if "//## File" in l:
            if not pending:
                chain = []
            pending = True
            chain += re.findall(r'"([^"]*)", line (\d+)', l)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            pending = False
            ph = "other"
            for f, n in chain:
                if f.endswith("engine_core.cuh") and int(n) >= 184:
                    ph = fn(int(n))
                    break
            a2p[int(m.group(1), 16)] = ph
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ie, ad = hdr.index("Instructions Executed"), hdr.index("Address")
    base = int(data[0][ad], 16)
    c = Counter()
    for r in data:
        c[a2p.get(int(r[ad], 16) - base, "?")] += float(r[ie] or 0)
    tot = sum(c.values())
    print(f"total {tot:.4g} warp instructions, {tot / events:.1f} per handler event")
    for k, v in c.most_common(30):
        print(f"{k:22s} {v / tot * 100:5.1f}%  {v / events:6.1f} inst/event")


if __name__ == "__main__":
    main()
