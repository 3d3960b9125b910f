"""Per-opcode executed-instruction mix of one kernel in an ncu report, per lattice cell.

python tools/sass_mix.py report.ncu-rep --cells N [--top 30]
"""
import argparse
import collections
import csv
import io
import re
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--cells", type=float, required=True, help="lattice updates of the profiled launch")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    op, stall = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+(\.[A-Z0-9_.]+)?)", r[iS].strip())
        o = m.group(2) if m else r[iS].strip()
        op[o] += int(r[iE] or 0)
        stall[o] += int(r[iW] or 0)
    warp_cells = a.cells / 32
    tot = sum(op.values())
    print(f"total {tot / warp_cells:.2f} thread-instructions per cell")
    for o, n in op.most_common(a.top):
        print(f"{o:34s} {n / warp_cells:7.2f}/cell  stall-samples {stall[o]}")


if __name__ == "__main__":
    main()
