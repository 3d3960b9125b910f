"""Summarise an ncu --set full report: time, DRAM bytes, throughputs, occupancy, top stall reasons.

python tools/ncu_summary.py report.ncu-rep [--json out.json] [--lups N]
"""
import argparse
import csv
import io
import json
import re
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
    "dram__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    return hdr, units, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    ap.add_argument("--lups", type=float, default=0.0, help="lattice updates of the profiled launch")
    ap.add_argument("--bytes", type=float, default=0.0, help="algorithmic bytes of the profiled launch")
    a = ap.parse_args()
    hdr, units, vals = load(a.report)
    res = []
    for v in vals:
        d = {"kernel": v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = v[i] + (" " + units[i] if units[i] else "")
        stalls = []
        for i, n in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio$", n)
            if m and v[i]:
                try:
                    stalls.append((float(v[i]), m.group(1)))
                except ValueError:
                    pass
        d["top_stalls"] = [f"{n}={x:.2f}" for x, n in sorted(stalls, reverse=True)[:6]]
        try:
            t = float(v[hdr.index("gpu__time_duration.sum")])
            tu = units[hdr.index("gpu__time_duration.sum")]
            t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}.get(tu, 1e-9)
            rb = float(v[hdr.index("dram__bytes_read.sum")])
            wb = float(v[hdr.index("dram__bytes_write.sum")])
            bu = units[hdr.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
            wscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[hdr.index("dram__bytes_write.sum")], 1)
            tot = rb * scale + wb * wscale
            d["dram_bytes_total"] = tot
            d["dram_GBps"] = tot / t_s / 1e9
            if a.lups:
                d["dram_bytes_per_lup"] = tot / a.lups
                d["glups"] = a.lups / t_s / 1e9
            if a.bytes:
                d["traffic_over_algorithmic"] = tot / a.bytes
        except (ValueError, KeyError):
            pass
        res.append(d)
    for d in res:
        for k, x in d.items():
            print(f"{k:70s} {x}")
        print()
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
