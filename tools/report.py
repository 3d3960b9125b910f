"""One CSV row per BASELINE.json config: the library's default plan timed on this GPU
(median of --reps stencil_run(T) calls, CUDA events on the grid's stream, SM clock and board power sampled
through NVML meanwhile) against the roofline of its plan -- min(HBM copy peak / (bytes per cell per block /
bt), FP64 peak / flops per LUP) -- and at bt = 1, with the ncu DRAM bytes per update of the plan's kernel
(profiles/traffic.json) and the parity / oracle facts the full-size GPU tests recorded
(tests/test_gpu_fullsize.py with STENCIL_REPORT_DIR set: G1 / G2 errors, oracle threads, seconds and
GLUP/s).  This tool never runs the oracle itself (only tests/ and bench.py's baseline legs may).

python tools/report.py [--workloads C1,C2,C3,C4,C5,C3A] [--reps 3] [--parity gpurun_out/parity.json] \
    > profiles/r02_report.csv
"""
import argparse
import csv
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402
from bench import (ClockSampler, FLOPS_PER_LUP, block_bytes_per_cell, cpu_model, load_fp64_peak,  # noqa: E402
                   load_peaks, load_traffic)
from synth import workloads  # noqa: E402

VARIANTS = {1: "naive", 2: "stream", 3: "pipe", 4: "coop"}
COLUMNS = ["kind", "workload", "nx", "ny", "nz", "T", "seed", "bt", "tile", "P", "variant", "seconds",
           "glups", "roof1_glups", "roof_bt_glups", "pct_roof_bt", "pct_roof1", "ncu_dram_bytes_per_lup",
           "compulsory_bytes_per_lup", "hbm_gbs", "pct_hbm", "bound", "fp64_util_pct", "sm_mhz", "clock_reasons",
           "power_w", "nj_per_lup", "g1_err", "g2_err", "parity_cells", "oracle_threads", "oracle_s",
           "oracle_glups", "cpu_model"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C1,C2,C3,C4,C5,C3A")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--parity", default=os.path.join(ROOT, "profiles", "r02_parity.json"))
    ap.add_argument("--fp64-util", default=os.path.join(ROOT, "profiles", "r02_fp64_util.json"),
                    help="ncu sm__pipe_fp64_cycles_active per workload (optional)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    hbm, _ = load_peaks()
    fp64, _ = load_fp64_peak()
    parity = json.load(open(a.parity)) if os.path.exists(a.parity) else {}
    util = json.load(open(a.fp64_util)) if os.path.exists(a.fp64_util) else {}
    by = {x.name.split("-")[0]: x for x in workloads.CONFIGS + workloads.EXTRA}
    out = csv.writer(sys.stdout)
    out.writerow(COLUMNS)
    for name in a.workloads.split(","):
        w = by[name]
        g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED)
        s = g.stream
        g.run(w.T)
        g.sync()
        ts = []
        with ClockSampler(torch.cuda.current_device()) as clk:
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                g.run(w.T)
                e1.record(s)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
        info = g.info()
        g.close()
        torch.cuda.empty_cache()
        ms = statistics.median(ts)
        glups = w.luops / ms / 1e6
        bt = info["bt"]
        bpc = block_bytes_per_cell(w.kind, bt)
        roof_hbm = hbm / (bpc / bt)
        roof_fp = fp64 * 1e3 / FLOPS_PER_LUP[w.kind]
        roof = min(roof_hbm, roof_fp)
        roof1 = min(hbm / block_bytes_per_cell(w.kind, 1), roof_fp)
        hbm_gbs = glups * bpc / bt  # algorithmic bytes moved per second
        tr = load_traffic(w.name, bt)
        c = clk.summary()
        pr = parity.get(w.name, {})
        out.writerow([synth.KIND_NAMES[w.kind], w.name, w.nx, w.ny, w.nz, w.T, synth.DEFAULT_SEED, bt,
                      f"{info['tile_x']}x{info['tile_y']}", 1, VARIANTS.get(info["variant"]), round(ms / 1e3, 5),
                      round(glups, 2), round(roof1, 1), round(roof, 1), round(100 * glups / roof, 1),
                      round(100 * glups / roof1, 1),
                      round(tr / (w.nx * w.ny * w.nz * bt), 2) if tr else None, round(bpc / bt, 2),
                      round(hbm_gbs, 1), round(100 * hbm_gbs / hbm, 1), "hbm" if roof_hbm <= roof_fp else "fp64",
                      util.get(w.name), c.get("sm_mhz"), "|".join(c.get("reasons") or []), c.get("power_w"),
                      round(c["power_w"] / glups, 3) if c.get("power_w") else None,
                      pr.get("g1_err"), pr.get("g2_err"), pr.get("g1_cells"), pr.get("oracle_threads"),
                      pr.get("oracle_s"), pr.get("oracle_glups"), cpu_model()])
        sys.stdout.flush()


if __name__ == "__main__":
    main()
