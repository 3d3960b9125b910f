"""One CSV row per BASELINE.json config: the library's default plan timed on
this GPU (median of --reps stencil_run(T) calls, CUDA events on the grid's stream, SM clock sampled
through NVML meanwhile) against the roofline of its plan -- min(HBM copy peak / (bytes per cell per
block / bt), FP64 peak / flops per LUP) -- and at bt = 1.  Parity of the same plans is in
tests/test_gpu_fullsize.py.

python tools/report.py [--workloads C1,C2,C3,C4,C5,C3A] [--reps 3] > profiles/rNN_report.csv
"""
import argparse
import csv
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402
from bench import ClockSampler, FLOPS_PER_LUP, block_bytes_per_cell, load_fp64_peak, load_peaks  # noqa: E402
from synth import workloads  # noqa: E402

VARIANTS = {1: "naive", 2: "stream", 3: "pipe", 4: "coop"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C1,C2,C3,C4,C5,C3A")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    hbm, _ = load_peaks()
    fp64, _ = load_fp64_peak()
    by = {x.name.split("-")[0]: x for x in workloads.CONFIGS + workloads.EXTRA}
    out = csv.writer(sys.stdout)
    out.writerow(["workload", "kind", "nx", "ny", "nz", "T", "variant", "bt", "tile", "ms_median", "glups",
                  "roof_bt_glups", "frac_roof_bt", "roof_bt1_glups", "frac_roof_bt1", "roof_fp64_glups",
                  "bound", "sm_mhz", "clock_reasons", "power_w", "nj_per_lup"])
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
        glups = w.nx * w.ny * w.nz * w.T / ms / 1e6
        bt = info["bt"]
        roof_hbm = hbm / (block_bytes_per_cell(w.kind, bt) / bt)
        roof_fp = fp64 * 1e3 / FLOPS_PER_LUP[w.kind]
        roof = min(roof_hbm, roof_fp)
        roof1 = min(hbm / block_bytes_per_cell(w.kind, 1), roof_fp)
        c = clk.summary()
        out.writerow([w.name, synth.KIND_NAMES[w.kind], w.nx, w.ny, w.nz, w.T, VARIANTS.get(info["variant"]), bt,
                      f"{info['tile_x']}x{info['tile_y']}", round(ms, 3), round(glups, 2), round(roof, 1),
                      round(glups / roof, 3), round(roof1, 1), round(glups / roof1, 3), round(roof_fp, 1),
                      "hbm" if roof_hbm <= roof_fp else "fp64", c.get("sm_mhz"), "|".join(c.get("reasons") or []),
                      c.get("power_w"), round(c["power_w"] / glups, 3) if c.get("power_w") else None])
        sys.stdout.flush()


if __name__ == "__main__":
    main()
