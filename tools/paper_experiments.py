"""The paper's measurement methodology on B200:

  * grid-size sweep (§6.2, Fig. 10): cubic grids in multiples of 64, every kind,
    the library's default plan -> GLUP/s and fraction of the HBM roofline of the plan's bt;
  * in-cache ceiling (§3.4): a grid whose arrays all fit in the 126 MB L2
    (64^3 .. 128^3), run long enough to amortise launches -> the ceiling once decoupled from HBM.

python tools/paper_experiments.py [--sizes 64,128,...] [--kinds 1,2,3,4,5] > table.md
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402

HBM = 6546.9


def bytes_per_cell(kind, b):
    if kind in synth.WAVE_KINDS:
        return (24 if b == 1 else 32) + 8 * synth.N_COEF_FIELDS[kind]
    return 16 + 8 * synth.N_COEF_FIELDS[kind]


def measure(kind, n, T, reps=3, **kw):
    s = torch.cuda.current_stream()
    with st.Grid(kind, n, n, n, seed=synth.DEFAULT_SEED, **kw) as g:
        g.run(T)
        g.sync()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.run(T)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        info = g.info()
    ms = statistics.median(ts)
    glups = n ** 3 * T / ms / 1e6
    return glups, info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,192,256,320,384,448,512,640")
    ap.add_argument("--kinds", default="1,2,3,4,5")
    ap.add_argument("--json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rows = []
    print("| kind | n^3 | T | bt | GLUP/s | roof(bt) GLUP/s | frac | fits L2 |")
    print("|---|---|---|---|---|---|---|---|")
    for kind in [int(k) for k in a.kinds.split(",")]:
        for n in [int(x) for x in a.sizes.split(",")]:
            R = synth.RADIUS[kind]
            arrays = 2 + synth.N_COEF_FIELDS[kind]
            bytes_ = arrays * (n + 2 * R) ** 3 * 8
            if bytes_ > 150e9:
                continue
            # long enough that launches amortise (>= ~50 ms of work at ~100 GLUP/s), at least 20 steps
            T = max(20, min(2000, int(5e9 / n ** 3)))
            glups, info = measure(kind, n, T)
            bt = info["bt"]
            roof = HBM / (bytes_per_cell(kind, bt) / bt)
            fits = bytes_ < 100e6
            rows.append({"kind": kind, "n": n, "T": T, "bt": bt, "glups": glups, "roof": roof, "fits_l2": fits})
            print(f"| {synth.KIND_NAMES[kind]} | {n} | {T} | {bt} | {glups:.1f} | {roof:.1f} | {glups / roof:.2f} | "
                  f"{'yes' if fits else 'no'} |", flush=True)
            torch.cuda.empty_cache()
    if a.json:
        json.dump(rows, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
