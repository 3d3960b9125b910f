"""Auto-tuner for the pipe kernel's plan (the paper's D_w / N_F search, P:808-822,
brute force after model pruning): for a workload, enumerate (bt, tile_cfg, zchunk) candidates that the
shared-memory/register footprint admits (the library rejects the rest), time short runs, and write the
best plan per workload to paper_1410_3060_b200/tuned.json, which `Grid(..., tuned=True)` applies.

python tools/tune.py --workloads C2,C3,C4 [--T 20]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402
from synth import workloads  # noqa: E402

TUNED = os.path.join(ROOT, "paper_1410_3060_b200", "tuned.json")
MAX_BT = {1: 8, 2: 4, 3: 2, 4: 1, 5: 1}
N_CFG = {1: 1, 2: 10, 3: 9, 4: 4, 5: 5}  # pipe tile configurations per kind (pipe.cu launch_pipe)


def time_plan(w, T, bt, cfg, zchunk, reps=3, variant=st.ST_VARIANT_PIPE, warm_s=0.0):
    s = torch.cuda.current_stream()
    g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, bt=bt, tile_cfg=cfg, zchunk=zchunk,
                variant=variant)
    try:
        g.run(T)
        g.sync()
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < warm_s:  # sustained mode: run into the board's power cap first
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
        return w.nx * w.ny * w.nz * T / statistics.median(ts) / 1e6
    finally:
        g.close()
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C1,C2,C3,C4")
    ap.add_argument("--T", type=int, default=0, help="steps per timed run (0: min(workload T, 24))")
    ap.add_argument("--sustained", type=float, default=0.0,
                    help="seconds of warm-up per plan before timing, at the workload's full T (the rate under "
                         "the 1 kW power cap, which short runs do not reach); 0 = short isolated runs")
    ap.add_argument("--bts", default="", help="restrict b_t candidates (comma list)")
    ap.add_argument("--cfgs", default="", help="restrict tile_cfg candidates")
    ap.add_argument("--zchunks", default="0,64,256")
    ap.add_argument("--out", default=TUNED)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    table = json.load(open(a.out)) if os.path.exists(a.out) else (json.load(open(TUNED)) if os.path.exists(TUNED) else {})
    names = {x.name.split("-")[0]: x for x in workloads.CONFIGS + workloads.EXTRA}
    for name in a.workloads.split(","):
        w = names[name]
        T = a.T or (w.T if a.sustained else min(w.T, 24))
        best = None
        # the cooperative all-steps kernel (one launch per stencil_run) as a candidate of its own
        g = time_plan(w, T, 0, 0, 0, variant=st.ST_VARIANT_COOP, warm_s=a.sustained)
        print(json.dumps({"workload": name, "variant": "coop", "glups": round(g, 2)}), flush=True)
        best = {"variant": st.ST_VARIANT_COOP, "bt": 1, "tile_cfg": 0, "zchunk": 0, "glups": round(g, 2), "T": T}
        bts = [int(x) for x in a.bts.split(",")] if a.bts else range(1, MAX_BT[w.kind] + 1)
        for bt in bts:
            cfgs = [int(x) for x in a.cfgs.split(",")] if a.cfgs else range(N_CFG[w.kind])
            for cfg in cfgs:
                for zc in [int(x) for x in a.zchunks.split(",")]:
                    try:
                        g = time_plan(w, T, bt, cfg, zc, warm_s=a.sustained)
                    except st.StencilError as e:
                        print(json.dumps({"workload": name, "bt": bt, "cfg": cfg, "error": str(e)[:80]}))
                        continue
                    print(json.dumps({"workload": name, "bt": bt, "cfg": cfg, "zchunk": zc, "glups": round(g, 2)}),
                          flush=True)
                    if best is None or g > best["glups"]:
                        best = {"variant": st.ST_VARIANT_PIPE, "bt": bt, "tile_cfg": cfg, "zchunk": zc,
                                "glups": round(g, 2), "T": T, "sustained_s": a.sustained}
        best["workload"] = w.name
        table[f"{w.kind}:{w.nx}x{w.ny}x{w.nz}"] = best
        print(json.dumps({"workload": name, "best": best}), flush=True)
    json.dump(table, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
