"""Auto-tuner for the library's plan (the paper's D_w / N_F search, with the
footprint model pruning the search the way the paper's Eq. 4.1/4.2 bounds its cache blocks):
for a workload, take every (bt, tile_cfg) plan the kernels instantiate (model.pipe_plans /
model.pipe25_plans, parsed from the sources), drop those whose on-chip footprint does not fit
(model.pipe_footprint / pipe25_footprint), rank the rest by the modeled energy per lattice update
(model.modeled_nj_per_lup -- the 1 kW board cap makes energy per update the rate limit), time the best
--top of them (plus the library's default plan and, for small grids, the cooperative kernel) under the
power cap, and write the fastest plan per workload to paper_1410_3060_b200/tuned.json, which
`Grid(...)` applies by default to a grid of exactly that kind and shape.

python tools/tune.py --workloads C2,C3,C4,C5 [--top 5] [--sustained 1.0]
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
from paper_1410_3060_b200 import model  # noqa: E402
from synth import workloads  # noqa: E402

TUNED = os.path.join(ROOT, "paper_1410_3060_b200", "tuned.json")


def candidates(kind):
    """[(modeled nJ/LUP, bt, tile_cfg, footprint)] of every fitting plan of the kind, cheapest first."""
    out = []
    for k, bt, cfg, a in model.pipe_plans():
        if k != kind or (kind == model.K25V and bt == 2):
            continue
        f = model.pipe_footprint(kind, bt, **a)
        if f["fits"]:
            out.append((model.modeled_nj_per_lup(kind, bt, f), bt, cfg, f))
    if kind == model.K25V:
        for cfg, TX, TY, D, CLU, SKEW in model.pipe25_plans():
            f = model.pipe25_footprint(TX, TY, D, CLU, SKEW)
            if f["fits"]:
                out.append((model.modeled_nj_per_lup(kind, 2, f), 2, cfg, f))
    return sorted(out, key=lambda c: c[0])


def time_plan(w, T, bt, cfg, zchunk, reps=3, variant=st.ST_VARIANT_PIPE, warm_s=0.0):
    s = torch.cuda.current_stream()
    g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, bt=bt, tile_cfg=cfg, zchunk=zchunk,
                variant=variant, tuned=False)
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
        return w.nx * w.ny * w.nz * T / statistics.median(ts) / 1e6, g.info()["bt"]
    finally:
        g.close()
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C1,C2,C3,C4,C5")
    ap.add_argument("--T", type=int, default=0, help="steps per timed run (0: the workload's T)")
    ap.add_argument("--top", type=int, default=5, help="plans timed per workload, by modeled energy")
    ap.add_argument("--sustained", type=float, default=1.0,
                    help="seconds of warm-up per plan before timing, at the workload's full T (the rate under "
                         "the 1 kW power cap, which short runs do not reach); 0 = short isolated runs")
    ap.add_argument("--zchunks", default="0")
    ap.add_argument("--out", default=TUNED)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    table = json.load(open(a.out)) if os.path.exists(a.out) else {}
    names = {x.name.split("-")[0]: x for x in workloads.CONFIGS + workloads.EXTRA}
    for name in a.workloads.split(","):
        w = names[name]
        T = a.T or w.T
        results = []
        cells = (w.nx + 2) * (w.ny + 2) * (w.nz + 2)
        if cells <= 3e6:  # small grids: the cooperative all-steps kernel is a candidate of its own
            g, _ = time_plan(w, T, 0, 0, 0, variant=st.ST_VARIANT_COOP, warm_s=a.sustained)
            results.append({"variant": st.ST_VARIANT_COOP, "bt": 1, "tile_cfg": 0, "zchunk": 0, "glups": round(g, 2)})
            print(json.dumps({"workload": name, **results[-1]}), flush=True)
        cand = candidates(w.kind)
        pick = cand[:a.top]
        # the library's own default plan is always timed
        g, bt0 = time_plan(w, T, 0, 0, 0, variant=st.ST_VARIANT_PIPE, warm_s=a.sustained)
        results.append({"variant": st.ST_VARIANT_PIPE, "bt": bt0, "tile_cfg": 0, "zchunk": 0, "glups": round(g, 2),
                        "note": "library default"})
        print(json.dumps({"workload": name, **results[-1]}), flush=True)
        for nj, bt, cfg, f in pick:
            for zc in [int(x) for x in a.zchunks.split(",")]:
                try:
                    g, _ = time_plan(w, T, bt, cfg, zc, warm_s=a.sustained)
                except st.StencilError as e:
                    print(json.dumps({"workload": name, "bt": bt, "cfg": cfg, "error": str(e)[:80]}))
                    continue
                results.append({"variant": st.ST_VARIANT_PIPE, "bt": bt, "tile_cfg": cfg, "zchunk": zc,
                                "glups": round(g, 2), "modeled_nj_per_lup": round(nj, 2)})
                print(json.dumps({"workload": name, **results[-1]}), flush=True)
        best = max(results, key=lambda r: r["glups"])
        best = {k: v for k, v in best.items() if k != "note"}
        best.update({"T": T, "sustained_s": a.sustained, "workload": w.name,
                     "pruned": f"{len(pick)} of {len(cand)} fitting plans timed (modeled nJ/LUP ranking)"})
        table[f"{w.kind}:{w.nx}x{w.ny}x{w.nz}"] = best
        print(json.dumps({"workload": name, "best": best}), flush=True)
    json.dump(table, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
