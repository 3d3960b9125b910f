"""Plan sweep on one GPU: GLUP/s of stencil_run(T) for each (workload, variant, bt, zchunk).

python tools/sweep.py [--workloads C2,C3] [--bts 1,2,3,4] [--zchunks 0,64,128] [--T 20]
Prints one JSON object per plan (CUDA-event timed, 1 warm-up + `--reps` timed runs, median).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
from bench import ClockSampler  # noqa: E402
import synth  # noqa: E402
from synth import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C1,C2,C3,C4")
    ap.add_argument("--bts", default="1,2,3,4,5,6")
    ap.add_argument("--zchunks", default="0")
    ap.add_argument("--variants", default="2")
    ap.add_argument("--cfgs", default="0")
    ap.add_argument("--T", type=int, default=0, help="override T (0 = the workload's)")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    for name in a.workloads.split(","):
        w = {x.name.split("-")[0]: x for x in workloads.CONFIGS + workloads.EXTRA}[name]
        T = a.T or w.T
        for variant in [int(v) for v in a.variants.split(",")]:
            for bt, zc, cfg in [(int(b), int(z), int(c)) for b in a.bts.split(",")
                                for z in a.zchunks.split(",") for c in a.cfgs.split(",")]:
                if True:
                    try:
                        g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, variant=variant,
                                    bt=bt, zchunk=zc, tile_cfg=cfg)
                    except st.StencilError as e:
                        print(json.dumps({"workload": name, "bt": bt, "error": str(e)}))
                        continue
                    info = g.info()
                    if bt and info["bt"] != bt and variant != 1:
                        g.close()
                        continue
                    g.run(T)
                    g.sync()
                    ts = []
                    clk = ClockSampler(torch.cuda.current_device())
                    clk.__enter__()
                    for _ in range(a.reps):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        g.run(T)
                        e1.record(s)
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    clk.__exit__()
                    ms = statistics.median(ts)
                    cs = clk.summary()
                    info = g.info()
                    g.close()
                    lups = w.nx * w.ny * w.nz * T
                    print(json.dumps({"workload": name, "variant": variant, "bt": info["bt"], "cfg": cfg,
                                      "zchunk": info["zchunk"], "tile": [info["tile_x"], info["tile_y"]],
                                      "ms": round(ms, 3), "glups": round(lups / ms / 1e6, 2),
                                      "sm_mhz": cs.get("sm_mhz"), "power_w": cs.get("power_w"),
                                      "reasons": cs.get("reasons")}), flush=True)
                    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
