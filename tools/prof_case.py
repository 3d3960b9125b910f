"""Small fixed case for ncu: create one workload grid, run T steps, exit.

python tools/prof_case.py --workload C2 [--bt 2] [--T 4] [--variant 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402
from synth import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
ap.add_argument("--bt", type=int, default=0)
ap.add_argument("--T", type=int, default=0)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--zchunk", type=int, default=0)
ap.add_argument("--cfg", type=int, default=0)
a = ap.parse_args()
torch.cuda.set_device(0)
w = {x.name.split("-")[0]: x for x in workloads.CONFIGS + workloads.EXTRA}[a.workload]
g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, variant=a.variant, bt=a.bt, zchunk=a.zchunk,
            tile_cfg=a.cfg)
bt = g.info()["bt"]
g.run(a.T or 2 * bt)
g.sync()
print("info", g.info())
g.close()
