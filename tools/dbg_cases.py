"""Run each (kind, shape, variant, bt, cfg, T) case in its own subprocess; report ok / error.

python tools/dbg_cases.py            # default case list
"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json
sys.path.insert(0, %r)
import torch, numpy as np
import paper_1410_3060_b200 as st, synth
torch.cuda.set_device(0)
kind, n, variant, bt, cfg, T = json.loads(sys.argv[1])
g = st.Grid(kind, *n, seed=5, variant=variant, bt=bt, tile_cfg=cfg)
g.run(T); g.sync()
a = g.read(0)
ref = st.Grid(kind, *n, seed=5, variant=st.ST_VARIANT_NAIVE)
ref.run(T); b = ref.read(0)
print(json.dumps({"equal_naive": bool(np.array_equal(a, b)), "info": g.info()["tile_x"]}))
""" % ROOT


def run(case):
    r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(case)], capture_output=True, text=True,
                       env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"), timeout=300)
    out = (r.stdout.strip().splitlines() or [""])[-1]
    err = [l for l in r.stderr.splitlines() if "Error" in l or "error" in l][-1:] if r.returncode else []
    print(json.dumps({"case": case, "rc": r.returncode, "out": out, "err": err}), flush=True)


def main():
    cases = []
    if len(sys.argv) > 1:
        cases = [json.loads(a) for a in sys.argv[1:]]
    else:
        for bt in range(1, 9):
            cases.append([1, [64, 64, 64], 3, bt, 0, bt])
            cases.append([1, [33, 19, 14], 3, bt, 0, bt])
        cases += [[1, [33, 40, 14], 3, 3, 0, 3], [1, [33, 40, 40], 3, 3, 0, 3]]
        for bt, cfg in itertools.product([1, 2, 3], [0, 1]):
            cases.append([2, [64, 64, 64], 3, bt, cfg, bt])
        cases += [[2, [128, 128, 128], 3, 1, 0, 1], [2, [512, 512, 64], 3, 1, 0, 1]]
        cases += [[3, [130, 37, 41], 3, 1, 0, 2], [4, [130, 37, 41], 3, 1, 0, 2], [3, [64, 20, 20], 3, 1, 1, 2]]
    for c in cases:
        run(c)


if __name__ == "__main__":
    main()
