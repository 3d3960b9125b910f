"""Repeatability stress: the default plans (and a small-z-chunk plan with many work items per CTA, i.e.
many item boundaries) re-run N times must give bitwise identical results (races would show up as
run-to-run differences)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402

torch.cuda.set_device(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cases = [(synth.K7V, (256, 200, 160), 12, dict(variant=3)), (synth.K7V, (256, 200, 160), 12, dict(variant=3, zchunk=5)),
         (synth.K7V, (256, 200, 160), 12, dict(variant=3, bt=4, zchunk=7)),
         (synth.K7V, (256, 200, 160), 12, dict(variant=3, bt=3, tile_cfg=9, zchunk=7)),  # cluster pairs
         (synth.K25W, (256, 120, 100), 6, dict(variant=3, zchunk=9)), (synth.K25V, (192, 100, 90), 5, dict(variant=3, zchunk=9)),
         (synth.K7C, (200, 200, 200), 17, dict(variant=3, zchunk=6))]
bad = 0
for kind, n, T, kw in cases:
    ref = None
    for r in range(N):
        with st.Grid(kind, *n, seed=8, **kw) as g:
            g.run(T)
            out = g.read(0)
        if ref is None:
            ref = out
        elif not np.array_equal(out, ref):
            bad += 1
            print("MISMATCH", kind, n, kw, "rep", r, flush=True)
    print("ok" if bad == 0 else "bad", synth.KIND_NAMES[kind], n, kw, flush=True)
print("stress done, mismatches:", bad)
sys.exit(1 if bad else 0)
