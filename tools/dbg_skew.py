"""Where do the skewed 25v tiles (tile_cfg 3) differ from the naive sweeps?  Prints mismatch statistics.
python tools/dbg_skew.py [nx ny nz T zchunk]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402

a = [int(x) for x in sys.argv[1:]] + [0] * 5
nx, ny, nz, T, zc = (a[0] or 130), (a[1] or 37), (a[2] or 41), (a[3] or 2), a[4]
K = synth.K25V
R = 4


def run(**kw):
    with st.Grid(K, nx, ny, nz, seed=21, tuned=False, **kw) as g:
        g.run(T)
        return g.read(0)


ref = run(variant=st.ST_VARIANT_NAIVE)
got = run(variant=st.ST_VARIANT_PIPE, bt=2, tile_cfg=3, zchunk=zc)
d = got != ref
print("shape", (nx, ny, nz), "T", T, "mismatches", int(d.sum()), "of", d.size)
if d.any():
    z, y, x = np.nonzero(d)
    print("z range", z.min(), z.max(), "y range", y.min(), y.max(), "x range", x.min(), x.max())
    print("y histogram", np.bincount(y, minlength=ny + 2 * R).tolist())
    print("(y - R) % 20 histogram", np.bincount((y - R) % 20, minlength=20).tolist())
    print("z histogram", np.bincount(z, minlength=nz + 2 * R).tolist())
    print("x histogram", np.bincount(x, minlength=nx + 2 * R).tolist()[:64])
    i = 0
    print("first", z[i], y[i], x[i], got[z[i], y[i], x[i]], ref[z[i], y[i], x[i]])
    print("max abs diff", float(np.abs(got - ref)[d].max()))
