import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1410_3060_b200 as st, synth
torch.cuda.set_device(0)
for n, T, bt, cfg in [((61, 70, 45), 7, 3, 9), ((61, 70, 45), 9, 4, 3), ((40, 33, 21), 5, 3, 9), ((256, 200, 100), 12, 3, 9)]:
    ref = None
    with st.Grid(synth.K7V, *n, seed=9, variant=1) as g:
        g.run(T); ref = g.read(0)
    with st.Grid(synth.K7V, *n, seed=9, variant=3, bt=bt, tile_cfg=cfg) as g:
        g.run(T); out = g.read(0); info = g.info()
    print(n, T, bt, cfg, info["tile_x"], info["tile_y"], "equal" if np.array_equal(out, ref) else "DIFF max %g" % np.max(np.abs(out - ref)), flush=True)
