"""Tiny cases for compute-sanitizer: every pipe/stream/naive kernel variant on small grids."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402

torch.cuda.set_device(0)
cases = [(synth.K7C, (40, 33, 21), [(3, b, 0) for b in (1, 2, 4)]),
         (synth.K7V, (40, 33, 21), [(3, 1, 0), (3, 1, 1), (3, 2, 0), (3, 2, 1), (3, 3, 0), (3, 3, 1), (2, 2, 0), (1, 1, 0)]),
         (synth.K25W, (70, 20, 19), [(3, 1, c) for c in range(4)] + [(2, 1, 0)]),
         (synth.K25V, (70, 20, 19), [(3, 1, c) for c in range(3)] + [(2, 1, 0)])]
for kind, n, plans in cases:
    for variant, bt, cfg in plans:
        with st.Grid(kind, *n, seed=3, variant=variant, bt=bt, tile_cfg=cfg) as g:
            g.run(2 * bt + 1)
            g.read(0)
    with st.Grid(kind, *n, seed=3, nranks=3, local_slabs=3) as g:
        g.run(5)
        g.read(0)
print("san_case done")
