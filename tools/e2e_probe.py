"""Time breakdown of one end-to-end step (create from pinned host arrays, run T, read, close)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402
from synth import workloads  # noqa: E402

w = workloads.BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "C2-7pt-var-512"]
torch.cuda.set_device(0)
t0 = time.perf_counter()
inp = synth.make_inputs(w.kind, w.nx, w.ny, w.nz)
print(f"make_inputs {time.perf_counter() - t0:.2f} s")
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
V = pin(inp.V)
U = pin(inp.U) if w.kind in synth.WAVE_KINDS else None
coeff = list(inp.scalars) + [pin(c) for c in inp.coef]
out = pin(np.empty_like(inp.V))
for rep in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    g = st.Grid(w.kind, w.nx, w.ny, w.nz, v0=V, u0=U, coeff=coeff)
    t.append(time.perf_counter())
    g.run(w.T)
    g.sync()
    t.append(time.perf_counter())
    g.read(0, out=out)
    t.append(time.perf_counter())
    g.close()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: create {d[0]:.1f} ms, run {d[1]:.1f} ms, read {d[2]:.1f} ms, close {d[3]:.1f} ms, "
          f"total {sum(d):.1f} ms -> {w.nx * w.ny * w.nz * w.T / sum(d) / 1e6:.1f} GLUP/s")
