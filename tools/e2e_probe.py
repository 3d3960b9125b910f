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

# two-deep pipeline (as bench.py's e2e): worker thread creates step k+1 on its own stream
from concurrent.futures import ThreadPoolExecutor  # noqa: E402

streams = [torch.cuda.Stream(), torch.cuda.Stream()]
outs = [out, pin(np.empty_like(out))]
T0 = time.perf_counter()
log = []


def create(k):
    torch.cuda.set_device(0)
    a = time.perf_counter() - T0
    g = st.Grid(w.kind, w.nx, w.ny, w.nz, v0=V, u0=U, coeff=coeff, stream=streams[k % 2])
    log.append((k, "create", a, time.perf_counter() - T0))
    return g


for rnd in range(2):
    T0 = time.perf_counter()
    log.clear()
    K = 6
    with ThreadPoolExecutor(1) as ex:
        fut = ex.submit(create, 0)
        for k in range(K):
            g = fut.result()
            if k + 1 < K:
                fut = ex.submit(create, k + 1)
            a = time.perf_counter() - T0
            g.run(w.T)
            g.sync()
            b = time.perf_counter() - T0
            g.read(0, out=outs[k % 2])
            c = time.perf_counter() - T0
            g.close()
            log.append((k, "run", a, b))
            log.append((k, "read", b, c))
    tot = time.perf_counter() - T0
    print(f"pipelined round {rnd}: {K} steps {tot * 1e3:.0f} ms -> {w.nx * w.ny * w.nz * w.T * K / tot / 1e9:.1f} GLUP/s")
    for e in sorted(log, key=lambda e: e[2]):
        print(f"  step {e[0]} {e[1]:6s} {e[2] * 1e3:8.1f} -> {e[3] * 1e3:8.1f} ms ({(e[3] - e[2]) * 1e3:.1f})")
