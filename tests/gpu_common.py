"""Helpers shared by the -m gpu tests: run the CUDA path through the C ABI and compare with oracle/."""
import numpy as np

import oracle
import paper_1410_3060_b200 as st
import synth

WAVE = synth.K25W
WAVES = synth.WAVE_KINDS


def interior(R):
    return (slice(R, -R),) * 3


def gpu_run(kind, nx, ny, nz, T, seed=synth.DEFAULT_SEED, variant=0, bt=0, zchunk=0, inputs=None,
            scalars=None, tile_cfg=0):
    """Run the CUDA path; returns (Omega^T, Omega^{T-1} or None, info)."""
    if inputs is None:
        g = st.Grid(kind, nx, ny, nz, seed=seed, scalars=scalars, variant=variant, bt=bt, zchunk=zchunk,
                    tile_cfg=tile_cfg)
    else:
        coeff = list(inputs.scalars) + list(inputs.coef)
        u0 = inputs.U if kind in WAVES else None
        g = st.Grid(kind, nx, ny, nz, v0=inputs.V, u0=u0, coeff=coeff, variant=variant, bt=bt,
                    zchunk=zchunk, tile_cfg=tile_cfg)
    with g:
        if T > 0:
            g.run(T)
        new = g.read(0)
        old = g.read(1) if kind in WAVES else None
        info = g.info()
    return new, old, info


def rel_err(g, o, R):
    I = interior(R)
    d = np.max(np.abs(g[I] - o[I]))
    return d / max(np.max(np.abs(o[I])), 1e-300)


def assert_parity(kind, g_new, g_old, o_new, o_old, R, tol, inputs=None):
    e = rel_err(g_new, o_new, R)
    assert e <= tol, f"normwise relative error {e:.3e} > {tol:.1e}"
    if kind in WAVES:
        e1 = rel_err(g_old, o_old, R)
        assert e1 <= tol, f"level-1 normwise relative error {e1:.3e} > {tol:.1e}"
    if inputs is not None:  # G5: ghosts bitwise untouched
        m = np.ones(g_new.shape, bool)
        m[interior(R)] = False
        assert np.array_equal(g_new[m], inputs.V[m])
        if kind in WAVES:
            assert np.array_equal(g_old[m], inputs.V[m])


def record(config, **values):
    """Append parity / oracle-timing facts of a full-size test to $STENCIL_REPORT_DIR/parity.json (read by
    tools/report.py for the SURVEY d.6 rows; nothing is recorded when the variable is unset)."""
    import json
    import os
    d = os.environ.get("STENCIL_REPORT_DIR")
    if not d:
        return
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, "parity.json")
    try:
        cur = json.load(open(path))
    except (OSError, ValueError):
        cur = {}
    cur.setdefault(config, {}).update({k: (float(v) if hasattr(v, "__float__") and not isinstance(v, (int, str))
                                           else v) for k, v in values.items()})
    json.dump(cur, open(path, "w"), indent=1, sort_keys=True)


def timed_oracle(inp, T):
    """oracle.run with its wall time and thread count (d.6 oracle_threads / oracle_s)."""
    import os
    import time
    n = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    out = oracle.run(inp, T, n)
    return out, time.perf_counter() - t0, n
