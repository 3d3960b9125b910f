"""Mutation tests: inject a fault into the CUDA path and check that the parity
and invariance checks used elsewhere in the suite catch it.  Faults (STENCIL_FAULT bits, test-only):
1 = multi-slab halo exchanged (or, fused, stored into the neighbour) one plane too shallow, 4 = the last plane of every z-chunk never written
(stale plane), 8 = work item 0 skipped (stale tile)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_common import gpu_run, rel_err

pytestmark = pytest.mark.gpu


def _parity_err(kind, n, T, **kw):
    inp = synth.make_inputs(kind, *n, seed=17)
    o_new, _ = oracle.run(inp, T)
    g_new, _, _ = gpu_run(kind, *n, T, seed=17, **kw)
    return rel_err(g_new, o_new, inp.R)


@pytest.mark.parametrize("kind", [synth.K7V, synth.K25V])
@pytest.mark.parametrize("fault,extra", [(4, {}), (8, {}), (1, {"nranks": 3, "local_slabs": 3}),
                                         (1, {"nranks": 3, "local_slabs": 3, "halo": 1})])
def test_injected_fault_is_detected(monkeypatch, kind, fault, extra):
    n = (40, 33, 37) if synth.RADIUS[kind] == 1 else (70, 20, 41)
    T = 12  # several full blocks at the default bt (4 for 7v, 2 for 25v here): the second reads the
    # deepest halo plane
    if "nranks" in extra:
        from paper_1410_3060_b200 import Grid
        import paper_1410_3060_b200 as st

        def run(**kw):
            with st.Grid(kind, *n, seed=17, **kw) as g:
                g.run(T)
                return g.read(0)
        ok = run(**extra)
        monkeypatch.setenv("STENCIL_FAULT", str(fault))
        bad = run(**extra)
        assert not np.array_equal(ok, bad), "fault not visible"
        return
    pipe = {"zchunk": 8, "variant": 3}  # the faults are injected into the pipe kernel
    assert _parity_err(kind, n, T, **pipe) <= 1e-13
    monkeypatch.setenv("STENCIL_FAULT", str(fault))
    assert _parity_err(kind, n, T, **pipe) > 1e-6
