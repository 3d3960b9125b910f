"""CPU-only checks of the C ABI boundary: the library loads, exports every symbol include/stencil.h
declares, the host-side slab plan is right, and without a GPU creation fails loudly (no fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1410_3060_b200 as st

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "stencil.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(stencil_[a-z_0-9]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(st.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = st.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", st.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (stencil_\w+)", out))
    assert set(header_functions()) <= exported
    assert "sm_100a" in st.stencil_version()


def test_library_contains_sm100a_code_and_no_oracle():
    out = subprocess.run(["cuobjdump", "--list-elf", st.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    syms = subprocess.run(["nm", "-D", st.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in syms


@pytest.mark.parametrize("nz,R,P", [(512, 1, 2), (1024, 4, 8), (1024, 4, 3), (7, 1, 7), (12, 4, 3), (1, 1, 1)])
@pytest.mark.parametrize("bt", [1, 2, 4])
def test_plan_slab_partition(nz, R, P, bt):
    plans = [st.stencil_plan_slab(nz, R, P, r, bt) for r in range(P)]
    # owned planes tile the padded grid exactly
    assert plans[0]["own_z0"] == 0 and plans[-1]["own_z1"] == nz + 2 * R
    for a, b in zip(plans, plans[1:]):
        assert a["own_z1"] == b["own_z0"]
    sizes = [p["own_z1"] - p["own_z0"] for p in plans]
    inner = [s for s in sizes]
    inner[0] -= R
    inner[-1] -= R
    assert sum(inner) == nz and max(inner) - min(inner) <= 1
    assert inner == sorted(inner, reverse=True)  # remainder to the lowest ranks
    b = plans[0]["bt"]
    assert all(p["bt"] == b for p in plans)
    if P > 1:
        assert R * b <= min(inner) and b <= max(1, bt)
    for r, p in enumerate(plans):
        lo_h = p["own_z0"] - p["store_z0"] if r > 0 else 0
        hi_h = p["store_z1"] - p["own_z1"] if r < P - 1 else 0
        if r > 0:
            assert lo_h == R * b
        if r < P - 1:
            assert hi_h == R * b
        assert p["store_z0"] >= 0 and p["store_z1"] <= nz + 2 * R


def test_plan_slab_rejects():
    with pytest.raises(st.StencilError):
        st.stencil_plan_slab(3, 1, 4, 0, 1)  # nz < nranks
    with pytest.raises(st.StencilError):
        st.stencil_plan_slab(8, 1, 2, 2, 1)  # rank out of range
    with pytest.raises(st.StencilError):
        st.stencil_plan_slab(10, 4, 3, 0, 1)  # slabs of 3 planes < R = 4


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(st.StencilError) as ei:
        st.stencil_create_seeded(st.ST_7PT_CONST, 4, 4, 4, 1)
    assert ei.value.code == st.ST_E_CUDA
    assert "no CPU fallback" in st.stencil_last_error()


def test_argument_validation_before_device():
    for args in [(9, 4, 4, 4, 1), (st.ST_7PT_CONST, 0, 4, 4, 1), (st.ST_7PT_CONST, 4, -1, 4, 1)]:
        with pytest.raises(st.StencilError) as ei:
            st.stencil_create_seeded(*args)
        assert ei.value.code == st.ST_E_INVAL
    with pytest.raises(st.StencilError) as ei:
        st.stencil_create_seeded(st.ST_7PT_VAR, 4, 4, 4, 1, scalars=[1.0])
    assert ei.value.code == st.ST_E_INVAL
    with pytest.raises(st.StencilError):
        st.stencil_run(None, 1)
    assert st.lib().stencil_destroy(None) == 0


@pytest.mark.parametrize("kind", [1, 2, 3, 4, 5])
def test_stencil_generate_equals_synth(kind):
    """The library's host generator (the device fill's bits, no device needed) equals synth's inputs."""
    import synth
    n = (7, 5, 6)
    inp = synth.make_inputs(kind, *n, seed=77)
    assert np.array_equal(st.stencil_generate(kind, *n, 77, 0), inp.V)
    if kind in synth.WAVE_KINDS:
        assert np.array_equal(st.stencil_generate(kind, *n, 77, 1), inp.U)
    for i, c in enumerate(inp.coef):
        assert np.array_equal(st.stencil_generate(kind, *n, 77, 2 + i), c)
    with pytest.raises(st.StencilError):
        st.stencil_generate(kind, *n, 77, 2 + len(inp.coef))
    if kind not in synth.WAVE_KINDS:
        with pytest.raises(st.StencilError):
            st.stencil_generate(kind, *n, 77, 1)


def test_host_slab_binding_checks():
    """st_opts.host_slab (a rank's host arrays hold only its stored planes): the binding sizes the arrays
    with stencil_plan_slab and refuses a missing bt, a single rank, and arrays of the wrong size -- all
    before any device work (the library repeats the bt / rank rule for C callers)."""
    import synth
    kind, n = synth.K7V, (8, 8, 12)
    o = st.stencil_opts_default()
    o.nranks, o.rank, o.host_slab = 2, 1, 1
    pl = st.stencil_plan_slab(n[2], 1, 2, 1, 2)
    box = ((pl["store_z0"], pl["store_z1"]), (0, 10), (0, 10))
    loc = synth.make_inputs(kind, *n, seed=1, box=box)
    full = synth.make_inputs(kind, *n, seed=1)
    with pytest.raises(ValueError):  # bt = 0: the stored range is not known in advance
        st.stencil_create(kind, *n, list(loc.coef), loc.V, None, o)
    o.bt = 2
    with pytest.raises(ValueError):  # the global arrays are not this rank's planes
        st.stencil_create(kind, *n, list(full.coef), full.V, None, o)
    o.nranks = 1
    with pytest.raises(ValueError):
        st.stencil_create(kind, *n, list(loc.coef), loc.V, None, o)
