"""GPU parity (G1-G6): the CUDA path through the C ABI against oracle/ on the same seeded
inputs, element by element, at sizes spanning several tiles with ragged tails; bitwise invariance of
the GPU results across kernel variants; ghosts untouched; degenerate extents; error codes."""
import numpy as np
import pytest

import oracle
import paper_1410_3060_b200 as st
import synth
from gpu_common import WAVES, assert_parity, gpu_run, interior, rel_err

pytestmark = pytest.mark.gpu

KINDS = [synth.K7C, synth.K7V, synth.K25W, synth.K25V, synth.K25WA]
# several tiles in x and y with ragged tails, several z-chunks (7-point output tiles 32x32 .. 16x16,
# 25-point output tiles 64 x 8 / 32 x 16 / 64 x 16; streaming variant 30 x 30 .. 22 x 22, 56 x 8)
SHAPES = {synth.K7C: (61, 70, 45), synth.K7V: (61, 70, 45), synth.K25W: (130, 37, 41),
          synth.K25V: (130, 37, 41), synth.K25WA: (130, 37, 41)}


def max_bt(kind, variant=st.ST_VARIANT_PIPE):
    if variant == st.ST_VARIANT_STREAM:
        return {synth.K7C: 6, synth.K7V: 4, synth.K25W: 1, synth.K25V: 1, synth.K25WA: 1}[kind]
    return {synth.K7C: 8, synth.K7V: 5, synth.K25W: 2, synth.K25V: 2, synth.K25WA: 1}[kind]


N_CFG = {synth.K7C: 1, synth.K7V: 10, synth.K25W: 9, synth.K25V: 4, synth.K25WA: 5}  # pipe tile configurations


@pytest.mark.parametrize("kind", KINDS)
def test_seeded_fill_matches_host_generator(kind):
    nx, ny, nz = 37, 20, 11
    new, old, _ = gpu_run(kind, nx, ny, nz, 0, seed=77)
    inp = synth.make_inputs(kind, nx, ny, nz, seed=77)
    assert np.array_equal(new, inp.V)
    if kind in WAVES:
        assert np.array_equal(old, inp.U)


@pytest.mark.parametrize("kind", KINDS)
def test_create_from_host_equals_seeded(kind):
    nx, ny, nz = 33, 19, 14
    inp = synth.make_inputs(kind, nx, ny, nz, seed=5)
    a = gpu_run(kind, nx, ny, nz, 7, seed=5)
    b = gpu_run(kind, nx, ny, nz, 7, inputs=inp)
    assert np.array_equal(a[0], b[0])
    if kind in WAVES:
        assert np.array_equal(a[1], b[1])


@pytest.mark.parametrize("kind", KINDS)
def test_parity_short_T_every_block_boundary(kind):
    """G3: T in {1, 2, bt-1, bt, bt+1, 2bt+1} against the oracle, normwise <= 1e-13; G5 ghosts."""
    nx, ny, nz = SHAPES[kind]
    inp = synth.make_inputs(kind, nx, ny, nz, seed=3)
    bts = sorted({1, 2, max_bt(kind)} & set(range(1, max_bt(kind) + 1)))
    for bt in bts:
        Ts = sorted({1, 2, max(1, bt - 1), bt, bt + 1, 2 * bt + 1})
        o_new, o_old = inp.V.copy(), inp.U.copy()
        done = 0
        for T in Ts:
            oracle.run_arrays(kind, nx, ny, nz, o_new, o_old, inp.coef, inp.scalars, T - done)
            done = T
            g_new, g_old, info = gpu_run(kind, nx, ny, nz, T, seed=3, bt=bt)
            assert info["bt"] == bt
            assert_parity(kind, g_new, g_old, o_new, o_old, inp.R, 1e-13, inputs=inp)


@pytest.mark.parametrize("kind", KINDS)
def test_parity_T20_default_plan(kind):
    """G1 at moderate T with the library's default plan (the benchmarked one)."""
    nx, ny, nz = SHAPES[kind]
    inp = synth.make_inputs(kind, nx, ny, nz, seed=1)
    T = 20
    o_new, o_old = oracle.run(inp, T)
    g_new, g_old, info = gpu_run(kind, nx, ny, nz, T, seed=1)
    assert_parity(kind, g_new, g_old, o_new, o_old, inp.R, 1e-11, inputs=inp)


@pytest.mark.parametrize("kind", [synth.K7C, synth.K7V, synth.K25V])
def test_shadow_scaled_per_cell(kind):  # needs non-negative weights: not the waves
    """G2: |g - o| <= 1e-11 * S(p), S = oracle on |inputs| (non-negative coefficients), T = 60."""
    n = (70, 66, 64) if synth.RADIUS[kind] == 1 else (72, 40, 48)
    inp = synth.make_inputs(kind, *n, seed=2)
    T = 60
    o_new, _ = oracle.run(inp, T)
    absinp = synth.Inputs(kind, *n, np.abs(inp.V), np.abs(inp.U), inp.coef, inp.scalars)
    S, _ = oracle.run(absinp, T)
    g_new, _, _ = gpu_run(kind, *n, T, seed=2)
    I = interior(inp.R)
    assert np.all(np.abs(g_new[I] - o_new[I]) <= 1e-11 * S[I])


@pytest.mark.parametrize("kind", KINDS)
def test_variants_bitwise_identical(kind):
    """G4: naive == streaming == TMA-pipelined (every bt, tile configs, several z-chunks) == cooperative
    all-steps kernel, bitwise."""
    nx, ny, nz = SHAPES[kind]
    T = 7
    ref = gpu_run(kind, nx, ny, nz, T, seed=9, variant=st.ST_VARIANT_NAIVE)
    plans = [(st.ST_VARIANT_STREAM, bt, zc, 0) for bt in range(1, max_bt(kind, st.ST_VARIANT_STREAM) + 1)
             for zc in (0, 5, 1000)]
    plans += [(st.ST_VARIANT_PIPE, bt, zc, cfg) for bt in range(1, max_bt(kind) + 1) for zc in (0, 5, 1000)
              for cfg in range(N_CFG[kind])]
    # all T steps in one cooperative launch: one sweep per grid barrier; 7-point Jacobi kinds also with
    # temporal blocking in shared memory (rounds of 5 + 2 levels)
    plans += [(st.ST_VARIANT_COOP, 1, 0, 0)]
    if kind in (synth.K7C, synth.K7V):
        plans += [(st.ST_VARIANT_COOP, 1, 0, 2)]
    for variant, bt, zchunk, cfg in plans:
        got = gpu_run(kind, nx, ny, nz, T, seed=9, variant=variant, bt=bt, zchunk=zchunk, tile_cfg=cfg)
        assert got[2]["bt"] == bt
        assert np.array_equal(got[0], ref[0]), (variant, bt, zchunk, cfg)
        if kind in WAVES:
            assert np.array_equal(got[1], ref[1]), (variant, bt, zchunk, cfg)


@pytest.mark.parametrize("kind", KINDS)
def test_degenerate_extents(kind):
    """G6: extents 1, 2, 3, 5, 17 in every axis (nz < R*bt included), T not a multiple of bt."""
    rng = np.random.default_rng(kind)
    shapes = [(1, 1, 1), (2, 3, 1), (1, 5, 17), (17, 1, 2), (3, 17, 5), (5, 2, 3)]
    shapes += [tuple(int(v) for v in rng.integers(1, 41, size=3)) for _ in range(3)]
    for (nx, ny, nz) in shapes:
        inp = synth.make_inputs(kind, nx, ny, nz, seed=4)
        T = 5
        o_new, o_old = oracle.run(inp, T)
        for variant, bt, cfg in sorted({(st.ST_VARIANT_PIPE, 1, 0), (st.ST_VARIANT_PIPE, max_bt(kind), 0),
                                        (st.ST_VARIANT_STREAM, max_bt(kind, st.ST_VARIANT_STREAM), 0),
                                        (st.ST_VARIANT_COOP, 1, 0)} |
                                       ({(st.ST_VARIANT_COOP, 1, 2)} if kind in (synth.K7C, synth.K7V) else set())):
            g_new, g_old, _ = gpu_run(kind, nx, ny, nz, T, seed=4, bt=bt, variant=variant, tile_cfg=cfg)
            assert_parity(kind, g_new, g_old, o_new, o_old, inp.R, 1e-13, inputs=inp)


@pytest.mark.parametrize("kind", [synth.K7C, synth.K7V])
@pytest.mark.parametrize("T", [1, 5, 12])
def test_coop_temporal_blocking_bitwise(kind, T):
    """G4 for the temporally blocked cooperative kernel (tile_cfg 2 forces it) on a grid with more
    output blocks (16 x 16 x 8) than SMs, so each CTA runs several blocks per round, ragged in every
    axis; rounds of 5 levels with a remainder round (T = 12)."""
    nx, ny, nz = 100, 90, 50
    ref = gpu_run(kind, nx, ny, nz, T, seed=21, variant=st.ST_VARIANT_NAIVE)
    got = gpu_run(kind, nx, ny, nz, T, seed=21, variant=st.ST_VARIANT_COOP, tile_cfg=2)
    assert got[2]["tile_x"] == 16 and got[2]["zchunk"] == 8
    assert np.array_equal(got[0], ref[0])


def test_repeatable_bitwise():
    """Five identical runs of a multi-tile, multi-chunk case give bitwise identical results: a race in
    the TMA/mbarrier rings or the shared level planes would show up as run-to-run differences
    (compute-sanitizer is not available on this pool)."""
    for kind in KINDS:
        nx, ny, nz = (96, 80, 70) if synth.RADIUS[kind] == 1 else (150, 60, 70)
        ref = gpu_run(kind, nx, ny, nz, 9, seed=13, zchunk=8)
        for _ in range(4):
            got = gpu_run(kind, nx, ny, nz, 9, seed=13, zchunk=8)
            assert np.array_equal(got[0], ref[0])


def test_checkpoint_resume_bitwise():
    """run(T1); read; create from the read state; run(T2) == run(T1 + T2), bitwise (all kinds)."""
    for kind in KINDS:
        nx, ny, nz = SHAPES[kind]
        inp = synth.make_inputs(kind, nx, ny, nz, seed=6)
        full = gpu_run(kind, nx, ny, nz, 9, seed=6)
        a_new, a_old, _ = gpu_run(kind, nx, ny, nz, 4, seed=6)
        res = synth.Inputs(kind, nx, ny, nz, a_new, a_old if kind in WAVES else a_new.copy(), inp.coef,
                           inp.scalars)
        b = gpu_run(kind, nx, ny, nz, 5, inputs=res)
        assert np.array_equal(b[0], full[0])
        if kind in WAVES:
            assert np.array_equal(b[1], full[1])


def test_error_codes_on_gpu():
    with pytest.raises(st.StencilError) as ei:
        st.Grid(synth.K7C, 0, 4, 4, seed=1)
    assert ei.value.code == st.ST_E_INVAL
    g = st.Grid(synth.K7V, 8, 8, 8, seed=1)
    with pytest.raises(st.StencilError) as ei:
        g.run(0)
    assert ei.value.code == st.ST_E_INVAL
    with pytest.raises(st.StencilError) as ei:
        g.read(1)  # level 1 is scratch for Jacobi kinds
    assert ei.value.code == st.ST_E_INVAL
    with pytest.raises(st.StencilError) as ei:
        st.stencil_read(g.h, 0, np.zeros(10))
    assert ei.value.code == st.ST_E_INVAL
    info = g.info()
    assert info["device_bytes"] > 0 and info["steps_done"] == 0
    g.run(3)
    g.sync()
    assert g.info()["steps_done"] == 3
    g.close()
    with pytest.raises(st.StencilError) as ei:
        st.Grid(synth.K25V, 4000, 4000, 4000, seed=1)  # 15 x 32 GB: does not fit
    assert ei.value.code == st.ST_E_NOMEM
    assert "bytes" in st.stencil_last_error()


@pytest.mark.parametrize("kind", [synth.K7C, synth.K7V, synth.K25V])
def test_multiblock_launch_bitwise(kind, monkeypatch):
    """All full blocks of a run in one pipe-kernel launch with dependency-driven scheduling across blocks
    (STENCIL_MULTIBLOCK=1; opt-in) == one launch per block, bitwise, including remainder blocks, a
    second run and the work-item-0 fault still terminating (its completion is published)."""
    nx, ny, nz = SHAPES[kind]
    plans = [(1, 5)]
    if kind != synth.K25V:  # the two-level 25-point kernel (pipe25.cu) runs one block per launch
        plans.append((max_bt(kind), 3 * max_bt(kind) + 1))
    for bt, T in plans:
        ref = gpu_run(kind, nx, ny, nz, T, seed=5, variant=st.ST_VARIANT_PIPE, bt=bt, zchunk=7)
        monkeypatch.setenv("STENCIL_MULTIBLOCK", "1")
        got = gpu_run(kind, nx, ny, nz, T, seed=5, variant=st.ST_VARIANT_PIPE, bt=bt, zchunk=7)
        monkeypatch.delenv("STENCIL_MULTIBLOCK")
        assert np.array_equal(got[0], ref[0]), bt
        assert got[2]["launches"] < ref[2]["launches"]


@pytest.mark.parametrize("T,bt", [(7, 3), (10, 3), (12, 4), (5, 1), (9, 2)])
def test_launch_schedule_matches_bench_accounting(T, bt):
    """bench.py counts the roofline's algorithmic bytes per fused block with bench.blocks_of(T, bt);
    the runtime must launch exactly those blocks (one pipe launch per block on a single slab)."""
    import bench
    with st.Grid(synth.K7V, 40, 36, 30, seed=2, variant=st.ST_VARIANT_PIPE, bt=bt) as g:
        l0 = g.info()["launches"]
        g.run(T)
        assert g.info()["launches"] - l0 == len(bench.blocks_of(T, bt))


@pytest.mark.parametrize("kind,n", [(synth.K7V, (8000, 3, 3)), (synth.K7V, (3, 5000, 5)),
                                    (synth.K7V, (4096, 4096, 2)), (synth.K25V, (2500, 9, 6)),
                                    (synth.K25W, (7, 3000, 9))])
def test_extreme_aspect_ratios_bitwise(kind, n):
    """G6 at the extremes: very long rows / columns and a 16.8 M-cell plane (64-bit plane offsets, TMA
    boxes at the far end of a row, one z-chunk per tile) -- the default plan equals the naive sweeps
    bitwise, and the oracle on the thin cases."""
    T = 3
    ref = gpu_run(kind, *n, T, seed=5, variant=st.ST_VARIANT_NAIVE)
    got = gpu_run(kind, *n, T, seed=5)
    assert np.array_equal(got[0], ref[0])
    if kind in WAVES:
        assert np.array_equal(got[1], ref[1])
    if n[0] * n[1] * n[2] <= 200000:
        inp = synth.make_inputs(kind, *n, seed=5)
        o_new, o_old = oracle.run(inp, T)
        assert_parity(kind, got[0], got[1], o_new, o_old, inp.R, 1e-13, inputs=inp)
