"""The 25-point variable-coefficient kind with two fused levels (pipe25.cu, SURVEY §8(a) row a7 for C4/C5):
bitwise equal to the naive sweeps (G4) at every T parity, z-chunk and tile position; oracle parity at short
T (G3) and ghosts untouched (G5); degenerate and ragged extents (G6); z-slabs with both halo modes."""
import numpy as np
import pytest

import oracle
import paper_1410_3060_b200 as st
import synth
from gpu_common import assert_parity, gpu_run

pytestmark = pytest.mark.gpu
K = synth.K25V

# output tile 24 x 16: shapes with ragged tails in x and y, and z-chunks from 1 plane to the whole slab
SHAPES = [(130, 37, 41), (24, 16, 9), (25, 17, 13), (71, 50, 30), (1, 1, 1), (3, 2, 5), (50, 3, 8), (2, 40, 17),
          (48, 150, 12)]


# tile_cfg: 0 = single CTA (24 x 16 output tiles), 1 = cluster pair (24 x 32), 2 = cluster of 4 (24 x 72),
# 3 = skewed single-CTA tiles (24 x 20, level-1 rows handed to the tile above through global memory)
CFGS = (0, 1, 2, 3)


@pytest.mark.parametrize("shape", SHAPES)
def test_bt2_bitwise_equal_naive(shape):
    for T in (1, 2, 3, 6):
        ref = gpu_run(K, *shape, T, seed=21, variant=st.ST_VARIANT_NAIVE)
        for cfg in CFGS:
            for zc in (0, 1, 3, 1000):
                got = gpu_run(K, *shape, T, seed=21, variant=st.ST_VARIANT_PIPE, bt=2, zchunk=zc, tile_cfg=cfg)
                assert got[2]["bt"] == 2
                assert np.array_equal(got[0], ref[0]), (shape, T, cfg, zc)


def test_bt2_oracle_short_T():
    nx, ny, nz = 130, 37, 41
    inp = synth.make_inputs(K, nx, ny, nz, seed=8)
    o_new, o_old = inp.V.copy(), inp.U.copy()
    done = 0
    for T in (1, 2, 3, 4, 5):
        oracle.run_arrays(K, nx, ny, nz, o_new, o_old, inp.coef, inp.scalars, T - done)
        done = T
        for cfg in CFGS:
            g_new, _, info = gpu_run(K, nx, ny, nz, T, seed=8, bt=2, tile_cfg=cfg)
            assert info["bt"] == 2
            assert_parity(K, g_new, None, o_new, None, inp.R, 1e-13, inputs=inp)


def test_bt2_consecutive_runs_and_odd_T():
    # runs of odd length end with a one-level block (the bt = 1 kernel); resuming must continue exactly
    nx, ny, nz = 61, 29, 23
    ref = gpu_run(K, nx, ny, nz, 9, seed=4, variant=st.ST_VARIANT_NAIVE)
    with st.Grid(K, nx, ny, nz, seed=4, bt=2) as g:
        for t in (3, 1, 5):
            g.run(t)
        assert np.array_equal(g.read(0), ref[0])


@pytest.mark.parametrize("cfg", [0, 3])
@pytest.mark.parametrize("halo", [st.ST_HALO_COPY, st.ST_HALO_PEER])
@pytest.mark.parametrize("P", [2, 3])
def test_bt2_loopback_slabs(halo, P, cfg):
    nx, ny, nz = 70, 33, 40
    ref = gpu_run(K, nx, ny, nz, 6, seed=6, variant=st.ST_VARIANT_NAIVE)
    with st.Grid(K, nx, ny, nz, seed=6, bt=2, nranks=P, local_slabs=P, halo=halo, tile_cfg=cfg, tuned=False) as g:
        g.run(6)
        assert g.info()["bt"] == 2
        assert np.array_equal(g.read(0), ref[0])


# ------------------------------------------------------------------ the wave (Fig. 1e) on the same kernel
W = synth.K25W


@pytest.mark.parametrize("shape", SHAPES)
def test_wave_bt2_bitwise_equal_naive(shape):
    """pipe25.cu's wave instance (tile_cfg 0; 1 and 2 = the round-1 generic kernel): both new levels
    (Omega^T and Omega^{T-1}) bitwise equal to the naive sweeps."""
    for T in (1, 2, 3, 6):
        ref = gpu_run(W, *shape, T, seed=23, variant=st.ST_VARIANT_NAIVE)
        for cfg in (0, 1):
            for zc in (0, 1, 3, 1000):
                got = gpu_run(W, *shape, T, seed=23, variant=st.ST_VARIANT_PIPE, bt=2, zchunk=zc, tile_cfg=cfg)
                assert got[2]["bt"] == 2
                assert np.array_equal(got[0], ref[0]), (shape, T, cfg, zc)
                assert np.array_equal(got[1], ref[1]), (shape, T, cfg, zc)


def test_wave_bt2_oracle_short_T():
    nx, ny, nz = 130, 37, 41
    inp = synth.make_inputs(W, nx, ny, nz, seed=8)
    o_new, o_old = inp.V.copy(), inp.U.copy()
    done = 0
    for T in (1, 2, 3, 4, 5):
        oracle.run_arrays(W, nx, ny, nz, o_new, o_old, inp.coef, inp.scalars, T - done)
        done = T
        g_new, g_old, info = gpu_run(W, nx, ny, nz, T, seed=8, bt=2)
        assert info["bt"] == 2
        assert_parity(W, g_new, g_old, o_new, o_old, inp.R, 1e-13, inputs=inp)


@pytest.mark.parametrize("halo", [st.ST_HALO_COPY, st.ST_HALO_PEER])
def test_wave_bt2_loopback_slabs(halo):
    nx, ny, nz = 70, 33, 40
    ref = gpu_run(W, nx, ny, nz, 6, seed=6, variant=st.ST_VARIANT_NAIVE)
    with st.Grid(W, nx, ny, nz, seed=6, bt=2, nranks=3, local_slabs=3, halo=halo) as g:
        g.run(6)
        assert np.array_equal(g.read(0), ref[0]) and np.array_equal(g.read(1), ref[1])
