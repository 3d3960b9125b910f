"""Randomised plans (tools/fuzz.py's generator: kind, extents, T -- sometimes split over consecutive
stencil_run calls -- variant, bt, tile_cfg, z-chunk, loopback slabs with copy or peer halos) checked
(a) bitwise against the naive sweeps (G4) and (b) against the CPU oracle at extents <= 40 (normwise
<= 1e-13), each for a bounded time with a fixed seed."""
import importlib.util
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

_spec = importlib.util.spec_from_file_location(
    "fuzz", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "fuzz.py"))
fuzz = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(fuzz)


def _oracle_check(kind, n, T, seed, got):
    R = synth.RADIUS[kind]
    o_new, o_old = oracle.run(synth.make_inputs(kind, *n, seed=seed), T, nthreads=1)
    I = (slice(R, -R),) * 3

    def close(g, o):
        return np.max(np.abs(g[I] - o[I])) <= 1e-13 * max(np.max(np.abs(o[I])), 1e-300)
    return close(got[0], o_new) and (got[1] is None or close(got[1], o_old))


def test_random_plans_bitwise_vs_naive():
    cases, bad = fuzz.fuzz(0.5, 11)
    assert cases > 100 and bad == 0


def test_random_plans_vs_oracle():
    cases, bad = fuzz.fuzz(0.75, 12, against=_oracle_check, max_extent=40)
    assert cases > 100 and bad == 0
