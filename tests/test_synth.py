"""Generator tests (reading Q6): determinism, golden values, numpy restatement == C fill,
sub-box == global (partition independence), moments of the drawn distributions."""
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "synth_golden.txt")


def test_golden_values_numpy_and_c():
    rows = [l.split() for l in open(GOLDEN) if not l.startswith("#")]
    assert len(rows) >= 40
    for seed, stream, idx, hexv in rows:
        seed, stream, idx = int(seed), int(stream), int(idx)
        want = float.fromhex(hexv)
        got = synth.numpy_unit(seed, stream, np.array([idx], dtype=np.uint64))[0]
        assert got == want
    # the C fill draws u at linear index idx of a flat (1, 1, n) grid; dist 1 with c = 1 -> u*1 = u
    for seed, stream, idx, hexv in rows:
        idx = int(idx)
        if idx > 5000:
            continue
        a = synth.fill_box(int(seed), int(stream), (1, 1, idx + 1), ((0, 1), (0, 1), (idx, idx + 1)), scale=1.0)
        assert a[0, 0, 0] == float.fromhex(hexv)


def test_c_fill_matches_numpy_restatement():
    dims = (7, 9, 11)
    for stream in (0, 1, 5):
        a = synth.fill_box(42, stream, dims)
        u = synth.numpy_unit(42, stream, np.arange(np.prod(dims)))
        assert np.array_equal(a.ravel(), 2.0 * u - 1.0)
        b = synth.fill_box(42, stream, dims, scale=1.0 / 7.0)
        assert np.array_equal(b.ravel(), u * (1.0 / 7.0))


def test_determinism_and_seed_sensitivity():
    a = synth.fill_box(3, 0, (5, 6, 7))
    b = synth.fill_box(3, 0, (5, 6, 7))
    c = synth.fill_box(4, 0, (5, 6, 7))
    d = synth.fill_box(3, 1, (5, 6, 7))
    assert np.array_equal(a, b)
    assert not np.any(a == c)
    assert not np.any(a == d)


def test_subbox_equals_global():
    dims = (12, 10, 9)
    g = synth.fill_box(9, 2, dims)
    box = ((3, 8), (1, 10), (2, 7))
    s = synth.fill_box(9, 2, dims, box)
    assert np.array_equal(s, g[3:8, 1:10, 2:7])
    for kind in (synth.K7C, synth.K7V, synth.K25W, synth.K25V):
        full = synth.make_inputs(kind, 5, 6, 7, seed=11)
        Z, Y, X = synth.padded_dims(kind, 5, 6, 7)
        bx = ((2, Z - 1), (0, Y), (3, X))
        sub = synth.make_inputs(kind, 5, 6, 7, seed=11, box=bx)
        sl = tuple(slice(a, b) for a, b in bx)
        assert np.array_equal(sub.V, full.V[sl])
        assert np.array_equal(sub.U, full.U[sl])
        for w, wf in zip(sub.coef, full.coef):
            assert np.array_equal(w, wf[sl])


def test_initial_state_rules():
    # Q1/Q8: U is a copy of V for Jacobi kinds; Q9: wave U interior from stream 1, ghosts from V.
    for kind in (synth.K7C, synth.K7V, synth.K25V):
        inp = synth.make_inputs(kind, 4, 5, 6, seed=5)
        assert np.array_equal(inp.U, inp.V)
    inp = synth.make_inputs(synth.K25W, 4, 5, 6, seed=5)
    R = 4
    interior = (slice(R, -R),) * 3
    assert not np.any(inp.U[interior] == inp.V[interior])
    m = np.ones(inp.V.shape, bool)
    m[interior] = False
    assert np.array_equal(inp.U[m], inp.V[m])


def test_moments():
    n = 2_000_000
    a = synth.fill_box(14103060, 0, (1, 1, n)).ravel()
    assert a.min() >= -1.0 and a.max() < 1.0
    sd = np.sqrt(1.0 / 3.0 / n)
    assert abs(a.mean()) < 4 * sd
    assert abs(a.var() - 1.0 / 3.0) < 2e-3
    w = synth.fill_box(14103060, 2, (1, 1, n), scale=1.0 / 7.0).ravel()
    assert w.min() >= 0.0 and w.max() < 1.0 / 7.0
    assert abs(w.mean() - 0.5 / 7.0) < 4 * (1.0 / 7.0) * np.sqrt(1.0 / 12.0 / n)
    w = synth.fill_box(14103060, 3, (1, 1, n), scale=1.0 / 25.0).ravel()
    assert w.max() < 1.0 / 25.0


def test_bad_box_rejected():
    with pytest.raises(ValueError):
        synth.fill_box(1, 0, (3, 3, 3), ((0, 4), (0, 3), (0, 3)))
