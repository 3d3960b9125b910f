"""Pins P1-P11: facts the paper and the mathematics fix, checked against oracle/.

None of these re-types the oracle's loop: each compares with a hand-computed value, a closed
form, an exact-rational brute force of the affine map, a symmetry, or a textbook solver.
"""
from fractions import Fraction
import itertools
import math

import numpy as np
import pytest

import oracle
import synth

K7C, K7V, K25W, K25V = synth.K7C, synth.K7V, synth.K25W, synth.K25V
U_RND = 2.0 ** -53


def mk(kind, nx, ny, nz, V, U=None, coef=(), scalars=()):
    return synth.Inputs(kind, nx, ny, nz, np.ascontiguousarray(V, dtype=np.float64),
                        np.ascontiguousarray(V if U is None else U, dtype=np.float64).copy(),
                        [np.ascontiguousarray(c, dtype=np.float64) for c in coef], tuple(scalars))


def ulps(a, b):
    return abs(a - b) / math.ulp(b)


# ---------------------------------------------------------------- P1 hand-computed points
def star_grid(R, centre, minus, plus):
    """1^3 interior, padded (2R+1)^3; V(axis a, -r) = minus(a, r), V(+r) = plus(a, r)."""
    n = 2 * R + 1
    V = np.zeros((n, n, n))
    V[R, R, R] = centre
    for a in range(3):
        for r in range(1, R + 1):
            for sgn, f in ((-1, minus), (1, plus)):
                idx = [R, R, R]
                idx[2 - a] += sgn * r  # axis 0 = x = last array index
                V[tuple(idx)] = f(a, r)
    return V


def test_P1a_7c_hand():
    # ghosts x-,x+,y-,y+,z-,z+ = 1..6, centre 1 (Fig. 1b)
    V = star_grid(1, 1.0, lambda a, r: 1.0 + 2 * a, lambda a, r: 2.0 + 2 * a)
    o, _ = oracle.run(mk(K7C, 1, 1, 1, V, scalars=(0.25, 0.125)), 1)
    assert o[1, 1, 1] == 2.875  # 1/4 + 1/8*(3 + 7 + 11), exact dyadic
    o, _ = oracle.run(mk(K7C, 1, 1, 1, V, scalars=(0.4, 0.1)), 1)
    assert ulps(o[1, 1, 1], 2.5) <= 2  # 0.4 + 0.1*21 = 2.5 in exact arithmetic


def test_P1b_7v_direction_map():
    # W_i = 2^-(i+1): 1/2 + 1/4*1 + 1/8*2 + 1/16*3 + 1/32*4 + 1/64*5 + 1/128*6 = 1.4375 (Fig. 1c)
    V = star_grid(1, 1.0, lambda a, r: 1.0 + 2 * a, lambda a, r: 2.0 + 2 * a)
    W = [np.full(V.shape, 2.0 ** -(i + 1)) for i in range(7)]
    o, _ = oracle.run(mk(K7V, 1, 1, 1, V, coef=W), 1)
    assert o[1, 1, 1] == 1.4375
    # swapping W1 and W2 (x- <-> x+) must change the answer to 1.5625
    W2 = list(W)
    W2[1], W2[2] = W[2], W[1]
    o, _ = oracle.run(mk(K7V, 1, 1, 1, V, coef=W2), 1)
    assert o[1, 1, 1] == 1.5625


def test_P1c_25v_radius_axis_indexing():
    # W0 = 1/2, W_{1+3(r-1)+a} = 2^-(2+3(r-1)+a), V(a,-r) = (a+1) r, V(a,+r) = 2 (a+1) r  -> 6535/2048
    V = star_grid(4, 1.0, lambda a, r: (a + 1.0) * r, lambda a, r: 2.0 * (a + 1) * r)
    W = [np.full(V.shape, 0.5)] + [np.full(V.shape, 2.0 ** -(2 + j)) for j in range(12)]
    o, _ = oracle.run(mk(K25V, 1, 1, 1, V, coef=W), 1)
    assert o[4, 4, 4] == 6535.0 / 2048.0


def test_P1d_25w_hand():
    # V centre 1, U centre 0.5, V(axis, +-r) = r; BASELINE.json config 3 constants:
    # 2*1 - 0.5 + 0.1*(w0 + sum_r w_r * 6 r) = 1.4072619047619048 (exact rational 1 ulp below)
    V = star_grid(4, 1.0, lambda a, r: float(r), lambda a, r: float(r))
    U = V.copy()
    U[4, 4, 4] = 0.5
    new, old = oracle.run(mk(K25W, 1, 1, 1, V, U, scalars=synth.SCALARS_25W), 1)
    assert ulps(new[4, 4, 4], 1.4072619047619048) <= 2
    assert old[4, 4, 4] == 1.0  # Omega^{T-1} = Omega^0 centre


def test_P1e_1d_degenerate_two_steps():
    # ny = nz = 1, weights (0.5, 0.25), ghosts 0, V = (1,2,3,4): T=1 -> (1,2,3,2.75); T=2 -> (1,2,2.6875,2.125)
    V = np.zeros((3, 3, 6))
    V[1, 1, 1:5] = [1, 2, 3, 4]
    o, prev = oracle.run(mk(K7C, 4, 1, 1, V, scalars=(0.5, 0.25)), 1)
    assert list(o[1, 1, 1:5]) == [1, 2, 3, 2.75]
    o, prev = oracle.run(mk(K7C, 4, 1, 1, V, scalars=(0.5, 0.25)), 2)
    assert list(o[1, 1, 1:5]) == [1, 2, 2.6875, 2.125]
    assert list(prev[1, 1, 1:5]) == [1, 2, 3, 2.75]


# ---------------------------------------------------------------- P2 constant field
@pytest.mark.parametrize("kind", [K7C, K7V, K25V])
def test_P2_constant_field_dyadic_bitwise(kind):
    R = synth.RADIUS[kind]
    n = (5, 6, 7)
    shape = tuple(d + 2 * R for d in n[::-1])
    V = np.full(shape, 0.75)
    if kind == K7C:
        inp = mk(kind, *n, V, scalars=(0.25, 0.125))
    elif kind == K7V:
        inp = mk(kind, *n, V, coef=[np.full(shape, 0.25)] + [np.full(shape, 0.125)] * 6)
    else:
        inp = mk(kind, *n, V, coef=[np.full(shape, 0.25)] + [np.full(shape, 1.0 / 32)] * 12)
    o, _ = oracle.run(inp, 9)
    assert np.all(o == 0.75)


def test_P2_constant_field_bj_weights():
    shape = (10, 9, 8)
    for c in (1.0, -0.7, 0.123456789, 0.3):
        o, _ = oracle.run(mk(K7C, 6, 7, 8, np.full(shape, c), scalars=synth.SCALARS_7C), 10)
        assert np.max(np.abs(o - c)) <= 8 * 10 * math.ulp(abs(c))


@pytest.mark.parametrize("kind", [K7V, K25V])
def test_P2_random_coefficients_summing_to_one(kind):
    R = synth.RADIUS[kind]
    n = (6, 5, 4)
    shape = tuple(d + 2 * R for d in n[::-1])
    rng = np.random.default_rng(0)
    k = synth.N_COEF_FIELDS[kind]
    W = [None] + [rng.uniform(0, 1.0 / (2 * k), shape) for _ in range(k - 1)]
    pair = 2 if kind == K25V else 1  # 25v weights multiply a pair sum
    W[0] = 1.0 - pair * sum(W[1:])
    T = 6
    o, _ = oracle.run(mk(kind, *n, np.full(shape, 0.5), coef=W), T)
    assert np.max(np.abs(o - 0.5)) <= 2 * T * 2 * k * U_RND * 4


def test_P2_wave_constant():
    shape = (14, 13, 12)
    o, prev = oracle.run(mk(K25W, 4, 5, 6, np.full(shape, 0.8), scalars=synth.SCALARS_25W), 100)
    assert np.max(np.abs(o - 0.8)) <= 1e-12
    assert np.max(np.abs(prev - 0.8)) <= 1e-12


# ---------------------------------------------------------------- P3 polynomial exactness
def poly_grid(R, n, fn):
    m = n + 2 * R
    z, y, x = np.meshgrid(np.arange(m, dtype=np.float64), np.arange(m, dtype=np.float64),
                          np.arange(m, dtype=np.float64), indexing="ij")
    return x, y, z, fn(x, y, z)


POLYS_8 = [  # (p, analytic Laplacian), per-axis degree <= 9
    (lambda x, y, z: x ** 9 - 3 * y ** 7 + 2 * z ** 8 + x ** 2 * y ** 3 * z,
     lambda x, y, z: 72 * x ** 7 - 126 * y ** 5 + 112 * z ** 6 + 2 * y ** 3 * z + 6 * x ** 2 * y * z),
    (lambda x, y, z: x ** 4 * y ** 5 - z ** 9,
     lambda x, y, z: 12 * x ** 2 * y ** 5 + 20 * x ** 4 * y ** 3 - 72 * z ** 7),
]


@pytest.mark.parametrize("pi", range(len(POLYS_8)))
def test_P3_wave_laplacian_exact_to_degree_9(pi):
    p, lap = POLYS_8[pi]
    x, y, z, P = poly_grid(4, 8, p)
    new, _ = oracle.run(mk(K25W, 8, 8, 8, P, P, scalars=synth.SCALARS_25W), 1)
    want = P + 0.1 * lap(x, y, z)
    I = (slice(4, -4),) * 3
    scale = np.max(np.abs(P))
    assert np.max(np.abs(new[I] - want[I])) / scale <= 1e-14


def test_P3_wave_degree_10_fails():
    x, y, z, P = poly_grid(4, 8, lambda x, y, z: x ** 10)
    new, _ = oracle.run(mk(K25W, 8, 8, 8, P, P, scalars=synth.SCALARS_25W), 1)
    want = P + 0.1 * 90 * x ** 8
    I = (slice(4, -4),) * 3
    assert np.max(np.abs(new[I] - want[I])) / np.max(np.abs(P)) > 1e-10


def test_P3_7c_exact_to_degree_3_and_heat8_25v():
    x, y, z, P = poly_grid(1, 9, lambda x, y, z: x ** 3 - 2 * y ** 2 * z + z ** 3 * x)
    o, _ = oracle.run(mk(K7C, 9, 9, 9, P, scalars=(0.4, 0.1)), 1)
    want = P + 0.1 * (6 * x - 4 * z + 6 * z * x)
    I = (slice(1, -1),) * 3
    assert np.max(np.abs(o[I] - want[I])) / np.max(np.abs(P)) <= 1e-14
    x, y, z, P = poly_grid(1, 9, lambda x, y, z: x ** 4)
    o, _ = oracle.run(mk(K7C, 9, 9, 9, P, scalars=(0.4, 0.1)), 1)
    assert np.max(np.abs(o[I] - (P + 0.1 * 12 * x ** 2)[I])) > 0.01  # 7-point fails at degree 4
    # 25v with "heat-8" coefficients W0 = 1 + alpha*w0, W_{r,a} = alpha*w_r
    w0, w1, w2, w3, w4, _ = synth.SCALARS_25W
    al = 0.125
    p, lap = POLYS_8[1]
    x, y, z, P = poly_grid(4, 8, p)
    W = [np.full(P.shape, 1 + al * w0)] + [np.full(P.shape, al * w) for w in (w1, w2, w3, w4) for _ in range(3)]
    o, _ = oracle.run(mk(K25V, 8, 8, 8, P, coef=W), 1)
    I = (slice(4, -4),) * 3
    assert np.max(np.abs(o[I] - (P + al * lap(x, y, z))[I])) / np.max(np.abs(P)) <= 1e-14


# ---------------------------------------------------------------- P4 exact affine-map power
def star_offsets(kind):
    """(weight-source, [(dz,dy,dx), ...]) terms of Fig. 1, written from the figure as a list."""
    if kind in (K7C, K7V):
        return [("c", [(0, 0, 0)]), ("x-", [(0, 0, -1)]), ("x+", [(0, 0, 1)]), ("y-", [(0, -1, 0)]),
                ("y+", [(0, 1, 0)]), ("z-", [(-1, 0, 0)]), ("z+", [(1, 0, 0)])]
    terms = [("c", [(0, 0, 0)])]
    for r in range(1, 5):
        terms += [(("x", r), [(0, 0, -r), (0, 0, r)]), (("y", r), [(0, -r, 0), (0, r, 0)]),
                  (("z", r), [(-r, 0, 0), (r, 0, 0)])]
    return terms


def exact_run(inp, T):
    """Exact-rational T steps of the affine map v_{t+1} = A v_t (+ ghosts), using Fractions."""
    kind, R = inp.kind, inp.R
    shape = inp.V.shape
    F = np.vectorize(Fraction, otypes=[object])
    cur, prev = F(inp.V), F(inp.U)
    W = [F(c) for c in inp.coef]
    s = [Fraction(v) for v in inp.scalars]
    terms = star_offsets(kind)
    for _ in range(T):
        nxt = prev.copy()
        for z, y, x in itertools.product(range(R, shape[0] - R), range(R, shape[1] - R), range(R, shape[2] - R)):
            acc = Fraction(0)
            for ti, (src, offs) in enumerate(terms):
                val = sum(cur[z + dz, y + dy, x + dx] for dz, dy, dx in offs)
                if kind == K7C:
                    w = s[0] if src == "c" else s[1]
                elif kind in (K7V, K25V):
                    w = W[ti][z, y, x]
                else:
                    w = s[0] if src == "c" else s[src[1]]
                acc += w * val
            if kind == K25W:
                acc = 2 * cur[z, y, x] - prev[z, y, x] + s[5] * acc
            nxt[z, y, x] = acc
        prev, cur = cur, nxt
    return cur, prev


@pytest.mark.parametrize("kind,n,T", [(K7C, (4, 3, 4), 6), (K7V, (3, 4, 4), 6), (K25W, (5, 4, 3), 5),
                                      (K25V, (5, 4, 3), 6)])
def test_P4_exact_rational_brute_force(kind, n, T):
    inp = synth.make_inputs(kind, *n, seed=3)
    o_new, o_old = oracle.run(inp, T)
    e_new, e_old = exact_run(inp, T)
    k = 25 if synth.RADIUS[kind] == 4 else 7
    for o, e in ((o_new, e_new), (o_old, e_old)):
        ef = e.astype(np.float64)
        err = np.max(np.abs(o - ef)) / np.max(np.abs(ef))
        assert err <= 2 * T * k * U_RND * (8 if kind == K25W else 1), err


# ---------------------------------------------------------------- P5 mirror symmetry
def mirror_inputs(kind, n, seed=4):
    inp = synth.make_inputs(kind, *n, seed=seed)
    # symmetrise V, U (and coefficients) under x -> mirror; 7v: W1 <-> W2 under the mirror
    V = 0.5 * (inp.V + inp.V[:, :, ::-1])
    U = V.copy() if kind != K25W else 0.5 * (inp.U + inp.U[:, :, ::-1])
    coef = inp.coef
    if kind == K7V:
        W = [0.5 * (c + c[:, :, ::-1]) for c in coef]
        W[1] = coef[1]
        W[2] = coef[1][:, :, ::-1].copy()
        coef = W
    elif kind == K25V:
        coef = [0.5 * (c + c[:, :, ::-1]) for c in coef]
    return mk(kind, *n, V, U, coef, inp.scalars)


@pytest.mark.parametrize("kind", [K7C, K7V, K25W, K25V])
def test_P5_mirror_symmetry(kind):
    inp = mirror_inputs(kind, (7, 5, 6))
    T = 5
    o, _ = oracle.run(inp, T)
    d = np.max(np.abs(o - o[:, :, ::-1]))
    if kind == K7V:
        assert d <= T * 7 * U_RND * np.max(np.abs(o)) * 4
    else:
        assert d == 0.0


def test_P5_axis_permutation_7c():
    inp = synth.make_inputs(K7C, 6, 6, 6, seed=8)
    V = inp.V
    Vs = (V + V.transpose(0, 2, 1)) / 2  # symmetric under x <-> y
    o, _ = oracle.run(mk(K7C, 6, 6, 6, Vs, scalars=synth.SCALARS_7C), 6)
    assert np.max(np.abs(o - o.transpose(0, 2, 1))) <= 6 * 7 * U_RND * 4


# ---------------------------------------------------------------- P6 plane-wave closed form
def test_P6_plane_wave_7c_and_wave():
    T = 5
    k = (0.3, 0.7, 1.1)
    for kind, R, n in ((K7C, 1, 30), (K25W, 4, 60)):
        m = n + 2 * R
        z, y, x = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
        phase = k[0] * x + k[1] * y + k[2] * z
        if kind == K7C:
            V = np.cos(phase)
            o, _ = oracle.run(mk(kind, n, n, n, V, scalars=(0.4, 0.1)), T)
            lam = 0.4 + 2 * 0.1 * sum(math.cos(kk) for kk in k)
            want = lam ** T * np.cos(phase)
        else:
            w = synth.SCALARS_25W
            Lam = w[0] + 2 * sum(w[r] * sum(math.cos(r * kk) for kk in k) for r in range(1, 5))
            a0, a1 = 0.6, 1.0
            V, U = a1 * np.cos(phase), a0 * np.cos(phase)
            o, _ = oracle.run(mk(kind, n, n, n, V, U, scalars=w), T)
            am, a = a0, a1
            for _ in range(T):
                am, a = a, (2 + w[5] * Lam) * a - am
            want = a * np.cos(phase)
        lo, hi = R + R * T, m - R - R * T
        I = (slice(lo, hi),) * 3
        assert np.max(np.abs(o[I] - want[I])) <= 1e-12


# ---------------------------------------------------------------- P7 linearity
@pytest.mark.parametrize("kind", [K7C, K7V, K25W, K25V])
def test_P7_linearity(kind):
    inp = synth.make_inputs(kind, 6, 5, 7, seed=2)
    T = 4
    o, op = oracle.run(inp, T)
    o2, op2 = oracle.run(mk(kind, 6, 5, 7, 2 * inp.V, 2 * inp.U, inp.coef, inp.scalars), T)
    assert np.array_equal(o2, 2 * o) and np.array_equal(op2, 2 * op)
    # superposition: o(v, g) = o(v, 0) + o(0, g)
    R = inp.R
    I = (slice(R, -R),) * 3
    Vi = np.zeros_like(inp.V); Vi[I] = inp.V[I]
    Ui = np.zeros_like(inp.U); Ui[I] = inp.U[I]
    a, _ = oracle.run(mk(kind, 6, 5, 7, Vi, Ui, inp.coef, inp.scalars), T)
    b, _ = oracle.run(mk(kind, 6, 5, 7, inp.V - Vi, inp.U - Ui, inp.coef, inp.scalars), T)
    tol = 2 * T * 25 * U_RND * (8 ** T if kind == K25W else 1) * 4
    assert np.max(np.abs(a + b - o)) <= tol


# ---------------------------------------------------------------- P8 special-case reductions
def test_P8_reductions():
    inp = synth.make_inputs(K7C, 6, 7, 5, seed=6)
    T = 5
    o7c, _ = oracle.run(inp, T)
    shape = inp.V.shape
    W = [np.full(shape, 0.4)] + [np.full(shape, 0.1)] * 6
    o7v, _ = oracle.run(mk(K7V, 6, 7, 5, inp.V, coef=W), T)
    assert np.max(np.abs(o7v - o7c)) <= T * 7 * U_RND * 4
    inp = synth.make_inputs(K25W, 5, 6, 7, seed=6)
    s0 = list(synth.SCALARS_25W)
    s0[5] = 0.0
    new, old = oracle.run(mk(K25W, 5, 6, 7, inp.V, inp.U, scalars=s0), 1)
    I = (slice(4, -4),) * 3
    assert np.array_equal(new[I], (2 * inp.V - inp.U)[I])


# ---------------------------------------------------------------- P9 locality cone
@pytest.mark.parametrize("kind,T", [(K7C, 3), (K7V, 4), (K25W, 2), (K25V, 2)])
def test_P9_locality_cone(kind, T):
    n = 21
    inp = synth.make_inputs(kind, n, n, n, seed=1)
    R = inp.R
    a, _ = oracle.run(inp, T)
    p = (R + 10, R + 10, R + 10)
    V = inp.V.copy(); V[p] += 1.0
    U = inp.U.copy()
    if kind != K25W:
        U[p] += 1.0  # keep U = V (Jacobi kinds' scratch buffer)
    b, _ = oracle.run(mk(kind, n, n, n, V, U, inp.coef, inp.scalars), T)
    changed = a != b
    m = n + 2 * R
    z, y, x = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    moves = sum(np.ceil(np.abs(c - pc) / R) for c, pc in zip((z, y, x), p))
    reach = moves <= T
    assert np.array_equal(changed, reach)


# ---------------------------------------------------------------- P10 determinism
def test_P10_thread_count_invariance():
    for kind in (K7V, K25W):
        inp = synth.make_inputs(kind, 9, 10, 23, seed=7)
        res = [oracle.run(inp, 4, nthreads=t)[0] for t in (1, 2, 8)]
        assert all(np.array_equal(res[0], r) for r in res[1:])


# ---------------------------------------------------------------- P11 steady state
def test_P11_steady_state_dirichlet():
    n = 4
    inp = synth.make_inputs(K7C, n, n, n, seed=9)
    o, _ = oracle.run(inp, 3000)
    V = inp.V
    idx = {c: i for i, c in enumerate(itertools.product(range(1, n + 1), repeat=3))}
    A = np.zeros((n ** 3, n ** 3))
    b = np.zeros(n ** 3)
    for (z, y, x), i in idx.items():
        A[i, i] = -6.0
        for dz, dy, dx in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
            q = (z + dz, y + dy, x + dx)
            if q in idx:
                A[i, idx[q]] += 1.0
            else:
                b[i] -= V[q]
    sol = np.linalg.solve(A, b)
    got = np.array([o[c] for c in idx])
    assert np.max(np.abs(got - sol)) <= 1e-12


# ---------------------------------------------------------------- misc contract
def test_oracle_rejects_bad_arguments():
    inp = synth.make_inputs(K7C, 3, 3, 3)
    with pytest.raises(ValueError):
        oracle.run(inp, 0)
    with pytest.raises(ValueError):
        oracle.run_arrays(K7C, 3, 3, 3, inp.V, inp.U, [], (0.4,), 1)


def test_run_cone_matches_full_run():
    for kind, n, T in ((K7V, (20, 18, 22), 4), (K25W, (22, 21, 20), 2), (K25V, (21, 20, 22), 2)):
        inp = synth.make_inputs(kind, *n, seed=12)
        full_new, full_old = oracle.run(inp, T)
        R = inp.R
        cells = [(R, R, R), (R + 9, R + 10, R + 11), (n[2] + R - 1, n[1] + R - 1, n[0] + R - 1),
                 (R + 3, n[1] + R - 2, R + 12)]
        new, old = oracle.run_cone(kind, *n, cells, T, seed=12)
        assert np.array_equal(new, np.array([full_new[c] for c in cells]))
        assert np.array_equal(old, np.array([full_old[c] for c in cells]))


# ---------------------------------------------------------------- kind 5: Fig. 1e with alpha_{z,y,x}
K25WA = synth.K25WA


def test_P8_alpha_field_constant_equals_scalar_wave():
    """A constant alpha field reproduces the scalar-alpha wave bitwise (same expression)."""
    inp = synth.make_inputs(K25W, 7, 6, 9, seed=3)
    o3, p3 = oracle.run(inp, 6)
    A = np.full(inp.V.shape, synth.SCALARS_25W[5])
    o5, p5 = oracle.run(mk(K25WA, 7, 6, 9, inp.V, inp.U, coef=[A], scalars=synth.SCALARS_25WA), 6)
    assert np.array_equal(o5, o3) and np.array_equal(p5, p3)


def test_P1f_alpha_field_hand_point():
    """V centre 1, U centre 0.5, V(axis, +-r) = r, alpha(centre) = 0.25 (dyadic), other alpha cells
    arbitrary: 1.5 + 0.25 * (w0 + 6 * sum_r r w_r), to 2 ulp."""
    V = star_grid(4, 1.0, lambda a, r: float(r), lambda a, r: float(r))
    U = V.copy()
    U[4, 4, 4] = 0.5
    A = np.full(V.shape, 7.0)
    A[4, 4, 4] = 0.25
    new, _ = oracle.run(mk(K25WA, 1, 1, 1, V, U, coef=[A], scalars=synth.SCALARS_25WA), 1)
    w0, w1, w2, w3, w4 = (Fraction(x) for x in synth.SCALARS_25WA)
    exact = Fraction(3, 2) + Fraction(1, 4) * (w0 + 6 * (1 * w1 + 2 * w2 + 3 * w3 + 4 * w4))
    assert ulps(new[4, 4, 4], float(exact)) <= 2


def test_P4_alpha_field_exact_rational():
    inp = synth.make_inputs(K25WA, 5, 4, 3, seed=8)
    T = 4
    o_new, o_old = oracle.run(inp, T)
    F = np.vectorize(Fraction, otypes=[object])
    cur, prev, A = F(inp.V), F(inp.U), F(inp.coef[0])
    w = [Fraction(x) for x in inp.scalars]
    R, sh = 4, inp.V.shape
    for _ in range(T):
        nxt = prev.copy()
        for z, y, x in itertools.product(range(R, sh[0] - R), range(R, sh[1] - R), range(R, sh[2] - R)):
            L = w[0] * cur[z, y, x]
            for r in range(1, 5):
                L += w[r] * (cur[z, y, x - r] + cur[z, y, x + r] + cur[z, y - r, x] + cur[z, y + r, x]
                             + cur[z - r, y, x] + cur[z + r, y, x])
            nxt[z, y, x] = 2 * cur[z, y, x] - prev[z, y, x] + A[z, y, x] * L
        prev, cur = cur, nxt
    for o, e in ((o_new, cur), (o_old, prev)):
        ef = e.astype(np.float64)
        assert np.max(np.abs(o - ef)) / np.max(np.abs(ef)) <= 2 * T * 25 * U_RND * 8


def test_P9_alpha_field_locality_and_linearity():
    n = 17
    inp = synth.make_inputs(K25WA, n, n, n, seed=2)
    a, _ = oracle.run(inp, 2)
    p = (12, 12, 12)
    V = inp.V.copy(); V[p] += 1.0
    b, _ = oracle.run(mk(K25WA, n, n, n, V, inp.U, inp.coef, inp.scalars), 2)
    m = n + 8
    z, y, x = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    reach = sum(np.ceil(np.abs(c - pc) / 4) for c, pc in zip((z, y, x), p)) <= 2
    assert np.array_equal(a != b, reach)
    c2, _ = oracle.run(mk(K25WA, n, n, n, 2 * inp.V, 2 * inp.U, inp.coef, inp.scalars), 2)
    assert np.array_equal(c2, 2 * a)
