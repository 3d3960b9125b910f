"""Randomised plan fuzzing on the GPU: random kind, extents, T and plan (variant, bt, tile_cfg, z-chunk,
z-slabs with copy / peer halos), each compared bitwise with the naive sweeps (G4).  Prints one line per
mismatch and a summary; exit code 1 if any plan disagrees.

python tools/fuzz.py [--minutes 5] [--seed 1]
"""
import argparse
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
import synth  # noqa: E402

N_CFG = {synth.K7C: 1, synth.K7V: 10, synth.K25W: 9, synth.K25V: 4, synth.K25WA: 5}
MAX_BT = {synth.K7C: 8, synth.K7V: 5, synth.K25W: 2, synth.K25V: 2, synth.K25WA: 1}


def run(kind, n, T, seed, **kw):
    with st.Grid(kind, *n, seed=seed, **kw) as g:
        for t in (T if isinstance(T, tuple) else (T,)):  # consecutive stencil_run calls
            g.run(t)
        new = g.read(0)
        old = g.read(1) if kind in synth.WAVE_KINDS else None
    return new, old


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=5.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-extent", type=int, default=0, help="largest extent per axis (0: 90, a fifth up to 300)")
    ap.add_argument("--max-cells", type=float, default=3e7, help="skip shapes with more interior cells")
    a = ap.parse_args()
    return fuzz(a.minutes, a.seed, max_extent=a.max_extent or None, max_cells=a.max_cells)[1]


def fuzz(minutes, seed0, against=None, max_extent=None, max_cells=3e7):
    """Run random plans for `minutes`; compare each with the naive sweeps, or -- when `against` is given
    (tests/test_gpu_fuzz.py passes the CPU oracle's checker; tools never import the oracle) -- with
    against(kind, n, T, seed, got).  Returns (cases, mismatches)."""
    from types import SimpleNamespace
    a = SimpleNamespace(minutes=minutes, seed=seed0, oracle=against is not None)
    torch.cuda.set_device(0)
    rnd = random.Random(a.seed)
    t_end = time.time() + 60 * a.minutes
    cases = bad = 0
    while time.time() < t_end:
        kind = rnd.choice(list(N_CFG))
        R = synth.RADIUS[kind]
        big = rnd.random() < 0.2 and not a.oracle
        n = tuple(rnd.randint(1, max_extent or (40 if a.oracle else (300 if big else 90))) for _ in range(3))
        if n[0] * n[1] * n[2] > max_cells:
            continue
        T = rnd.randint(1, 13)
        if rnd.random() < 0.3:  # the same steps split over 2-3 runs (state and remainder blocks carry over)
            cuts = sorted(rnd.sample(range(1, T), min(T - 1, rnd.randint(1, 2)))) if T > 1 else []
            T = tuple(b - a for a, b in zip([0] + cuts, cuts + [T]))
        seed = rnd.randint(1, 10**6)
        v = rnd.choice(["pipe", "pipe", "pipe", "stream", "coop", "slabs"])
        kw = {}
        if v == "pipe":
            kw = dict(variant=st.ST_VARIANT_PIPE, bt=rnd.randint(1, MAX_BT[kind]), tile_cfg=rnd.randrange(N_CFG[kind]),
                      zchunk=rnd.choice([0, 0, rnd.randint(1, 64)]))
        elif v == "stream":
            kw = dict(variant=st.ST_VARIANT_STREAM, bt=rnd.randint(1, 2), zchunk=rnd.choice([0, rnd.randint(1, 64)]))
        elif v == "coop":
            kw = dict(variant=st.ST_VARIANT_COOP, tile_cfg=2 if kind in (synth.K7C, synth.K7V) and rnd.random() < 0.3 else 0)
        else:
            P = rnd.randint(2, 5)
            if n[2] < P * R:
                continue
            kw = dict(nranks=P, local_slabs=P, halo=rnd.choice([st.ST_HALO_COPY, st.ST_HALO_PEER]),
                      bt=rnd.randint(1, MAX_BT[kind]))
        try:
            got = run(kind, n, T, seed, **kw)
        except st.StencilError as e:  # plans the library rejects (e.g. slabs thinner than R) are fine
            print(f"rejected {synth.KIND_NAMES[kind]} {n} T={T} {kw}: {str(e)[:90]}", flush=True)
            continue
        Tt = sum(T) if isinstance(T, tuple) else T
        cases += 1
        if a.oracle:
            ok = against(kind, n, Tt, seed, got)
        else:
            ref = run(kind, n, Tt, seed, variant=st.ST_VARIANT_NAIVE)
            ok = np.array_equal(got[0], ref[0]) and (got[1] is None or np.array_equal(got[1], ref[1]))
        if not ok:
            bad += 1
            print(f"MISMATCH {synth.KIND_NAMES[kind]} {n} T={T} seed={seed} {kw}", flush=True)
        torch.cuda.empty_cache()
    print(f"fuzz done: {cases} plans, {bad} mismatches", flush=True)
    return cases, bad


if __name__ == "__main__":
    sys.exit(1 if main() else 0)
