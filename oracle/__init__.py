"""TEST INFRASTRUCTURE ONLY -- the CPU oracle of PAPER.md Fig. 1 (see oracle.c's header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this module.  The product path (paper_1410_3060_b200/) never imports it and shares no code
with it; the two meet only through the seeded inputs of synth/.

Functions:
  run(inputs, T)          -- full naive sweeps (oracle.c:oracle_run) on copies of the inputs.
  run_cone(...)           -- the same naive sweeps on a sub-box around sample cells; exact for a
                             cell at L1/axis distance >= R*T from the sub-box's artificial faces
                             (each step moves information at most R cells along one axis,
                             PAPER.md Fig. 1: star stencils of radius R), so it returns the
                             oracle's value of single cells of a large grid one by one.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

import synth

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build() -> str:
    src = os.path.join(_HERE, "oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB_PATH, src])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_run.restype = ctypes.c_int
        L.oracle_run.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                 ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int]
        _lib = L
    return _lib


def run_arrays(kind, nx, ny, nz, V, U, coef, scalars, T, nthreads=0):
    """In place: V <- Omega^T, U <- Omega^{T-1}.  Arrays are C-contiguous float64 padded grids."""
    R = synth.RADIUS[kind]
    shape = (nz + 2 * R, ny + 2 * R, nx + 2 * R)
    for a in [V, U, *coef]:
        if a.shape != shape or a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ValueError(f"array shape {a.shape} dtype {a.dtype}; want {shape} float64 C-contiguous")
    cptr = (ctypes.c_void_p * max(1, len(coef)))(*[a.ctypes.data for a in coef])
    sc = np.ascontiguousarray(np.array(scalars, dtype=np.float64))
    rc = lib().oracle_run(kind, nx, ny, nz, V.ctypes.data, U.ctypes.data,
                          ctypes.cast(cptr, ctypes.c_void_p) if coef else None, len(coef),
                          sc.ctypes.data if len(scalars) else None, len(scalars), T, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_run failed rc={rc}")
    return V, U


def run(inp: "synth.Inputs", T: int, nthreads: int = 0):
    """Return (V, U) = (Omega^T, Omega^{T-1}) over the padded grid, inputs untouched."""
    V, U = inp.V.copy(), inp.U.copy()
    run_arrays(inp.kind, inp.nx, inp.ny, inp.nz, V, U, inp.coef, inp.scalars, T, nthreads)
    return V, U


def run_cone(kind, nx, ny, nz, cells, T, seed=synth.DEFAULT_SEED, nthreads=0, scalars=None):
    """Oracle values (Omega^T, Omega^{T-1}) at padded-grid `cells` [(z,y,x), ...] of a large grid.

    Each cell is computed on its own sub-box: the box extends R*T + R cells around the cell along
    every axis, clipped to the global padded grid.  Cells of the sub-box's outermost R layer are
    held fixed as ghosts; where that layer is inside the global interior the values there are
    wrong after step 1, but the error travels at most R cells per step, so the cell (>= R*T + R
    away) is exact.  Inputs come from synth.make_inputs(box=...) -- bitwise the global draws.
    """
    R = synth.RADIUS[kind]
    dims = synth.padded_dims(kind, nx, ny, nz)
    out_new, out_old = [], []
    m = R * T + R
    for (z, y, x) in cells:
        box = tuple((max(0, c - m), min(d, c + m + 1)) for c, d in zip((z, y, x), dims))
        inp = synth.make_inputs(kind, nx, ny, nz, seed=seed, box=box, scalars=scalars)
        bz, by, bx = (b[1] - b[0] - 2 * R for b in box)
        if min(bz, by, bx) < 1:
            raise ValueError("cell box has no interior")
        V, U = inp.V, inp.U
        run_arrays(kind, bx, by, bz, V, U, inp.coef, inp.scalars, T, nthreads)
        lz, ly, lx = z - box[0][0], y - box[1][0], x - box[2][0]
        out_new.append(V[lz, ly, lx])
        out_old.append(U[lz, ly, lx])
    return np.array(out_new), np.array(out_old)
