"""Seeded synthetic inputs shared by the oracle harness and the CUDA path (input synthesis only).

Holds none of the stencil method's arithmetic: it draws the numbers (synth.h, reading Q6 in
DESIGN.md), composes the initial state (readings Q1, Q8, Q9) and names the BASELINE.json workloads.
Both sides of a parity test take their inputs from here; the CUDA library fills on the device
with the same header (synth/synth.h), and a test checks the two fills agree bitwise.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")

# Stencil kinds (SURVEY.md §8(b) numbering; Fig. 1b/1c/1e/1d).
K7C, K7V, K25W, K25V, K25WA = 1, 2, 3, 4, 5
KIND_NAMES = {K7C: "7pt-const", K7V: "7pt-var", K25W: "25pt-wave", K25V: "25pt-var",
              K25WA: "25pt-wave-alpha-field"}
RADIUS = {K7C: 1, K7V: 1, K25W: 4, K25V: 4, K25WA: 4}
N_COEF_FIELDS = {K7C: 0, K7V: 7, K25W: 0, K25V: 13, K25WA: 1}
N_SCALARS = {K7C: 2, K7V: 0, K25W: 6, K25V: 0, K25WA: 5}
WAVE_KINDS = (K25W, K25WA)
# U[0, c) scale of the coefficient fields (BASELINE.json configs 2, 4, 5).  The alpha field of the
# NEXT-1 wave (Fig. 1e as printed, not a BASELINE.json config) is drawn from U[0, 0.2): the leapfrog
# update is stable for alpha * max|Laplacian symbol| = alpha * 19.505 < 4, i.e. alpha < 0.205.
COEF_SCALE = {K7V: 1.0 / 7.0, K25V: 1.0 / 25.0, K25WA: 0.2}

# Scalar weights of the constant kinds (BASELINE.json configs 1 and 3; reading Q3).
SCALARS_7C = (0.4, 0.1)  # w_c (centre), w_n (each neighbour)
SCALARS_25W = (3.0 * (-205.0 / 72.0), 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0, 0.1)  # w0,a1..a4,alpha
SCALARS_25WA = SCALARS_25W[:5]  # w0, w1..w4 (alpha is a field)

DEFAULT_SEED = 14103060  # reading Q7

STREAM_V, STREAM_U = 0, 1


def stream_w(i: int) -> int:
    return 2 + i


def _build() -> None:
    src = os.path.join(_HERE, "synth.c")
    subprocess.check_call(
        ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _LIB_PATH, src]
    )


_lib_handle = None


def lib():
    global _lib_handle
    if _lib_handle is None:
        src = os.path.join(_HERE, "synth.c")
        hdr = os.path.join(_HERE, "synth.h")
        if (not os.path.exists(_LIB_PATH)
                or os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(src), os.path.getmtime(hdr))):
            _build()
        L = ctypes.CDLL(_LIB_PATH)
        L.synth_fill_box.restype = ctypes.c_int
        L.synth_fill_box.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_double] + \
            [ctypes.c_int64] * 9 + [ctypes.c_void_p]
        _lib_handle = L
    return _lib_handle


def fill_box(seed: int, stream: int, dims, box=None, scale: float | None = None,
             out: np.ndarray | None = None) -> np.ndarray:
    """Draw stream `stream` over `box` = ((z0,z1),(y0,y1),(x0,x1)) of a global padded grid `dims`=(Z,Y,X).

    scale None -> U[-1,1); else U[0, scale).  out: a C-contiguous float64 array of the box's shape to
    fill in place (e.g. pinned host memory); default a new array.
    """
    Z, Y, X = dims
    if box is None:
        box = ((0, Z), (0, Y), (0, X))
    (z0, z1), (y0, y1), (x0, x1) = box
    shape = (z1 - z0, y1 - y0, x1 - x0)
    if out is None:
        out = np.empty(shape, dtype=np.float64)
    elif out.shape != shape or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float64 array of shape {shape}")
    rc = lib().synth_fill_box(seed, stream, 0 if scale is None else 1, 0.0 if scale is None else scale,
                              Z, Y, X, z0, z1, y0, y1, x0, x1, out.ctypes.data)
    if rc != 0:
        raise ValueError(f"bad box {box} for dims {dims}")
    return out


# ---- pure-numpy restatement of synth.h, for the cross-check test only ----
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _np_mix(z):
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def numpy_unit(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        key = _np_mix(np.array([seed ^ ((0x9E3779B97F4A7C15 * (stream + 1)) & 0xFFFFFFFFFFFFFFFF)],
                               dtype=np.uint64))[0]
        h = _np_mix(key + np.uint64(0xD1B54A32D192ED03) * (idx.astype(np.uint64) + np.uint64(1)))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


# ---- the initial state (readings Q1, Q8, Q9) ----
@dataclass
class Inputs:
    kind: int
    nx: int
    ny: int
    nz: int
    V: np.ndarray                      # Omega^0 over the padded box (ghosts included)
    U: np.ndarray                      # second buffer: copy of V, interior = Omega^{-1} for the wave
    coef: list = field(default_factory=list)   # padded-extent fields W_i (variable kinds)
    scalars: tuple = ()                # scalar weights (constant kinds)

    @property
    def R(self):
        return RADIUS[self.kind]


def padded_dims(kind: int, nx: int, ny: int, nz: int):
    R = RADIUS[kind]
    return (nz + 2 * R, ny + 2 * R, nx + 2 * R)


def make_inputs(kind: int, nx: int, ny: int, nz: int, seed: int = DEFAULT_SEED, box=None,
                scalars=None) -> Inputs:
    """Seeded inputs of one configuration over the padded box `box` (default: whole padded grid).

    V = stream 0 everywhere (Q1: ghosts ~ U[-1,1], fixed).  U = copy of V (Q8); for the wave kind
    U's *global interior* cells come from stream 1 (Q9: U holds Omega^{-1}).  W_i = stream 2+i ~ U[0,c).
    """
    R = RADIUS[kind]
    dims = padded_dims(kind, nx, ny, nz)
    if box is None:
        box = tuple((0, d) for d in dims)
    V = fill_box(seed, STREAM_V, dims, box)
    U = V.copy()
    if kind in WAVE_KINDS:
        # interior of the global grid intersected with the box
        lo = [max(b[0], R) for b in box]
        hi = [min(b[1], d - R) for b, d in zip(box, dims)]
        if all(l < h for l, h in zip(lo, hi)):
            sub = ((lo[0], hi[0]), (lo[1], hi[1]), (lo[2], hi[2]))
            U[lo[0] - box[0][0]:hi[0] - box[0][0], lo[1] - box[1][0]:hi[1] - box[1][0],
              lo[2] - box[2][0]:hi[2] - box[2][0]] = fill_box(seed, STREAM_U, dims, sub)
    coef = []
    if N_COEF_FIELDS[kind]:
        c = COEF_SCALE[kind]
        coef = [fill_box(seed, stream_w(i), dims, box, scale=c) for i in range(N_COEF_FIELDS[kind])]
    if scalars is None:
        scalars = {K7C: SCALARS_7C, K25W: SCALARS_25W, K25WA: SCALARS_25WA}.get(kind, ())
    return Inputs(kind, nx, ny, nz, V, U, coef, tuple(scalars))
