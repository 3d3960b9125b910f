"""The performance model of the hot path (§3.3): code balance
(compulsory memory bytes per lattice update) and the roofline min(bandwidth / code balance, FP64 peak /
flops per update).  Host logic only; bench.py and tools/report.py take their rooflines from here, and
tests/test_model.py pins it to the numbers the paper prints.

Kinds: 1 = 7-point constant (Fig. 1b), 2 = 7-point variable (Fig. 1c), 3 = 25-point wave with a scalar
alpha (Fig. 1e, BASELINE.json config 3), 4 = 25-point variable (Fig. 1d), 5 = the wave with the
domain-sized alpha field as printed.
"""
K7C, K7V, K25W, K25V, K25WA = 1, 2, 3, 4, 5
WAVE_KINDS = (K25W, K25WA)
COEF_FIELDS = {K7C: 0, K7V: 7, K25W: 0, K25V: 13, K25WA: 1}  # domain-sized read-only streams
FLOPS_PER_LUP = {K7C: 8, K7V: 13, K25W: 30, K25V: 37, K25WA: 30}  # FMA = 2 (SURVEY d.2)
WORD = 8  # fp64


def code_balance(kind: int, bt: int = 1, write_allocate: bool = False) -> float:
    """Compulsory bytes per lattice update of a fused block of bt levels.

    Per block every state level is read once and written once and every coefficient field read once
    (the N_D streams cross memory once per block).  Jacobi kinds: read Omega^t, write
    Omega^{t+bt}; with write-allocate (the paper's CPU without non-temporal stores) the
    written line is read first.  The wave: at bt = 1 Omega^{t+1} overwrites Omega^{t-1} in
    place (read both levels, write one; no write-allocate since the line was just read); at bt >= 2
    both levels are read and both written.  Divided by bt: updates per block."""
    if bt < 1:
        raise ValueError("bt >= 1")
    coef = WORD * COEF_FIELDS[kind]
    if kind in WAVE_KINDS:
        state = 3 * WORD if bt == 1 else 4 * WORD
    else:
        state = 2 * WORD + (WORD if write_allocate else 0)
    return (state + coef) / bt


def roofline_glups(kind: int, bandwidth_gbs: float, bt: int = 1, fp64_tflops: float = float("inf"),
                   write_allocate: bool = False) -> float:
    """min(bandwidth / code balance, FP64 peak / flops per update) in GLUP/s (BASELINE.json north star)."""
    mem = bandwidth_gbs / code_balance(kind, bt, write_allocate)
    return min(mem, fp64_tflops * 1e3 / FLOPS_PER_LUP[kind])
