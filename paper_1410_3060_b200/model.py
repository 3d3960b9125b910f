"""The performance model of the hot path (§3.3): code balance
(compulsory memory bytes per lattice update) and the roofline min(bandwidth / code balance, FP64 peak /
flops per update).  Host logic only; bench.py and tools/report.py take their rooflines from here, and
tests/test_model.py pins it to the numbers the paper prints.

Kinds: 1 = 7-point constant (Fig. 1b), 2 = 7-point variable (Fig. 1c), 3 = 25-point wave with a scalar
alpha (Fig. 1e, BASELINE.json config 3), 4 = 25-point variable (Fig. 1d), 5 = the wave with the
domain-sized alpha field as printed.
"""
import math
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


# ---------------------------------------------------------------------------------------------------------
# On-chip footprint of one CTA's z-stream: the GPU counterpart of the paper's wavefront
# cache-block size, Eq. 4.1 / 4.2.  The paper's cache block of a thread group is
#     N_xb * [N_D * D_w * (D_w/2 - R + N_F + 1) + 2R (D_w + W_w)]
# bytes: the domain-sized streams (N_D) over the diamond area plus the wavefront's state rows.  On B200 a
# CTA plays the thread group: its "cache block" is what its rings keep on chip -- the state planes
# (the Omega^t footprint of the level-1 extent grown by R) and the N_D coefficient fields over the
# level-1 extent, each times its ring depth -- held in shared memory (227 KB per CTA), tensor memory
# (512 columns x 128 lanes x 4 B) and registers.  These functions mirror the kernels' layouts exactly
# (pipe.cu PipeCfg, pipe25.cu P25Cfg); tests/test_model.py pins them to the configuration tables in the
# sources, and the GPU tests to the shared memory the launches really request.
SMEM_LIMIT = 227 * 1024   # opt-in dynamic shared memory per CTA (sm_100a)
TMEM_COLUMNS = 512        # 32-bit columns per lane, 128 lanes
RADIUS = {K7C: 1, K7V: 1, K25W: 4, K25V: 4, K25WA: 4}


def _ceil16(n):
    return (n + 15) // 16 * 16


def pipe_footprint(kind, bt, TX, TY, CX, CY, DV, DC, WIN, CLU=1):
    """Footprint of pipe.cu's pipe_kernel<kind, bt, TX, TY, CX, CY, DV, DC, WIN, MINB, UNR, CLU>: shared
    memory bytes (the kernel's PipeCfg::SMEM), TMEM columns, threads, output tile, and the level work per
    output update (overlapped-tile redundancy, sum over levels of the level-k extent / (bt * output))."""
    R, NC, wave = RADIUS[kind], COEF_FIELDS[kind], kind in WAVE_KINDS
    NS, LPR = TY // CY, TX // CX
    NCONS = LPR * NS
    FX, FY = TX + 2 * R, TY + 2 * R
    OX = TX - 2 * R * (bt - 1)
    OYP = CLU * TY - 2 * R * (bt - 1)
    SHV = R & 1
    FXB = (FX + SHV + 1) // 2 * 2
    EXB = TX + (2 if R == 1 else 0)
    VELEMS, CFIELD = FXB * FY, EXB * TY
    FOFF = 1 if wave else 0
    NCF = FOFF + NC
    CF0 = _ceil16(CFIELD) if FOFF else 0
    CELEMS = CF0 + CFIELD * NC
    VSLOT, CSLOT = _ceil16(VELEMS), _ceil16(CELEMS)
    NPL = bt - 1
    XROW = TX * R
    doubles = DV * VSLOT + (DC * CSLOT if NCF > 0 else 0) + NPL * 2 * TX * TY + (NPL * 8 * XROW if CLU == 2 else 0)
    smem = 8 * doubles + 8 * (2 * (DV + DC) + 8 + (12 if CLU == 2 else 0)) + (8 if CLU == 2 else 4) * 4 + 128
    tmem = 0
    if WIN < 0:  # TMEM coefficient window: NSL slots of CY * 32 columns per warp, WPQ warps per quadrant
        NSL = (bt - 1) * R + 1
        WPQ = (NCONS // 32 + 3) // 4
        tmem = WPQ * NSL * CY * 32
    # the ring-depth and window rules of PipeCfg's static_asserts: the V ring holds the R + 2 planes a
    # step reads, the coefficient ring keeps a plane CLAG = (bt - 1 - WIN) * R steps after level 1 (0 for
    # the wave and the TMEM window), a TMEM window slot holds a cell row's NC * CX coefficients
    TW = WIN < 0
    CLAG = 0 if (wave or TW) else (bt - 1 - WIN) * R
    # a register window (WIN = k > 0) keeps k*R coefficient planes of the thread's cells in registers:
    # at most 32 doubles (64 of the 255 registers; the configured windows use 28)
    REGWIN = max(WIN, 0) * R * NC * CX * CY
    valid = (DV >= R + 2 and (NCF == 0 or DC >= CLAG + 2) and -1 <= WIN <= bt - 1 and (WIN == 0 or NC > 0)
             and (not TW or (not wave and bt >= 2 and 2 * NC * CX <= 32)) and REGWIN <= 32 and OX > 0 and OYP > 0)
    # level-k extent (TX - 2R(k-1)) x (CLU*TY - 2R(k-1)): a cluster pair shrinks only at its outer rows
    work = sum((TX - 2 * R * (k - 1)) * (CLU * TY - 2 * R * (k - 1)) for k in range(1, bt + 1))
    return {"smem": smem, "tmem_cols": tmem, "threads": NCONS + 32, "out_tile": (OX, OYP),
            "level_work": work / (bt * OX * OYP), "level1_ratio": TX * CLU * TY / (OX * OYP),
            "fits": valid and smem <= SMEM_LIMIT and tmem <= TMEM_COLUMNS, "valid": valid,
            "ring_bytes": {"state": 8 * DV * VSLOT, "coef": 8 * DC * CSLOT if NCF > 0 else 0,
                           "level_planes": 8 * NPL * 2 * TX * TY}}


def pipe25_footprint(TX, TY, D, CLU, SKEW=0):
    """Footprint of pipe25.cu's two-level 25-point kernel pipe25_kernel<K25V, TX, TY, D, CLU, SKEW> (P25Cfg).
    SKEW: parallelogram tiles in y -- level 2 runs R rows below level 1, box C reaches R
    rows lower, box I brings 2R level-1 rows from the tile underneath; output rows = TY."""
    R, NC = 4, 13
    NCONS = (TX // 2) * (TY // 2)
    CR, IEL = (R, 2 * R * TX) if SKEW else (0, 0)
    AEL, BEL = TX * TY, (TX + 2 * R) * (TY + 2 * R)
    SLOT = _ceil16(AEL) + _ceil16(BEL) + _ceil16(NC * TX * (TY + CR)) + _ceil16(IEL)
    NRX = 4 if CLU > 1 else 0
    STASH = 2 * 32 * 4 * 5 if CLU > 1 else 0
    NPB = 2 if SKEW else 3
    smem = 8 * (D * SLOT + NPB * TX * TY + 2 * NRX * R * TX + STASH) + 8 * (2 * D + 8 + 2 * NRX + 8) + 4 * 8 + 128
    OX, OYP = TX - 2 * R, (TY if SKEW else CLU * TY - 2 * R)
    work = (TX * CLU * TY + OX * OYP) / (2 * OX * OYP)  # level 1 over every CTA's rows, level 2 = output
    return {"smem": smem, "tmem_cols": 512, "threads": NCONS + 32, "out_tile": (OX, OYP), "level_work": work,
            "level1_ratio": TX * CLU * TY / (OX * OYP),
            "fits": smem <= SMEM_LIMIT, "coef_box_bytes_per_output": 8 * NC * TX * (TY + CR) * CLU / (OX * OYP),
            "ring_bytes": {"slot": 8 * SLOT, "slots": D}}


def l2_retention_steps(out_tile, bt, kind, ctas=148, l2_bytes=126 * 2 ** 20):
    """z-steps for which the L2 holds what all CTAs streamed from DRAM: the drift two neighbouring tiles'
    z-streams may have and still find each other's overlapping boxes in L2 (the coefficient and state
    halos overlapped tiles share).  Fresh DRAM bytes per CTA and step = one plane of its output tile at the
    block's compulsory bytes per cell."""
    per_step = ctas * out_tile[0] * out_tile[1] * code_balance(kind, bt) * bt
    return l2_bytes / per_step


def lockstep_tile_blocks(ntx, out_tile, conc=148):
    """(tblk_w, tblk_h) of the lockstep tile order the launchers pick (pipe.cu / pipe25.cu: blocks of about
    sqrt(conc * OY / OX) tile columns, sized so that a tile row splits into equal blocks)."""
    OX, OY = out_tile
    target = math.sqrt(conc * OY / OX)
    nb = max(1, int(ntx / target + 0.5))
    bw = max(1, min((ntx + nb - 1) // nb, ntx))
    return bw, max(1, (conc + bw - 1) // bw)


def lockstep_dram_bytes_per_lup(kind, bt, shape, out_tile, conc=148, granule=128):
    """DRAM bytes per lattice update of one lockstep launch of bt fused levels over a grid of `shape`
     if the L2 keeps everything a round streams and nothing across rounds.  Per round (conc
    consecutive tiles of the blocked order, `sm100.cuh` decode, blocks from lockstep_tile_blocks): the union
    of the coefficient boxes (the level-1 extent, i.e. the output tile grown by R per fused level beyond
    the first; NC fields, the wave's Omega^{t-1} as one) and of the state boxes (the level-0 footprint, R
    wider again) over the padded plane, taken in aligned `granule`-byte pieces of each row (the DRAM fetch
    granularity; interior column x = R starts a 128-byte line, `runtime.cu`); every tile streams the
    nz + 2R planes of the padded z extent; plus one write per cell (two for the wave at bt >= 2).  The
    excess over code_balance is the re-read of halos across round-patch boundaries, the ghost cells and
    the partial lines at patch and grid edges; what ncu measures beyond it is lost inside a round."""
    import numpy as np
    R, NC = RADIUS[kind], COEF_FIELDS[kind] + (1 if kind in WAVE_KINDS else 0)
    nx, ny, nz = shape
    OX, OY = out_tile
    ntx, nty = -(-nx // OX), -(-ny // OY)
    bw, bh = lockstep_tile_blocks(ntx, out_tile, conc)
    H = R * (bt - 1)  # the level-1 extent reaches H beyond the output tile, the footprint H + R
    ext_tile, foot_tile = (OX + 2 * H, OY + 2 * H), (OX + 2 * H + 2 * R, OY + 2 * H + 2 * R)
    X, Y = nx + 2 * R, ny + 2 * R
    g = max(1, granule // 8)  # doubles per granule
    xoff = 16 - R               # raw column of padded column 0
    XR = (xoff + X + g - 1) // g * g

    def span(lo, hi):  # raw columns of the granules covering padded columns [lo, hi)
        lo, hi = max(lo, 0), min(hi, X)
        return (xoff + lo) // g * g, -(-(xoff + hi) // g) * g

    ext, foot = 0, 0
    items = ntx * nty
    for r0 in range(0, items, conc):
        mc = np.zeros((Y, XR), bool)
        mv = np.zeros((Y, XR), bool)
        for t in range(r0, min(items, r0 + conc)):
            by, rem = divmod(t, ntx * bh)
            h = min(bh, nty - by * bh)
            bx, rem2 = divmod(rem, bw * h)
            w = min(bw, ntx - bx * bw)
            tx, ty = bx * bw + rem2 % w, by * bh + rem2 // w
            x0, y0 = R + tx * OX - H, R + ty * OY - H
            a, b = span(x0, x0 + ext_tile[0])
            mc[max(y0, 0):y0 + ext_tile[1], a:b] = True
            fx, fy = x0 - (foot_tile[0] - ext_tile[0]) // 2, y0 - (foot_tile[1] - ext_tile[1]) // 2
            a, b = span(fx, fx + foot_tile[0])
            mv[max(fy, 0):fy + foot_tile[1], a:b] = True
        ext += int(mc.sum())
        foot += int((mv | mc).sum())
    cells = nx * ny
    zpad = (nz + 2 * R) / nz
    return (zpad * (8 * NC * ext + 8 * foot) + 8 * cells * (2 if kind in WAVE_KINDS and bt >= 2 else 1)) / (bt * cells)


# ---------------------------------------------------------------------------------------------------------
# The plan tables of the kernels (parsed from the sources, so the model and the tuner can never drift from
# what launch_pipe / launch_pipe25v2 really instantiate) and a modeled cost per lattice update used to
# prune the tuner's candidates (tools/tune.py).
_CSRC = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)), "csrc")
_KINDS = {"K7C": K7C, "K7V": K7V, "K25W": K25W, "K25V": K25V, "K25WA": K25WA}


def pipe_plans():
    """[(kind, bt, tile_cfg, footprint args)] of pipe.cu's launch_pipe table, tile_cfg numbered as the
    launcher does (explicit `cfg == k` entries, the last entry of each (kind, bt) is cfg 0)."""
    import re
    src = open(__import__("os").path.join(_CSRC, "pipe.cu")).read()
    body = src[src.index("cudaError_t launch_pipe("):src.index("#undef CFG")]
    out = []
    for line in body.splitlines():
        m = re.search(r"(?:if \(cfg == (\d+)\) )?(CFG[UC]?)\((K\w+),\s*([-\d,\s]+)\);", line)
        if not m:
            continue
        cfg = int(m.group(1)) if m.group(1) else 0
        bt, TX, TY, CX, CY, DV, DC, WIN, _minb = (int(x) for x in m.group(4).split(","))
        out.append((_KINDS[m.group(3)], bt, cfg, dict(TX=TX, TY=TY, CX=CX, CY=CY, DV=DV, DC=DC, WIN=WIN,
                                                       CLU=2 if m.group(2) == "CFGC" else 1)))
    return out


def pipe25_plans():
    """[(tile_cfg, TX, TY, D, CLU, SKEW)] of pipe25.cu's launch_pipe25v2 table (the default entry is cfg 0)."""
    import re
    src = open(__import__("os").path.join(_CSRC, "pipe25.cu")).read()
    body = src[src.index("cudaError_t launch_pipe25v2("):]
    out = []
    for m in re.finditer(r"(case (\d+)|default): return run_pipe25<K25V,\s*([\d,\s]+)>", body[:body.index("cudaError_t launch_pipe25w2(")]):
        cfg = int(m.group(2)) if m.group(2) else 0
        out.append((cfg,) + tuple(int(x) for x in m.group(3).split(",")))
    return out


def modeled_nj_per_lup(kind, bt, footprint, pj_dram=91.0, pj_l2=23.0, pj_smem=5.9, nj_level=0.6):
    """Modeled dynamic energy per lattice update of a plan (the board's 1 kW cap makes energy per update
    the rate limit): compulsory DRAM bytes, L2->SM bytes of the overlapped boxes (each
    level-1 cell's coefficients and state cross L2 once per block), shared-memory write + read of those
    bytes, and per-level SM work (redundant trapezoid cells included).  Constants: the round-1 energy probe
    (profiles/r01_energy_probe.json); nj_level fitted to the C2/C4 power measurements.  A ranking tool,
    not a prediction to the percent."""
    R, NC = RADIUS[kind], COEF_FIELDS[kind]
    W = footprint["level_work"]  # level-k cells per output update, averaged over the bt levels
    # each level-1 cell brings its coefficients and state on chip once per block
    per_cell = 8 * (NC + (1 if kind in WAVE_KINDS else 0) + 1)
    l2_bytes = per_cell * footprint["level1_ratio"] / bt
    dram = code_balance(kind, bt)
    return (pj_dram * dram + pj_l2 * l2_bytes + 2 * pj_smem * l2_bytes) / 1e3 + nj_level * W
