"""The performance model (paper_1410_3060_b200/model.py) against the numbers PAPER.md prints (SURVEY.md §4
item 2) and the GPU code balances DESIGN.md derives."""
import json
import os
import re

import pytest

from paper_1410_3060_b200 import model as m


def test_paper_cpu_code_balances():
    # P:338 (7-point constant, with write-allocate), P:344-345 (16 with non-temporal stores),
    # P:456 (7-point variable: 80), P:458 (25-point variable: 128), P:1140 (120 without write-allocate),
    # P:418 (25-point "constant" wave with the domain-sized alpha of Fig. 1e: 32)
    assert m.code_balance(m.K7C, write_allocate=True) == 24
    assert m.code_balance(m.K7C) == 16
    assert m.code_balance(m.K7V, write_allocate=True) == 80
    assert m.code_balance(m.K25V, write_allocate=True) == 128
    assert m.code_balance(m.K25V) == 120
    assert m.code_balance(m.K25WA) == 32


def test_paper_rooflines_at_40_gbs():
    # 1.67 and 1.25 GLUP/s at the measured 40 GB/s
    assert m.roofline_glups(m.K7C, 40.0, write_allocate=True) == pytest.approx(1.67, abs=0.005)
    assert m.roofline_glups(m.K25WA, 40.0) == pytest.approx(1.25, abs=0.005)


def test_gpu_code_balances_and_temporal_blocking():
    # DESIGN.md §5 table (no write-allocate): 16 / 72 / 24 (32 at bt >= 2) / 120 per block
    assert [m.code_balance(k) for k in (m.K7C, m.K7V, m.K25W, m.K25V)] == [16, 72, 24, 120]
    assert m.code_balance(m.K25W, 2) == 16 and m.code_balance(m.K25W, 4) == 8
    assert m.code_balance(m.K7V, 3) == 24  # the C2 default plan
    assert m.roofline_glups(m.K7V, 6536.7, 3) == pytest.approx(272.36, abs=0.01)
    assert m.roofline_glups(m.K25V, 6536.7) == pytest.approx(54.47, abs=0.01)


def test_fp64_bound_takes_over():
    # the FP64 bound caps the roofline once bt is large enough (SURVEY d.2: crossover bt* for C3 = 6)
    assert m.roofline_glups(m.K25W, 6546.9, 8, fp64_tflops=37.0) == pytest.approx(37.0e3 / 30)
    assert m.roofline_glups(m.K25W, 6546.9, 2, fp64_tflops=37.0) < 37.0e3 / 30
    with pytest.raises(ValueError):
        m.code_balance(m.K7C, 0)


# ------------------------------------------------------------------ footprint model

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = {"K7C": m.K7C, "K7V": m.K7V, "K25W": m.K25W, "K25V": m.K25V, "K25WA": m.K25WA}


def _plans():
    src = open(os.path.join(ROOT, "paper_1410_3060_b200", "csrc", "pipe.cu")).read()
    body = src[src.index("cudaError_t launch_pipe("):]
    plans = []
    for mac, kind, args in re.findall(r"\b(CFG[UC]?)\((K\w+),\s*([-\d,\s]+)\);", body):
        bt, TX, TY, CX, CY, DV, DC, WIN, MINB = (int(x) for x in args.split(","))
        plans.append(dict(kind=KINDS[kind], bt=bt, TX=TX, TY=TY, CX=CX, CY=CY, DV=DV, DC=DC, WIN=WIN,
                          CLU=2 if mac == "CFGC" else 1))
    return plans


def _plans25():
    src = open(os.path.join(ROOT, "paper_1410_3060_b200", "csrc", "pipe25.cu")).read()
    body = src[src.index("cudaError_t launch_pipe25v2("):src.index("cudaError_t launch_pipe25w2(")]
    return [tuple(int(x) for x in a.split(",")) for a in re.findall(r"run_pipe25<K25V,\s*([\d,\s]+)>", body)]


def test_every_configured_plan_fits_on_chip():
    plans = _plans()
    assert len(plans) >= 40  # the whole table was parsed
    for p in plans:
        f = m.pipe_footprint(p["kind"], p["bt"], p["TX"], p["TY"], p["CX"], p["CY"], p["DV"], p["DC"], p["WIN"],
                             p["CLU"])
        assert f["fits"], (p, f)
        if p["WIN"] < 0:  # TMEM-window plans also keep a second CTA off the SM (pipe.cu static_assert)
            assert f["smem"] > 116 * 1024 and f["tmem_cols"] <= 512, (p, f)
    p25 = _plans25()
    assert len(p25) == 4
    for TX, TY, D, CLU, SKEW in p25:
        f = m.pipe25_footprint(TX, TY, D, CLU, SKEW)
        assert f["fits"] and f["out_tile"][0] == TX - 8, f
        assert f["out_tile"][1] == (TY if SKEW else CLU * TY - 8), f


def test_footprint_rules_out_what_the_design_says():
    # DESIGN.md §5/§8: in the generic pipe kernel a 25-point variable bt = 2 plan needs (R + 2) coefficient
    # slots of 13 fields over the level-1 extent -- over the shared memory for any tile with an output
    f = m.pipe_footprint(m.K25V, 2, 32, 24, 2, 2, 6, 6, 0)
    assert not f["fits"] and f["ring_bytes"]["coef"] > 320 * 1024
    # ... while the two-level kernel that carries the z chains in TMEM needs one slot per step
    assert m.pipe25_footprint(32, 24, 2, 1)["fits"]
    # a 7v bt = 4 TMEM window of 3 warps per lane quadrant would need 576 of the 512 columns
    f = m.pipe_footprint(m.K7V, 4, 32, 36, 2, 2, 4, 2, -1)
    assert f["tmem_cols"] > 512 and not f["fits"]


def test_level_work_matches_the_trapezoid():
    # C2 default bt = 3: level-1 extent 32 x 28, output 28 x 24 -> (32*28 + 30*26 + 28*24) / (3 * 28 * 24)
    f = m.pipe_footprint(m.K7V, 3, 32, 28, 2, 2, 4, 3, -1)
    assert f["out_tile"] == (28, 24)
    assert f["level_work"] == pytest.approx((32 * 28 + 30 * 26 + 28 * 24) / (3 * 28 * 24))
    # the cluster pair shares the y halo: less redundant work than two single tiles
    assert m.pipe25_footprint(32, 20, 2, 2)["level_work"] < m.pipe25_footprint(32, 24, 2, 1)["level_work"]
    # the 25v bt = 2 single tile 32 x 24 -> 24 x 16: (768 + 384) / (2 * 384) = 1.5
    assert m.pipe25_footprint(32, 24, 2, 1)["level_work"] == pytest.approx(1.5)


def test_l2_retention():
    # C4 at bt = 2 with 24 x 16 output tiles: 148 CTAs stream 148 * 384 cells * 120 B of fresh DRAM bytes
    # per z-step, so the 126 MiB L2 holds ~19 steps of them
    assert m.l2_retention_steps((24, 16), 2, m.K25V) == pytest.approx(126 * 2 ** 20 / (148 * 384 * 120))
    assert m.l2_retention_steps((24, 32), 2, m.K25V) == pytest.approx(m.l2_retention_steps((24, 16), 2, m.K25V) / 2)


def test_lockstep_dram_model_single_round_is_compulsory_plus_ghosts():
    # one round covering every tile, byte granules: each padded cell of every field crosses DRAM once
    n, R = 64, 4
    X = n + 2 * R
    got = m.lockstep_dram_bytes_per_lup(m.K25V, 2, (n, n, n), (24, 16), conc=10 ** 6, granule=8)
    want = ((n + 2 * R) / n * (8 * 13 * X * X + 8 * X * X) + 8 * n * n) / (2 * n * n)
    assert abs(got - want) < 1e-9
    # rounds of fewer tiles re-read the halos at their patch boundaries; coarser granules add partial lines
    small = m.lockstep_dram_bytes_per_lup(m.K25V, 2, (n, n, n), (24, 16), conc=4, granule=8)
    assert small > got
    assert m.lockstep_dram_bytes_per_lup(m.K25V, 2, (n, n, n), (24, 16), conc=4, granule=128) > small


def test_lockstep_dram_model_reproduces_ncu():
    # the model with 148 concurrent tiles and 128-byte lines against ncu's DRAM bytes per update of the
    # default plans (profiles/traffic.json, one launch each): the two-level 25v kernel to 0.5 %, the generic
    # pipe kernel (C2 bt = 4, C3 bt = 1) to 3 %
    t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    cases = [("C4-25pt-var-512/bt2", m.K25V, 2, 512, (24, 16), 0.005),
             ("C5-25pt-var-1024/bt2", m.K25V, 2, 1024, (24, 16), 0.005),
             ("C2-7pt-var-512/bt4", m.K7V, 4, 512, (26, 22), 0.03),
             ("C3-25pt-wave-512/bt1", m.K25W, 1, 512, (64, 14), 0.03)]
    for key, kind, bt, n, tile, tol in cases:
        e = t[key]
        meas = e["dram_bytes_per_lup"] if isinstance(e, dict) else e / (n ** 3 * bt)
        mod = m.lockstep_dram_bytes_per_lup(kind, bt, (n, n, n), tile)
        assert abs(mod - meas) / meas < tol, (key, mod, meas)
        assert mod > m.code_balance(kind, bt)


def test_footprint_rules_for_deeper_7v_blocks():
    # PipeCfg's static_asserts as model rules: a 5-level TMEM window of 2x2-cell warps needs 640 columns;
    # a shared-memory coefficient ring keeps each plane (bt - 1 - WIN) * R steps and needs that + 2 slots;
    # a register window is capped at 32 doubles per thread
    f = m.pipe_footprint(m.K7V, 5, 32, 28, 2, 2, 4, 2, -1)
    assert f["tmem_cols"] == 640 and not f["fits"]
    assert not m.pipe_footprint(m.K7V, 5, 32, 20, 2, 2, 4, 2, 0)["valid"]   # CLAG 4 needs DC >= 6
    assert m.pipe_footprint(m.K7V, 5, 32, 20, 2, 2, 4, 6, 0)["valid"]
    assert not m.pipe_footprint(m.K7V, 5, 32, 20, 2, 2, 4, 4, 2)["valid"]   # 2 planes x 7 x 4 cells = 56
    # the b_t = 5 plan pipe.cu instantiates: 2x1 cells, 3 warps per lane quadrant, 480 columns
    f = m.pipe_footprint(m.K7V, 5, 32, 24, 2, 1, 4, 2, -1)
    assert f["fits"] and f["tmem_cols"] == 480 and f["out_tile"] == (24, 16)
