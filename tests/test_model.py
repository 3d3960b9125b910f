"""The performance model (paper_1410_3060_b200/model.py) against the numbers PAPER.md prints (SURVEY.md §4
item 2) and the GPU code balances DESIGN.md derives."""
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
