"""The C ABI used from plain C: examples/stencil_c_api.c compiles against include/stencil.h and links
libstencil.so; without a GPU it exercises the host-only plan and error paths and reports ST_E_CUDA;
with a GPU it runs a grid and its checksum equals the Python binding's."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build():
    exe = os.path.join(ROOT, "build", "stencil_c_api")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    lib = os.path.join(ROOT, "paper_1410_3060_b200")
    subprocess.check_call(["cc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "stencil_c_api.c"), "-L", lib, "-lstencil",
                           f"-Wl,-rpath,{lib}", "-o", exe])
    return exe


def test_c_example_builds_and_runs():
    out = subprocess.run([build(), "20", "18", "16", "5"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "slab 3: owns planes [13,18)" in out.stdout
    assert "ST_E_INVAL" in out.stdout
    assert "checksum" in out.stdout or "no CUDA device" in out.stdout


@pytest.mark.gpu
def test_c_example_matches_binding():
    import paper_1410_3060_b200 as st
    out = subprocess.run([build(), "33", "21", "17", "7"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = [l for l in out.stdout.splitlines() if "checksum" in l][0]
    c_sum = float(line.split("checksum=")[1])
    with st.Grid(st.ST_7PT_VAR, 33, 21, 17, seed=14103060) as g:
        g.run(7)
        py_sum = 0.0
        for v in g.read(0).ravel().tolist():  # the C loop's left-to-right order
            py_sum += v
    assert c_sum == py_sum
