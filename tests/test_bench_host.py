"""Host-side logic of bench.py (no GPU): the fused-block schedule the roofline's byte count assumes, the
N-GPU workloads, and the compulsory bytes per launch."""
import bench
import synth
from synth import workloads


def test_blocks_of_matches_the_runtime_schedule():
    # runtime.cu: full blocks of bt; a remainder shorter than bt is merged with the last full block and
    # split evenly (T = 100 at bt = 3 -> 32 blocks of 3, then 2 + 2)
    assert bench.blocks_of(100, 3) == [3] * 32 + [2, 2]
    assert bench.blocks_of(100, 4) == [4] * 25
    assert bench.blocks_of(10, 1) == [1] * 10
    assert bench.blocks_of(7, 3) == [3, 2, 2]
    assert bench.blocks_of(5, 8) == [5]
    for T in range(1, 60):
        for bt in range(1, 9):
            b = bench.blocks_of(T, bt)
            assert sum(b) == T and max(b) <= bt and min(b) >= 1


def test_block_bytes_per_cell():
    # C2 at bt = 3: 16 B of state + 56 B of coefficients per cell per launch = 24 B per update
    assert bench.block_bytes_per_cell(synth.K7V, 3) == 72
    assert bench.block_bytes_per_cell(synth.K7V, 1) == 72
    assert bench.block_bytes_per_cell(synth.K25V, 1) == 120
    assert bench.block_bytes_per_cell(synth.K25W, 2) == 32  # both levels in (16 B) and out (16 B)
    assert bench.block_bytes_per_cell(synth.K25W, 1) == 24  # V, U in; U out (in place)


def test_pick_workload_weak_and_strong():
    w = bench.pick_workload("C2", 4, "weak")
    assert (w.nx, w.ny, w.nz, w.T) == (512, 512, 2048, 100)
    w = bench.pick_workload("C2", 4, "strong")
    assert (w.nx, w.ny, w.nz) == (512, 512, 512)
    w = bench.pick_workload("C5", 8, "weak")  # BASELINE.json's weak variant: 1024 x 1024 x 256N
    assert (w.nx, w.ny, w.nz, w.T) == (1024, 1024, 2048, 200)
    assert bench.pick_workload("C2", 1) is workloads.C2 or bench.pick_workload("C2", 1).nz == 512


def test_slowdown_reasons_trigger_a_second_measurement():
    assert {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} <= bench.SLOWDOWN_REASONS
    assert "sw_power_cap" not in bench.SLOWDOWN_REASONS  # kept and noted, not re-measured


def test_observed_limiter():
    assert bench.observed_limiter({"reasons": ["sw_power_cap"], "power_w": 1040.0}, "hbm") == "board_power_cap"
    assert bench.observed_limiter({"reasons": ["sw_power_cap"], "power_w": 480.0}, "hbm") == "hbm"  # a 1-s average
    assert bench.observed_limiter({"reasons": [], "power_w": 1000.0}, "hbm") == "hbm"
    assert bench.observed_limiter({}, "fp64") == "fp64"


def test_default_headline_is_the_metric_config():
    # BASELINE.json quotes GLUP/s "at 1/2/4/8 B200" on config 5 (C5, 1024^3, T = 200)
    w = bench.pick_workload(bench.DEFAULT_WORKLOAD, 1)
    assert w is workloads.C5 and (w.nx, w.ny, w.nz, w.T) == (1024, 1024, 1024, 200)
    w = bench.pick_workload(bench.DEFAULT_WORKLOAD, 4, "strong")
    assert (w.nx, w.ny, w.nz) == (1024, 1024, 1024)


def test_both_arms_share_the_config_keys():
    w = bench.pick_workload("C5", 2, "weak")
    c = bench.workload_config(w, 2, "weak")
    assert c["workload"] == w.name and c["nz"] == 512 and c["T"] == 200
    assert c["parallelism"] == "z-slab x2"
    assert c == bench.workload_config(bench.pick_workload("C5", 2, "weak"), 2, "weak")


def test_oracle_sample_is_a_bounded_z_slab():
    # C5's 1024^3 inputs need 132 GB of host memory: the oracle is timed on whole xy planes of a z-slab
    assert bench.sample_planes(workloads.C5) == 96
    assert bench.sample_planes(workloads.C2) == 384
    assert bench.sample_planes(workloads.C1) == 64  # small grids: the full grid


def test_gpus_2_spawns_two_ranks():
    # `bench.py --gpus 2` without torchrun re-launches itself as 2 ranks (here: gloo, no GPU work)
    import json
    import os
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--gpus", "2", "--probe-launch"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["world"] == 2 and sorted(lines[0]["ranks"]) == [0, 1]


def test_modeled_dram_reports_the_round_model_for_pipe_plans_only():
    # bench.py's roofline carries model.lockstep_dram_bytes_per_lup for the plan that ran (next to ncu's
    # measured bytes); the cooperative and naive plans have no lockstep rounds
    import paper_1410_3060_b200 as st
    from paper_1410_3060_b200 import model
    info = {"variant": st.ST_VARIANT_PIPE, "bt": 2, "tile_x": 24, "tile_y": 16}
    got = bench.modeled_dram(st, workloads.C4, info)
    assert got == round(model.lockstep_dram_bytes_per_lup(model.K25V, 2, (512, 512, 512), (24, 16)), 2)
    assert 60.0 < got < 75.0
    assert bench.modeled_dram(st, workloads.C4, dict(info, variant=st.ST_VARIANT_COOP)) is None


def test_energy_split_adds_up():
    e = bench.energy_split(16.98, 58.7, 70.31)
    assert e is not None and abs(e["idle_nj"] + e["dram_nj"] + e["rest_nj"] - 16.98) < 0.02
    assert 4.0 < e["idle_nj"] < 5.0 and 6.0 < e["dram_nj"] < 7.0
