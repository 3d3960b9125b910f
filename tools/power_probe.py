"""Board-power model of the hot path: instantaneous power, SM clock and DRAM rate per plan.

python tools/power_probe.py [--secs 2.0]

For a plain HBM copy (torch, the MEASURED_PEAKS recipe) and for C2 / C3 plans at several b_t, run
each for about `--secs` seconds of sustained work and print one JSON line per case: GLUP/s (or GB/s),
the median instantaneous board power under load (NVML_FI_DEV_POWER_INSTANT), the median SM clock,
the throttle reasons and the energy per lattice update.  With the DRAM bytes per update from
profiles/traffic.json this separates the DRAM share of the 1 kW budget from the SM share
(profiles/r01_summary.md "power").
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1410_3060_b200 as st  # noqa: E402
from bench import ClockSampler  # noqa: E402
import synth  # noqa: E402
from synth import workloads  # noqa: E402


def sustained(fn, secs):
    """Run fn() back to back until `secs` of device time have passed; returns (seconds, calls, clocks)."""
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    e1.synchronize()
    one = e0.elapsed_time(e1) / 1e3
    n = max(1, int(secs / max(one, 1e-6)))
    fn()  # bring the board to its steady power state before sampling
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device())
    e0.record(s)
    with clk:
        for _ in range(n):
            fn()
        e1.record(s)
        e1.synchronize()
    return e0.elapsed_time(e1) / 1e3, n, clk.summary()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--secs", type=float, default=2.0)
    ap.add_argument("--cases", default="copy,C2:1,C2:2,C2:3,C2:4,C3:1,C3:2")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    idle = ClockSampler(0)
    with idle:
        time.sleep(0.5)
    print(json.dumps({"case": "idle", **idle.summary()}), flush=True)
    for case in a.cases.split(","):
        if case == "copy":
            n = 1 << 29  # 4 GiB per buffer (fp64)
            x = torch.empty(n, dtype=torch.float64, device="cuda")
            y = torch.empty_like(x)
            x.fill_(1.0)
            secs, calls, cs = sustained(lambda: y.copy_(x), a.secs)
            gbs = 2 * 8 * n * calls / secs / 1e9
            print(json.dumps({"case": "copy", "gbs": round(gbs, 1), **cs,
                              "pj_per_byte": round(cs.get("power_w", 0) / (gbs * 1e9) * 1e12, 1)
                              if cs.get("power_w") else None}), flush=True)
            del x, y
            torch.cuda.empty_cache()
            continue
        name, bt = case.split(":")
        bt = int(bt)
        w = {x.name.split("-")[0]: x for x in workloads.CONFIGS}[name]
        g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, variant=3, bt=bt)
        T = 6 * bt * 4
        secs, calls, cs = sustained(lambda: g.run(T), a.secs)
        info = g.info()
        g.close()
        torch.cuda.empty_cache()
        lups = w.nx * w.ny * w.nz * T * calls
        glups = lups / secs / 1e9
        out = {"case": case, "workload": w.name, "bt": info["bt"], "tile": [info["tile_x"], info["tile_y"]],
               "glups": round(glups, 2), **cs}
        if cs.get("power_w"):
            out["nj_per_lup"] = round(cs["power_w"] / (glups * 1e9) * 1e9, 3)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
