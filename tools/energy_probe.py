"""Energy per operation of the SM's data paths on this B200 (the power model of DESIGN.md §6).

python tools/energy_probe.py [--secs 2.0] > profiles/rNN_energy_probe.json

Each kernel of tools/energy_probe.cu keeps one path of every SM busy (FP64 FMA, shared memory, L2,
HBM, TMEM) for about --secs seconds while NVML's instantaneous board power and the SM clock are sampled.
Energy per unit = (board power - idle power) / rate.  A run that reaches the 1 kW cap is marked: its
clock drops, the energy per unit stays meaningful.
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402

KINDS = {0: ("fp64_fma", "flop"), 1: ("shared_memory", "byte"), 2: ("l2", "byte"), 3: ("hbm_copy", "byte"),
         4: ("tmem_ld", "byte")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--secs", type=float, default=2.0)
    a = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = ctypes.CDLL(os.path.join(root, "build", "libenergy_probe.so"))
    lib.ep_run.restype = ctypes.c_double
    lib.ep_run.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_longlong,
                           ctypes.POINTER(ctypes.c_double)]
    torch.cuda.set_device(0)
    n = 1 << 29  # 4 GiB of doubles: HBM halves of 2 GiB; L2 probe reads the first 32 MiB
    buf = torch.ones(n, dtype=torch.float64, device="cuda")
    idle = ClockSampler(0)
    with idle:
        time.sleep(1.0)
    p_idle = idle.summary().get("power_w")
    print(json.dumps({"case": "idle", **idle.summary()}), flush=True)
    units = ctypes.c_double()
    for kind, (name, unit) in KINDS.items():
        nn = (32 << 20) // 8 if kind == 2 else n
        iters = 16
        while True:  # calibrate on a run long enough that launch overhead does not matter
            ms = lib.ep_run(kind, iters, ctypes.c_void_p(buf.data_ptr()), nn, ctypes.byref(units))
            if ms < 0 or ms > 200:
                break
            iters *= 4
        if ms < 0:
            print(json.dumps({"case": name, "error": ms}), flush=True)
            continue
        iters = max(1, int(iters * a.secs * 1e3 / ms))
        lib.ep_run(kind, max(1, iters // 4), ctypes.c_void_p(buf.data_ptr()), nn, ctypes.byref(units))  # warm
        clk = ClockSampler(0)
        with clk:
            ms = lib.ep_run(kind, iters, ctypes.c_void_p(buf.data_ptr()), nn, ctypes.byref(units))
        cs = clk.summary()
        rate = units.value / (ms / 1e3)
        out = {"case": name, "unit": unit, "rate_per_s": rate, "ms": ms, **cs}
        if cs.get("power_w") and p_idle:
            out["pj_per_unit"] = (cs["power_w"] - p_idle) / rate * 1e12
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
