#!/usr/bin/env python
"""Benchmark of the stencil hot path (BASELINE.json metric: GLUP/s, fp64 lattice updates per second).

A step = one pass of the whole hot path over one batch of synthetic input: stencil_run(T) of the
workload (T time steps, i.e. ceil(T/bt) fused-level kernel launches), inputs resident in HBM.

  N = 1   : C5 = BASELINE.json configs[4], the configuration the metric is quoted on ("at 1/2/4/8 B200"):
            25-point variable coefficients, 1024^3 interior, T = 200 (135 GB of device memory).  C2, C3
            and C4 (configs[1..3]) are timed after it with their default plans and reported under
            "secondary" (not the headline); --workload picks another headline (C1..C5, C3A).
  N > 1   : one rank per GPU.  Launched by the driver through torchrun; `python bench.py --gpus N`
            without torchrun re-launches itself under torch.distributed.run (127.0.0.1).  --scaling weak
            (default): BASELINE.json's C5 weak variant, 1024 x 1024 x 256N (per-GPU work fixed);
            --scaling strong: the 1024^3 grid split over the N GPUs.  z-slabs with R*bt-deep halos;
            --halo copy (default): edge kernels + NCCL send/recv overlapped with the interior kernel
            (SURVEY.md §8(e)); --halo peer: the kernel stores the neighbours' halo planes straight into
            their memory (CUDA IPC).  value = all ranks' LUPs / max-over-ranks device time.
  --impl reference : the CPU oracle (oracle/, test infrastructure) timed on this host's cores on a
            bounded z-slab sample of the same workload (this tier's reference arm; rank 0 only).

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from synth import workloads  # noqa: E402

METRIC = "GLUP/s"
DEFAULT_WORKLOAD = "C5"
SECONDARY = ("C2", "C3", "C4")


# compulsory HBM bytes per lattice cell per fused block of b levels:
# state read once + written once per block, coefficients read once per block, no write-allocate.
def block_bytes_per_cell(kind, b):
    """Compulsory HBM bytes per lattice cell per fused block of b levels (paper_1410_3060_b200.model)."""
    from paper_1410_3060_b200 import model
    return model.code_balance(kind, b) * b


def blocks_of(T, bt):
    """Fused-block lengths stencil_run(T) uses (runtime.cu): full blocks of bt; a remainder shorter than
    bt is merged with the last full block and split evenly."""
    out, left = [], T
    while left > 0:
        b = (left + 1) // 2 if bt < left < 2 * bt else min(bt, left)
        out.append(b)
        left -= b
    return out


from paper_1410_3060_b200.model import FLOPS_PER_LUP  # noqa: E402


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


SLOWDOWN_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "hw_power_brake_slowdown"}


class ClockSampler:
    """Samples SM clock, board power and throttle reasons through NVML while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.power = [], set(), []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _power_w(self):
        # Instantaneous board power (NVML_FI_DEV_POWER_INSTANT, mW).  nvmlDeviceGetPowerUsage is a 1-s
        # moving average: it lags a sub-second timed region and under-reads the 1 kW cap.
        try:
            v = self.nv.nvmlDeviceGetFieldValues(self.h, [self.nv.NVML_FI_DEV_POWER_INSTANT])[0]
            if v.nvmlReturn == 0:
                return v.value.uiVal / 1000.0
        except Exception:
            pass
        return self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.power.append(self._power_w())
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "note": "NVML unavailable"}
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power:
            out["power_w"] = round(statistics.median(self.power), 1)
        return out


def observed_limiter(clocks, bound):
    """'board_power_cap' when the timed region sat at the board's power limit with sw_power_cap active,
    else the roofline's own bound."""
    if "sw_power_cap" in (clocks.get("reasons") or []) and (clocks.get("power_w") or 0) >= 900:
        return "board_power_cap"
    return bound


def load_fp64_peak():
    """Measured FP64 FMA throughput (tools/fp64_peak.cu -> profiles/fp64_peak.json), TFLOP/s."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        return float(d["fp64_tflops"]), "measured (profiles/fp64_peak.json, tools/fp64_peak.cu)"
    except Exception:
        return 37.2, "nominal (64 FP64 FMA lanes per SM x 148 SMs x 1.965 GHz)"


def energy_split(energy_nj, glups_per_gpu, dram_bytes_per_lup):
    """Board energy per update split with round 1's probe (profiles/r01_energy_probe.json, tools/
    energy_probe.py): idle power / rate, DRAM bytes x the streaming copy's incremental pJ per byte, the rest
    (SM, L2, shared memory, TMEM at the plan's clock).  None without the probe file or the ncu bytes."""
    try:
        probe = {}
        for line in open(os.path.join(ROOT, "profiles", "r01_energy_probe.json")):
            if line.strip():
                d = json.loads(line)
                probe[d["case"]] = d
        idle = probe["idle"]["power_w"] / glups_per_gpu
        dram = dram_bytes_per_lup * probe["hbm_copy"]["pj_per_unit"] / 1e3
    except Exception:
        return None
    return {"idle_nj": round(idle, 2), "dram_nj": round(dram, 2), "rest_nj": round(energy_nj - idle - dram, 2),
            "source": "profiles/r01_energy_probe.json (idle W, HBM copy pJ/B) and the ncu DRAM bytes per update"}


def pick_workload(name, n_gpus, scaling="weak"):
    """The workload of an N-GPU run.  weak: per-GPU work fixed (the global nz grows with N; C5 uses
    BASELINE.json's weak variant 1024 x 1024 x 256N); strong: the configuration's global grid split over N."""
    w = workloads.BY_NAME.get(name) or {x.name.split("-")[0]: x
                                        for x in workloads.CONFIGS + workloads.EXTRA}.get(name)
    if w is None:
        raise SystemExit(f"unknown workload {name}")
    if n_gpus > 1 and scaling == "weak":
        if w is workloads.C5:
            return workloads.weak_c5(n_gpus)
        w = workloads.Workload(f"{w.name}-weak-x{n_gpus}", w.kind, w.nx, w.ny, w.nz * n_gpus, w.T)
    return w


def workload_config(w, n_gpus, scaling):
    """The `config` object of the JSON line: what the workload IS (identical in both arms; the plan the
    library chose is reported separately under "plan")."""
    return {"workload": w.name, "kind": synth.KIND_NAMES[w.kind], "nx": w.nx, "ny": w.ny, "nz": w.nz,
            "T": w.T, "luops_per_step": w.nx * w.ny * w.nz * w.T,
            "parallelism": f"z-slab x{n_gpus}" if n_gpus > 1 else "single GPU",
            "scaling": scaling, "l2": "inputs larger than L2 (no flush needed)"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def sample_planes(w, target_cells=96 * 2 ** 20):
    """Interior planes of the z-slab sample the oracle times (whole xy planes of the workload): the
    full grid when it has at most ~100 M cells, else enough planes for ~100 M cells (C5: 96 of 1024)."""
    return max(1, min(w.nz, target_cells // (w.nx * w.ny)))


def oracle_sample(w, target_s=12.0, max_steps=None):
    """Time the oracle (test infrastructure: allowed in the cpu_baseline / reference legs only) on a
    z-slab sample of the workload: planes [R, R + nzs) of the global grid (its own seeded values, the
    planes around it as the fixed boundary), for as many time steps as fit ~target_s."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    R = synth.RADIUS[w.kind]
    nzs = sample_planes(w)
    dims = synth.padded_dims(w.kind, w.nx, w.ny, w.nz)
    box = ((0, nzs + 2 * R), (0, dims[1]), (0, dims[2]))
    inp = synth.make_inputs(w.kind, w.nx, w.ny, w.nz, box=box)
    cells = w.nx * w.ny * nzs
    V, U = inp.V, inp.U
    t0 = time.perf_counter()
    oracle.run_arrays(w.kind, w.nx, w.ny, nzs, V, U, inp.coef, inp.scalars, 1, cores)
    t1 = time.perf_counter() - t0
    steps = max(1, min(max_steps or w.T, int(target_s / max(t1, 1e-9))))
    t0 = time.perf_counter()
    oracle.run_arrays(w.kind, w.nx, w.ny, nzs, V, U, inp.coef, inp.scalars, steps, cores)
    dt = time.perf_counter() - t0
    where = "the full grid" if nzs == w.nz else f"a {w.nx}x{w.ny}x{nzs} z-slab (planes 1..{nzs} of {w.nz})"
    return {"value": cells * steps / dt / 1e9, "unit": METRIC, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{steps} of T={w.T} time steps of {where} of {w.name} ({cells * steps:.3g} LUPs, "
                      f"{dt:.2f} s, {cores} OpenMP threads)",
            "sample_planes": nzs, "T_sampled": steps, "seconds": dt}


def run_reference(args):
    """This tier's reference arm: the CPU oracle as it stands, on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    n = max(world, args.gpus)
    w = pick_workload(args.workload, n, args.scaling)
    import oracle
    cores = len(os.sched_getaffinity(0))
    R = synth.RADIUS[w.kind]
    nzs = sample_planes(w)
    dims = synth.padded_dims(w.kind, w.nx, w.ny, w.nz)
    inp = synth.make_inputs(w.kind, w.nx, w.ny, w.nz, box=((0, nzs + 2 * R), (0, dims[1]), (0, dims[2])))
    cells = w.nx * w.ny * nzs
    t0 = time.perf_counter()
    oracle.run_arrays(w.kind, w.nx, w.ny, nzs, inp.V, inp.U, inp.coef, inp.scalars, 1, cores)
    t1 = time.perf_counter() - t0
    # each step: a bounded sample of s time steps on the z-slab, sized so the whole run stays short
    budget = 150.0 / max(1, args.steps + args.warmup)
    s = max(1, min(w.T, int(budget / max(t1, 1e-9))))
    for _ in range(args.warmup):
        oracle.run_arrays(w.kind, w.nx, w.ny, nzs, inp.V, inp.U, inp.coef, inp.scalars, s, cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.run_arrays(w.kind, w.nx, w.ny, nzs, inp.V, inp.U, inp.coef, inp.scalars, s, cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = cells * s * args.steps / tot / 1e9
    where = "the full grid" if nzs == w.nz else f"a {w.nx}x{w.ny}x{nzs} z-slab of the grid"
    sample = f"{s} of T={w.T} time steps per step on {where} ({cells * s:.3g} LUPs per step)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth/ seeded generator)",
        "config": workload_config(w, n, args.scaling),
        "sample": {"T_sampled": s, "planes_sampled": nzs, "luops_per_step": cells * s},
        "cpu_baseline": {"value": value, "unit": METRIC, "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def load_traffic(workload, bt):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum of one bt-level launch over the local grid
    (profiles/traffic.json, written from the committed --set full captures)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        v = d.get(f"{workload}/bt{bt}")
        return v.get("bytes") if isinstance(v, dict) else v
    except Exception:
        return None


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(n):
    """`bench.py --gpus N` without torchrun: run the same command line as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", str(max(1, len(os.sched_getaffinity(0)) // n)))
    return subprocess.call(cmd, env=env)


def probe_launch(args):
    """--probe-launch (tests): every rank reports (rank, world) over a gloo group; no GPU work."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
        got = [None] * world
        dist.all_gather_object(got, rank)
        dist.destroy_process_group()
    else:
        got = [0]
    if rank == 0:
        print(json.dumps({"probe": True, "world": world, "ranks": got, "gpus": args.gpus}))


def time_plan(st, torch, w, steps, warmup, local, **kw):
    """Create a seeded grid with plan kw, warm up, time `steps` stencil_run(T) calls with CUDA events on
    the library's stream; returns (GLUP/s, info, clocks summary, summed kernel ms, timed launches)."""
    g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, **kw)
    try:
        for _ in range(warmup):
            g.run(w.T)
        g.sync()
        g.set_timing(True)
        g.kernel_time(reset=True)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            ea.record(g.stream)
            for _ in range(steps):
                g.run(w.T)
            eb.record(g.stream)
            eb.synchronize()
        kern_ms, kern_n = g.kernel_time(reset=True)
        info = g.info()
    finally:
        g.close()
        torch.cuda.empty_cache()
    return w.luops * steps / (ea.elapsed_time(eb) / 1e3) / 1e9, info, clk.summary(), kern_ms, kern_n


def roofline_of(w, bt, value_per_gpu, kern_ms, kern_steps, cells_local, peak, fp64):
    """Roofline object of the dominant (fused-level) kernel: algorithmic bytes of the timed launches / their
    summed device time (CUDA events around every launch on the library's stream)."""
    per_step_bytes = cells_local * sum(block_bytes_per_cell(w.kind, b) for b in blocks_of(w.T, bt))
    achieved = per_step_bytes * kern_steps / (kern_ms / 1e3) / 1e9 if kern_ms else 0.0
    roof_bt = peak / (block_bytes_per_cell(w.kind, bt) / bt)
    roof_bt1 = peak / block_bytes_per_cell(w.kind, 1)
    roof_fp64 = fp64 * 1e3 / FLOPS_PER_LUP[w.kind]
    tr = load_traffic(w.name, bt)
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": tr, "bytes_per_cell_per_launch": block_bytes_per_cell(w.kind, bt), "bt": bt,
            "roof_glups_bt": roof_bt, "roof_glups_bt1": roof_bt1,
            # BASELINE.json's second bound: FP64 peak / flops per LUP (the lower one is the roofline)
            "fp64_tflops": fp64, "flops_per_lup": FLOPS_PER_LUP[w.kind], "roof_glups_fp64": roof_fp64,
            "roof_glups": min(roof_bt, roof_fp64),
            # SURVEY 8(d) anti-gaming rule: the rate against roof(1) and roof(bt), and the measured DRAM
            # bytes per lattice update (ncu, one launch of bt levels over the local grid) next to B_C / bt
            "frac_of_roof_bt": value_per_gpu / min(roof_bt, roof_fp64),
            "frac_of_roof_bt1": value_per_gpu / roof_bt1,
            "compulsory_bytes_per_lup": block_bytes_per_cell(w.kind, bt) / bt,
            "dram_bytes_per_lup": tr / (cells_local * bt) if tr else None}


def modeled_dram(st, w, info):
    """DRAM bytes per update the lockstep round model predicts for the plan that ran (model.py
    lockstep_dram_bytes_per_lup: round-patch halo re-reads, ghosts, 128-byte lines), next
    to ncu's `dram_bytes_per_lup`; None for plans without lockstep rounds."""
    if info["variant"] != st.ST_VARIANT_PIPE:
        return None
    from paper_1410_3060_b200 import model
    return round(model.lockstep_dram_bytes_per_lup(w.kind, info["bt"], (w.nx, w.ny, w.nz),
                                                   (info["tile_x"], info["tile_y"])), 2)


def alloc_pinned(shape, torch):
    """A page-locked host array (numpy view of a pinned torch tensor)."""
    n = int(np.prod(shape))
    return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy().reshape(shape)


def host_mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--bt", type=int, default=0)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--tile-cfg", type=int, default=0)
    ap.add_argument("--zchunk", type=int, default=0)
    ap.add_argument("--slabs", type=int, default=1,
                    help="single GPU only: run the z-slab plan with this many slabs on the one device "
                         "(loopback halo copies; measures the multi-GPU plan's overhead)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = per-GPU work fixed (default; C5: 1024x1024x256N), strong = the "
                         "configuration's global grid split over the N GPUs")
    ap.add_argument("--halo", default="copy", choices=["copy", "peer"],
                    help="z-slab halo exchange: copy = edge kernels + NCCL send/recv (device copies in "
                         "loopback) overlapped with the interior kernel (default); peer = fused into the "
                         "kernel, which stores the neighbours' halo planes straight into their memory "
                         "(CUDA IPC over NVLink across processes)")
    ap.add_argument("--alt-bt", type=int, default=-1,
                    help="also time the plan at this time-block depth (-1: the default bt + 1; 0: off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--probe-launch", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if args.probe_launch:
        return probe_launch(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1410_3060_b200 as st

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = world
    w = pick_workload(args.workload, n, args.scaling)
    nccl_id = None
    if world > 1:
        obj = [st.stencil_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    def barrier():
        if world > 1:
            dist.barrier()

    slabs = args.slabs if world == 1 else 1
    halo = st.ST_HALO_PEER if args.halo == "peer" else st.ST_HALO_COPY
    halo_note = None
    plan_kw = dict(variant=args.variant, bt=args.bt, zchunk=args.zchunk, tile_cfg=args.tile_cfg)
    if slabs > 1:
        g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, nranks=slabs, local_slabs=slabs,
                    halo=halo, **plan_kw)
    else:
        g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, rank=rank, nranks=world,
                    nccl_id=nccl_id, halo=halo, wire_peers=False, **plan_kw)
        if world > 1 and halo == st.ST_HALO_PEER:
            # wire the neighbours' memory (CUDA IPC); if any rank cannot, every rank falls back to the
            # NCCL halo exchange together (a half-wired job would wait forever on a flag)
            ok, halo_note = g.wire_peers(timeout_ms=20000)
            if not ok:
                g.close()
                halo, args.halo = st.ST_HALO_COPY, "copy"
                g = st.Grid(w.kind, w.nx, w.ny, w.nz, seed=synth.DEFAULT_SEED, rank=rank, nranks=world,
                            nccl_id=nccl_id, **plan_kw)
    stream = g.stream
    for _ in range(args.warmup):
        g.run(w.T)
    g.sync()

    def timed_region():
        info0 = g.info()
        barrier()
        torch.cuda.synchronize()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.set_timing(True)
        g.kernel_time(reset=True)
        with ClockSampler(local) as clk:
            barrier()
            torch.cuda.synchronize()
            start.record(stream)
            for _ in range(args.steps):
                g.run(w.T)
            end.record(stream)
            end.synchronize()
            torch.cuda.synchronize()
        barrier()
        kern = g.kernel_time(reset=True)
        g.set_timing(False)
        return start.elapsed_time(end), kern, g.info()["launches"] - info0["launches"], clk

    ms, (kern_ms, kern_launches), launches, clk = timed_region()
    # a timed region that saw a hardware or thermal slowdown is measured once more (any rank's verdict)
    # (or whose SM clock sat far below its maximum with no throttle reason: a leftover clock lock)
    cs0 = clk.summary()
    stuck = (not cs0.get("reasons") and cs0.get("sm_mhz") and cs0.get("sm_max_mhz")
             and cs0["sm_mhz"] < 0.75 * cs0["sm_max_mhz"])
    bad = torch.tensor([int(bool(set(cs0.get("reasons", [])) & SLOWDOWN_REASONS) or bool(stuck))], device=dev)
    if world > 1:
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    remeasured = None
    if int(bad.item()):
        remeasured = {"first_ms": ms, "first_reasons": clk.summary().get("reasons")}
        ms, (kern_ms, kern_launches), launches, clk = timed_region()
    info = g.info()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    luops = w.luops * args.steps  # all ranks' LUPs (global grid)
    value = luops / (ms_max / 1e3) / 1e9

    bt = info["bt"]
    peak, peak_src = load_peaks()
    fp64, fp64_src = load_fp64_peak()
    cells_local = w.nx * w.ny * (info["own_z1"] - info["own_z0"] - (2 * info["R"] if world == 1 else 0))
    if world > 1:  # owned planes minus the global ghost planes on the edge ranks
        R = info["R"]
        cells_local = w.nx * w.ny * ((info["own_z1"] - info["own_z0"]) - (R if rank == 0 else 0)
                                     - (R if rank == world - 1 else 0))
    roofline = roofline_of(w, bt, value / world, kern_ms, args.steps, cells_local, peak, fp64)
    roofline.update({"peak_source": peak_src, "fp64_source": fp64_src,
                     "avg_launch_ms": kern_ms / max(1, kern_launches),
                     "kernel_share_of_step": kern_ms / ms if ms else None})
    if world == 1 and slabs == 1:
        roofline["modeled_dram_bytes_per_lup"] = modeled_dram(st, w, info)
    plan = {"bt": bt, "variant": info["variant"], "tile": [info["tile_x"], info["tile_y"]],
            "zchunk": info["zchunk"], "halo": args.halo if (world > 1 or slabs > 1) else None,
            "halo_note": halo_note, "device_bytes": info["device_bytes"],
            "slabs_on_one_gpu": slabs if slabs > 1 else None}

    g.close()
    del g
    torch.cuda.empty_cache()

    # Alternative plan at a deeper time block (single GPU, default plan only): its measured rate next to
    # its own (higher) roofline, so a reader sees both sides of the b_t choice
    alt = None
    alt_bt = args.alt_bt if args.alt_bt >= 0 else (bt + 1 if args.bt == 0 else 0)
    if world == 1 and slabs == 1 and alt_bt > bt:
        try:
            va, ia, ca, _, _ = time_plan(st, torch, w, max(1, min(args.steps, 3)), 1, local, variant=args.variant,
                                         bt=alt_bt)
        except st.StencilError:
            ia = None
        if ia is not None and ia["bt"] == alt_bt:
            roof_a = min(peak / (block_bytes_per_cell(w.kind, alt_bt) / alt_bt), fp64 * 1e3 / FLOPS_PER_LUP[w.kind])
            alt = {"bt": alt_bt, "value": va, "roof_glups_bt": roof_a, "frac": va / roof_a,
                   "tile": [ia["tile_x"], ia["tile_y"]], "sm_mhz": ca.get("sm_mhz"),
                   "note": "same workload, next deeper time block; not the headline plan"}

    # The other BASELINE.json configurations (single GPU, default plans): secondary numbers, not the headline
    secondary = None
    if world == 1 and slabs == 1 and not args.no_secondary and args.workload == DEFAULT_WORKLOAD:
        secondary = {}
        for name in SECONDARY:
            ws = pick_workload(name, 1)
            try:
                vs, is_, cs_, kms, _ = time_plan(st, torch, ws, 3, 2, local)
            except st.StencilError as e:
                secondary[ws.name] = {"error": str(e)}
                continue
            cl = ws.nx * ws.ny * ws.nz
            rs = roofline_of(ws, is_["bt"], vs, kms, 3, cl, peak, fp64)
            secondary[ws.name] = {"value": vs, "unit": METRIC, "bt": is_["bt"],
                                  "tile": [is_["tile_x"], is_["tile_y"]],
                                  "frac_of_roof_bt": rs["frac_of_roof_bt"], "roof_glups_bt": rs["roof_glups_bt"],
                                  "frac_of_roof_bt1": rs["frac_of_roof_bt1"], "hbm_frac": rs["frac"],
                                  "dram_bytes_per_lup": rs["dram_bytes_per_lup"],
                                  "modeled_dram_bytes_per_lup": modeled_dram(st, ws, is_),
                                  "sm_mhz": cs_.get("sm_mhz"), "power_w": cs_.get("power_w")}

    # e2e: through the public API with HOST buffers: create from pinned host inputs (H2D), run T,
    # read the newest level (D2H), every step.
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, st, torch, dist, w, info, rank, world, local, dev, nccl_id, halo, barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(w)
        cpu.pop("seconds", None)

    if rank == 0:
        clocks = clk.summary()
        if remeasured:
            clocks["remeasured"] = remeasured
        # what actually limits the timed region: the roofline above is HBM / FP64; a run that sat at the
        # board's power limit with sw_power_cap active is power-bound (DESIGN.md §6's power model)
        roofline["observed_limiter"] = observed_limiter(clocks, roofline["bound"])
        if clocks.get("power_w"):  # board energy per lattice update on this GPU (cf. the paper's Table 1)
            clocks["energy_nj_per_lup"] = round(clocks["power_w"] / (value / world), 3)
            if roofline.get("dram_bytes_per_lup"):
                clocks["energy_split"] = energy_split(clocks["energy_nj_per_lup"], value / world,
                                                      roofline["dram_bytes_per_lup"])
        line = {
            "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (synth/ counter-based generator, seed 14103060, drawn on the device)",
            "config": workload_config(w, n, args.scaling),
            "plan": plan,
            "roofline": roofline,
            "alt_plan": alt,
            "secondary": secondary,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, st, torch, dist, w, info, rank, world, local, dev, nccl_id, halo, barrier):
    """Same metric end to end through the C ABI: every step stencil_create from pinned HOST arrays (H2D
    inside the timed region), stencil_run(T), stencil_read of the newest level (D2H)."""
    # multi-rank: every rank holds (and uploads) only the planes it stores, and reads back the planes it
    # owns (st_opts.host_slab) -- no rank ever materialises the global inputs in host memory
    pl = None
    R = synth.RADIUS[w.kind]
    dims = synth.padded_dims(w.kind, w.nx, w.ny, w.nz)
    if world > 1:
        pl = st.stencil_plan_slab(w.nz, R, world, rank, info["bt"])
        box = ((pl["store_z0"], pl["store_z1"]), (0, dims[1]), (0, dims[2]))
    else:
        box = ((0, dims[0]), (0, dims[1]), (0, dims[2]))
    shape = (box[0][1] - box[0][0], dims[1], dims[2])
    out_shape = shape if pl is None else (pl["own_z1"] - pl["own_z0"],) + shape[1:]
    nf = synth.N_COEF_FIELDS[w.kind]
    wave = w.kind in synth.WAVE_KINDS
    arr_bytes = int(np.prod(shape)) * 8
    # host memory: V (+U) + the coefficient fields + the result, on every rank of this node; when that
    # exceeds ~60 % of the available RAM the coefficient fields share one pinned buffer (the step still
    # copies every field host->device; the values of fields 1.. are then field 0's -- a throughput run)
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    need = (1 + (1 if wave else 0) + nf + 1) * arr_bytes * local_ranks
    shared_coef = nf > 1 and need > 0.6 * host_mem_available()
    # fill the pinned arrays in place with the seeded generator (no second host copy)
    V = alloc_pinned(shape, torch)
    synth.fill_box(synth.DEFAULT_SEED, synth.STREAM_V, dims, box, out=V)
    U = None
    if wave:
        U = alloc_pinned(shape, torch)
        inp = synth.make_inputs(w.kind, w.nx, w.ny, w.nz, box=box)
        U[...] = inp.U
        del inp
    fields = []
    for i in range(nf if not shared_coef else 1):
        f = alloc_pinned(shape, torch)
        synth.fill_box(synth.DEFAULT_SEED, synth.stream_w(i), dims, box, scale=synth.COEF_SCALE[w.kind], out=f)
        fields.append(f)
    if shared_coef:
        fields = fields * nf
    coeff = list({synth.K7C: synth.SCALARS_7C, synth.K25W: synth.SCALARS_25W,
                  synth.K25WA: synth.SCALARS_25WA}.get(w.kind, ())) + fields
    out = alloc_pinned(out_shape, torch)
    h2d = arr_bytes * (1 + (1 if wave else 0) + nf)
    d2h = out.nbytes

    def make_grid(stream=None):
        return st.Grid(w.kind, w.nx, w.ny, w.nz, v0=V, u0=U, coeff=coeff, variant=args.variant,
                       bt=info["bt"] if world > 1 else args.bt, zchunk=args.zchunk, tile_cfg=args.tile_cfg,
                       rank=rank, nranks=world, nccl_id=nccl_id, halo=halo, stream=stream, host_slab=world > 1)

    def read_result(ge, o):
        if pl is None:
            ge.read(0, out=o)
        else:
            st.stencil_read_planes(ge.h, 0, pl["own_z0"], pl["own_z1"], o)

    # Single GPU with room for two grids: a two-deep pipeline -- a host thread creates (uploads) step
    # k+1's grid on its own stream while step k runs and reads back on the other; every step still moves
    # its own inputs host->device and its result device->host.
    free_b, _ = torch.cuda.mem_get_info(dev)
    pipelined = world == 1 and free_b > 2.2 * info["device_bytes"]
    ek = max(1, min(2 * args.steps, 8) if pipelined else min(args.steps, 3))
    outs = [out, alloc_pinned(out_shape, torch)] if pipelined else [out, out]
    # the pipeline's two streams live across the warm-up and the timed steps: torch's caching allocator
    # keeps freed device memory per stream, so new streams would allocate afresh
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]

    def e2e_run(k_steps):
        if not pipelined:
            for _ in range(k_steps):
                with make_grid() as ge:
                    ge.run(w.T)
                    read_result(ge, out)
            return
        from concurrent.futures import ThreadPoolExecutor

        def create(k):
            torch.cuda.set_device(dev)
            return make_grid(streams[k % 2])
        with ThreadPoolExecutor(1) as ex:
            fut = ex.submit(create, 0)
            for k in range(k_steps):
                ge = fut.result()
                if k + 1 < k_steps:
                    fut = ex.submit(create, k + 1)
                ge.run(w.T)
                read_result(ge, outs[k % 2])
                ge.close()
    e2e_run(2 if pipelined else 1)  # warm-up: both pipeline slots' device memory cached
    barrier()
    t0 = time.perf_counter()
    e2e_run(ek)
    torch.cuda.synchronize()
    barrier()
    et = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e = {"value": w.luops * ek / float(et.item()) / 1e9, "unit": METRIC,
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": ek,
           "note": ("stencil_create from pinned host arrays + stencil_run(T) + stencil_read of the newest "
                    "level every step, wall clock" +
                    ("; each rank holds, uploads and reads back only its own planes (st_opts.host_slab)"
                     if world > 1 else "") +
                    ("; two-deep pipeline (step k+1's upload on a second stream overlaps step k's "
                     "run and readback)" if pipelined else "") +
                    (f"; the {nf} coefficient fields are uploaded from ONE shared pinned host buffer (all "
                     f"{nf} host->device copies happen; host RAM holds {need / 1e9:.0f} GB otherwise)"
                     if shared_coef else ""))}
    # the e2e's own bound: this GPU's pinned host->device bandwidth (a 1 GiB copy, best of 3) carrying the
    # step's inputs -- the step can be no faster than its upload
    hb = torch.from_numpy(V.reshape(-1)[: (1 << 27)])
    db = torch.empty(hb.numel(), dtype=torch.float64, device=dev)
    best = None
    for _ in range(3):
        t1 = time.perf_counter()
        db.copy_(hb, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        best = dt if best is None or dt < best else best
    h2d_gbs = hb.numel() * 8 / best / 1e9
    bound = w.luops / (h2d / (h2d_gbs * 1e9)) / 1e9 * world
    e2e.update({"h2d_gbs": h2d_gbs, "bound_glups": bound, "frac_of_bound": e2e["value"] / bound})
    return e2e


if __name__ == "__main__":
    main()
