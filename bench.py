#!/usr/bin/env python
"""Benchmark of the DPD solvent step (Mirheo, arXiv:1911.04712) on B200.

Metric (BASELINE.json): DPD particle-steps/s (whole job), plus the HBM-roofline fraction
of the step (SURVEY §8d byte model) and the dominant kernel's roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config eq64] [--impl reference]

N = 1 runs the BASELINE config 2 (64^3, rho = 8, 2,097,152 particles, P:483, P:489 params).
N > 1 (under torchrun): BASELINE config 4, weak scaling, one 128^3 subdomain per GPU
(16,777,216 particles, same parameters) on a 3D rank grid, NCCL.  One GPU runs both sizes at
the same per-particle rate (profiles/r01_bench_weak128.json), so the driver's efficiency
from the per-N values measures the decomposition cost.  `--config strong256 --scaling strong`
runs BASELINE config 5 instead: the fixed 256^3 box split over the N GPUs.
Prints ONE JSON line on rank 0.  See DESIGN.md §8 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "DPD particle-steps/s"
UNIT = "particle-steps/s"
BYTES_PER_PARTICLE_STEP = 192.0  # bin 56 + scan ~1 + scatter 88 + force 48 (rounded model)


_RESULT_OUT = sys.stdout  # main() re-points it at a duplicate of the original fd 1
# The synthetic input (uniform positions, Maxwell-Boltzmann velocities) is an ideal gas; the
# benchmarked workload is the equilibrium DPD fluid (BASELINE config 2).  Its
# density fluctuations relax within ~100 steps at dt = 0.002, and the force pass is ~3 %
# faster on the equilibrated fluid (more uniform cell occupancy and list lengths:
# DESIGN §8), so every bench workload is equilibrated, untimed, before the W warm-up steps.
EQUIL_STEPS = 200


def rank_grid(n):
    return {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(n) or _factor3(n)


def _factor3(n):
    best = None
    for a in range(1, n + 1):
        if n % a:
            continue
        for b in range(1, n // a + 1):
            if (n // a) % b:
                continue
            c = n // a // b
            key = max(a, b, c) - min(a, b, c)
            if best is None or key < best[0]:
                best = (key, (a, b, c))
    return best[1]


# Algorithmic work model, in scalar lane-instructions.  Per unordered
# interacting pair (C-7 Philox2x32-10, k = 1/2): Philox words 10 x (IMAD.WIDE + LOP3) + id
# min/max = 22; Box-Muller 2 I2F + FFMA + LG2 + SQRT + 2 FMUL + COS + FMUL = 9; geometry
# dx (3) + r^2 (3) + RSQ + r + w + SQRT(w) = 10; dissipative dot product 6; magnitude and
# scalar 6; fixed-point quantise and Newton-3 accumulation 3 FFMA + 6 IADD + 3 ATOMS = 12;
# operand loads (entry, j position x3, j velocity+id) 5 -> 70.  Per candidate pair of the
# half stencil a distance test of 7 (3 FADD, 3 FMUL/FFMA, 1 FSETP).
INSTR_PER_PAIR = 70.0
INSTR_PER_CANDIDATE = 7.0
# bytes per particle and launch, SURVEY §8d byte model
KERNEL_BYTES = {"bin": 56.0, "scatter": 88.0, "force": 48.0, "pack": 40.0, "gather": 60.0}


def kernel_roofline(name, ms_per_launch, cfg, n_local, peaks, src):
    sec = ms_per_launch * 1e-3
    if name == "force":
        vol = 4.0 * math.pi / 3.0 * cfg.rc ** 3
        pairs = n_local * cfg.rho * vol / 2.0
        cand = n_local * cfg.rho * 13.5 * cfg.rc ** 3
        inst = pairs * INSTR_PER_PAIR + cand * INSTR_PER_CANDIDATE
        clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        peak = 148 * 128 * clk / 1e12  # lane-instructions / s: 148 SMs x 4 SMSP x 32 lanes, 1 instr/cycle
        ach = inst / sec / 1e12
        return {"kernel": name, "bound": "alu", "achieved": ach, "peak": peak, "unit": "Tinst/s",
                "frac": ach / peak, "traffic": None,
                "work_model": f"{INSTR_PER_PAIR:g} instr/pair x {pairs:.4g} pairs + {INSTR_PER_CANDIDATE:g} "
                              f"instr/candidate x {cand:.4g} candidates per launch",
                "peak_source": "148 SM x 128 lanes x sm_max_mhz (%s)" % src,
                "hbm_view": {"bytes_per_particle": 48.0,
                             "achieved_gbs": 48.0 * n_local / sec / 1e9, "peak_gbs": float(peaks["hbm_gbs"])}}
    b = KERNEL_BYTES.get(name, 0.0) * n_local
    ach = b / sec / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
            "frac": ach / float(peaks["hbm_gbs"]), "traffic": None, "peak_source": src}


def kernel_traffic():
    """DRAM bytes per launch from the committed `ncu --set full` capture (tools/ncu_traffic.py);
    None when absent."""
    path = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    if not os.path.exists(path):
        return {}, None
    with open(path) as fh:
        d = json.load(fh)
    return d.get("per_launch", {}), "profiles/kernel_traffic.json (" + d.get("source", "?") + ")"


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent sampling via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index=0, period=0.01):
        self.samples = []
        self.reasons = 0
        self.period = period
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml-unavailable"]}
        reasons = [name for bit, name in self.REASONS.items() if self.reasons & bit and name != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference): the oracle as it stands, fp64 cell-list
# mode (C-2 item 7) on a bounded sub-box sample of the same workload (same rho / params).
# ------------------------------------------------------------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_probe(cfg_name):
    """The CPU legs of cpu_baseline, run in a child process with the
    oracle built -O3 -march=native for this host (DPD_ORACLE_NATIVE=1; same source as the
    parity build): brute force (the plain definition, C-1) on config 1 at 1 thread and at all
    threads, and the fp64 cell-list mode (C-2 item 7) on the bench workload itself, full size,
    all threads.  Each leg is bounded (a few seconds); prints one JSON object."""
    import oracle
    oracle.build(force=True)  # -march=native for the host this runs on
    nthreads = oracle.num_threads()

    def rate(cfg, celllist, budget_s, max_steps):
        p = oracle.DPDParams(box=cfg.box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power,
                             dt=cfg.dt, seed=cfg.seed, body_f=cfg.body_f)
        pos, vel = workloads.make_config(cfg)
        st = oracle.State(p, pos, vel, celllist=celllist)
        n = pos.shape[0]
        if not celllist:
            st.step(2)  # thread-pool warm-up (the cell-list leg's step is seconds long)
        t0 = time.perf_counter()
        st.step(1)
        dt1 = time.perf_counter() - t0
        k = int(max(1, min(max_steps, budget_s / max(dt1, 1e-9))))
        t0 = time.perf_counter()
        st.step(k)
        el = time.perf_counter() - t0
        return {"value": n * k / el, "particles": n, "steps": k, "seconds": el}

    c1 = workloads.CONFIGS["parity"]
    cl = rate(workloads.CONFIGS[cfg_name], True, 12.0, 20)
    bfn = rate(c1, False, 3.0, 400)
    oracle.set_num_threads(1)
    bf1 = rate(c1, False, 3.0, 200)
    oracle.set_num_threads(nthreads)
    print(json.dumps({"bf1": bf1, "bfn": bfn, "cl": cl, "threads": nthreads, "cpu_model": cpu_model(),
                      "nproc": os.cpu_count(), "flags": " ".join(oracle.FLAGS)}), flush=True)


def oracle_sample_rate(cfg):
    """cpu_baseline: oracle_probe in a child process (its own -O3 -march=native oracle)."""
    import subprocess
    env = dict(os.environ, DPD_ORACLE_NATIVE="1")
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-probe", cfg.name], env=env,
                       capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-400:])
    d = json.loads(r.stdout.strip().splitlines()[-1])
    cl, bf1, bfn = d["cl"], d["bf1"], d["bfn"]
    return {"value": cl["value"], "unit": UNIT, "cores": d["threads"], "kind": "oracle",
            "sample": f"oracle fp64 cell-list mode (C-2 item 7), {cl['steps']} steps of '{cfg.name}' itself "
                      f"({cl['particles']} particles, full size), {d['threads']} threads",
            "cpu_model": d["cpu_model"], "nproc": d["nproc"], "build": f"gcc {d['flags']} -fopenmp (same source "
            "as the parity build, -O2)",
            "brute_force_config1": {"workload": "parity: 8^3, rho=3, 1536 particles, O(N^2) all pairs (C-1)",
                                    "threads_1": bf1["value"], f"threads_{d['threads']}": bfn["value"],
                                    "unit": UNIT}}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ["DPD_ORACLE_NATIVE"] = "1"  # the same source, -O3 -march=native for this host
    import oracle
    oracle.build(force=True)
    box = tuple(min(float(b), 24.0) for b in cfg.box)
    p = oracle.DPDParams(box=box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power, dt=cfg.dt,
                         seed=cfg.seed, body_f=cfg.body_f)
    pos, vel = workloads.make_particles(box, cfg.rho, cfg.kT)
    st = oracle.State(p, pos, vel, celllist=True)
    n = pos.shape[0]
    st.step(args.warmup)
    t0 = time.perf_counter()
    st.step(args.steps)
    el = time.perf_counter() - t0
    value = n * args.steps / el
    sample = (f"oracle fp64 cell-list mode, each step a {box[0]:g}^3 sub-box ({n} particles) of '{cfg.name}' "
              f"(same rho and parameters)")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_block(cfg, args, int(os.environ.get("WORLD_SIZE", "1"))),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), file=_RESULT_OUT, flush=True)
    return 0


def rank_boxes(cfg, world, scaling):
    """(global box, subdomain) of an N-GPU run: weak = the config's box per GPU, strong = the
    config's box split over the GPUs (rank grid as rank_grid)."""
    grid = rank_grid(world)
    gbox = tuple(cfg.box[k] if scaling == "strong" else cfg.box[k] * grid[k] for k in range(3))
    return gbox, tuple(gbox[k] / grid[k] for k in range(3))


def rank_particles(cfg, world, rank, scaling="weak"):
    """This rank's own particles (global coordinates inside its subdomain, float32), velocities
    and globally unique ids; rank -> subdomain coordinates as the library's (x fastest)."""
    grid = rank_grid(world)
    sub = rank_boxes(cfg, world, scaling)[1]
    coord = (rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1]))
    pos, vel = workloads.make_particles(sub, cfg.rho, cfg.kT, init_seed=1 + rank)
    pos = (pos + np.array([coord[k] * sub[k] for k in range(3)], np.float32)).astype(np.float32)
    for k in range(3):  # the shift can round up onto the next subdomain's face: keep it local
        hi = np.float32((coord[k] + 1) * sub[k])
        pos[pos[:, k] >= hi, k] = np.nextafter(hi, np.float32(0.0))
    n_local = pos.shape[0]
    ids = (np.arange(n_local, dtype=np.int64) + rank * n_local).astype(np.int32)
    return pos, vel, ids, coord, sub


def weak_point(capi, stream, torch, steps, warmup, loopback=False, equilibrate=EQUIL_STEPS):
    """BASELINE config 4 (128^3, rho = 8) on this one GPU: particle-steps/s over `steps`
    device-timed steps after `warmup`, inputs resident.  loopback: the same box as ONE
    subdomain of a 3D decomposition whose six faces are exchanged through NCCL with the rank
    itself (dpd_create_loopback: ghost pack, NCCL send/recv, ghost sort and halo forces,
    migration) -- the per-GPU step of the 8-GPU weak series, on one GPU."""
    cfg = workloads.CONFIGS["weak128"]
    if loopback:
        ctx = capi.dpd_create_loopback(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed,
                                       (1, 1, 1))
    else:
        ctx = capi.dpd_create(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    try:
        capi.dpd_set_stream(ctx, stream.cuda_stream)
        pos, vel = workloads.make_config(cfg)
        capi.dpd_set_particles_ex(ctx, pos, vel, None, 0)
        capi.dpd_step(ctx, equilibrate + warmup)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        capi.dpd_step_async(ctx, steps)
        e1.record(stream)
        capi.dpd_sync(ctx)
        ms = e0.elapsed_time(e1)
        if loopback:
            return {"value": cfg.n * steps / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
                    "workload": "weak128 as one subdomain of a 3D decomposition (split x, y, z), all six faces "
                                "exchanged through NCCL send/recv with the rank itself (dpd_create_loopback): "
                                "the per-GPU step of the N = 8 weak-scaling line without the NVLink transfer time"}
        return {"value": cfg.n * steps / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
                "workload": "weak128: 128^3 rho=8 (16,777,216 particles), BASELINE config 4 on one GPU -- the "
                            "per-GPU workload of the N > 1 weak-scaling lines"}
    finally:
        capi.dpd_destroy(ctx)


def config_block(cfg, args, world):
    g = rank_grid(world)
    strong = getattr(args, "scaling", "weak") == "strong"
    where = "in total, split over the GPUs" if strong else "per GPU"
    return {"workload": f"{cfg.name}: periodic DPD box {cfg.box[0]:g}x{cfg.box[1]:g}x{cfg.box[2]:g} {where}, "
                        f"rho={cfg.rho:g}, a={cfg.a:g}, gamma={cfg.gamma:g}, kT={cfg.kT:g}, k={cfg.power:g}, "
                        f"dt={cfg.dt:g}, rc={cfg.rc:g}",
            "particles_per_gpu": cfg.n // world if strong else cfg.n,
            "particles_total": cfg.n if strong else cfg.n * world,
            "rank_grid": list(g), "parallelism": f"domain-decomposition {g[0]}x{g[1]}x{g[2]}",
            "l2": "inputs larger than L2: double-buffered state ~%.0f MB > 126 MB L2; no flush" %
                  (cfg.n * 96 / 1e6),
            "equilibration_steps": int(getattr(args, "equilibrate", 0) or 0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default=None, help="workloads.CONFIGS name (default: eq64 at N = 1, weak128 at N > 1)")
    ap.add_argument("--impl", default="dpd", choices=["dpd", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the config's box per GPU (default); strong: the config's box split over the GPUs "
                         "(BASELINE config 5: --config strong256 --scaling strong)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-weak-point", action="store_true", help="skip the 128^3 N = 1 weak-series point")
    ap.add_argument("--equilibrate", type=int, default=EQUIL_STEPS,
                    help="untimed steps that equilibrate the synthetic input before the warm-up (BASELINE config 2 "
                         "is an equilibrium run; SURVEY 8(d): discard 200 warm-up steps before timing)")
    ap.add_argument("--force-kernel", type=int, default=None, help="0 tiled, 1 reference, 2 cell-warp")
    ap.add_argument("--option", action="append", default=[], help="engine option name=value (dpd_set_option)")
    ap.add_argument("--oracle-probe", default=None, help=argparse.SUPPRESS)  # cpu_baseline child process
    args = ap.parse_args()
    if args.oracle_probe:
        oracle_probe(args.oracle_probe)
        return 0
    # stdout carries exactly one JSON line: native code writes to fd 1 on its own (NCCL's
    # version banner at communicator init), so fd 1 points at stderr for the run and the
    # result line goes through a private duplicate of the original stdout
    global _RESULT_OUT
    sys.stdout.flush()
    _RESULT_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args.warmup = max(args.warmup, 3)
    if args.config is None:
        args.config = "eq64" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "weak128"
    cfg = workloads.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_1911_04712_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    grid = rank_grid(world)
    gbox = rank_boxes(cfg, world, args.scaling)[0]
    stream = torch.cuda.Stream()

    # --- build the context and the workload -------------------------------------------------
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (np.zeros(128, np.uint8))
            code = capi.load().dpd_nccl_unique_id(capi._ptr(buf))
            if code != 0:
                raise RuntimeError("dpd_nccl_unique_id failed")
            uid = torch.from_numpy(buf)
        uid = uid.cuda()
        dist.broadcast(uid, 0)
        uidh = uid.cpu().numpy().astype(np.uint8)
        ctx = capi.dpd_create_dist(gbox, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, rank, world,
                                   grid, uidh)
    else:
        ctx = capi.dpd_create(gbox, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    capi.dpd_set_stream(ctx, stream.cuda_stream)
    if args.force_kernel is not None:
        capi.dpd_set_option(ctx, "force_kernel", args.force_kernel)
    for opt in args.option:
        name, val = opt.split("=")
        capi.dpd_set_option(ctx, name, int(val))
    if cfg.body_f:
        capi.dpd_set_body_force(ctx, cfg.body_f)
    pos, vel, ids = rank_particles(cfg, world, rank, args.scaling)[:3]
    n_local = pos.shape[0]
    pos_h = torch.from_numpy(pos).pin_memory()
    vel_h = torch.from_numpy(vel).pin_memory()
    ids_h = torch.from_numpy(ids).pin_memory()
    capi.dpd_set_particles_ex(ctx, pos_h, vel_h, ids_h if world > 1 else None, 0)
    n_total = n_local * world
    if args.equilibrate > 0:
        # equilibrate the synthetic input (untimed), then take the equilibrated state as the
        # host input of the end-to-end leg as well
        capi.dpd_step(ctx, args.equilibrate)
        if world > 1:
            cnt = capi.dpd_get_count(ctx)
            pos_h = torch.empty((cnt, 3), dtype=torch.float32).pin_memory()
            vel_h = torch.empty((cnt, 3), dtype=torch.float32).pin_memory()
            ids_h = torch.empty((cnt,), dtype=torch.int32).pin_memory()
            capi.dpd_get_particles_ex(ctx, pos_h, vel_h, ids_h)
            n_local = cnt
        else:
            capi.dpd_get_particles(ctx, pos_h, vel_h)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # --- warm-up -----------------------------------------------------------------------
    capi.dpd_step(ctx, args.warmup)

    # --- timed region: K steps, inputs resident in HBM ----------------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = capi.dpd_get_launch_count(ctx)
    barrier()
    # all K steps are enqueued before the NVML sampler starts: its driver queries then run
    # while the GPU drains the queued steps (still inside the timed region) and cannot delay
    # a kernel launch (an NVML call contending with the launches cost up to ~3 % in a run)
    ev0.record(stream)
    capi.dpd_step_async(ctx, args.steps)
    ev1.record(stream)
    with ClockSampler(local_rank) as clocks:
        capi.dpd_sync(ctx)
    barrier()
    launches = capi.dpd_get_launch_count(ctx) - l0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_per_step = ms / args.steps
    value = n_total * args.steps / (ms * 1e-3)

    # --- per-kernel times (CUDA events around each launch, same stream), K steps ----------
    capi.dpd_set_timing(ctx, True)
    capi.dpd_step(ctx, args.steps)
    ktimes = capi.dpd_get_timing(ctx)
    capi.dpd_set_timing(ctx, False)
    per_kernel = {k: {"ms_per_launch": v[0] / max(v[1], 1), "launches": v[1]} for k, v in ktimes.items() if v[1]}
    step_kernel_ms = sum(v[0] for k, v in ktimes.items()) / args.steps

    # --- e2e: public API with host buffers (set -> step(K) -> get), copies inside ---------
    e2e = None
    if not args.no_e2e:
        out_pos = torch.empty((n_local, 3), dtype=torch.float32).pin_memory()
        out_vel = torch.empty((n_local, 3), dtype=torch.float32).pin_memory()
        out_ids = torch.empty((n_local * 2 + 1024,), dtype=torch.int32).pin_memory()
        big_p = big_v = None
        if world > 1:
            big_p = torch.empty((n_local * 2 + 1024, 3), dtype=torch.float32).pin_memory()
            big_v = torch.empty((n_local * 2 + 1024, 3), dtype=torch.float32).pin_memory()

        def fetch():
            if world > 1:
                capi.dpd_get_particles_ex(ctx, big_p, big_v, out_ids)
            else:
                capi.dpd_get_particles(ctx, out_pos, out_vel)

        # warm-up of the API path (first-touch of the pinned buffers and the copy engines),
        # untimed, as the device-timed region is warmed up
        capi.dpd_set_particles_ex(ctx, pos_h, vel_h, ids_h if world > 1 else None, 0)
        capi.dpd_step(ctx, 1)
        fetch()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        capi.dpd_set_particles_ex(ctx, pos_h, vel_h, ids_h if world > 1 else None, 0)
        capi.dpd_step_async(ctx, args.steps)
        fetch()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        te = torch.tensor([ems], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        h2d = n_local * (24 + (4 if world > 1 else 0))
        d2h = n_local * 24
        e2e = {"value": n_total * args.steps / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d * world / args.steps, "d2h_bytes_per_step": d2h * world / args.steps,
               "note": "set_particles(pinned host) + dpd_step(K) + get_particles(pinned host); "
                       "bytes amortised over the K steps of one call sequence"}

    # --- roofline --------------------------------------------------------------------------
    peaks, peaks_src = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    step_bytes_gbs = BYTES_PER_PARTICLE_STEP * (n_total / world) / (ms_per_step * 1e-3) / 1e9
    dom = max(per_kernel.items(), key=lambda kv: kv[1]["ms_per_launch"] * kv[1]["launches"])[0] if per_kernel else None
    roof = None
    if dom:
        roof = kernel_roofline(dom, per_kernel[dom]["ms_per_launch"], cfg, n_local, peaks, peaks_src)
        traffic, tsrc = kernel_traffic()
        t = traffic.get(dom)
        if t and t.get("workload") == cfg.name and int(t.get("n_local", -1)) == int(n_local):
            roof["traffic"] = t["dram_bytes"]
            roof["traffic_source"] = tsrc
            roof["traffic_vs_algorithmic"] = t["dram_bytes"] / (48.0 * n_local) if dom == "force" else \
                t["dram_bytes"] / max(1.0, KERNEL_BYTES.get(dom, 0.0) * n_local)
            if dom == "force" and t.get("smem_wavefronts"):
                # the co-limiting resource of the force kernel: shared-memory
                # wavefronts of the ncu capture over this run's launch time, against one
                # wavefront per cycle per SM
                clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
                sec = per_kernel[dom]["ms_per_launch"] * 1e-3
                wf = float(t["smem_wavefronts"])
                roof["smem_view"] = {"wavefronts_per_launch": wf, "achieved_wf_per_s": wf / sec,
                                     "peak_wf_per_s": 148 * clk, "frac": wf / sec / (148 * clk),
                                     "warp_instr_per_launch": t.get("warp_instr"),
                                     "issue_frac": (t["warp_instr"] / sec / (148 * 4 * clk)) if t.get("warp_instr") else None,
                                     "peak_source": "148 SM x 1 shared wavefront/cycle x sm_max_mhz"}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
           "vs_baseline": None, "dtype": "f32",
           "data": "synthetic: uniform positions, Maxwell-Boltzmann velocities, equilibrated for %d untimed steps"
                   % args.equilibrate,
           "config": config_block(cfg, args, world), "clocks": clocks.summary(), "gpu_launches": launches,
           "roofline": roof,
           "step_roofline": {"bound": "hbm", "bytes_per_particle_step": BYTES_PER_PARTICLE_STEP,
                             "achieved": step_bytes_gbs, "peak": hbm, "unit": "GB/s",
                             "frac": step_bytes_gbs / hbm, "peak_source": peaks_src},
           "kernels": per_kernel, "kernel_ms_per_step": step_kernel_ms, "e2e": e2e,
           "force_fallback_tiles": capi.dpd_get_stat(ctx, "fallback_tiles")}

    # --- the weak series' N = 1 point: the driver's scaling run times this same command at N =
    # 1 (BASELINE config 2, 64^3) and N > 1 (config 4, one 128^3 subdomain per GPU); the
    # config-4 workload on this one GPU, same timing rules, is recorded beside it
    if world == 1 and args.config == "eq64" and not args.no_weak_point:
        out["weak128_n1"] = weak_point(capi, stream, torch, max(5, min(args.steps, 20)), args.warmup,
                                       equilibrate=args.equilibrate)
        try:
            out["weak128_loopback_n1"] = weak_point(capi, stream, torch, max(5, min(args.steps, 20)), args.warmup,
                                                    loopback=True, equilibrate=args.equilibrate)
        except Exception as exc:  # noqa: BLE001  (a library built without NCCL)
            out["weak128_loopback_n1"] = {"error": repr(exc)}

    if rank == 0 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = oracle_sample_rate(cfg)
        except Exception as exc:  # noqa: BLE001
            out["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(out), file=_RESULT_OUT, flush=True)
    capi.dpd_destroy(ctx)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
