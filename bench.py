#!/usr/bin/env python
"""Benchmark: MPCRTile mixed-precision tiled Cholesky TFLOP/s on B200.

Default workload (north star: "n=131072 ... on 1 B200 with >=6x strong
scaling at 8 GPUs"; BASELINE.json configs[3]): n = 131072, tile 1024,
exponential (Matern nu=0.5) covariance of the first n points of a 363x363
unit grid, range 0.03; tile precision by band |i-j|: < b64 -> FP64, < b32 ->
FP32, else FP16 (default b64=1, b32=2).  The same n at every N, so the
driver's per-N values measure strong scaling (fixed total work).
configs[2] (n = 65536) is `--n 65536`.

A step is one full factorization chol(A) of the resident matrix (n^3/3
flops).  Inputs are restored from a pristine device copy before every step,
outside the CUDA-event pair; the 35 GB of tiles are far larger than the
126 MB L2, so no flush is needed.  e2e repeats the step through the public
C ABI from host buffers: host point coordinates -> device Matern generation
-> chol -> logdet read back.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python bench.py --workload gemm --prec half --n 8192     (config 2 lines)

Multi-GPU (torchrun, N > 1): BASELINE.json configs[3] — ONE n = 131072
matrix (--n overrides) 2D block-cyclic over a P x Q process grid
(P = largest divisor of N <= sqrt(N)), panel tiles broadcast by NCCL
(csrc/dist.cpp); strong scaling: value = n^3/3 / (max over ranks of the
step time).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def write_results(path, records, fmt=None):
    """BenchRecord-compatible results (io.hpp:11-20, io.cpp:97-126): CSV header
    op,n,precision,placement,reps,median_seconds,rel_frob_err with %.17g
    numbers, or a JSON array of the same objects (extra keys carry the
    roofline fields).  rel_frob_err is NaN / null where it was not measured."""
    fmt = fmt or ("json" if path.endswith(".json") else "csv")
    keys = ["op", "n", "precision", "placement", "reps", "median_seconds", "rel_frob_err"]
    if fmt == "csv":
        with open(path, "w") as f:
            f.write(",".join(keys) + "\n")
            for r in records:
                def num(v):
                    return "nan" if v is None else "%.17g" % v
                f.write(f"{r['op']},{r['n']},{r['precision']},{r['placement']},{r['reps']},"
                        f"{num(r['median_seconds'])},{num(r.get('rel_frob_err'))}\n")
    else:
        with open(path, "w") as f:
            json.dump(records, f, indent=2)
            f.write("\n")


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f), "measured"
    except OSError:
        return FALLBACK, "fallback"


def band_map(nt, b64, b32):
    i, j = np.indices((nt, nt))
    d = np.abs(i - j)
    return np.where(d < b64, 2, np.where(d < b32, 1, 0)).astype(np.int32)


def grid_points(n):
    side = int(np.ceil(np.sqrt(n)))
    side = max(side, 2)
    p = np.arange(n)
    return (p % side) / (side - 1), (p // side) / (side - 1), side


def flops_by_precision(nt, nb, g):
    """Algorithmic flops of the tiled right-looking Cholesky by destination
    tile precision: POTRF nb^3/3, TRSM nb^3, SYRK nb^3, GEMM 2 nb^3
    (SURVEY.md §8d).  Sums to n^3/3 up to O(n^2)."""
    f = np.zeros(3)
    b3 = float(nb) ** 3
    for k in range(nt):
        f[g[k, k]] += b3 / 3
        for i in range(k + 1, nt):
            f[g[i, k]] += b3
            f[g[i, i]] += b3
            for j in range(k + 1, i):
                f[g[i, j]] += 2 * b3
    return f


PIPES = ("tc_f16", "int8_digits", "dmma")


def flops_by_pipe(nt, nb, g):
    """The same algorithmic flops (SURVEY §8d counts) split by the pipe the
    scheduler (csrc/tile.cpp) runs each task on:
      tc_f16      FP16-destination GEMM/SYRK, FP32-destination updates whose two
                  panel tiles are FP16 (exact products, FP32 accumulate), the
                  FP16 panel TRSM (tcgen05 kind::f16);
      int8_digits FP64-destination updates with two FP16 panel tiles (exact
                  INT8 digit products, tcgen05 kind::i8) and FP32-destination
                  updates with FP32 (or FP32 + FP16) panel tiles (the same
                  digits; MPCR_OZAKI32=0 sends these to DMMA);
      dmma        every other FP32/FP64-destination update (panel tiles widened
                  exactly, FP64 accumulate), the FP32 and FP64 panel TRSM,
                  POTRF (mma.sync .f64)."""
    f = dict.fromkeys(PIPES, 0.0)
    oz32 = os.environ.get("MPCR_OZAKI32", "1") != "0"
    b3 = float(nb) ** 3
    for k in range(nt):
        f["dmma"] += b3 / 3
        for i in range(k + 1, nt):
            f["tc_f16" if g[i, k] == 0 else "dmma"] += b3
            for j in range(k + 1, i + 1):
                w = b3 if i == j else 2 * b3
                d, pa, pb = g[i, j], g[i, k], g[j, k]
                if d == 0:
                    f["tc_f16"] += w
                elif d == 1:
                    if pa == 0 and pb == 0:
                        f["tc_f16"] += w
                    elif oz32 and pa <= 1 and pb <= 1:
                        f["int8_digits"] += w
                    else:
                        f["dmma"] += w
                else:
                    f["int8_digits" if pa == 0 and pb == 0 else "dmma"] += w
    return f


def pipe_peaks(pk):
    """Per-pipe sustained peaks (TFLOP/s; INT8 in TOPS) for the blended
    roofline: the measured sustained BF16 GEMM rate (MEASURED_PEAKS.json) is
    the FP16 pipe; INT8 scales it by the tcgen05 kind::i8 / kind::f16 issue-rate
    ratio measured by tools/micro/tc_peak.cu (profiles/r02_pipe_peaks.json,
    clocks recorded); DMMA is the measured FP64 peak
    (tools/micro/fp64_peak.cu, same file)."""
    f16 = pk["bf16_tflops_sustained"]
    try:
        with open(os.path.join(ROOT, "profiles", "r02_pipe_peaks.json")) as fh:
            mp = json.load(fh)
        src = "profiles/r02_pipe_peaks.json"
    except (OSError, ValueError):
        mp, src = {"f16_burst": 1.0, "tf32_burst": 0.5, "i8_burst": 2.0, "dmma_tflops": 37.1}, "nominal ratios"
    r = {"tc_f16": f16, "int8_tops": f16 * mp["i8_burst"] / mp["f16_burst"], "dmma": mp["dmma_tflops"]}
    return r, src


class ClockSampler:
    """SM clocks, power and throttle reasons sampled DURING the timed region:
    NVML polled every 20 ms from a thread (short timed regions still get
    samples), else nvidia-smi -lms 200."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80}

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, power_w, reasons bitmask)
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.nvml = (pynvml, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((sm, mx, pw, rs))
            except Exception:  # noqa: BLE001
                pass
            self.stop.wait(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.nvml:
            sm = [x[0] for x in self.samples]
            mx = max([x[1] for x in self.samples], default=0)
            reasons = {nm for x in self.samples for nm, bit in self.BITS.items() if x[3] & bit}
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                    "reasons": sorted(reasons), "samples": len(sm),
                    "power_w_max": max([x[2] for x in self.samples], default=None), "source": "nvml 20 ms"}
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 200 ms"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def dist_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified mpnum library): bounded sample
# ---------------------------------------------------------------------------
def cpu_reference_chol(args, budget_s=20.0, steps=None):
    from oracle import oracle as orc

    if os.path.exists(orc.REF_SO):
        o, kind = orc.Ref(), "reference"
        cores = os.cpu_count() or 1
        o.set_num_threads(cores)
    else:
        o, kind, cores = orc.Port(), "port", 1
    n, nb = args.cpu_n, args.cpu_nb
    x, y, side = grid_points(n)
    if kind == "reference":
        cov = o.grid_matern(side, n, 0.5, args.range, 1.0, 2)
    else:
        d = np.hypot(x[:, None] - x[None], y[:, None] - y[None])
        cov = np.exp(-d / args.range)
    cov = cov + args.nugget * np.eye(n)
    g = band_map(n // nb, args.b64, args.b32)
    times = []
    t_end = time.perf_counter() + budget_s
    while True:
        t0 = time.perf_counter()
        o.tile_chol(n, nb, g, cov)
        times.append(time.perf_counter() - t0)
        if steps is not None and len(times) >= steps:
            break
        if steps is None and (time.perf_counter() > t_end or len(times) >= 5):
            break
    t = float(np.median(times))
    return {"value": n ** 3 / 3 / t / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind,
            "sample": f"MPCRTile chol n={n} nb={nb} (same band map and covariance family), "
                      f"median of {len(times)} runs, {t:.3f} s each",
            "seconds": t}, times


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's CPU tiled Cholesky on host cores."""
    if rank != 0:
        return
    from oracle import oracle as orc

    # warmup + timed steps, each one factorization of the bounded sample
    _, wt = cpu_reference_chol(args, steps=max(args.warmup, 1))
    base, times = cpu_reference_chol(args, steps=args.steps)
    n = args.cpu_n
    tot = float(np.sum(times))
    val = n ** 3 / 3 * len(times) / tot / 1e12
    base["value"] = val
    line = {
        "impl": "reference",
        "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / len(times) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "mixed(f64/f32/f16-storage, f32/f64 compute)", "data": "synthetic",
        "config": {"workload": f"MPCRTile mixed-precision Cholesky (CPU reference sample n={n}, "
                               f"tile {args.cpu_nb})", "n": n, "nb": args.cpu_nb,
                   "precision_map": f"|i-j|<{args.b64}:FP64, <{args.b32}:FP32, else FP16",
                   "matern_range": args.range},
        "cpu_baseline": base,
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_library": os.path.basename(orc.REF_SO) if base["kind"] == "reference" else "port",
    }
    print(json.dumps(line))


METRIC = "mixed-precision tiled Cholesky TFLOP/s"


def run_chol(args, world, rank, local):
    import paper_2406_02701_b200 as mp

    ctx = mp.Context(local)
    n = args.n or 131072
    nb = args.nb
    nt = n // nb
    g = band_map(nt, args.b64, args.b32)
    x, y, side = grid_points(n)
    grid = None
    if world > 1:
        import torch.distributed as tdist

        P = max(d for d in range(1, int(world ** 0.5) + 1) if world % d == 0)
        Q = world // P
        obj = [mp.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        grid = mp.ProcessGrid(rank, world, P, Q, obj[0], ctx)
    A0 = mp.MPCRTile(n, n, nb, nb, None, g, ctx, grid=grid)
    A = mp.MPCRTile(n, n, nb, nb, None, g, ctx, grid=grid)
    A0.fill_matern_points(x, y, 0.5, args.range, 1.0, args.nugget)
    ctx.synchronize()

    import torch

    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    def factor():
        mp.tile_chol(A)

    # warm-up
    for _ in range(args.warmup):
        A.copy_from(A0)
        factor()
    ctx.synchronize()
    # timed region (profiler off: the factorization replays as one CUDA graph)
    l0 = ctx.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    dist_barrier(world)
    torch.cuda.synchronize(local)
    ctx.synchronize()
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        for k in range(args.steps):
            A.copy_from(A0)
            ev[k][0].record(stream)
            factor()
            ev[k][1].record(stream)
        ctx.synchronize()
        torch.cuda.synchronize(local)
        t_wall = time.perf_counter() - t_wall0
    dist_barrier(world)
    launches = ctx.launch_count() - l0
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    ms_max = dist_max(ms, world)
    # one extra, profiled factorization (eager launches, per-kernel-class
    # event pairs) for the breakdown and the dominant kernel's rate
    A.copy_from(A0)
    ctx.synchronize()
    ctx.prof_reset()
    ctx.prof_enable(True)
    pe = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    pe[0].record(stream)
    factor()
    pe[1].record(stream)
    ctx.synchronize()
    prof_step_ms = pe[0].elapsed_time(pe[1])
    prof_pairs = ctx.prof_digit_products()
    ctx.prof_enable(False)
    cls_names = ["gemm_f16", "gemm_f32", "gemm_f64", "potrf_trtri", "trsm", "cast", "other", "gemm_f64_int8"]
    prof = {}
    for c, nm in enumerate(cls_names):
        t, cnt, work = ctx.prof_query(c)
        if cnt:
            prof[nm] = {"ms": t, "launches": cnt, "work": work,
                        "rate": work / (t * 1e-3) / 1e12 if t > 0 else None}
    logdet = A.logdet()
    accuracy = None if args.no_check else check_factor(args, A, g, x, y, n, nb, ctx, world, grid)
    # e2e through the C ABI from host buffers
    e2e_ms = None
    if not args.no_e2e:
        xs = np.ascontiguousarray(x)
        ys = np.ascontiguousarray(y)
        e2e = []
        for _ in range(max(1, args.steps)):
            ctx.synchronize()
            t0 = time.perf_counter()
            A.fill_matern_points(xs, ys, 0.5, args.range, 1.0, args.nugget)  # H2D + generate
            mp.tile_chol(A)
            A.logdet()  # D2H of the step's result (synchronises)
            e2e.append(time.perf_counter() - t0)
        e2e_ms = dist_max(float(np.mean(e2e)) * 1e3, world)
    pk, src = peaks()
    flops = n ** 3 / 3
    fp = flops_by_precision(nt, nb, g)
    fpipe = flops_by_pipe(nt, nb, g)
    f16 = prof.get("gemm_f16")
    roof = None
    if f16:
        # dominant kernel: the tcgen05 FP16 pair GEMM (trailing update, FP32 tiles
        # fed by FP16 panels, FP16 panel TRSM); algorithmic flops of exactly
        # those tasks (TRSM at nb^3) / the class's event-timed duration
        ach = fpipe["tc_f16"] / world / (f16["ms"] * 1e-3) / 1e12
        peak = pk["bf16_tflops_sustained"]
        traffic, tnote = None, None
        # the ncu capture of this n's bulk launch when one is committed
        tpath = None
        for cand in (f"r02_ncu_traffic_n{n}.json", f"r01_ncu_traffic_n{n}.json", "r01_ncu_traffic.json"):
            tpath = os.path.join(ROOT, "profiles", cand)
            if os.path.exists(tpath):
                break
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj["traffic_bytes_per_launch"]
            tnote = (f"dram read+write of one captured bulk launch ({tj['duration_us']} us, "
                     f"{tj.get('tiles', '?')} tiles), algorithmic "
                     f"{tj['algorithmic_bytes_per_launch']:.3g} B; {os.path.basename(tpath)}")
        except (OSError, KeyError, ValueError):
            pass
        roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "traffic": traffic, "traffic_note": tnote,
                "kernel": "gemm_tc2_kernel (tcgen05 kind::f16 cta_group::2: trailing update, FP32 tiles "
                          "fed by FP16 panels, FP16 panel TRSM)",
                "algorithmic_flops": fpipe["tc_f16"] / world,
                "peak_source": f"{src} bf16_tflops_sustained (FP16 = BF16 tensor rate)",
                "share_of_step": f16["ms"] / prof_step_ms}
    # Blended roofline: every algorithmic flop charged at the pipe that runs it
    # (flops_by_pipe); the INT8-digit FP64 tiles at the INT8 rate divided by
    # the digit-pair products the kernel actually issued (device counter).
    pp, pp_src = pipe_peaks(pk)
    pairs, ptiles = prof_pairs
    avg_pairs = pairs / ptiles if ptiles else 36.0
    t_pipe = {"tc_f16": fpipe["tc_f16"] / (pp["tc_f16"] * 1e12),
              "int8_digits": fpipe["int8_digits"] * avg_pairs / (pp["int8_tops"] * 1e12),
              "dmma": fpipe["dmma"] / (pp["dmma"] * 1e12)}
    tmin = sum(t_pipe.values()) / world
    value = flops / (ms_max * 1e-3) / 1e12  # one matrix over all ranks (strong scaling)
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "mixed(f64/f32/f16 tiles; f16: tcgen05 f16 f32-acc; f32: tcgen05 f16 (f16 panels) / "
                 "DMMA; f64: exact INT8 digits (f16 panels) / DMMA)",
        "data": "synthetic",
        "config": {"workload": f"MPCRTile mixed-precision Cholesky n={n}, tile {nb}" +
                               (f", 2D block-cyclic {grid.P}x{grid.Q}" if grid else ", 1 GPU"),
                   "n": n, "nb": nb, "precision_map": f"|i-j|<{args.b64}:FP64, <{args.b32}:FP32, else FP16",
                   "tiles_by_precision": {p: int((g == i).sum()) for i, p in enumerate(["f16", "f32", "f64"])},
                   "covariance": f"Matern nu=0.5 range {args.range} sigma2 1 nugget {args.nugget}, "
                                 f"first {n} points of a {side}x{side} unit grid",
                   "fp32_method": "FP16 panels: tcgen05 kind::f16 (exact products, FP32 accumulate); "
                                  + ("FP32 panels: 7-bit digits of the FP16/FP32 panel rows (exact to 2^-41 of "
                                     "the row max), tcgen05 kind::i8, FP64 combination, one rounding"
                                     if os.environ.get("MPCR_OZAKI32", "1") != "0" else
                                     "FP32 panels: DMMA (widened exactly, FP64 accumulate, one rounding)"),
                   "steps": "paired (two panels per tensor-core tile pass)"
                            if os.environ.get("MPCR_PAIR_STEPS", "1") != "0" else "one panel per pass",
                   "fp64_method": "FP16 panels: exact 7-bit digit slicing, tcgen05 kind::i8 (Ozaki); "
                                  "FP32/FP64 panels: DMMA",
                   "l2": "inputs 8+ GB >> 126 MB L2 (no flush needed)",
                   "parallelism": f"2D block-cyclic {grid.P}x{grid.Q}, NCCL panel broadcast"
                                  if grid else "single GPU"},
        "roofline": roof,
        "blended_roofline": {"t_min_ms": tmin * 1e3, "frac": tmin / (ms_max * 1e-3),
                             "flops_by_pipe": fpipe, "t_min_ms_by_pipe": {k: v * 1e3 / world for k, v in t_pipe.items()},
                             "flops_by_dest_precision": {"f16": fp[0], "f32": fp[1], "f64": fp[2]},
                             "peaks": {"tc_f16_tflops": pp["tc_f16"], "int8_tops": pp["int8_tops"],
                                       "dmma_tflops": pp["dmma"]},
                             "int8_digit_pairs_per_tile_product": avg_pairs,
                             "peak_source": f"{src} bf16 sustained x tcgen05 kind ratios ({pp_src})",
                             "note": "T_min = sum over pipes of algorithmic flops / that pipe's sustained peak "
                                     "(INT8-digit FP64 tiles: flops x digit pairs issued / INT8 peak); "
                                     "frac = T_min / step time"},
        "breakdown": {"note": "one extra eager (non-graph) factorization with per-launch event "
                              "pairs; classes overlap in time across the three streams",
                      "step_ms": prof_step_ms, "classes": prof},
        "gpu_launches": launches,
        "wall_ms_per_step": t_wall / args.steps * 1e3,
        "logdet": logdet,
        "accuracy": accuracy,
        "rel_err": accuracy["sampled_backward_error"] if accuracy else None,
        "clocks": clk.summary(),
    }
    if e2e_ms is not None:
        line["e2e"] = {"value": flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                       "h2d_bytes_per_step": 2 * n * 8, "d2h_bytes_per_step": 8,
                       "ms_per_step": e2e_ms,
                       "path": "host (x,y) -> mp_tile_fill_matern_points -> mp_tile_chol -> mp_tile_logdet"}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"], _ = cpu_reference_chol(args)
    if rank == 0:
        print(json.dumps(line))
        if args.results:
            steps_s = sorted(a.elapsed_time(b) * 1e-3 for a, b in ev)
            write_results(args.results, [{
                "op": "tile_chol", "n": n, "precision": f"mixed(b64={args.b64};b32={args.b32})",
                "placement": f"gpu:{world}", "reps": args.steps,
                "median_seconds": steps_s[len(steps_s) // 2],
                "rel_frob_err": accuracy["sampled_backward_error"] if accuracy else None,
                "tflops": value, "blended_roofline_frac": line["blended_roofline"]["frac"],
                "roofline_frac": (line["roofline"] or {}).get("frac"),
                "e2e_tflops": line.get("e2e", {}).get("value")}])
    ctx.synchronize()


def check_factor(args, A, g, x, y, n, nb, ctx, world, grid):
    """Error attached to the timing (mpnum_cli.cpp:59-63,174 writes rel_frob_err
    with every bench record): the factor is 9-35 GB, so it is checked on a
    sample (paper_2406_02701_b200/verify.py):
      * sampled backward error ||(LL^T - A)[R,R]||_F / ||A[R,R]||_F over 256 rows
        (clusters spread over the matrix, the last tile row included, + random);
      * the leading m x m block (m = min(n, 8192)) equal bit for bit to a
        separate factorization of the leading sub-problem, which
        tests/test_gpu_tile_nb1024.py checks against the CPU oracle."""
    import paper_2406_02701_b200 as mp
    from paper_2406_02701_b200 import verify

    t0 = time.perf_counter()
    rows = verify.sample_rows(n, nb, clusters=16, width=8, extra=128)
    Lr = A.get_rows(rows)
    if world > 1:  # every rank holds its own tiles, zeros elsewhere
        import torch
        import torch.distributed as tdist

        tt = torch.from_numpy(Lr).cuda()
        tdist.all_reduce(tt)
        Lr = tt.cpu().numpy()
    res = verify.sampled_residual(None, x, y, rows, nb, g, args.range, 1.0, args.nugget, L_rows=Lr)
    m = min(n, 8192 // nb * nb)
    lead = rows[rows < m]
    same = None
    if m < n and lead.size:
        sub = mp.MPCRTile(m, m, nb, nb, None, g[:m // nb, :m // nb], ctx)
        sub.fill_matern_points(x[:m], y[:m], 0.5, args.range, 1.0, args.nugget)
        mp.tile_chol(sub)
        same = verify.leading_rows_equal(Lr[np.searchsorted(rows, lead)], sub.get_rows(lead))
        sub.close()
    return {"sampled_backward_error": res["normwise"], "max_entry_backward_error": res["max_entry"],
            "sample_rows": res["rows"], "sample_entries": res["entries"],
            "leading_block": m, "leading_block_bitwise_equal": same,
            "check_seconds": time.perf_counter() - t0,
            "note": "normwise ||(LL^T-A)[R,R]||_F/||A[R,R]||_F on the sample R; the leading block is the "
                    "factor of the leading sub-problem (checked vs the CPU oracle in "
                    "tests/test_gpu_tile_nb1024.py); bound there: 4*(n/8192)*oracle value at n=8192"}


def cpu_info():
    """Host CPU model and the thread count a reference run may use."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def _ref_lib():
    """The reference CPU library for a cpu_baseline leg (oracle/_ref, else the port)."""
    from oracle import oracle as orc

    if os.path.exists(orc.REF_SO):
        o = orc.Ref()
        o.set_num_threads(cpu_info()[1])
        return o, "reference", cpu_info()[1]
    return orc.Port(), "port", 1


class L2Flush:
    """Writes a 512 MB buffer (> the 126 MB L2) between timed iterations of a
    workload whose operands fit in L2."""

    def __init__(self, enabled, stream):
        import torch

        self.buf = torch.empty(256 << 20, dtype=torch.float16, device="cuda") if enabled else None
        self.stream = stream

    def __call__(self):
        if self.buf is not None:
            import torch

            with torch.cuda.stream(self.stream):
                self.buf.fill_(0.0)


GEMM_PEAK_NOTE = {0: "tcgen05 kind::f16: measured bf16 burst (MEASURED_PEAKS.json)",
                  1: "3xTF32: measured bf16 burst x tcgen05 tf32/f16 ratio / 3 (profiles/r02_pipe_peaks.json)",
                  2: "DMMA: measured FP64 peak (profiles/r02_pipe_peaks.json)"}


def gemm_peak(p, pc, pk):
    try:
        with open(os.path.join(ROOT, "profiles", "r02_pipe_peaks.json")) as fh:
            mp_ = json.load(fh)
    except (OSError, ValueError):
        mp_ = {"f16_burst": 1.0, "tf32_burst": 0.5, "i8_burst": 2.0, "dmma_tflops": 37.1}
    if p == 0 and pc == 2:
        return pk["bf16_tflops"] * mp_["i8_burst"] / mp_["f16_burst"], "INT8 digits: measured bf16 burst x i8/f16 ratio (TOPS; FP64-equivalent divides by the digit pairs)"
    if p == 0:
        return pk["bf16_tflops"], GEMM_PEAK_NOTE[0]
    if p == 1:
        return pk["bf16_tflops"] * mp_["tf32_burst"] / mp_["f16_burst"] / 3, GEMM_PEAK_NOTE[1]
    return mp_["dmma_tflops"], GEMM_PEAK_NOTE[2]


def run_gemm(args, world, rank, local):
    """BASELINE.json configs[0] / [1]: linalg::gemm (linalg.cpp:316-357) on
    n x n x n MPArrays, C = A B (alpha 1, beta 0, NN: mpnum_cli.cpp:117-120).
    Inputs are the reference's acceptance-test stream (acceptance.cpp:30-36,
    :158-162): A = the first n^2 draws of Rng(1000 + n) column-major, B the
    next n^2, rounded to the precision on upload.  rel_frob_err is against the
    same product at double precision (mpnum_cli.cpp:59-63,174 does the same)."""
    import torch

    import paper_2406_02701_b200 as mp

    ctx = mp.Context(local)
    n = args.n or 8192
    p = mp.parse_precision(args.prec)
    pc = mp.parse_precision(args.cprec) if args.cprec else p
    A = mp.random_uniform_matrix(n, n, 1000 + n)
    B = mp.random_uniform_matrix(n, n, 1000 + n, skip=n * n)
    dA, dB = mp.MPArray.from_numpy(A, p, ctx), mp.MPArray.from_numpy(B, p, ctx)
    dC = mp.MPArray.zeros_matrix(n, n, pc, ctx)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))
    es = {0: 2, 1: 4, 2: 8}
    in_l2 = 2 * n * n * es[int(p)] + n * n * es[int(pc)] < 126e6
    flush = L2Flush(in_l2, stream)
    for _ in range(args.warmup):
        mp.linalg.gemm(dA, dB, dC)
    ctx.synchronize()
    l0 = ctx.launch_count()
    evs = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mp.linalg.gemm(dA, dB, dC)
            e1.record(stream)
            evs.append((e0, e1))
        ctx.synchronize()
    launches = ctx.launch_count() - l0
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    tf = 2 * n ** 3 / (ms * 1e-3) / 1e12
    # error as mpnum_cli reports it: vs the same product at double precision
    d64 = mp.MPArray.zeros_matrix(n, n, mp.Precision.Double, ctx)
    mp.linalg.gemm(mp.MPArray.from_numpy(A, p, ctx).converted(mp.Precision.Double),
                   mp.MPArray.from_numpy(B, p, ctx).converted(mp.Precision.Double), d64)
    C64, Cg = d64.to_numpy(), dC.to_numpy()
    rel = float(np.linalg.norm(Cg - C64) / np.linalg.norm(C64))
    # e2e: host doubles -> device (set_linear rounding) -> gemm -> host doubles
    e2e = []
    for _ in range(max(1, min(args.steps, 10))):
        ctx.synchronize()
        t0 = time.perf_counter()
        a_ = mp.MPArray.from_numpy(A, p, ctx)
        b_ = mp.MPArray.from_numpy(B, p, ctx)
        c_ = mp.MPArray.zeros_matrix(n, n, pc, ctx)
        mp.linalg.gemm(a_, b_, c_)
        c_.to_numpy()
        e2e.append(time.perf_counter() - t0)
        for h in (a_, b_, c_):
            h.close()
    e2e_s = float(np.median(e2e))
    pk, src = peaks()
    peak, peak_src = gemm_peak(int(p), int(pc), pk)
    ach = tf
    line = {"metric": "per-precision GEMM TFLOP/s", "value": tf, "unit": "TFLOP/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "replicas only", "vs_baseline": None, "dtype": f"{args.prec}" + (f"->{args.cprec}" if args.cprec else ""),
            "data": "synthetic (reference Rng(1000+n) uniform stream, acceptance.cpp:158-162)",
            "config": {"workload": f"linalg::gemm {n}x{n}x{n} {mp.Precision(p).name} inputs, "
                                   f"{mp.Precision(pc).name} C, NN, alpha 1 beta 0", "n": n,
                       "l2": "flushed between iterations (512 MB write)" if in_l2 else "operands > 126 MB L2"},
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s" if not (p == 0 and pc == 2) else "TOPS",
                         "frac": ach / peak if not (p == 0 and pc == 2) else None, "peak_source": f"{src}: {peak_src}",
                         "traffic": None},
            "rel_frob_err": rel, "gpu_launches": launches, "clocks": clk.summary(),
            "e2e": {"value": 2 * n ** 3 / e2e_s / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 2 * n * n * 8,
                    "d2h_bytes_per_step": n * n * 8, "ms_per_step": e2e_s * 1e3,
                    "path": "host doubles -> mp_array_from_doubles (x2) -> mp_gemm -> mp_array_to_doubles"}}
    if not args.no_cpu:
        o, kind, cores = _ref_lib()
        ns = min(n, args.cpu_n if args.cpu_n else 2048)
        As, Bs = A[:ns, :ns].copy(order="F"), B[:ns, :ns].copy(order="F")
        from oracle.oracle import round_to
        As, Bs = round_to(As, int(p)), round_to(Bs, int(p))
        ts = []
        t_end = time.perf_counter() + 20
        while len(ts) < 3 and (not ts or time.perf_counter() < t_end):
            t0 = time.perf_counter()
            o.gemm(int(p), int(p), int(pc), As, Bs, np.zeros((ns, ns)))
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        model, _ = cpu_info()
        line["cpu_baseline"] = {"value": 2 * ns ** 3 / t / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind,
                                "cpu": model,
                                "sample": f"reference linalg::gemm {ns}^3 same precisions, median of {len(ts)}: {t:.3f} s"
                                          + ("" if ns == n else f"; n^3 projection to n={n}: {t * (n / ns) ** 3:.1f} s (projected, not run)")}
    print(json.dumps(line))


def sample_gp_gpu(ctx, x, y, n, nb, range_, nugget):
    """sample_gp (workloads.cpp:41-49) at the reference's criterion-6 / CLI seed
    (acceptance.cpp:325-326, mpnum_cli.cpp:397): z = L eps, L the FP64 Cholesky
    factor of the true covariance, eps = Rng(4).normal() (the reference stream,
    mp_rng_normal).  The factor runs on the GPU (all-FP64 MPCRTile) since the
    host cannot factor n = 65536; returns z and the exact-factor NLL
    0.5 (eps'eps + logdet) + 0.5 n log 2 pi (w = L^-1 z = eps)."""
    import paper_2406_02701_b200 as mp

    nt = n // nb
    t64 = mp.MPCRTile(n, n, nb, nb, None, np.full((nt, nt), 2, np.int32), ctx)
    t64.fill_matern_points(x, y, 0.5, range_, 1.0, nugget)
    mp.tile_chol(t64)
    ld64 = t64.logdet()
    eps = mp.rng_normal(4, n)
    e = mp.MPCRTile(n, 1, nb, 1, eps, np.full((nt, 1), 2, np.int32), ctx)
    z_t = mp.MPCRTile(n, 1, nb, 1, None, np.full((nt, 1), 2, np.int32), ctx)
    mp.tile_gemm(t64, e, z_t, False, False, 1.0, 0.0)
    z = z_t.to_numpy().ravel()
    for h in (t64, e, z_t):
        h.close()
    nll64 = 0.5 * float(eps @ eps) + 0.5 * ld64 + 0.5 * n * np.log(2 * np.pi)
    return z, nll64, ld64


def run_nll(args, world, rank, local):
    """BASELINE.json configs[4]: Gaussian log-likelihood of a Matern GP at the
    given locations (workloads.cpp:74-87): covariance generated on the device
    from the points -> jittered mixed-precision tiled Cholesky -> forward solve
    -> logdet + quadratic form -> nll to the host.  One step = one likelihood
    evaluation; z = sample_gp(cov_true, Rng(4)) as in the reference."""
    import torch

    import paper_2406_02701_b200 as mp

    ctx = mp.Context(local)
    n = args.n or 65536
    nb = args.nb
    g = band_map(n // nb, args.b64, args.b32)
    x, y, side = grid_points(n)
    z, nll64, ld64 = sample_gp_gpu(ctx, x, y, n, nb, args.range, args.nugget)
    A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    st = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    def step():
        A.fill_matern_points(x, y, 0.5, args.range, 1.0, args.nugget)
        return mp.gaussian_nll(z, A, jitter=1e-6, max_jitter=1e-3)

    for _ in range(args.warmup):
        r = step()
    ctx.synchronize()
    l0 = ctx.launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(st)
            r = step()  # returns after the nll is on the host
            e1.record(st)
            ctx.synchronize()
            times.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    launches = ctx.launch_count() - l0
    ms = float(np.mean([t[0] for t in times]))
    wall = float(np.mean([t[1] for t in times]))
    flops = n ** 3 / 3
    line = {
        "metric": "Gaussian log-likelihood evaluation (Matern -> tiled chol -> solve -> logdet) TFLOP/s",
        "value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "mixed(f64/f32/f16 tiles)",
        "data": "synthetic: z = sample_gp(cov_true, Rng(4)) (workloads.cpp:41-49; reference Rng stream)",
        "config": {"workload": f"gaussian_nll n={n}, tile {nb}, Matern nu=0.5 range {args.range}, "
                               f"jitter 1e-6 (x10 up to 1e-3)",
                   "n": n, "nb": nb, "precision_map": f"|i-j|<{args.b64}:FP64, <{args.b32}:FP32, else FP16",
                   "l2": "covariance regenerated in HBM every step (> 126 MB L2)"},
        "nll": r["nll"], "logdet": r["logdet"], "jitter_used": r["jitter"],
        "nll_fp64_factor": nll64, "rel_err": abs(r["nll"] - nll64) / abs(nll64),
        "rel_err_note": "vs the NLL of the exact (all-FP64) factor of the same covariance",
        "gpu_launches": launches,
        "e2e": {"value": flops / (wall * 1e-3) / 1e12, "unit": "TFLOP/s",
                "h2d_bytes_per_step": 3 * n * 8, "d2h_bytes_per_step": 32, "ms_per_step": wall,
                "path": "host (x, y, z) -> mp_tile_fill_matern_points -> mp_tile_gaussian_nll -> nll"},
        "clocks": clk.summary(),
    }
    if not args.no_cpu:
        o, kind, cores = _ref_lib()
        if kind == "reference":
            ns = min(n, 2048)
            xs, ys, sside = grid_points(ns)
            cov = np.exp(-np.hypot(xs[:, None] - xs[None], ys[:, None] - ys[None]) / args.range)
            zs = z[:ns].copy()
            ts = []
            while len(ts) < 3:
                t0 = time.perf_counter()
                o.gaussian_nll(1, zs, cov)
                ts.append(time.perf_counter() - t0)
            t = float(np.median(ts))
            line["cpu_baseline"] = {
                "value": ns ** 3 / 3 / t / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind, "cpu": cpu_info()[0],
                "sample": f"reference stats::gaussian_nll(z, cov, single) n={ns} dense (chol single-threaded "
                          f"in the reference), median of 3: {t:.3f} s; n^3 projection to n={n}: "
                          f"{t * (n / ns) ** 3 / 3600:.1f} h (projected, not run)"}
    print(json.dumps(line))


def run_mle(args, world, rank, local):
    """matern_mle (workloads.cpp:89-110) with every likelihood
    evaluated on the GPU: Nelder-Mead (host, deterministic) over (log range,
    log sigma2), start log(range/2), log(0.5).  One step = one full fit."""
    import torch  # noqa: F401

    import paper_2406_02701_b200 as mp

    ctx = mp.Context(local)
    n = args.n or 65536
    nb = args.nb
    g = band_map(n // nb, args.b64, args.b32)
    x, y, side = grid_points(n)
    z = np.random.default_rng(5).standard_normal(n)  # white-noise observations (synthetic)
    A = mp.MPCRTile(n, n, nb, nb, None, g, ctx)
    fits = []
    for _ in range(max(1, min(args.steps, 20))):
        ctx.synchronize()
        t0 = time.perf_counter()
        r = mp.matern_mle(A, x, y, z, np.log(args.range / 2), np.log(0.5), max_iter=200, tol=1e-4)
        fits.append((time.perf_counter() - t0, r))
    secs = float(np.median([f[0] for f in fits]))
    r = fits[-1][1]
    print(json.dumps({
        "metric": "matern_mle fit time (Nelder-Mead, GPU likelihood)", "value": secs, "unit": "s",
        "n_gpus": 1, "steps": len(fits), "warmup": 0, "ms_per_step": secs * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "mixed(f64/f32/f16 tiles)", "data": "synthetic",
        "config": {"workload": f"matern_mle n={n}, tile {nb}, nu=0.5", "n": n, "nb": nb,
                   "precision_map": f"|i-j|<{args.b64}:FP64, <{args.b32}:FP32, else FP16"},
        "result": r,
    }))


def run_cast(args, world, rank, local):
    """BASELINE.json configs[1] cast line: MPArray::converted (array.cpp:187-191)
    of an n x n array, pin -> pout, as an HBM stream (n^2 (s_in + s_out) bytes).
    Input values: the reference Rng(1000 + n) uniform stream scaled to span
    the destination's range, so FP16 destinations see normals, subnormals and
    overflow to inf (bit-exactness over every pattern is in the tests)."""
    import torch

    import paper_2406_02701_b200 as mp

    ctx = mp.Context(local)
    n = args.n or 8192
    pin, pout = (mp.parse_precision(x) for x in args.cast.split(":"))
    es = {0: 2, 1: 4, 2: 8}
    u = mp.rng_uniform(1000 + n, n * n)
    vals = np.ldexp(u - 0.5, (np.floor(u * 1e6) % 48 - 24).astype(np.int32))  # |x| from 2^-25 to 2^23
    with np.errstate(over="ignore"):
        raw = {0: vals.astype(np.float16).view(np.uint16), 1: vals.astype(np.float32), 2: vals}[int(pin)]
    a = mp.MPArray.from_storage(raw.reshape((n, n), order="F"), n, n, pin, ctx)
    b = mp.MPArray.zeros_matrix(n, n, pout, ctx)
    lib, C = mp.lib(), __import__("ctypes")
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))
    for _ in range(args.warmup):
        lib.mp_convert(ctx.h, a.h, b.h)
    ctx.synchronize()
    l0 = ctx.launch_count()
    evs = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            lib.mp_convert(ctx.h, a.h, b.h)
            e1.record(stream)
            evs.append((e0, e1))
        ctx.synchronize()
    launches = ctx.launch_count() - l0
    ms = float(np.mean([x.elapsed_time(y) for x, y in evs]))
    byts = n * n * (es[int(pin)] + es[int(pout)])
    gbs = byts / (ms * 1e-3) / 1e9
    # e2e through the public API: raw source storage up, convert, raw result down
    e2e = []
    for _ in range(max(1, min(args.steps, 20))):
        ctx.synchronize()
        t0 = time.perf_counter()
        a_ = mp.MPArray.from_storage(raw.reshape((n, n), order="F"), n, n, pin, ctx)
        b_ = a_.converted(pout)
        b_.storage()
        e2e.append(time.perf_counter() - t0)
        a_.close()
        b_.close()
    e2e_s = float(np.median(e2e))
    pk, src = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_casts.json")) as fh:
            traffic = json.load(fh).get(f"{args.cast}@{n}", {}).get("dram_bytes")
    except (OSError, ValueError):
        pass
    line = {"metric": "precision conversion GB/s", "value": gbs, "unit": "GB/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "replicas only", "vs_baseline": None, "dtype": args.cast.replace(":", "->"),
            "data": "synthetic (reference Rng(1000+n) stream, scaled)",
            "config": {"workload": f"MPArray::converted {n}x{n} {args.cast}", "n": n, "bytes_per_step": byts,
                       "l2": "operands > 126 MB L2" if byts > 126e6 else "operands fit L2 (small n)"},
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / pk["hbm_gbs"], "peak_source": f"{src} hbm_gbs (copy)",
                         "algorithmic_bytes": byts, "traffic": traffic},
            "gpu_launches": launches, "clocks": clk.summary(),
            "e2e": {"value": byts / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": n * n * es[int(pin)],
                    "d2h_bytes_per_step": n * n * es[int(pout)], "ms_per_step": e2e_s * 1e3,
                    "path": "host raw -> mp_array_upload -> mp_convert -> mp_array_download"}}
    if not args.no_cpu:
        o, kind, _ = _ref_lib()
        ts = []
        flat = np.ascontiguousarray(raw.ravel())
        while len(ts) < 3:
            t0 = time.perf_counter()
            o.convert(int(pin), int(pout), flat)
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        line["cpu_baseline"] = {"value": byts / t / 1e9, "unit": "GB/s", "cores": 1, "kind": kind, "cpu": cpu_info()[0],
                                "sample": f"reference MPArray::converted on the same {n}x{n} array (single-threaded "
                                          f"in the reference), median of 3: {t:.3f} s"}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="chol", choices=["chol", "gemm", "cast", "nll", "mle"])
    ap.add_argument("--cast", default="double:half")
    ap.add_argument("--n", type=int, default=None,
                    help="matrix order (default 131072 for the chol at every N; per-workload defaults otherwise)")
    ap.add_argument("--nb", type=int, default=1024)
    ap.add_argument("--b64", type=int, default=1)
    ap.add_argument("--b32", type=int, default=2)
    ap.add_argument("--range", type=float, default=0.03)
    ap.add_argument("--nugget", type=float, default=0.0)
    ap.add_argument("--prec", default="half")
    ap.add_argument("--cprec", default=None, help="gemm: C precision (default: --prec)")
    ap.add_argument("--ta", action="store_true")
    ap.add_argument("--tb", action="store_true")
    ap.add_argument("--beta", type=float, default=0.0)
    ap.add_argument("--cpu-n", type=int, default=2048)
    ap.add_argument("--cpu-nb", type=int, default=256)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the sampled accuracy check")
    ap.add_argument("--results", default=None,
                    help="also write a BenchRecord CSV/JSON (io.hpp:11-20) to this path")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
    elif args.workload == "gemm":
        run_gemm(args, world, rank, local)
    elif args.workload == "cast":
        run_cast(args, world, rank, local)
    elif args.workload == "nll":
        run_nll(args, world, rank, local)
    elif args.workload == "mle":
        run_mle(args, world, rank, local)
    else:
        run_chol(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
