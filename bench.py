#!/usr/bin/env python3
"""Benchmark: convective columns/s (deep + shallow, fp64) on B200.

One step = one pass of the hot path (trigger + compaction, deep plume,
shallow + deep zero-fill) over the whole column block, inputs resident in
HBM.  At N GPUs (torchrun, one rank per GPU) the f02 grid is partitioned into
N contiguous ranges balanced by estimated cost (cvg_plan_partition); there is
no collective on the data path -- torch.distributed/NCCL is used only for the
barrier and the max-over-ranks of the device timings.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's own
CPU implementation (oracle/_ref: physics.cpp + sched.cpp compiled from the
reference sources, run through its run_parallel dynamic scheduler on all host
threads) on the same workload and prints the same line with impl=reference.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "convective columns/sec (deep+shallow, fp64)"
UNIT = "columns/s"
HBM_FALLBACK_GBS = 6650.0
L2_BYTES = 126 * 2 ** 20


# ---------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws, backend):
    if ws <= 1:
        return None
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend=backend)
    return dist


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# FLOP / byte model; per-column integers come from the
# step's own outputs (work_units, exited_early), which match the oracle's.
def flop_model(L, deep_work, deep_exited, sh_work, sh_exited):
    trig = deep_exited == 0
    U = deep_work[trig].astype(np.float64)
    deep_flops = float(np.sum(159.0 * L + 37.0 * U))
    P = (sh_work // L).astype(np.float64)
    surv = (sh_exited == 0)
    sh_flops = float(np.sum(P * (9 * L + 8 + 29) + (P >= 2) * L * (3 + 29) + surv * (6 * L + 3 + 29)))
    return deep_flops, sh_flops, int(trig.sum())


def bytes_model(n, L, n_trig):
    per_col = 8 + 2 * 8 * L + 2 * (2 * 8 * L + 8 + 8 + 1)   # 1,482 B at L = 30
    deep_only = n_trig * (8 + 2 * 8 * L + 2 * 8 * L + 8 + 8 + 1)
    return n * per_col, per_col, deep_only


# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self._nv:
            return None
        r = [name for bit, name in self.REASONS.items() if self.reasons & bit and name != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": r, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def cpu_reference_time(s, T, q, thr, threads, variant=0, reps=3, warm=1):
    """Reference run_parallel (Dynamic, omp_chunk 1) deep + shallow wall time,
    median of `reps` after `warm` warm-ups."""
    import oracle as O
    opts = O.Options(variant=variant, activity_threshold=thr)
    walls = []
    for i in range(warm + reps):
        w = O.ref_time_run_parallel(s, T, q, opts, n_threads=threads, strategy=2, omp_chunk=1)
        if i >= warm:
            walls.append(w["deep"] + w["shallow"])
    return float(np.median(walls))


def cpu_port_time(s, T, q, thr, variant=0):
    import oracle as O
    opts = O.Options(variant=variant, activity_threshold=thr)
    t0 = time.perf_counter()
    O.convection("deep", s, T, q, opts)
    O.convection("shallow", s, T, q, opts)
    return time.perf_counter() - t0


def strided_sample(s, T, q, stride):
    idx = np.arange(0, s.size, stride)
    return np.ascontiguousarray(s[idx]), np.ascontiguousarray(T[:, idx]), np.ascontiguousarray(q[:, idx])


def cpu_baseline(s, T, q, thr, variant, target_s=10.0):
    """Bounded sample of the workload on the host cores (rank 0, N=1)."""
    import oracle as O
    threads = os.cpu_count() or 1
    if O.ref_available():
        # calibrate on a small strided sample, then size the sample so one
        # timed rep is ~target_s / 4 seconds of wall
        cal_stride = max(1, s.size // 20000)
        cs, cT, cq = strided_sample(s, T, q, cal_stride)
        t = cpu_reference_time(cs, cT, cq, thr, threads, variant, reps=1, warm=0)
        rate = cs.size / max(t, 1e-6)
        want = int(min(s.size, max(2000, rate * target_s / 4)))
        stride = max(1, s.size // want)
        ss, sT, sq = strided_sample(s, T, q, stride)
        wall = cpu_reference_time(ss, sT, sq, thr, threads, variant, reps=3, warm=1)
        return {"value": ss.size / wall, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"every {stride}th column of the same grid ({ss.size} columns), reference "
                          f"run_parallel Dynamic(omp_chunk=1) deep+shallow, median of 3 after 1 warm-up",
                "wall_s": wall}
    stride = max(1, s.size // 20000)
    ss, sT, sq = strided_sample(s, T, q, stride)
    wall = cpu_port_time(ss, sT, sq, thr, variant)
    return {"value": ss.size / wall, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"every {stride}th column ({ss.size} columns), serial C oracle", "wall_s": wall}


def workload_config(args, n_columns, levels, thr):
    """The `config` dict -- identical in both arms (the driver compares it)."""
    return {"workload": args.config, "n_columns": int(n_columns), "levels": int(levels),
            "activity_threshold": float(thr), "variant": int(args.variant)}


def serial_reference(s, T, q, thr, variant, target_s=2.0):
    """The reference's serial chunk drivers deep_convection + shallow_convection
    (physics.cpp:227-245) on one core, on a strided sample (BASELINE.md 2:
    the serial number beside run_parallel); median of 3."""
    import oracle as O
    opts = O.Options(variant=variant, activity_threshold=thr)
    stride = max(1, s.size // 20000)
    cs, cT, cq = strided_sample(s, T, q, stride)
    t0 = time.perf_counter()
    O.ref_convection("deep", cs, cT, cq, opts)
    O.ref_convection("shallow", cs, cT, cq, opts)
    rate = cs.size / max(time.perf_counter() - t0, 1e-6)
    stride = max(1, s.size // int(min(s.size, max(2000, rate * target_s))))
    ss, sT, sq = strided_sample(s, T, q, stride)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        O.ref_convection("deep", ss, sT, sq, opts)
        O.ref_convection("shallow", ss, sT, sq, opts)
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    return {"value": ss.size / wall, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"every {stride}th column ({ss.size} columns), reference serial deep_convection + "
                      f"shallow_convection, median of 3"}


def parity_against_reference(s, T, q, thr, variant, deep, sh, stats):
    """The step's outputs (full grid) against the reference's own run_parallel
    outputs on the same grid (the north star's rule: flags and work_units
    exact, fp64 fields within 1e-10 relative or 1e-14 absolute)."""
    import oracle as O
    opts = O.Options(variant=variant, activity_threshold=thr)
    rec = {"columns": int(s.size), "rule": "flags and work_units exact; tend_T, tend_q, precip within 1e-10 "
                                           "relative or 1e-14 absolute; every column, no exemption",
           "exempt_columns": 0, "rederived_levels": int(stats.n_recomputed),
           "rewritten_patches": int(stats.n_corrected)}
    ok = True
    for kernel, got in (("deep", deep), ("shallow", sh)):
        ref, _ = O.ref_run_parallel(kernel, s, T, q, opts)
        flags = int((got[4] != ref.exited).sum())
        work = int((got[3] != ref.work).sum())
        viol, worst = 0, 0.0
        for a, b in ((got[0], ref.tend_T), (got[1], ref.tend_q), (got[2], ref.precip)):
            d = np.abs(a - b)
            viol += int((d > np.maximum(1e-10 * np.abs(b), 1e-14)).sum())
            nz = np.abs(b) > 0
            if nz.any():
                worst = max(worst, float((d[nz] / np.abs(b[nz])).max()))
        rec[kernel] = {"flag_mismatch": flags, "work_mismatch": work, "tolerance_violations": viol,
                       "max_rel_err": worst}
        ok = ok and flags == 0 and work == 0 and viol == 0
    rec["work_mismatch"] = rec["deep"]["work_mismatch"] + rec["shallow"]["work_mismatch"]
    rec["ok"] = ok
    return rec


# ---------------------------------------------------------------------------
def run_reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    from paper_1711_00289_b200 import gridgen
    import oracle as O
    thr = gridgen.config_threshold(args.config)
    s, T, q = gridgen.make_config(args.config, seed=args.seed)
    threads = os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    # size one step's sample to ~1.5 s of wall so K+W steps stay within minutes
    cal_stride = max(1, s.size // 20000)
    cs, cT, cq = strided_sample(s, T, q, cal_stride)
    if kind == "reference":
        t = cpu_reference_time(cs, cT, cq, thr, threads, args.variant, reps=1, warm=0)
    else:
        t = cpu_port_time(cs, cT, cq, thr, args.variant)
        threads = 1
    rate = cs.size / max(t, 1e-6)
    stride = max(1, s.size // int(min(s.size, max(2000, rate * 1.5))))
    ss, sT, sq = strided_sample(s, T, q, stride)
    opts = O.Options(variant=args.variant, activity_threshold=thr)
    walls = []
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            w = O.ref_time_run_parallel(ss, sT, sq, opts, n_threads=threads, strategy=2, omp_chunk=1)
            wall = w["deep"] + w["shallow"]
        else:
            wall = cpu_port_time(ss, sT, sq, thr, args.variant)
        if i >= args.warmup:
            walls.append(wall)
    tot = float(np.sum(walls))
    value = ss.size * len(walls) / tot
    sample = (f"every {stride}th column of {args.config} ({ss.size} columns) per step; "
              + ("reference run_parallel Dynamic(omp_chunk=1) deep then shallow" if kind == "reference"
                 else "serial C oracle"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(walls),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, gridgen.py)",
        "config": workload_config(args, s.size, T.shape[0], thr),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_gpu_arm(args):
    import torch
    import paper_1711_00289_b200 as P
    from paper_1711_00289_b200 import gridgen

    ws, rank, local = dist_env()
    # BENCH_DIST_BACKEND / BENCH_DEVICE: functional check of the N > 1 path
    # on a one-GPU box (every rank on one device, gloo) -- not a measurement
    dist = init_dist(ws, os.environ.get("BENCH_DIST_BACKEND", "nccl"))
    if os.environ.get("BENCH_DEVICE") is not None:
        local = int(os.environ["BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    thr = gridgen.config_threshold(args.config)
    s, T, q = gridgen.make_config(args.config, seed=args.seed)
    L, n_total = T.shape
    opts = P.KernelOptions(variant=args.variant, activity_threshold=thr)

    # partition: contiguous ranges balanced by estimated cost (multigpu.py)
    from paper_1711_00289_b200 import multigpu
    hbm_gbs, hbm_src = measured_peaks()
    if args.slice:
        # diagnostic: one rank's share of a W-way partition, run alone on this GPU
        pr, pw = (int(x) for x in args.slice.split("/"))
        bounds = multigpu.rank_bounds(s, thr, pw, args.partition, L, hbm_gbs)
        lo, hi = int(bounds[pr]), int(bounds[pr + 1])
    else:
        bounds = multigpu.rank_bounds(s, thr, ws, args.partition, L, hbm_gbs)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    n = hi - lo
    s_r, T_r, q_r = s[lo:hi], np.ascontiguousarray(T[:, lo:hi]), np.ascontiguousarray(q[:, lo:hi])

    ctx = P.Context(local)
    # level rows pitched to a multiple of 32 columns (256-byte aligned rows)
    ldp = (n + 31) // 32 * 32

    def rows(a=None):
        t = torch.empty((L, ldp), dtype=torch.float64, device=dev)[:, :n]
        if a is not None:
            t.copy_(torch.from_numpy(a))
        return t

    ds = torch.from_numpy(s_r).to(dev)
    dT = rows(T_r)
    dq = rows(q_r)

    def alloc_out():
        return (rows(), rows(),
                torch.empty(n, dtype=torch.float64, device=dev),
                torch.empty(n, dtype=torch.int64, device=dev),
                torch.empty(n, dtype=torch.uint8, device=dev))

    deep_o, sh_o = alloc_out(), alloc_out()
    stream = torch.cuda.Stream(device=dev)

    def step():
        ctx.convect_async(ds, dT, dq, deep_o, sh_o, opts, P.BOTH, first_col=lo, stream=stream)

    # warm-up (W >= 3 enforced) and error check
    W = max(3, args.warmup)
    for _ in range(W):
        step()
    st = ctx.check(stream)
    n_trig_local = st.n_triggered

    # timed region: K steps, barrier + sync on both sides, device events on the launching stream
    K = args.steps
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(K):
            step()
        ev1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_local = ev0.elapsed_time(ev1)
    step_stats = ctx.check(stream)
    deep_kernel = ctx.last_deep_kernel
    shallow_kernel = ctx.last_shallow_kernel

    def timed_pass(o, k=K):   # ms per step of k steps with options o (untimed by the contract)
        for _ in range(2):
            ctx.convect_async(ds, dT, dq, deep_o, sh_o, o, P.BOTH, first_col=lo, stream=stream)
        ev0.record(stream)
        for _ in range(k):
            ctx.convect_async(ds, dT, dq, deep_o, sh_o, o, P.BOTH, first_col=lo, stream=stream)
        ev1.record(stream)
        stream.synchronize()
        ctx.check(stream)
        return ev0.elapsed_time(ev1) / k

    # median of >= 5 repetitions of the same K-step region
    reps5 = [timed_pass(opts) for _ in range(5)]
    # the exactness trade beside the headline: the same step without the FP32
    # far phase, and with the reference's rounding in every Newton update
    paths_ms = {"default": float(np.median(reps5)),
                "no_far32": timed_pass(P.KernelOptions(variant=args.variant, activity_threshold=thr, far32=False)),
                "strict": timed_pass(P.KernelOptions(variant=args.variant, activity_threshold=thr, strict=True))}
    step()   # outputs of the default path for the model counts and the parity check
    ctx.check(stream)
    if os.environ.get("BENCH_DEBUG"):   # diagnostic: three more timed passes to stderr (run-to-run spread)
        print(f"debug: lo={lo} hi={hi} n={n} ms/step={ms_local / K:.4f}", file=sys.stderr)
        for rep in range(3):
            ev0.record(stream)
            for _ in range(K):
                step()
            ev1.record(stream)
            stream.synchronize()
            print(f"debug: rep {rep} ms/step={ev0.elapsed_time(ev1) / K:.4f}", file=sys.stderr)
    # per-kernel breakdown from a separate, untimed pass with event pairs
    # between the kernels (kept out of the timed region: the extra event
    # records cost a few us per step, which shows at small per-GPU shares)
    ctx.profile_begin(K)
    for _ in range(K):
        step()
    stream.synchronize()
    kern = ctx.profile_end(K)  # [K][3] trigger, deep, shallow (ms)
    ctx.check(stream)

    # max over ranks
    t = torch.tensor([ms_local, n_trig_local, n], dtype=torch.float64, device=dev)
    if dist:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
        ms_total, n_trig = float(tmax[0]), int(tsum[1])
    else:
        ms_total, n_trig = ms_local, n_trig_local
    ms_step = ms_total / K
    value = (n if args.slice else n_total) * K / (ms_total * 1e-3)

    # model FLOPs from this rank's outputs (work_units / exit flags match the oracle)
    dw = deep_o[3].cpu().numpy()
    dx = deep_o[4].cpu().numpy()
    sw = sh_o[3].cpu().numpy()
    sx = sh_o[4].cpu().numpy()
    deep_flops, sh_flops, trig_r = flop_model(L, dw, dx, sw, sx)

    # FP64 peak measured live on this device
    fp64_peak = ctx.fp64_peak_tflops(5)
    deep_ms = float(np.mean(kern[:, 1])) if len(kern) else float("nan")
    trig_ms = float(np.mean(kern[:, 0])) if len(kern) else float("nan")
    # overlap mode: the shallow kernel runs on a side stream beside the deep
    # kernel; this is the time from the deep kernel's end to the shallow's end
    sh_ms = float(np.mean(np.maximum(kern[:, 2], 0.0))) if len(kern) else float("nan")
    achieved = deep_flops / (deep_ms * 1e-3) / 1e12
    traffic = None
    step_traffic = None
    tf = os.path.join(ROOT, "profiles", "deep_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                d = json.load(f)
            # only for the kernel this run launched, profiled on this workload
            if d.get("config") == args.config and d.get("kernel_desc") == deep_kernel and ws == 1 and not args.slice:
                traffic = d.get("dram_bytes_per_launch")
                # the range capture (kernels overlapped) when there is one, else the serialised sum
                step_traffic = d.get("step_dram_bytes_overlapped", d.get("step_dram_bytes"))
        except Exception:
            pass
    deep_bytes_alg = trig_r * (8 + 2 * 8 * L + 2 * 8 * L + 8 + 8 + 1)
    bytes_step, per_col, deep_bytes = bytes_model(n, L, trig_r)
    # roofline of the whole job per GPU: total FLOPs and bytes over all
    # ranks, divided over the N GPUs (the slower of the two bounds)
    tot = torch.tensor([deep_flops + sh_flops, float(bytes_step)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    flops_job, bytes_job = float(tot[0]), float(tot[1])
    nper = 1 if args.slice else ws
    t_flop = flops_job / nper / (fp64_peak * 1e12)
    t_hbm = bytes_job / nper / (hbm_gbs * 1e9)
    t_roof = max(t_flop, t_hbm)

    # ---- end-to-end through the public host API (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        pin = [P.PinnedArray(a.shape, a.dtype) for a in (s_r, T_r, q_r)]
        for pa, a in zip(pin, (s_r, T_r, q_r)):
            pa.array[...] = a

        def pinned_out():
            arrs = [P.PinnedArray((L, n)), P.PinnedArray((L, n)), P.PinnedArray((n,)),
                    P.PinnedArray((n,), np.int64), P.PinnedArray((n,), np.uint8)]
            return arrs, P.ColumnOutputs(*[a.array for a in arrs])

        pdo, out_d = pinned_out()
        pso, out_s = pinned_out()
        for _ in range(2):
            ctx.convect(pin[0].array, pin[1].array, pin[2].array, opts, P.BOTH, lo, out_d, out_s)
        Ke = max(1, min(K, args.e2e_steps))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(Ke):
            ctx.convect(pin[0].array, pin[1].array, pin[2].array, opts, P.BOTH, lo, out_d, out_s)
        el = time.perf_counter() - t0
        stt = ctx.last_stats
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te[0])
        # bytes moved per step by the whole job (all ranks)
        tb = torch.tensor([float(stt.h2d_bytes), float(stt.d2h_bytes)], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        e2e = {"value": n_total * Ke / el, "unit": UNIT, "h2d_bytes_per_step": int(tb[0]),
               "d2h_bytes_per_step": int(tb[1]), "steps": Ke,
               "ms_per_step": 1e3 * el / Ke,
               # the last step on rank 0 (cvg_stats): copy times summed over the pipeline's chunks (they
               # overlap one another and the kernels, so they add up to more than the step) and the span
               # from the first chunk's first kernel to the last chunk's last (CUDA events)
               "split_ms": {"h2d_sum": float(stt.h2d_ms), "d2h_sum": float(stt.d2h_ms),
                            "device_span": float(stt.device_ms)},
               "note": "cvg_convect (C ABI) on pinned host SoA buffers: H2D inputs, compute, D2H all outputs, per step; wall clock, max over ranks"}
        for a in pin + pdo + pso:
            a.free()

    # ---- device-resident feedback loop (cvg_timestep): the
    # per-step cost is the difference of a 42-step and a 2-step call (the
    # state's H2D / D2H and the buffer set-up happen once per call and cancel)
    loop = None
    if not args.no_loop and ws == 1:
        def loop_s(k):   # the call's stepping region, CUDA events (cvg_stats.device_ms), seconds
            ctx.timestep(s_r, T_r, q_r, opts, P.DEEP, k)
            return 1e-3 * ctx.last_stats.device_ms
        loop_s(1)
        a2, a42 = min(loop_s(2) for _ in range(3)), min(loop_s(42) for _ in range(3))
        per = (a42 - a2) / 40
        loop = None if per <= 0 else {"kernel": "deep", "ms_per_step": 1e3 * per, "columns_per_s": n_total / per,
                "note": "cvg_timestep: per step the deep kernel advances the state in place (T += tend_T, "
                        "q += tend_q) with check_finite latched on the device, guard-band re-derivation applied "
                        "to the state; the host checks every 16 steps (first failing step reported); state "
                        "resident in HBM; (t(42 steps) - t(2 steps)) / 40 over the calls' stepping regions, CUDA events"}

    cpu = None
    parity = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(s, T, q, thr, args.variant)
        import oracle as O
        if O.ref_available():
            cpu["serial"] = serial_reference(s, T, q, thr, args.variant)
            host = lambda o: [t.cpu().numpy() for t in o]   # noqa: E731
            parity = parity_against_reference(s, T, q, thr, args.variant, host(deep_o), host(sh_o), step_stats)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator, paper_1711_00289_b200/gridgen.py)",
        "config": workload_config(args, n_total, L, thr),
        "workload_notes": {"triggered_deep": int(n_trig), "partition": args.partition if ws > 1 else "single",
                           "l2": "inputs (432 MB) + outputs (879 MB) exceed the 126 MB L2; no flush needed",
                           "parallelism": f"column partition x{ws}, no collective"},
        "ms_per_step_median_of_5": paths_ms["default"],
        "paths_ms_per_step": {**paths_ms, "note": "default = relaxed Newton update with FP32 far phase and the "
                                                  "guard-band re-derivation (work_units exact); no_far32 = FP64 "
                                                  "relaxed update only; strict = the reference's rounding in every "
                                                  "update (bit-identical roots and counts)"},
        "parity": parity,
        "roofline": {"bound": "fp64",
                     "kernel": deep_kernel,
                     "achieved": achieved,
                     "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                     "traffic": traffic,
                     "peak_source": "live DFMA probe on this GPU (cvg_fp64_peak); MEASURED_PEAKS.json has no FP64 figure",
                     "flops_per_launch": deep_flops, "ms_per_launch": deep_ms,
                     "algorithmic_bytes_per_launch": deep_bytes_alg,
                     "model": "159*L + 37*U_c FLOP per triggered column (SURVEY 8d), U_c from the step's work_units"},
        "step_roofline": {"flops": flops_job, "bytes": bytes_job, "bytes_per_column": per_col,
                          "t_fp64_ms": 1e3 * t_flop, "t_hbm_ms": 1e3 * t_hbm,
                          "hbm_peak_gbs": hbm_gbs, "hbm_source": hbm_src,
                          "fp64_peak_tflops": fp64_peak,
                          "bound": "fp64" if t_flop >= t_hbm else "hbm",
                          "roofline_ms": 1e3 * t_roof, "frac": 1e3 * t_roof / (ms_total / K),
                          "frac_fp64_model": 1e3 * t_flop / (ms_total / K), "frac_hbm": 1e3 * t_hbm / (ms_total / K),
                          # the north star's nominal 8 TB/s beside the measured copy bandwidth (both)
                          "frac_hbm_nominal_8tbs": 1e3 * (bytes_job / nper / 8.0e12) / (ms_total / K),
                          "achieved_hbm_gbs": bytes_job / nper / (ms_total / K * 1e-3) / 1e9,
                          "traffic": step_traffic,
                          "note": "job FLOPs and bytes over all ranks / N GPUs; frac = roofline time / max-over-ranks step time; "
                                  "traffic = ncu DRAM bytes of one step, range capture with the kernels overlapped (profiles/deep_traffic.json, N=1 only)"},
        "kernels_ms": {"trigger_groups": trig_ms, "deep": deep_ms, "shallow_tail_after_deep": sh_ms,
                       "deep_kernel": deep_kernel, "shallow_kernel": shallow_kernel,
                       "schedule": "trigger/group compaction -> deep (main stream, programmatic dependent launch) || "
                                   "shallow + zero-fill of untriggered groups (side stream, concurrent)"},
        # per step: reset of the per-call words, trigger/compaction, deep, the
        # guard-band re-derivation kernel (relaxed path, calls of >= 100k
        # columns; smaller calls re-derive inside the deep kernel), shallow
        "gpu_launches": (5 if args.variant != 2 and n >= 100000 else 4) * K,
        "e2e": e2e,
        "feedback_loop": loop,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if rank == 0:
        # the reference's pinned BenchRecord CSV (bench.hpp:30-43): one run-gpu
        # row per run, by default into the scratch directory gpurun_out/
        rec_path = None
        if args.records == "auto" and not args.slice:
            rec_path = os.path.join(ROOT, "gpurun_out", "run_gpu_records.csv")
        elif args.records not in (None, "auto", "none"):
            rec_path = args.records
        if rec_path:
            try:
                from paper_1711_00289_b200 import records
                os.makedirs(os.path.dirname(os.path.abspath(rec_path)), exist_ok=True)
                records.append_records(rec_path, [records.run_gpu_record(line)])
                line["records"] = os.path.relpath(rec_path, ROOT)
            except OSError as e:   # a read-only tree: the JSON line is the result
                line["records"] = f"not written ({e.__class__.__name__})"
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["ref", "c1", "c2", "c3", "c4", "c5_05", "c5_50", "c5_95"])
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--partition", default="balanced", choices=["balanced", "overlap", "model", "naive"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-loop", action="store_true", help="skip the feedback-loop measurement")
    ap.add_argument("--records", default="auto",
                    help="append a run-gpu BenchRecord row (reference CSV schema) to this file "
                         "(default: gpurun_out/run_gpu_records.csv; 'none' to skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--slice", default=None,
                    help="diagnostic R/W: time rank R's share of a W-way partition alone on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
