#!/usr/bin/env python
"""Benchmark: forward DGT on a nonseparable lattice (shear algorithm) on B200.

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl ours|reference] [--config k]
One "step" = one pass of the whole hot path (Alg. 1: chirp/FFT front end, Zak/factorisation
DGT, phase + remap) over this rank's shard of the config's batch, inputs resident in HBM.
Default workload: BASELINE.json config 5 (L=262144, a=128, M=512, lambda=1/2, W=1024,
complex64).  Multi-GPU: the signals are independent units, so each rank transforms its own
batch of W signals (signals [rank W, (rank + 1) W) of the seeded stream; "scaling": "weak",
value = all ranks' coefficients / max-over-ranks time); --scaling strong splits one batch of
W contiguously instead.  There is no data-path collective.  Rank 0 prints ONE JSON line.
For N > 1 the driver launches torchrun (one process per GPU, NCCL); a plain
``python bench.py --gpus N`` re-executes itself under torch.distributed.run with N ranks.
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "DGT coefficients/sec (W*M*N per s)"
METRIC_INV = "DGT synthesis (inverse) coefficients/sec (W*M*N per s)"
UNIT = "coefficients/s"


def dist_setup(n_gpus):
    from paper_1307_4569_b200 import dist as pd
    return pd.init()


def shard(W, ws, rank, scaling="weak"):
    """This rank's signals [w0, w1): weak scaling -- every rank its own batch of W signals;
    strong -- one batch of W split contiguously."""
    from paper_1307_4569_b200 import dist as pd
    if scaling == "weak":
        return rank * W, (rank + 1) * W
    return pd.shard(W, ws, rank)


def spawn_ranks(n):
    """Re-execute this script under torch.distributed.run with n ranks on 127.0.0.1 (used when
    ``--gpus N > 1`` is given without a torchrun environment).  Returns the launcher's exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def barrier(ws):
    from paper_1307_4569_b200 import dist as pd
    pd.barrier()


def allreduce_max(x, ws):
    from paper_1307_4569_b200 import dist as pd
    return pd.allreduce(x, "max")


def allreduce_sum(x, ws):
    from paper_1307_4569_b200 import dist as pd
    return pd.allreduce(x, "sum")


class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index):
        self.samples = []
        self.reasons = 0
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

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
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            mp = json.load(fh)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy b/w)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


def ncu_traffic(workload, kernel):
    """Per-launch DRAM bytes from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(workload, {}).get(kernel)
    except Exception:  # noqa: BLE001
        return None


def fp_peak(dtype):
    """Measured CUDA-core FMA peak in TFLOP/s (2 flops per FMA) for the working precision:
    profiles/r01_microbench.json (tools/microbench.cu on a B200 of this pool)."""
    key = "fp32_ffma_reg_Tinstr_s" if dtype == "c64" else "fp64_dfma_reg_Tinstr_s"
    try:
        with open(os.path.join(ROOT, "profiles", "r01_microbench.json")) as fh:
            return 2.0 * float(json.load(fh)[key]), f"measured ({key} x 2, profiles/r01_microbench.json)"
    except Exception:  # noqa: BLE001
        return (74.4 if dtype == "c64" else 37.2), "nominal (148 SMs x 128 FP32 / 64 FP64 lanes x 2 x 1.965 GHz)"


def ncu_traffic_chain(workload, stats):
    """Summed per-chunk DRAM bytes of a multi-kernel chain, if every kernel has a capture."""
    vals = [ncu_traffic(workload, k["name"]) for k in stats]
    return None if any(v is None for v in vals) else float(sum(vals))


def oracle_sample(wl, budget_s, max_signals=None):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload.
    Returns (coefs/s, cores, description)."""
    import numpy as np

    import oracle
    from synthetic import batch, window
    g = window(wl)
    # all host cores, also under torchrun (which sets OMP_NUM_THREADS=1 for its ranks)
    cores = len(os.sched_getaffinity(0))
    variant = "literal" if wl.L * wl.M <= 4096 * 64 else "regrouped"
    # probe: one signal on a column subset to size the sample
    ncol = min(wl.N, 64)
    cols = np.arange(ncol)
    f1 = batch(wl, 0, 1)
    t0 = time.perf_counter()
    oracle.dgt(f1, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols, variant=variant, nthreads=cores)
    tp = time.perf_counter() - t0
    per_col = max(tp / ncol, 1e-7)
    ncols_total = int(max(1, min(wl.N * (max_signals or wl.W), budget_s / per_col)))
    nsig = max(1, min(wl.W if max_signals is None else max_signals, math.ceil(ncols_total / wl.N)))
    cols_per_sig = min(wl.N, max(1, ncols_total // nsig))
    f = batch(wl, 0, nsig)
    cols = np.arange(cols_per_sig)
    t0 = time.perf_counter()
    oracle.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols, variant=variant, nthreads=cores)
    dt = time.perf_counter() - t0
    coefs = nsig * wl.M * cols_per_sig
    desc = (f"oracle {'O1 literal' if variant == 'literal' else 'O2 regrouped'} sum (fp64, OpenMP), "
            f"{nsig} signal(s) x {cols_per_sig} of {wl.N} columns x all {wl.M} channels of {wl.name}")
    return coefs / dt, cores, desc, dt


def oracle_sample_inverse(wl, budget_s):
    """Time the CPU oracle's synthesis (S2 regrouped, as it stands) on whole signals of the
    workload until ~budget_s (at least one signal).  Returns (coefs/s, cores, description, s)."""
    import numpy as np

    import oracle
    from synthetic import window
    g = window(wl)
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(0)
    c = rng.standard_normal((1, wl.M, wl.N)) + 1j * rng.standard_normal((1, wl.M, wl.N))
    n, t0 = 0, time.perf_counter()
    while n == 0 or (time.perf_counter() - t0 < budget_s and n < wl.W):
        oracle.idgt(c, g, wl.a, wl.M, wl.lam1, wl.lam2, variant="regrouped", nthreads=cores)
        n += 1
    dt = time.perf_counter() - t0
    desc = f"oracle S2 regrouped synthesis (fp64, OpenMP), {n} whole signal(s) of {wl.name}"
    return n * wl.M * wl.N / dt, cores, desc, dt


def run_reference(args, wl, ws, rank):
    """--impl reference: the oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    from synthetic import batch  # noqa: F401
    # size each step to ~4 s of CPU work so W + K steps finish in minutes
    per_step = max(1.0, min(6.0, 150.0 / max(1, args.steps + args.warmup)))
    times, vals = [], []
    desc, cores = "", 0
    sample = oracle_sample_inverse if args.inverse else oracle_sample
    for i in range(args.warmup + args.steps):
        v, cores, desc, dt = sample(wl, per_step)
        if i >= args.warmup:
            times.append(dt)
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC_INV if args.inverse else METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, synthetic/workloads.py)",
        "config": {"workload": wl.name, "L": wl.L, "a": wl.a, "M": wl.M, "lambda": [wl.lam1, wl.lam2],
                   "W": wl.W, "parallelism": "host cores (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, help="BASELINE.json config (1-based)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--force-generic", action="store_true")
    ap.add_argument("--max-chunk", type=int, default=0)
    ap.add_argument("--inverse", action="store_true",
                    help="time the synthesis (dgt_execute_inverse, c -> f) instead of the forward DGT")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: W signals per rank (default); strong: W signals split over the ranks")
    ap.add_argument("--dry-run", action="store_true",
                    help="bring up the ranks and print the shard plan only (no GPU work; tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)

    from synthetic import config
    wl = config(args.config)
    ws, rank, local = dist_setup(args.gpus)
    if args.dry_run:
        import torch.distributed as dist
        w0, w1 = shard(wl.W, ws, rank, args.scaling)
        parts = [None] * ws
        if ws > 1:
            dist.all_gather_object(parts, (rank, w0, w1))
            dist.destroy_process_group()
        else:
            parts = [(rank, w0, w1)]
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": ws, "requested_gpus": args.gpus, "scaling": args.scaling,
                              "workload": wl.name, "shards": [list(p) for p in parts]}), flush=True)
        return 0

    if args.impl == "reference":
        rc = run_reference(args, wl, ws, rank)
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return rc

    import numpy as np
    import torch

    import paper_1307_4569_b200 as nsdgt
    from synthetic import batch, window

    dev = torch.device("cuda", torch.cuda.current_device())
    w0, w1 = shard(wl.W, ws, rank, args.scaling)
    Wr = w1 - w0
    g = window(wl)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=wl.real_input,
                      force_generic=args.force_generic, max_chunk=args.max_chunk)
    f_host = torch.from_numpy(batch(wl, w0, w1)).pin_memory()
    f_dev = f_host.to(dev)
    cdt = torch.complex64 if wl.dtype == "c64" else torch.complex128
    c_dev = torch.empty((Wr, wl.M, wl.N), dtype=cdt, device=dev)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()

    if args.inverse:
        # synthesis: the step maps the coefficients of this rank's shard back to signals
        plan.execute(f_dev, out=c_dev)
        fo_dev = torch.empty((Wr, wl.L), dtype=cdt, device=dev)

        def step():
            plan.inverse(c_dev, out=fo_dev)
    else:
        def step():
            plan.execute(f_dev, out=c_dev)

    # warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # timed region: K steps bracketed by barrier + synchronize, CUDA events on the launch stream;
    # kernel durations recorded with event pairs around every launch on the same stream.
    # SURVEY 8(d) algorithmic bytes of this rank's step; a step that moves less than ~4x the
    # 126 MB L2 could be served from L2 across iterations, so then L2 is flushed (a 512 MB
    # memset) between steps, outside per-step event pairs, and the step times are summed
    # (synthesis writes complex signals even for real-input plans)
    step_bytes = Wr * (wl.L * (8 if wl.dtype == "c64" else 16) // (2 if wl.real_input and not args.inverse else 1)
                       + wl.M * wl.N * (8 if wl.dtype == "c64" else 16)) + wl.L * (8 if wl.dtype == "c64" else 16)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if step_bytes <= 4 * 126e6 else None
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)] if flush is not None else []
    sampler = ClockSampler(torch.cuda.current_device())
    # per-kernel event pairs cost a few us per launch and stop consecutive kernels from
    # overlapping (PDL): inside the timed region for one-kernel steps (configs 3, 5: one event
    # pair around one long kernel), in a second identical pass for multi-kernel chains
    # (config 4) and the L2-flushed small steps (configs 1-2)
    prof_in_loop = flush is None and plan.launches(Wr) <= 2
    if prof_in_loop:
        plan.profile_begin()
    barrier(ws)
    torch.cuda.synchronize()
    with sampler:
        e0.record(stream)
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
                pairs[i][0].record(stream)
            step()
            if flush is not None:
                pairs[i][1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    if not prof_in_loop:
        plan.profile_begin()
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            step()
        torch.cuda.synchronize()
    stats = plan.profile_end()
    ms_total = e0.elapsed_time(e1) if flush is None else sum(a.elapsed_time(b) for a, b in pairs)
    ms_total_max = allreduce_max(ms_total, ws)
    ms_per_step = ms_total_max / args.steps
    coefs_per_step = (w1 - w0) * wl.M * wl.N
    coefs_all = allreduce_sum(coefs_per_step, ws)   # every rank's units (weak: ws x W signals)
    value = coefs_all / (ms_per_step * 1e-3)

    # Roofline: SURVEY 8(d)'s algorithmic bytes per signal (input + coefficients, window once)
    # over the time of the kernels that move them.  The fused path is one kernel per step; a
    # multi-kernel path (config 4: cuFFT + zak_ct + out_f4096 per chunk of signals) is charged
    # the summed time of its whole chain per chunk -- intermediates are not algorithmic bytes.
    dom = max(stats, key=lambda s: s["ms"])
    chain_ms = sum(k["ms"] for k in stats)
    launches_per_step = dom["launches"] / args.steps   # chunks per step (one launch of each kind per chunk)
    per_launch_bytes = step_bytes / launches_per_step
    per_chunk_ms = chain_ms / dom["launches"]
    achieved = per_launch_bytes / (per_chunk_ms * 1e-3) / 1e9
    peak, peak_src = measured_peaks()
    fpk, fpk_src = fp_peak(wl.dtype)
    chain_flops = sum(k["flops"] for k in stats)
    traffic = ncu_traffic(wl.name, dom["name"]) if len(stats) == 1 else ncu_traffic_chain(wl.name, stats)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom["name"] if len(stats) == 1 else "+".join(k["name"] for k in stats),
                "peak_source": peak_src,
                "kernel_ms_per_launch": per_chunk_ms, "algorithmic_bytes_per_launch": per_launch_bytes,
                "dominant_kernel": dom["name"],
                "kernel_share_of_step": chain_ms / ms_total if ms_total > 0 else None,
                "kernel_events": "inside the timed region" if prof_in_loop else
                                 "a second pass of the same K steps (L2 flushed; event pairs would perturb the timed one)",
                "model_tflops": chain_flops / (chain_ms * 1e-3) / 1e12,
                "compute_peak_tflops": fpk, "compute_peak_source": fpk_src,
                "compute_frac": chain_flops / (chain_ms * 1e-3) / 1e12 / fpk,
                "kernels": stats}
    step_gbs = step_bytes / (ms_total / args.steps * 1e-3) / 1e9

    # end to end through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and not args.inverse:
        c_host = torch.empty((Wr, wl.M, wl.N), dtype=cdt, pin_memory=True)
        plan.execute_host(f_host, out=c_host)  # allocate staging outside the timed region
        ee0 = torch.cuda.Event(enable_timing=True)
        ee1 = torch.cuda.Event(enable_timing=True)
        barrier(ws)
        torch.cuda.synchronize()
        ee0.record(stream)
        for _ in range(args.e2e_steps):
            plan.execute_host(f_host, out=c_host)
            _ = float(c_host.reshape(-1)[-1].real)  # the step's result read on the host
        ee1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        e2e_ms = allreduce_max(ee0.elapsed_time(ee1), ws) / args.e2e_steps
        e2e = {"value": coefs_all / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(allreduce_sum(f_host.numel() * f_host.element_size(), ws)),
               "d2h_bytes_per_step": int(allreduce_sum(c_host.numel() * c_host.element_size(), ws)),
               "ms_per_step": e2e_ms, "steps": args.e2e_steps,
               "path": "dgt_execute_host: pinned host f -> H2D (stream 1) -> kernels -> D2H (stream 2), chunked"}
        del c_host

    # our kernels only (the frequency-shear cuFFT calls are library launches)
    launches = (sum(k["launches"] for k in stats if k["name"] != "front_fft_cufft") if args.inverse
                else args.steps * plan.launches(Wr))
    launches_total = int(allreduce_sum(launches, ws))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, cores, desc, dt = (oracle_sample_inverse if args.inverse else oracle_sample)(wl, args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc, "seconds": dt}

    clocks = sampler.summary()
    if rank == 0:
        info = plan.info
        line = {
            "metric": METRIC_INV if args.inverse else METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic (seeded, synthetic/workloads.py)",
            "config": {"workload": wl.name, "L": wl.L, "a": wl.a, "M": wl.M, "N": wl.N,
                       "lambda": [wl.lam1, wl.lam2], "W": wl.W,
                       "global_batch": wl.W * ws if args.scaling == "weak" else wl.W,
                       "signals_per_rank": w1 - w0,
                       "parallelism": f"dp{ws} (independent signals per rank, no collective on the data path)",
                       "branch": nsdgt.BRANCH_NAMES[info["branch"]], "shear": [info["s0"], info["s1"]],
                       "inner": {"a": info["ia"], "M": info["iM"], "c": info["c"], "d": info["d"],
                                 "p": info["p"], "q": info["q"]},
                       "chunk": info["chunk"], "kernel_path": info["kernel_path"],
                       "l2": "inputs+outputs per step exceed the 126 MB L2 (no flush needed)"
                       if flush is None else "L2 flushed between steps (512 MB memset outside the per-step events)"},
            "roofline": roofline,
            "step_hbm_gbs": step_gbs,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_total,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
