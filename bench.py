#!/usr/bin/env python
"""bench.py -- -2logL evaluations/s on the B200 engine (BASELINE.json metric, config C3).

A step = one pass of the hot path over one batch: B=100 theta candidates (one GA
generation) through ProfileEvaluator::eval semantics (likelihood.hpp:108-141):
R assembly (K1), jitter-ladder Cholesky with the bordered solves (K2), deviance (K3).
Weak scaling: every rank evaluates its own 100-candidate batch (candidates are
independent; no data-path collective). Inputs (design table, thetas) are resident in
HBM when the timed region starts; the per-step working set (100 x 69 MB factor tiles)
is far larger than L2, so no extra flush is needed.

  python bench.py [--gpus N --steps K --warmup W]          # our arm
  python bench.py --impl reference [...]                    # the reference CPU path
  torchrun --nproc-per-node N bench.py --gpus N ...         # multi-GPU (one rank per GPU)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "-2logL evals/sec at n=4096,d=10 (C3: batch of 100 thetas per GPU per step)"
UNIT = "evals/s"
FP64_PEAK_FALLBACK = 37.0  # TFLOP/s, DMMA m8n8k4 measured on this pool (profiles/fp64_peak.json)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # (long names: torchrun would take --n / --d / --p as abbreviations of its own options)
    ap.add_argument("--size", dest="n", type=int, default=4096)
    ap.add_argument("--dims", dest="d", type=int, default=10)
    ap.add_argument("--power", dest="p", type=float, default=1.95)
    ap.add_argument("--batch", type=int, default=100)
    ap.add_argument("--seed", type=int, default=20120306)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fit", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-single", action="store_true",
                    help="skip the informational single-precision (FP32 engine) rate")
    ap.add_argument("--cpu-sample", type=int, default=0, help="evals in the CPU sample (0: auto)")
    return ap.parse_args()


# ----------------------------------------------------------------- inputs
def random_lhd(n, d, rng):
    """Random Latin hypercube (experiment.hpp:36-50 semantics, numpy RNG)."""
    X = np.empty((n, d))
    for k in range(d):
        X[:, k] = (rng.permutation(n) + rng.random(n)) / n
    return X


def smooth_response(X):
    """test_helpers.hpp:47-53, defined for any d."""
    k = np.arange(X.shape[1])
    return (np.sin(3.0 * X + 0.37 * k) + 0.5 * X * X).sum(1)


def lhs_thetas(d, count, rng, lo=1e-6, hi=12.0):
    """GA initial population over the log10 box (optimizer.hpp:62-80 semantics)."""
    g = np.empty((count, d))
    for k in range(d):
        g[:, k] = (rng.permutation(count) + rng.random(count)) / count
    return 10.0 ** (math.log10(lo) + (math.log10(hi) - math.log10(lo)) * g)


def make_inputs(args, rank):
    rng = np.random.default_rng(args.seed)
    X = random_lhd(args.n, args.d, rng)
    y = smooth_response(X)
    trng = np.random.default_rng(args.seed + 1000 * (rank + 1))
    batches = [lhs_thetas(args.d, args.batch, trng) for _ in range(max(args.steps, args.warmup, 1))]
    return X, y, batches


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock / max clock / clock-event reasons sampled every 20 ms during the timed region:
    NVML in a background thread (in-process, nothing buffered), else an `nvidia-smi -lms`
    subprocess. One sample is also taken on entry and exit, so a short region still has
    evidence."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self.lines = []

    def _nvml_sample(self):
        nv = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        masks = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        self.samples.append((float(sm), float(mx), {n for n, m in zip(self.NAMES, masks) if bits & m}))

    def _loop(self):
        while not self.stop.wait(0.02):
            try:
                self._nvml_sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import threading
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            try:  # the CUDA device's PCI address (CUDA and NVML may enumerate differently)
                import torch
                pr = torch.cuda.get_device_properties(self.index)
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(
                    f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml_sample()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=2)
            try:
                self._nvml_sample()
                self.nvml.nvmlShutdown()
            except Exception:
                pass
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                self.samples.append((float(f[0]), float(f[1]),
                                     {n for n, v in zip(self.NAMES, f[3:7]) if v.lower() == "active"}))
            except (ValueError, IndexError):
                continue

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set().union(*(r for _, _, r in self.samples))
        return {"sm_mhz": statistics.median(s for s, _, _ in self.samples),
                "sm_max_mhz": max(m for _, m, _ in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ----------------------------------------------------------------- reference arm
def cpu_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def run_reference_arm(args, rank, world):
    """The reference's own CPU path (oracle/_ref = unmodified reference headers, native
    flags, ParallelBackend on all host threads), same metric/config as our arm."""
    if rank != 0:
        return None
    from oracle.oracle import RefLib, ref_available
    if not ref_available(fast=True):
        return {"impl": "reference", "unavailable": "oracle/_ref/libgpemu_ref_fast.so not built"}
    ref = RefLib(fast=True)
    X, y, batches = make_inputs(args, 0)
    per_step = args.cpu_sample or 4
    th = batches[0]
    ref.eval_batch_timed(X, y, th[:1], args.p)  # page-in; the plan is excluded from timing below
    evals, secs, plan_s = 0, 0.0, 0.0
    for s in range(args.warmup + args.steps):
        sl = th[(s * per_step) % len(th):(s * per_step) % len(th) + per_step]
        _, sp, se = ref.eval_batch_timed(X, y, sl, args.p, threads=0)
        if s >= args.warmup:
            evals += len(sl)
            secs += se
            plan_s = sp
    value = evals / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_threads(), "kind": "reference",
                         "sample": f"{per_step} evals per step x {args.steps} steps of the step-0 "
                                   f"theta batch; ParallelBackend(hardware_concurrency); "
                                   f"plan construction ({plan_s:.2f} s) excluded"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def bench_config(args, world):
    """The workload description both arms print (the reference arm runs the same config)."""
    n, B = args.n, args.batch
    return {"workload": f"C3: n={n}, d={args.d}, p={args.p}; {B} theta candidates per GPU "
                        "per step (one GA generation); random LHD design, smooth_response y, "
                        "thetas from the GA's LHS over the log10 box [1e-6, 12]^d",
            "n": n, "d": args.d, "p": args.p, "batch_per_gpu": B, "global_batch": B * world,
            "parallelism": f"candidate sharding x{world} (weak)",
            "l2": "inputs larger than L2 (per-step working set ~%.1f GB)" % (
                B * (n / 128) * (n / 128 + 1) / 2 * 128 * 128 * 8 / 1e9)}


# ----------------------------------------------------------------- our arm
# Collectives backend for the multi-rank path: NCCL (one rank per GPU, the contract). The
# test-only override GPEMU_BENCH_DIST=gloo runs the same host logic with CPU collectives and
# maps ranks onto the visible GPUs, so the world > 1 code path can be exercised on one GPU
# (ranks never wait on each other's kernels: the work is independent candidate batches).
DIST_BACKEND = os.environ.get("GPEMU_BENCH_DIST", "nccl")


def rank_device(local_rank):
    import torch
    return local_rank if DIST_BACKEND == "nccl" else local_rank % max(1, torch.cuda.device_count())


def max_over_ranks(x, dev):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev if DIST_BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1203_1269_b200.gpemu as g
    local_rank = rank_device(local_rank)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    X, y, batches = make_inputs(args, rank)
    ctx = g.Context(local_rank, "dag")
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    be = g.Backend(ctx)
    ev = g.ProfileEvaluator(g.new_dataset(X, y), args.p, 0.0, be, max_batch=args.batch)
    B = args.batch
    d_th = [torch.from_numpy(b).to(dev) for b in batches]
    d_out = torch.empty(B * 8, dtype=torch.float64, device=dev)

    def step(s):
        ev.eval_batch_device(d_th[s % len(d_th)].data_ptr(), B, d_out.data_ptr())

    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ev.set_profiling(True)
    launches0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        e0.record(stream)
        for s in range(args.steps):
            step(s)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count - launches0
    chol_ms, chol_n = ev.phase_ms(1)
    asm_ms, _ = ev.phase_ms(0)
    fin_ms, _ = ev.phase_ms(2)
    ev.set_profiling(False)
    rec = d_out.view(B, 8).cpu().numpy()
    status = rec[:, 5]
    ms_max = max_over_ranks(ms, dev) if dist is not None else ms
    value = world * B * args.steps / (ms_max / 1e3)

    # ---- e2e: the public API with pinned host buffers (H2D thetas, D2H records) ----
    e2e = None
    if not args.no_e2e:
        h_th = [torch.from_numpy(b).pin_memory() for b in batches]
        outs = {k: torch.empty(B, dtype=torch.float64).pin_memory()
                for k in ("neg2", "mu", "sigma2", "jitter", "log_det")}
        st = torch.empty(B, dtype=torch.int32).pin_memory()
        L = g.lib()

        def api_step(s):
            th = h_th[s % len(h_th)]
            dp = lambda t: g.C.cast(g._vp(t.data_ptr()), g._dp)  # noqa: E731
            g._check(L.gpemu_eval_batch(ev.handle, dp(th), B,
                                        *[dp(outs[k]) for k in
                                          ("neg2", "mu", "sigma2", "jitter", "log_det")],
                                        g.C.cast(g._vp(st.data_ptr()), g._ip)))
        for s in range(args.warmup):
            api_step(s)
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for s in range(args.steps):
            api_step(s)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = f0.elapsed_time(f1)
        if dist is not None:
            ems = max_over_ranks(ems, dev)
        e2e = {"value": world * B * args.steps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": B * args.d * 8, "d2h_bytes_per_step": B * (5 * 8 + 4),
               "api": "gpemu_eval_batch (C-ABI, host buffers)"}

    out = {"value": value, "ms": ms_max, "status_ok": int(np.sum(status == 0)), "launches": launches,
           "chol_ms": chol_ms, "chol_launches": chol_n, "asm_ms": asm_ms, "fin_ms": fin_ms,
           "clocks": clk.summary(), "e2e": e2e, "ev": ev, "be": be, "ctx": ctx, "X": X, "y": y,
           "batches": batches}
    return out


def load_profile_traffic():
    p = os.path.join(ROOT, "profiles", "chol_dag_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except (OSError, ValueError):
            return None
    return None


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        try:
            return float(json.load(open(p))["dmma_tflops"]), "profiles/fp64_peak.json (DMMA m8n8k4 microbench, this pool)"
        except (OSError, ValueError, KeyError):
            pass
    return FP64_PEAK_FALLBACK, "tools/microbench/fp64_peak.cu measurement (37.0 TF DMMA)"


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)

    if args.impl == "reference":
        line = run_reference_arm(args, rank, world)
        if rank == 0 and line is not None:
            print(json.dumps(line))
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        if DIST_BACKEND == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(DIST_BACKEND)

    r = run_ours(args, rank, world, local_rank)
    B, n = args.batch, args.n
    flops_per_launch = B * n ** 3 / 3.0  # algorithmic Cholesky flops
    chol_avg_ms = r["chol_ms"] / max(1, r["chol_launches"])
    achieved = flops_per_launch / (chol_avg_ms / 1e3) / 1e12
    peak, peak_src = fp64_peak()
    traffic = load_profile_traffic()
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, world),
        "roofline": {"kernel": "chol_dag_kernel", "bound": "tensor", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": peak_src + " (FP64: MEASURED_PEAKS.json has bf16/HBM only)",
                     "algorithmic_flops_per_launch": flops_per_launch,
                     "avg_launch_ms": chol_avg_ms,
                     "traffic": traffic.get("bytes_per_launch") if traffic else None},
        "phases_ms_per_step": {"assemble": r["asm_ms"] / args.steps,
                               "cholesky": r["chol_ms"] / args.steps,
                               "finalize": r["fin_ms"] / args.steps},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "e2e": r["e2e"],
        "candidates_ok": r["status_ok"],
    }
    # ---- informational: the same batches on the single-precision engine (Precision::kSingle) ----
    if rank == 0 and world == 1 and not args.no_single:
        import torch
        import paper_1203_1269_b200.gpemu as g
        evs = g.ProfileEvaluator(g.new_dataset(r["X"], r["y"]), args.p, 0.0, r["be"],
                                 max_batch=B, precision="single")
        for b in r["batches"][:2]:
            evs.eval_batch(b)
        evs.set_profiling(True)
        t0 = time.time()
        for s in range(args.steps):
            evs.eval_batch(r["batches"][s % len(r["batches"])])
        wall = time.time() - t0
        sc_ms, _ = evs.phase_ms(1)
        evs.set_profiling(False)
        line["single_precision"] = {
            "value": B * args.steps / wall, "unit": UNIT, "chol_ms_per_step": sc_ms / args.steps,
            "note": "informational: FP32 engine (float R/factor/solves, dots in double) on the same "
                    "batches, host-timed through eval_batch; the headline value is FP64"}
        evs.close()
    # ---- fit wall time (GA 100 x 20 on the same design) ----
    if rank == 0 and world == 1 and not args.no_fit:
        import paper_1203_1269_b200.gpemu as g
        cfg = g.FitConfig(ga=g.GaConfig(population=B, generations=20), seed=1, p=args.p)
        t = time.time()
        fr = g.fit_gp_detailed(g.new_dataset(r["X"], r["y"]), cfg, r["be"], evaluator=r["ev"])
        line["fit"] = {"gpu_wall_s": time.time() - t, "evals": cfg.ga.budget(),
                       "neg2": fr.model.neg2_log_lik, "ga": f"{B}x20"}
    # ---- CPU baseline: the reference itself on the host cores (bounded sample) ----
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.oracle import RefLib, ref_available
        if ref_available(fast=True):
            ref = RefLib(fast=True)
            S = args.cpu_sample or 16
            th = r["batches"][0][:S]
            neg2, sp, se = ref.eval_batch_timed(r["X"], r["y"], th, args.p, threads=0)
            cpu_v = S / se
            line["cpu_baseline"] = {
                "value": cpu_v, "unit": UNIT, "cores": cpu_threads(), "kind": "reference",
                "sample": f"{S} of the step-0 thetas (n={n}, d={args.d}), reference ParallelBackend "
                          f"on all host threads, {se:.1f} s of evals; plan {sp:.2f} s excluded"}
            if "fit" in line:
                line["fit"]["cpu_wall_s_extrapolated"] = sp + line["fit"]["evals"] / cpu_v
        else:
            line["cpu_baseline"] = None
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
