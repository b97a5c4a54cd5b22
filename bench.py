#!/usr/bin/env python
"""Benchmark of the mM-Parareal hot path (BASELINE.json metric: fine-propagator
particle-steps/s and Parareal iteration time at 1/2/4/8 B200).

Workload (BASELINE config 4, the weak-scaling sweep the metric is quoted on):
linear mean-field OU dX = (-X + 0.5 E[X]) dt + 0.5 dW, X0 ~ N(1, 0.1^2),
P = 1e5 particles per slice, dt = 1e-3 (S = 100 steps per slice, T0 = 0.1),
N = 64 slices per GPU (N = 64 G), K = 5 iterations, coarse = exact-closure
mean/variance ODE with forward Euler dt = 1e-2, FROZEN numpy-exact noise,
seed 0, fp64.  One "step" = one complete run_micro_macro (noise generation,
iteration 0, K iterations), so value = K*N*P*S / run time (all GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs one process per GPU over NCCL: under torchrun as launched by the
driver, or relaunched through torch.distributed.run by this script when
started without one.  Both multi-GPU drivers run (per-iteration kernels with
NCCL collectives; the iteration pipeline with peer-memory hand-offs), their
traces are compared bit for bit and the faster verified one is `value`.
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-propagator particle-steps/s (mM-Parareal run, BASELINE config 4)"
UNIT = "particle-steps/s"
SLICES_PER_GPU, P, S, DT, K_ITER, SEED = 64, 100_000, 100, 1e-3, 5, 0


def workload(G: int) -> dict:
    return {"workload": "config4: linear mean-field OU weak-scaling sweep (dX=(-X+0.5E[X])dt+0.5dW, "
                        "X0~N(1,0.1^2)), coarse exact-closure moment ODE, forward Euler dt=1e-2",
            "slices": SLICES_PER_GPU * G, "slices_per_gpu": SLICES_PER_GPU, "particles_per_slice": P,
            "steps_per_slice": S, "dt": DT, "iterations": K_ITER, "noise": "frozen, numpy-exact Philox stream",
            "step": "one full run_micro_macro", "parallelism": f"slices sharded over {G} GPU(s)",
            "l2": "inputs larger than L2 (5.1 GB of increments per GPU per run)"}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


# SURVEY 8(d) canonical FP64 accounting of the Philox-mode fine propagator:
# I_fp64 = dynamics (OU: fma drift 1 + update 2 + mean 1 = 4) + the dynamic
# FP64 instruction count of curand_normal2_double per normal, measured on
# B200 with dev/curand_fp64.cu under ncu (31.0); peak = measured FP64 issue
# rate, dev/fp64_peak.cu (63.7 DADD/clk/SM) x 148 SMs x the run's SM clock.
FP64_DYNAMICS = 4
FP64_PER_NORMAL = 31.0
FP64_PER_CLK_SM = 63.7
N_SM = 148


def fp64_canonical(psteps_per_s, sm_mhz):
    peak = FP64_PER_CLK_SM * N_SM * sm_mhz * 1e6
    achieved = psteps_per_s * (FP64_DYNAMICS + FP64_PER_NORMAL)
    return {"achieved": achieved, "peak": peak, "unit": "FP64 instr/s", "frac": achieved / peak,
            "model": "SURVEY 8(d): particle-steps/s x (4 dynamics + 31.0 curand_normal2_double FP64 instr per "
                     "normal, dev/curand_fp64.cu) vs measured 63.7 FP64/clk/SM (dev/fp64_peak.cu) at the run's "
                     "SM clock; whole run (noise generation and all sweeps)"}


def ncu_traffic(name="fine_sweep_ncu.json"):
    """Per-launch DRAM bytes of a kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def pipeline_bytes(N, K):
    """Algorithmic HBM bytes of one mmpr_parareal_pipeline launch: the
    increments of every (k, n) fine unit (S*P*8), plus per unit the input
    ensemble read (lifted row 0, ens0 or F^{k-1}_{n-1}), the fine output
    written (K*N) and the matched snapshot written (K*(N+1)), P*8 each."""
    return 8 * P * (K * N * S + N + K * (N + 1) + K * N + K * (N + 1))


# ---------------------------------------------------------------------------
# CPU legs: the unmodified reference (baseline/_ref, pip-installed from
# /root/reference) when it is present, else the oracle's restatement of it
# ---------------------------------------------------------------------------
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def reference_kind() -> str:
    """'reference' when the unmodified mcparareal package is importable from
    baseline/_ref, else 'port' (oracle/mm_oracle.py)."""
    if os.path.isdir(os.path.join(REF_PATH, "mcparareal")):
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        try:
            import mcparareal  # noqa: F401
            return "reference"
        except Exception:  # noqa: BLE001 -- a broken install falls back to the port
            return "port"
    return "port"


def _cpu_slice(args):
    """propagate_fine of slice n of config 4 (noise included), seconds."""
    n, kind = args
    if kind == "reference":
        import mcparareal as R
        model = R.make_perturbed_ou(R.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
        plan = R.NoisePlan(SEED)
        ens = R.sample_initial(R.InitialDistribution.normal(1.0, 0.01), plan, P)
        t = time.perf_counter()
        R.propagate_fine(model, ens, n, n * S * DT, R.StepConfig(DT, S), plan)
        return time.perf_counter() - t
    from oracle import mm_oracle as O
    m = O.model_ou(-1.0, 0.5, 0.5)
    x0 = O.sample_normal_initial(SEED, 1.0, 0.01, P)
    t = time.perf_counter()
    xi = O.slice_noise(SEED, n, S, P)
    O.propagate_fine(m, x0, n, n * S * DT, DT, S, xi)
    return time.perf_counter() - t


def _what(kind):
    return ("the unmodified reference's mcparareal.propagate_fine (baseline/_ref)" if kind == "reference"
            else "the oracle's numpy restatement of propagate_fine")


def cpu_baseline(seconds: float) -> dict:
    """Single-core propagate_fine (noise included) on slices of the workload
    until ~`seconds` of CPU work."""
    kind = reference_kind()
    done, elapsed = 0, 0.0
    while elapsed < seconds and done < SLICES_PER_GPU:
        elapsed += _cpu_slice((done, kind))
        done += 1
    value = done * P * S / elapsed
    return {"value": value, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{done} slice(s) x {S} EM steps x {P} particles of config 4 through {_what(kind)} "
                      f"(numpy Philox/ziggurat noise included), one core, {elapsed:.1f} s"}


def reference_loop(cores: int) -> dict:
    """The reference's own loop (engine.py:127-259), unmodified, on config 4
    with K = 1 (iteration 0 + one Parareal iteration) and its default DP5(4)
    coarse (the reference has no forward-Euler integrator), workers = 1 and
    workers = cores (its GIL-bound thread pool), retain_snapshots=False."""
    import mcparareal as R
    model = R.make_perturbed_ou(R.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    out = {"config": "config 4 (N=64, P=1e5, S=100), K=1, reference default DP5(4) coarse, retain_snapshots=False"}
    for workers in (1, cores):
        cfg = R.PararealConfig(n_slices=SLICES_PER_GPU, iterations=1, slice_length=S * DT, particles=P,
                               step=R.StepConfig(DT, S), workers=workers, retain_snapshots=False)
        t = time.perf_counter()
        R.run_micro_macro(model, R.unimodal_rhs(model), R.InitialDistribution.normal(1.0, 0.01), cfg,
                          R.NoisePlan(SEED))
        el = time.perf_counter() - t
        out[f"run_micro_macro_workers{workers}_s"] = el
        out[f"workers{workers}_particle_steps_per_s"] = SLICES_PER_GPU * P * S / el
    return out


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    kind = reference_kind()
    G = args.gpus
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_cpu_slice, [(n, kind) for n in range(cores)])
        t = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_cpu_slice, [(n, kind) for n in range(cores)])
        elapsed = time.perf_counter() - t
    value = args.steps * cores * P * S / elapsed
    sample = (f"per step: {cores} slices of config 4 ({S} steps x {P} particles each) propagated in parallel by "
              f"{cores} processes running {_what(kind)} (noise included; BASELINE.md section 3, driver 3)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": G,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload(G),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if kind == "reference" and not args.no_reference_loop:
        line["reference_loop"] = reference_loop(cores)
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def _trace_arrays(tr):
    """Per-run trace arrays the drivers must agree on bit for bit."""
    import numpy as np
    return (np.array([[st.packed() for st in row] for row in tr.macro]),
            np.array([[st.packed() for st in row] for row in tr.micro_stats]))


def our_arm(args):
    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch N > 1 through torchrun "
                         "or let bench.py relaunch itself)")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G = world
    import paper_2310_11365_b200 as mm
    from paper_2310_11365_b200 import _lib, distributed

    N = SLICES_PER_GPU * G
    spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
    model = mm.make_perturbed_ou(spec)
    ode = mm.unimodal_rhs(model)
    cfg = mm.PararealConfig(n_slices=N, iterations=K_ITER, slice_length=S * DT, particles=P,
                            step=mm.StepConfig(DT, S), integrator=mm.EulerConfig(1e-2), retain_snapshots=False)
    plan = mm.NoisePlan(SEED)
    init = mm.InitialDistribution.normal(1.0, 0.01)
    ens0_dev = mm.sample_initial(init, plan, P)                    # device-resident input
    ens0_host = ens0_dev.device_positions.cpu().pin_memory()        # pinned host input (e2e)

    def run(ens, timings=False):
        if world > 1:
            return distributed.run_micro_macro_sharded(model, ode, ens, cfg, plan, record_timings=timings)
        return mm.run_micro_macro(model, ode, ens, cfg, plan, record_timings=timings)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    def all_max(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def measure():
        """W warm-up runs, then K timed runs between barriers (CUDA events,
        max over ranks); returns (ms per run, launches, clocks, last trace)."""
        for _ in range(max(args.warmup, 0)):
            run(ens0_dev)
        barrier()
        launches0 = _lib.launch_count["total"]
        with ClockSampler(local) as clocks:
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                tr = run(ens0_dev)
            e1.record()
            barrier()
        return all_max(e0.elapsed_time(e1) / args.steps), _lib.launch_count["total"] - launches0, \
            clocks.summary(), tr

    # ---- device-resident timing, per multi-GPU driver --------------------------
    # G > 1: the per-iteration kernels with NCCL collectives, and the
    # iteration pipeline on every GPU with the rank hand-offs through peer
    # memory (MMPR_SHARDED_PIPELINE=1).  Both run the same inputs; their
    # traces must agree bit for bit, and the faster verified one is `value`.
    drivers = {}
    if G == 1:
        drivers["engine"] = measure()
    else:
        os.environ["MMPR_SHARDED_PIPELINE"] = "0"
        drivers["nccl_per_iteration"] = measure()
        os.environ["MMPR_SHARDED_PIPELINE"] = "1"
        try:
            res = measure()
            ok = 1 if distributed.last_run_info.get("pipeline") else 0
        except Exception as exc:  # noqa: BLE001 -- collective decision below
            print(f"rank {rank}: peer-memory pipeline failed: {exc}", file=sys.stderr, flush=True)
            res, ok = None, 0
        t = torch.tensor([ok], dtype=torch.int32, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
        if int(t.item()) == 1:
            ref_arrays = _trace_arrays(drivers["nccl_per_iteration"][3])
            same = all(np.array_equal(a, b) for a, b in zip(ref_arrays, _trace_arrays(res[3])))
            t = torch.tensor([1 if same else 0], dtype=torch.int32, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
            if int(t.item()) == 1:
                drivers["peer_pipeline"] = res
            else:
                print("peer-memory pipeline trace differs from the NCCL driver's: not reported",
                      file=sys.stderr, flush=True)
    best = min(drivers, key=lambda d: drivers[d][0])
    if G > 1:
        os.environ["MMPR_SHARDED_PIPELINE"] = "1" if best == "peer_pipeline" else "0"
    ms_all, launches, clock_summary, _ = drivers[best]
    # per-launch kernel durations (CUDA events on the launching stream) from
    # two eager runs of the same configuration, for the roofline
    stage_ms = {}
    for _ in range(2):
        tr_t = run(ens0_dev, timings=True)
        for key, vals in tr_t.stage_timings.items():
            if isinstance(vals, list):
                stage_ms.setdefault(key, []).extend(1e3 * v for v in vals)
    fine_ms = stage_ms.get("fine", [])
    psteps = K_ITER * N * P * S
    value = psteps / (ms_all / 1e3)

    # ---- end to end through the public API from pinned host memory ----------
    # warm the host-input path exactly as the timed loop uses it (the previous
    # step's trace still alive when the next run starts: the first such reuse
    # allocates the plan's copy-on-reuse buffers once, ~10 ms)
    for _ in range(max(args.warmup, 3) + 2):
        barrier()
        ens = mm.ParticleEnsemble(ens0_host.to("cuda", non_blocking=True))
        tr = run(ens)
        barrier()
    e2e_times = []
    import gc
    gc.collect()  # (a generation-2 collection landing in the loop costs one sample ~0.5 ms)
    gc.disable()
    for _ in range(args.steps):
        barrier()
        t = time.perf_counter()
        ens = mm.ParticleEnsemble(ens0_host.to("cuda", non_blocking=True))
        tr = run(ens)  # returns after the trace arrays reached host memory
        barrier()
        e2e_times.append(time.perf_counter() - t)
    gc.enable()
    e2e_s = all_max(sum(e2e_times) / len(e2e_times))
    print("e2e ms per step: " + " ".join(f"{1e3 * t:.2f}" for t in e2e_times), file=sys.stderr, flush=True)
    d2h = int(getattr(tr, "d2h_bytes", 0))
    h2d = 8 * P + 8 * (N + 1)  # ens0 from pinned memory + the slice start times

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    peak, peak_src = measured_peak_hbm()
    Ng = SLICES_PER_GPU
    if stage_ms.get("iterations"):
        # iterations 1..K as one persistent kernel: the dominant launch
        kern_bytes = pipeline_bytes(Ng, K_ITER)
        kern_ms = statistics.mean(stage_ms["iterations"])
        roof = {"kernel": "pipeline_kernel (mmpr_parareal_pipeline: iterations 1..K)",
                "traffic": ncu_traffic("pipeline_ncu.json"),
                "bytes_model": "per (k, n) unit: 8 B increment read per particle-step; 8 B per particle for the "
                               "unit's input read, the fine output and the matched snapshot written"}
    else:
        kern_bytes = Ng * S * P * 8 + 2 * Ng * P * 8
        kern_ms = statistics.mean(fine_ms) if fine_ms else float("nan")
        roof = {"kernel": "fine_sweep_kernel (mmpr_fine_sweep)", "traffic": ncu_traffic(),
                "bytes_model": "8 B increment read per particle-step + 16 B per particle per slice (x in/out)"}
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_all, "parareal_iteration_ms": ms_all / K_ITER, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload(G),
        "roofline": {"kernel": roof["kernel"], "bound": "hbm", "achieved": achieved,
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": roof["traffic"], "algorithmic_bytes_per_launch": kern_bytes,
                     "avg_launch_ms": kern_ms, "bytes_model": roof["bytes_model"]},
        "e2e": {"value": psteps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clock_summary,
        "fp64_canonical": fp64_canonical(value / G, clock_summary.get("sm_mhz") or 1965.0),
        "stage_ms_per_run": {k: round(sum(v) / 2, 4) for k, v in stage_ms.items() if v},
    }
    if G > 1:
        line["driver"] = best
        line["drivers"] = {d: {"ms_per_step": r[0], "value": psteps / (r[0] / 1e3), "gpu_launches": r[1]}
                           for d, r in drivers.items()}
        line["drivers_bitwise_equal"] = len(drivers) == 2
    if G == 1 and not args.no_configs:
        line["other_configs"] = other_configs(mm, torch)
    if G == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def other_configs(mm, torch, reps: int = 3) -> dict:
    """The other BASELINE workloads on this GPU, graph-replayed, measured in
    the same run (CUDA events around each full run_micro_macro; mean of
    `reps` after one warm-up): configs 1, 2, 3, config 5 at one GPU's share
    of its 8-GPU run (N = 32 of 256 slices, full P = 2^20, S = 200, K = 10),
    configs 4 and 5 in the counter-based Philox noise mode, and config 4
    with FRESH noise (numpy-exact streams regenerated every iteration vs
    counter-based increments in registers)."""
    import math as _m

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ou = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5))
    init1 = mm.InitialDistribution.normal(1.0, 0.01)
    cub = mm.CubicMeanFieldSpec(1.0, 1.0, 1.0, 0.4)
    mc = mm.make_cubic_meanfield(cub)
    dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
    mdw = mm.make_double_well(dw)
    part = dw.default_partition()
    dw5 = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.3 * _m.sqrt(1.8))
    m5 = mm.make_double_well_multiplicative(dw5, 0.3)
    part5 = dw5.default_partition()
    bim = mm.bimodal_initial(-1.0, 1.0, 0.2)

    def cfg(N, K, T0, P, dt, S, euler, partition=mm.SINGLE_REGION):
        return mm.PararealConfig(n_slices=N, iterations=K, slice_length=T0, particles=P, step=mm.StepConfig(dt, S),
                                 partition=partition, integrator=mm.EulerConfig(euler), retain_snapshots=False)

    cases = [
        ("config1", "linear mean-field OU, N=10, P=1e4, S=100, K=5", cfg(10, 5, 0.1, 10_000, 1e-3, 100, 1e-2),
         ou, mm.unimodal_rhs(ou), init1, mm.NoisePlan(0)),
        ("config2", "cubic mean field, Gaussian closure, N=32, P=1e5, S=64, K=8",
         cfg(32, 8, 0.0625, 100_000, 2.0 ** -10, 64, 2.0 ** -6), mc, mm.gaussian_closure_rhs(cub),
         mm.InitialDistribution.normal(0.5, 0.04), mm.NoisePlan(0)),
        ("config3", "bimodal double well, two regions, N=32, P=1e5, S=64, K=10",
         cfg(32, 10, 0.0625, 100_000, 2.0 ** -10, 64, 2.0 ** -6, part), mdw,
         mm.multimodal_rhs(mdw, part, dw.potential, dw.sigma), bim, mm.NoisePlan(0)),
        ("config5_one_gpu_share", "multiplicative-noise double well, N=32 of 256, P=2^20, S=200, K=10",
         cfg(32, 10, 0.1, 1 << 20, 5e-4, 200, 1e-2, part5), m5,
         mm.multimodal_rhs(m5, part5, dw5.potential, dw5.sigma), bim, mm.NoisePlan(0)),
        ("config4_philox_noise", "config 4 with NoiseMode.PHILOX (increments in registers)",
         cfg(64, 5, 0.1, 100_000, 1e-3, 100, 1e-2), ou, mm.unimodal_rhs(ou), init1,
         mm.NoisePlan(0, mm.NoiseMode.PHILOX)),
        ("config4_fresh_numpy_noise", "config 4 with NoiseMode.FRESH (new numpy-exact streams every iteration)",
         cfg(64, 5, 0.1, 100_000, 1e-3, 100, 1e-2), ou, mm.unimodal_rhs(ou), init1,
         mm.NoisePlan(0, mm.NoiseMode.FRESH)),
        ("config4_philox_fresh_noise", "config 4 with NoiseMode.PHILOX_FRESH (new counter-based increments every "
                                       "iteration, in registers)",
         cfg(64, 5, 0.1, 100_000, 1e-3, 100, 1e-2), ou, mm.unimodal_rhs(ou), init1,
         mm.NoisePlan(0, mm.NoiseMode.PHILOX_FRESH)),
        ("config5_one_gpu_share_philox_noise", "config 5's one-GPU share with NoiseMode.PHILOX (increments in registers)",
         cfg(32, 10, 0.1, 1 << 20, 5e-4, 200, 1e-2, part5), m5,
         mm.multimodal_rhs(m5, part5, dw5.potential, dw5.sigma), bim, mm.NoisePlan(0, mm.NoiseMode.PHILOX)),
    ]
    out = {}
    for name, desc, c, model, ode, init, plan in cases:
        ens = mm.sample_initial(init, mm.NoisePlan(0), c.particles)
        ms = timed(lambda: mm.run_micro_macro(model, ode, ens, c, plan))
        ps = c.iterations * c.n_slices * c.particles * c.step.steps_per_slice
        out[name] = {"workload": desc, "ms_per_run": round(ms, 4), "value": ps / (ms / 1e3), "unit": UNIT,
                     "pipeline": bool(mm.engine.last_run_info.get("pipeline"))}
        mm.engine.clear_graph_cache()
        torch.cuda.empty_cache()
    return out


def relaunch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: run this script
    as N NCCL ranks, one per GPU (torch.distributed.run, 127.0.0.1)."""
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the timings of the other BASELINE configs (one GPU)")
    ap.add_argument("--no-reference-loop", action="store_true",
                    help="reference arm: skip the one-off timing of the reference's own run_micro_macro")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
