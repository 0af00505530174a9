#!/usr/bin/env python
"""Benchmark of the sampled-trajectory MPPI core on B200.

Metric (BASELINE.json): rollout state-steps/s (K*T/s) and MPC-iteration
latency.  Default workload = BASELINE config 1: cartpole closed-loop MPC,
K=65536 samples, T=100, BASELINE noise model (sigma=10 N force noise,
Bernoulli(nu dt) theta-dot jumps N(1, 0.5^2), O(1)); one "step" = one
control step on the device (rollout + weighting/update + plant + shift, one
CUDA-graph replay).  fp32, in-kernel Philox noise, synthetic (the configs are
fully synthetic).  Between timed steps a 256 MiB memset evicts the 126 MB L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg1|cfg0|cfg2|cfg3]
                  [--noise philox|hbm] [--precision f32|f64] [--impl ours|reference]

--impl reference times the reference's own CPU path (jump_mppi.mppi_iteration
from baseline/_ref, unmodified) on the host cores, on the reference-expressible
twin of the same config (control-channel jumps; same K, T, model and per
state-step work), one process per core.
N > 1 (torchrun): weak scaling (K samples per GPU) by default, strong scaling
(BASELINE config 3: K in total, K/N per GPU) for cfg3 or --scaling strong;
global sample indices; per control step one all_gather of the reduced
(rho, Z, sum w^2, N[T*m]) record of each rank over NCCL (JM_EXCHANGE=p2p: the
peer-memory exchange), then every rank merges and applies the same update and
plant step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import tempfile
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# algorithmic work per state-step (frozen as the roofline numerator)
FLOPS_PER_STATE_STEP = {"cartpole": 53, "quadrotor": 126}
SFU_OPS_PER_STATE_STEP = {"cartpole": 3, "quadrotor": 7}
# HBM bytes per state-step in noise-from-memory mode (fp32 eps_d + jump tensor, BASELINE noise model)
HBM_BYTES_PER_STATE_STEP = {"cartpole": 8, "quadrotor": 28}
FLUSH_BYTES = 256 << 20

WORKLOADS = {
    "cfg0": dict(index=0, loop=False),
    "cfg1": dict(index=1, loop=True),
    "cfg2": dict(index=2, loop=False),
    "cfg3": dict(index=3, loop=True),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--workload", default="cfg1", choices=sorted(WORKLOADS))
    p.add_argument("--noise", default="philox", choices=["philox", "hbm"])
    p.add_argument("--precision", default="f32", choices=["f32", "f64"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--samples", type=int, default=None, help="override K (per GPU under weak scaling)")
    p.add_argument("--scaling", default=None, choices=["weak", "strong"],
                   help="N > 1: weak = K per GPU (default), strong = K in total, K/N per GPU (default for cfg3)")
    p.add_argument("--horizon", type=int, default=None, help="override T")
    p.add_argument("--block", type=int, default=0, help="override the rollout tile (block_threads, tuning)")
    p.add_argument("--nu", type=float, default=None, help="override the jump rate (tuning; 0 = no jumps)")
    p.add_argument("--jump-process", default=None, choices=["bernoulli", "poisson"], help="override the jump process")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--profile", action="store_true", help="ncu mode: no clock settle, e2e or CPU legs")
    return p.parse_args()


# ---------------------------------------------------------------- reference CPU path
def _ref_import():
    ref = ROOT / "baseline" / "_ref"
    if (ref / "jump_mppi").exists():
        sys.path.insert(0, str(ref))
        import jump_mppi  # noqa: F401

        return jump_mppi, "reference"
    return None, "port"


def _twin_reference_objects(jm, system, K, T):
    """The control-channel twin of a BASELINE config in the reference's own classes."""
    import numpy as np

    if system == "cartpole":
        dt = 0.02
        model = jm.cartpole_dynamics(jm.CartpoleModel(1.0, 0.1, 0.5, 9.81))
        running = jm.CartpoleStateCost(w_pos=1.0, w_vel=0.1, w_angle=10.0, w_avel=0.1)
        cost = jm.CostModel(running, jm.ScaledTerminalCost(running, 10.0), 0.01 * np.eye(1), 1.0, 1.0)
        cfg = jm.MppiConfig(1.0, 1.0, 100.0 * dt, 100.0 * dt, 0.5, dt, T, K, np.zeros(1))
        x0 = np.array([0.0, 0.0, np.pi, 0.0])
    else:
        dt = 0.01
        model = jm.quadrotor_dynamics(jm.QuadrotorModel(1.0, 0.2, (0.0082, 0.0082, 0.0149), 9.81))
        running = jm.QuadrotorStateCost((4.0, 4.0, 2.0), 10.0, 1.0, 5.0, 0.1)
        cost = jm.CostModel(running, jm.ScaledTerminalCost(running, 10.0), 0.01 * np.eye(4), 1.0, 1.0)
        sd = np.diag(np.array([2.0, 0.1, 0.1, 0.1]) ** 2) * dt
        cfg = jm.MppiConfig(1.0, 1.0, sd, sd, 1.0, dt, T, K, np.array([9.81, 0, 0, 0]))
        x0 = np.zeros(12)
    return model, cost, cfg, x0


def _cpu_step_fn(spec):
    """One reference iteration (+ shift) on this process's share of the samples."""
    jm, kind = _ref_import()
    if jm is None:  # oracle port (numpy restatement) -- only when baseline/_ref is absent
        from oracle import mppi as om
        import numpy as np

        from paper_1807_06108_b200 import experiment

        task, cfg = experiment.baseline_config(1 if spec["system"] == "cartpole" else 2, mode="control",
                                               K=spec["K"], T=spec["T"])
        ospec = om.spec_from_plugins(task.model, task.cost_model, cfg)
        u = np.tile(cfg.u_init, (cfg.horizon_n, 1))

        def one(it):
            noise = om.sample_noise_batch_ref(spec["seed"], it, ospec)
            om.mppi_iteration_oracle(ospec, task.x0, u, noise)
    else:
        model, cost, cfg, x0 = _twin_reference_objects(jm, spec["system"], spec["K"], spec["T"])
        ctrl = jm.initial_controller_state(cfg)

        def one(it):
            seq, _ = jm.mppi_iteration(jm.ControllerState(ctrl.nominal_controls, it, cfg), model, cost, x0,
                                       master_seed=spec["seed"])
            jm.warm_start_shift(seq, cfg.u_init)

    return one, kind


def _cpu_proc(spec, barrier, times, kinds, slot):
    """Worker of run_cpu: every step starts and ends at a barrier across all workers, so
    worker 0's clock around (barrier, step, barrier) is the wall clock of the whole step."""
    one, kind = _cpu_step_fn(spec)
    kinds[slot] = 1 if kind == "reference" else 0
    one(0)  # warm-up (imports, allocator)
    for it in range(spec["iters"]):
        barrier.wait()
        t0 = time.perf_counter()
        one(it + 1)
        barrier.wait()
        if slot == 0:
            times[it] = time.perf_counter() - t0


def run_cpu(system, K, T, iters, procs, seed=0):
    """`procs` single-thread reference processes, each on K/procs samples, stepping in lockstep:
    the step time is the synchronised wall clock of the slowest process, not a per-process timer."""
    import multiprocessing as mp

    kp = max(1, K // procs)
    spec = {"system": system, "K": kp, "T": T, "iters": iters, "seed": seed}
    keys = {"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1", "CUDA_VISIBLE_DEVICES": ""}
    saved = {k: os.environ.get(k) for k in keys}
    os.environ.update(keys)  # inherited by the spawned workers (fresh interpreters: no CUDA state)
    try:
        ctx = mp.get_context("spawn")
        barrier = ctx.Barrier(procs)
        times = ctx.Array("d", iters)
        kinds = ctx.Array("i", procs)
        t0 = time.perf_counter()
        ps = [ctx.Process(target=_cpu_proc, args=(spec, barrier, times, kinds, i)) for i in range(procs)]
        for p in ps:
            p.start()
        for p in ps:
            p.join()
        wall = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    if any(p.exitcode != 0 for p in ps):
        raise RuntimeError(f"cpu worker failed (exit codes {[p.exitcode for p in ps]})")
    return list(times), ("reference" if kinds[0] else "port"), kp * procs, wall


def _host_cpu():
    """CPU model and logical core count of the box (state the host)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count()}


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = WORKLOADS[a.workload]
    system = "cartpole" if w["index"] in (0, 1) else "quadrotor"
    from paper_1807_06108_b200.experiment import BASELINE_SHAPES  # shapes only, no CUDA

    K = a.samples or BASELINE_SHAPES[w["index"]]["K"]
    T = a.horizon or BASELINE_SHAPES[w["index"]]["T"]
    procs = os.cpu_count() or 1
    # bounded sample: all cores, K split across them (capped so one step stays < ~1 s)
    Ks = min(K, procs * (8192 if system == "cartpole" else 2048))
    n = a.warmup + a.steps
    per_step, kind, Kdone, _ = run_cpu(system, Ks, T, n, procs)
    timed = per_step[a.warmup:]
    ms = 1e3 * statistics.mean(timed)
    val = Kdone * T / (ms * 1e-3)
    sample = (f"reference jump_mppi.mppi_iteration + warm_start_shift ({'baseline/_ref' if kind == 'reference' else 'oracle port'}), "
              f"control-channel twin of {a.workload}: {procs} processes x {Kdone // procs} samples x T={T} per step "
              f"(K={Kdone} of {K}), 1 thread each, lockstep (barrier per step: synchronised wall clock)")
    line = {
        "impl": "reference", "metric": "rollout state-steps/sec (K*T/s)", "value": val, "unit": "state-steps/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{a.workload} (control-channel twin)", "system": system, "K": Kdone, "T": T},
        "cpu_baseline": {"value": val, "unit": "state-steps/s", "cores": procs, "kind": kind, "sample": sample,
                         "host": _host_cpu()},
        "e2e": {"value": val, "unit": "state-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = Path(tempfile.gettempdir()) / f"jm_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return None
        rows = []
        for ln in self.path.read_text().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                rows.append((float(f[0]), float(f[1]), float(f[2]), float(f[3]), f[4:8]))
            except ValueError:
                continue
        if not rows:
            return None
        busy = [r for r in rows if r[3] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i, v in enumerate(r[4]) if v.lower() == "active"})
        self.path.unlink(missing_ok=True)
        return {"sm_mhz": statistics.median(r[0] for r in busy), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(busy), "power_w_max": max(r[2] for r in rows)}


# ---------------------------------------------------------------- ours
def kernel_source_hash():
    """sha256 over the CUDA sources of libjmppi.so (csrc/*.cu, *.cuh, internal.h, include/jmppi.h):
    the stamp profiles/kernel_counters.json carries, so a capture of an older kernel is refused."""
    import hashlib

    h = hashlib.sha256()
    src = ROOT / "paper_1807_06108_b200" / "csrc"
    files = sorted(list(src.glob("*.cu")) + list(src.glob("*.cuh")) + [src / "internal.h", ROOT / "include" / "jmppi.h"])
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def counters_from_profiles(workload, precision, noise, K):
    """ncu counters of the rollout kernel of this workload (dram bytes, warp instructions per
    launch) from profiles/kernel_counters.json -- only if the capture was taken from the kernel
    sources of this tree (src_hash) and at this K; else (None, reason)."""
    f = ROOT / "profiles" / "kernel_counters.json"
    try:
        d = json.loads(f.read_text())
    except (ValueError, OSError):
        return None, "no profiles/kernel_counters.json"
    e = d.get("captures", {}).get(f"{workload}/{precision}/{noise}/K={K}")
    if e is None:
        return None, "no ncu capture of this workload"
    if e.get("src_hash") != kernel_source_hash():
        return None, f"stale: captured at kernel sources {e.get('src_hash')}, this tree is {kernel_source_hash()}"
    return e, None


def ours_arm(a):
    import ctypes as C

    import numpy as np

    import paper_1807_06108_b200 as jb
    from paper_1807_06108_b200 import _lib as L
    from paper_1807_06108_b200 import engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or os.environ.get("JM_SHARDED_BENCH"):  # (the env var: exercise the sharded path at N=1)
        from paper_1807_06108_b200 import distributed as jd

        return jd.bench_sharded(a, world, rank, local, clock_sampler=ClockSampler,
                                flops_per_state_step=FLOPS_PER_STATE_STEP)

    w = WORKLOADS[a.workload]
    idx = w["index"]
    task, cfg = jb.baseline_config(idx, K=a.samples, T=a.horizon)
    if a.nu is not None or a.jump_process is not None:
        import dataclasses

        cfg = dataclasses.replace(cfg, nu=cfg.nu if a.nu is None else a.nu,
                                  jump_process=a.jump_process or cfg.jump_process)
    system = task.name
    K, T = cfg.samples_m, cfg.horizon_n
    hbm = a.noise == "hbm"
    use_loop = w["loop"] and not hbm
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision=a.precision, hbm=hbm, device=local,
                             block_threads=a.block)
    lib = ctx.lib
    peaks = engine.microbench(local)

    def ck(rc):
        ctx.check(rc)

    n_total = a.warmup + a.steps
    step_ms = np.zeros(a.steps)
    roll_ms = np.zeros(a.steps)
    x0 = np.ascontiguousarray(task.x0, float)
    u0 = np.ascontiguousarray(np.tile(cfg.u_init, (T, 1)), float)
    ck(lib.jm_upload_inputs(ctx.h, L.dptr(x0), L.dptr(u0)))  # device-resident inputs for jm_bench_iteration

    def settle():
        if a.profile:
            return
        # ~1 s of back-to-back device iterations (not timed) so the clock record covers a loaded GPU
        buf = np.zeros(64)
        t_end = time.time() + 1.0
        while time.time() < t_end:
            ck(lib.jm_bench_iteration(ctx.h, 64, 0, L.dptr(buf), None))

    if use_loop:
        ui = np.ascontiguousarray(cfg.u_init, float)
        cap = 2 * n_total + 64

        def init():
            ck(lib.jm_loop_init(ctx.h, L.dptr(x0), L.dptr(ui), C.c_uint64(0), C.c_uint64(0), cap))

        def check_running():
            xs = np.zeros(ctx.N)
            it, stp, halted, status = C.c_uint64(), C.c_int32(), C.c_int32(), C.c_int32()
            ck(lib.jm_loop_read(ctx.h, L.dptr(xs), C.byref(it), C.byref(stp), C.byref(halted), C.byref(status)))
            if halted.value:
                raise RuntimeError(f"closed loop halted during the bench (status {status.value}, step {stp.value})")

        init()
        wbuf = np.zeros(max(1, a.warmup))
        if a.warmup:
            ck(lib.jm_bench_loop(ctx.h, a.warmup, FLUSH_BYTES, 2, L.dptr(wbuf), None))
        with ClockSampler(local) as clk:
            settle()
            ck(lib.jm_bench_loop(ctx.h, a.steps, FLUSH_BYTES, 2, L.dptr(step_ms), None))
        check_running()
        # kernel-level pass: the same control steps with direct launches, events around the rollout kernel
        init()
        if a.warmup:
            ck(lib.jm_bench_loop(ctx.h, a.warmup, FLUSH_BYTES, 0, L.dptr(wbuf), None))
        ck(lib.jm_bench_loop(ctx.h, a.steps, FLUSH_BYTES, 0, L.dptr(np.zeros(a.steps)), L.dptr(roll_ms)))
        check_running()
        launches = 2 * a.steps
    else:
        wbuf = np.zeros(max(1, a.warmup))
        if a.warmup:
            ck(lib.jm_bench_iteration(ctx.h, a.warmup, FLUSH_BYTES, L.dptr(wbuf), None))
        with ClockSampler(local) as clk:
            settle()
            ck(lib.jm_bench_iteration(ctx.h, a.steps, FLUSH_BYTES, L.dptr(step_ms), None))
        # kernel-level pass: events around the rollout kernel alone
        ck(lib.jm_bench_iteration(ctx.h, a.steps, FLUSH_BYTES, L.dptr(np.zeros(a.steps)), L.dptr(roll_ms)))
        launches = 2 * a.steps
    ms = float(np.mean(step_ms))
    rms = float(np.mean(roll_ms))
    clocks = clk.summary()
    value = K * T / (ms * 1e-3)
    flops = FLOPS_PER_STATE_STEP[system] * K * T
    achieved = flops / (rms * 1e-3) / 1e12
    peak = peaks["fp32_tflops"]
    roof = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": None,
            "kernel": ctx.lib.jm_kernel_name(ctx.h).decode(), "kernel_ms": rms, "kernel_share_of_step": rms / ms,
            "flops_per_state_step": FLOPS_PER_STATE_STEP[system],
            "peak_source": "live FFMA microbenchmark (jm_microbench), no FP32 entry in MEASURED_PEAKS.json",
            "mufu_peak_tops": peaks["mufu_tops"], "fp64_peak_tflops": peaks["fp64_tflops"]}
    # SFU view: the algorithmic MUFU-class ops per state-step (SURVEY Appendix C:
    # sin, cos, rcp for the cartpole; 6 trig + rcp for the quadrotor) against the
    # live MUFU microbenchmark peak
    sfu_ops = SFU_OPS_PER_STATE_STEP[system] * K * T / (rms * 1e-3) / 1e12
    roof["sfu"] = {"ops_per_state_step": SFU_OPS_PER_STATE_STEP[system], "achieved_tops": sfu_ops,
                   "peak_tops": peaks["mufu_tops"], "frac": sfu_ops / peaks["mufu_tops"]}
    # issue-slot view of the same kernel: warp-instructions per state-step from the
    # committed ncu capture, and the rate at which 4 schedulers/SM issuing every
    # cycle would retire them -- what bounds this FP32-light, latency-bound loop
    cap, why = counters_from_profiles(a.workload, a.precision, a.noise, K)
    if cap is None:
        roof["traffic_note"] = why
    else:
        roof["traffic"] = cap.get("dram_bytes")
        roof["traffic_source"] = cap.get("source")
    ninst = cap.get("warp_instructions") if cap else None
    if ninst:
        ips = ninst / (K * T / 32.0)
        import torch
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        ceil = sms * 4 * mhz * 1e6 * 32 / ips
        roof["issue_slots"] = {"warp_instructions_per_state_step": ips, "ceiling_state_steps_per_s": ceil,
                               "achieved_state_steps_per_s": K * T / (rms * 1e-3),
                               "frac": K * T / (rms * 1e-3) / ceil,
                               "source": f"smsp__inst_executed of {cap.get('source')}; 4 issue slots/SM/cycle"}
    if hbm:
        bpss = HBM_BYTES_PER_STATE_STEP[system] * (2 if a.precision == "f64" else 1)
        gbs = bpss * K * T / (rms * 1e-3) / 1e9
        meas = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
        roof["hbm"] = {"achieved": gbs, "peak": meas, "unit": "GB/s", "frac": gbs / meas,
                       "bytes_per_state_step": bpss}

    line = {
        "metric": "rollout state-steps/sec (K*T/s)", "value": value, "unit": "state-steps/s", "n_gpus": 1,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": a.precision, "data": "synthetic",
        "config": {"workload": f"{a.workload}: BASELINE config {idx} ({system}, K={K}, T={T}, "
                               f"{'closed-loop control step' if use_loop else 'single MPC iteration'}, "
                               f"state-space jumps, {a.noise} noise)",
                   "K": K, "T": T, "system": system, "noise": a.noise, "nu": cfg.nu, "jump_process": cfg.jump_process,
                   "l2": "flushed (256 MiB memset) before each timed step",
                   "step": "rollout+weighting/update+plant+shift; the K timed steps are one CUDA graph (per step: L2 flush, event, 2 kernels, event)" if use_loop else "rollout+weighting/update"},
        "mpc_iteration_latency_ms": ms,
        "roofline": roof,
        "gpu_launches": launches,
    }
    if clocks:
        line["clocks"] = clocks

    # ---- e2e through the public drop-in API with host buffers
    if not (a.no_e2e or a.profile):
        ctrl = jb.initial_controller_state(cfg)
        x0 = np.asarray(task.x0, float)
        e2e = []
        b0 = (C.c_int64(), C.c_int64())
        b1 = (C.c_int64(), C.c_int64())
        for i in range(a.warmup + a.steps):
            if i == a.warmup:
                lib.jm_transfer_bytes(C.byref(b0[0]), C.byref(b0[1]))
            t0 = time.perf_counter()
            seq, diag = jb.mppi_iteration(ctrl, task.model, task.cost_model, x0, 0, precision=a.precision,
                                          device=local)
            ctrl = jb.ControllerState(jb.warm_start_shift(seq, cfg.u_init), ctrl.iteration_index + 1, cfg)
            e2e.append(time.perf_counter() - t0)
        e_ms = 1e3 * statistics.mean(e2e[a.warmup:])
        # bytes the library moved during the timed iterations (jm_transfer_bytes counts every
        # copy it issues): one staged block [x0|u_nom|mapping|u_init] in and one block
        # [u_new|norms|diag|status|u_shift] out per iteration; the per-sample weights stay on the
        # GPU until UpdateDiagnostics.weights is read
        lib.jm_transfer_bytes(C.byref(b1[0]), C.byref(b1[1]))
        h2d = (b1[0].value - b0[0].value) // a.steps
        d2h = (b1[1].value - b0[1].value) // a.steps
        line["e2e"] = {"value": K * T / (e_ms * 1e-3), "unit": "state-steps/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
                       "path": "paper_1807_06108_b200.mppi_iteration + warm_start_shift (numpy in/out), "
                               "the reference's `jump-mppi bench` loop (cli.py:157-183)"}

    # ---- CPU baseline (rank 0, N=1): the reference on one host core, bounded sample
    if not (a.no_cpu_baseline or a.profile):
        try:
            per_step, kind, Kdone, _ = run_cpu(system, min(K, 65536 if system == "cartpole" else 8192), T, 3, 1)
            cs = statistics.mean(per_step)
            line["cpu_baseline"] = {
                "value": Kdone * T / cs, "unit": "state-steps/s", "cores": 1, "kind": kind, "host": _host_cpu(),
                "sample": f"3 x jump_mppi.mppi_iteration+warm_start_shift at K={Kdone}, T={T}, control-channel twin "
                          f"of {a.workload}, 1 thread ({cs:.3f} s/iteration)"}
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(exc)[:300]}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
        return
    ours_arm(a)


if __name__ == "__main__":
    main()
