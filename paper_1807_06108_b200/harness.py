"""Closed-loop MPC on the device, mirroring jump_mppi.harness.run_trial
(/root/reference/pkg/src/jump_mppi/harness.py:108-153).

Each control step -- mppi_iteration, u0 = clamp(u[0]), plant noise (Sigma_D,
jumps always on), Euler plant step with divergence check, warm_start_shift,
iteration += 1 -- is one replay of a CUDA graph of two kernels (rollout;
finalize, whose last CTA runs the plant step and the shift); the loop never
returns to the host until the trial ends.  Plant noise comes from the device
Philox plant slot keyed on the trial seed (the reference's
RngStream(seed, PLANT_STREAM_ID) role).

run_batch (harness.py:197-233) replaces the reference's process pool with a
trial dimension on the GPU: every trial of every controller variant advances
in the same two launches per control step (grid.y = variant x trial, the
"old" variant's sampler drawing no jumps), each trial bit-identical to its
own run_trial.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from . import engine
from .errors import ControllerError

SLOW_ITERATION_MS = 20.0  # harness.py:27


@dataclass(frozen=True)
class Task:
    """harness.py:69-80."""

    name: str
    model: object
    cost_model: object
    x0: np.ndarray
    duration_steps: int
    success: Optional[Callable[[np.ndarray], bool]] = None
    state_names: Tuple[str, ...] = ()
    control_names: Tuple[str, ...] = ()


@dataclass(frozen=True)
class TrialRecord:
    """harness.py:83-92."""

    config_id: str
    seed: int
    states: np.ndarray
    controls: np.ndarray
    jump_indicators: np.ndarray
    success: bool
    wall_time_per_iteration: np.ndarray
    diverged: bool = False


def run_trial(task: Task, cfg, seed: int, config_id: str = "", *, precision=None,
              device=None) -> TrialRecord:
    """One closed-loop trial of task.duration_steps control steps on the GPU.

    wall_time_per_iteration is the device-clock time of each mppi_iteration
    (rollout start to update ready), the role of harness.py:132-134.
    """
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision=precision, device=device)
    steps = int(task.duration_steps)
    states, controls, jumps, step_ns, div, status = ctx.closed_loop(task.x0, cfg.u_init, seed, steps)
    if status == L.JM_ERR_NO_VIABLE:
        raise ControllerError("no viable rollout")
    diverged = div >= 0
    ok = False
    if not diverged and task.success is not None:
        ok = bool(task.success(np.asarray(states, dtype=float)))
    return TrialRecord(config_id, seed, states, controls, jumps, ok, step_ns * 1e-9, diverged)


@dataclass(frozen=True)
class BatchSummary:
    """harness.py:95-100."""

    success_rate: float
    mean_states: np.ndarray     # (T+1, n)
    ci_halfwidth: np.ndarray    # (T+1, n), 1.96 * sd / sqrt(trials)
    total_variance: float


def trial_seed(base_seed: int, trial_index: int) -> int:
    """Per-trial master seed, identical across controller variants (harness.py:156-159)."""
    ss = np.random.SeedSequence(base_seed, spawn_key=(trial_index,))
    return int(ss.generate_state(1, np.uint64)[0])


def total_variance(trials: Sequence[TrialRecord]) -> float:
    """harness.py:162-167."""
    if len(trials) < 2:
        raise ValueError("variance undefined for fewer than 2 trials")
    stacked = np.stack([t.states for t in trials])
    return float(np.var(stacked, axis=0, ddof=1).sum())


def summarize(trials: Sequence[TrialRecord]) -> BatchSummary:
    """harness.py:170-182."""
    stacked = np.stack([t.states for t in trials])
    k = stacked.shape[0]
    mean = stacked.mean(axis=0)
    if k >= 2:
        sd = stacked.std(axis=0, ddof=1)
        ci = 1.96 * sd / np.sqrt(k)
        tot_var = float(np.var(stacked, axis=0, ddof=1).sum())
    else:
        ci = np.zeros_like(mean)
        tot_var = 0.0
    rate = float(np.mean([t.success for t in trials]))
    return BatchSummary(rate, mean, ci, tot_var)


def run_batch(task: Task, cfg, n_trials: int, base_seed: int, variants: Sequence[str] = ("old", "new"),
              n_workers: Optional[int] = None, config_id: str = "", *, precision=None,
              device=None) -> Dict[str, Tuple[List[TrialRecord], BatchSummary]]:
    """Paired trials per controller variant, summarised (harness.py:197-233).

    Trial k uses the same master seed for every variant (paired plant noise).
    The jobs the reference fans out over its pool -- variants x trials
    (harness.py:215-221) -- run as ONE batch on the GPU (jm_batch_loop_host,
    grid.y = variant x trial; an "old" trial's sampler draws no jumps, exactly
    what jump_sampling_enabled=False does); n_workers is accepted for
    signature compatibility and has no effect -- as in the reference,
    results do not depend on it."""
    if n_trials < 1:
        raise ValueError("trial count must be >= 1")
    for v in variants:
        if v not in ("old", "new"):
            raise ValueError(f"unknown variant {v!r}")
    seeds = [trial_seed(base_seed, k) for k in range(n_trials)]
    steps = int(task.duration_steps)
    # one context whose sampler can draw jumps ("new"), unless only "old" runs
    bcfg = replace(cfg, jump_sampling_enabled=("new" in variants))
    ctx = engine.get_context(task.model, task.cost_model, bcfg, precision=precision, device=device)
    job_seeds = [s for _ in variants for s in seeds]
    flags = [1 if v == "new" else 0 for v in variants for _ in seeds]
    states, controls, jumps, step_ns, div, status = ctx.batch_loop(task.x0, bcfg.u_init, job_seeds, steps,
                                                                    sampler_jumps=flags)
    if np.any(status == L.JM_ERR_NO_VIABLE):
        raise ControllerError("no viable rollout")  # run_trial would raise inside the pool
    out: Dict[str, Tuple[List[TrialRecord], BatchSummary]] = {}
    for vi, variant in enumerate(variants):
        cid = f"{config_id}/{variant}" if config_id else variant
        recs = []
        for k, seed in enumerate(seeds):
            b = vi * n_trials + k
            diverged = bool(div[b] >= 0)
            ok = False
            if not diverged and task.success is not None:
                ok = bool(task.success(np.asarray(states[b], dtype=float)))
            recs.append(TrialRecord(cid, seed, states[b], controls[b], jumps[b], ok, step_ns[b] * 1e-9, diverged))
        out[variant] = (recs, summarize(recs))
    return out
