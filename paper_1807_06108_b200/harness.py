"""Closed-loop MPC on the device, mirroring jump_mppi.harness.run_trial
(/root/reference/pkg/src/jump_mppi/harness.py:108-153).

Each control step -- mppi_iteration, u0 = clamp(u[0]), plant noise (Sigma_D,
jumps always on), Euler plant step with divergence check, warm_start_shift,
iteration += 1 -- is one replay of a CUDA graph of three kernels (rollout,
finalize, plant+shift); the loop never returns to the host until the trial
ends.  Plant noise comes from the device Philox plant slot keyed on the trial
seed (the reference's RngStream(seed, PLANT_STREAM_ID) role).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

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
