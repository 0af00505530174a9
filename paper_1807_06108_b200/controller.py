"""Drop-in controller API, mirroring jump_mppi.controller
(/root/reference/pkg/src/jump_mppi/controller.py).

Every numeric step runs in libjmppi.so on the GPU:

    mppi_iteration   controller.py:103-181  -> jm_iteration_host
    compute_weights  controller.py:62-71    -> jm_compute_weights_host
    update_controls  controller.py:81-93    -> jm_update_controls_host
    warm_start_shift controller.py:96-100   -> jm_shift_host

`mppi_iteration` accepts the reference's own plugin objects as well as this
package's.  Keyword-only extensions:
  noise=      fed noise tensors (eps_d, indicators, eps_j, eps_combined), shapes
              (K,N,m), (K,N), (K,N,q), (K,N,m) as sample_noise_batch returns
              them -> the HBM (noise-from-memory) mode used for oracle parity;
              default: in-kernel Philox keyed on (master_seed, iteration_index).
  precision=  "f32" (default, JM_B200_PRECISION overrides) or "f64".
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import ctypes as C
import numpy as np

from . import _lib as L
from . import engine
from .errors import ControllerError
from .types import ControlSequence, NoiseRealization, RolloutResult, StateTrajectory

__all__ = [
    "ControllerError", "ControllerState", "UpdateDiagnostics", "initial_controller_state",
    "compute_weights", "update_controls", "warm_start_shift", "mppi_iteration",
]


@dataclass(frozen=True)
class ControllerState:
    """Nominal sequence + the iteration counter that seeds sampling (controller.py:35-45)."""

    nominal_controls: ControlSequence
    iteration_index: int
    config: object

    def __post_init__(self):
        if len(self.nominal_controls) != self.config.horizon_n:
            raise ValueError("nominal_controls length must equal config.horizon_n")


class UpdateDiagnostics:
    """controller.py:48-53: weights (M,), min_cost, effective_sample_size,
    per_step_update_norm (N,).

    The per-sample weights of a drop-in iteration stay on the GPU until first
    read (a K-double download per iteration otherwise dominates the call);
    `weights` then downloads them once and caches the array."""

    __slots__ = ("_weights", "_ctx", "_handle", "_z", "min_cost", "effective_sample_size",
                 "per_step_update_norm", "__weakref__")

    def __init__(self, weights=None, min_cost=0.0, effective_sample_size=0.0, per_step_update_norm=None,
                 *, _ctx=None, _handle=0, _z=0.0):
        self._weights = None if weights is None else np.asarray(weights)
        self._ctx = _ctx
        self._handle = _handle
        self._z = _z
        self.min_cost = min_cost
        self.effective_sample_size = effective_sample_size
        self.per_step_update_norm = per_step_update_norm

    @property
    def weights(self) -> np.ndarray:
        if self._weights is None and self._handle:
            w = self._ctx.stash_fetch(self._handle, self.min_cost, self._z)
            w.setflags(write=False)
            self._ctx.stash_release(self._handle)
            self._handle = 0
            self._ctx = None
            self._weights = w
        return self._weights

    def __del__(self):
        if getattr(self, "_handle", 0):
            try:
                self._ctx.stash_release(self._handle)
            except Exception:
                pass

    def __repr__(self):
        return (f"UpdateDiagnostics(min_cost={self.min_cost!r}, "
                f"effective_sample_size={self.effective_sample_size!r})")


def _device() -> int:
    import os

    return int(os.environ.get("JM_B200_DEVICE", "0"))


def initial_controller_state(cfg) -> ControllerState:
    """Nominal sequence filled with u_init (controller.py:56-59)."""
    controls = np.tile(np.atleast_1d(cfg.u_init), (cfg.horizon_n, 1))
    return ControllerState(ControlSequence(controls, cfg.dt), 0, cfg)


def compute_weights(costs, lambda_: float) -> np.ndarray:
    """Softmax weights, +inf costs -> exactly 0, all non-finite -> ControllerError."""
    costs = np.ascontiguousarray(costs, dtype=float).reshape(-1)
    w = np.empty_like(costs)
    rc = L.load().jm_compute_weights_host(_device(), costs.shape[0], L.dptr(costs), float(lambda_), L.dptr(w))
    engine.raise_status(rc)
    return w


def update_controls(ctrl: ControllerState, rollouts: Sequence[RolloutResult], mapping=None) -> ControlSequence:
    """Weighted perturbation average applied to the nominal sequence."""
    costs = np.ascontiguousarray([r.cost for r in rollouts], dtype=float)
    eps = np.ascontiguousarray(np.stack([r.noise.eps_combined for r in rollouts]), dtype=float)
    K, T, m = eps.shape
    u_nom = np.ascontiguousarray(ctrl.nominal_controls.controls, dtype=float)
    u_new = np.empty_like(u_nom)
    mp = None if mapping is None else np.ascontiguousarray(mapping, dtype=float)
    rc = L.load().jm_update_controls_host(
        _device(), K, T, m, L.dptr(costs), L.dptr(eps), float(ctrl.config.lambda_), float(ctrl.config.dt),
        L.dptr(u_nom), L.dptr(mp), L.dptr(u_new), None)
    engine.raise_status(rc)
    return ControlSequence(u_new, ctrl.config.dt)


def warm_start_shift(controls: ControlSequence, u_init) -> ControlSequence:
    """Drop u_0, shift forward, refill the tail with u_init.

    A sequence returned by mppi_iteration already carries its shift for the
    config's u_init, computed by the iteration's finalize kernel; any other
    sequence / u_init is shifted by a device kernel."""
    pre = getattr(controls, "_shifted", None)
    if pre is not None and (u_init is pre[0] or np.array_equal(np.atleast_1d(np.asarray(u_init, float)), pre[0])):
        return ControlSequence._adopt(pre[1], controls.dt)
    u = np.ascontiguousarray(controls.controls, dtype=float)
    T, m = u.shape
    ui = np.ascontiguousarray(np.atleast_1d(np.asarray(u_init, dtype=float)).reshape(m))
    out = np.empty_like(u)
    rc = L.load().jm_shift_host(_device(), T, m, L.dptr(u), L.dptr(ui), L.dptr(out))
    engine.raise_status(rc)
    return ControlSequence(out, controls.dt)


def _unpack_noise(noise):
    if isinstance(noise, (tuple, list)):
        eps_d, ind, eps_j, eps_c = noise
    else:
        eps_d, ind, eps_j, eps_c = noise.eps_d, noise.jump_indicator, noise.eps_j, noise.eps_combined
    return (np.asarray(eps_d, float), np.asarray(ind), np.asarray(eps_j, float), np.asarray(eps_c, float))


def mppi_iteration(
    ctrl: ControllerState,
    model,
    cost_model,
    x0: np.ndarray,
    master_seed: int,
    mapping: Optional[np.ndarray] = None,
    return_rollouts: bool = False,
    *,
    noise=None,
    precision: Optional[str] = None,
    device: Optional[int] = None,
):
    """One sampling-and-update pass from x0 on the GPU (controller.py:103-181).

    Deterministic given (master_seed, ctrl.iteration_index).  Returns
    (ControlSequence, UpdateDiagnostics[, list[RolloutResult]]).
    """
    if master_seed < 0 or ctrl.iteration_index < 0:
        raise ValueError("master_seed and stream_id must be nonnegative")  # noise.py:46-47
    cfg = ctrl.config
    ctx = engine.get_context(model, cost_model, cfg, precision=precision, hbm=noise is not None,
                             device=device)
    K, T, m = ctx.K, ctx.T, ctx.M
    eps_arg = jump_arg = None
    if noise is not None:
        eps_d, ind, eps_j, eps_c = _unpack_noise(noise)
        if eps_c.shape != (K, T, m):
            raise ValueError(f"eps_combined must have shape {(K, T, m)}, got {eps_c.shape}")
        eps_arg = ctx.step_major(eps_c, m)
        if ctx.mdesc.jump_channel == L.JM_JUMP_STATE:
            q = ctx.Q
            # indicator (or Poisson count: eps_j already sums the step's marks) * mark
            jump = (np.asarray(ind) != 0).astype(float).reshape(K, T, 1) * np.asarray(eps_j, float).reshape(K, T, q)
            jump_arg = ctx.step_major(jump, q)
    u_init = np.atleast_1d(np.asarray(cfg.u_init, dtype=float))
    if noise is None and mapping is None and not return_rollouts:
        # the drop-in fast path: one compact C call (jm_iteration_dropin)
        u_new, norms, (mc, ess, z, _), u_shift, handle = ctx.iteration_dropin(
            x0, ctrl.nominal_controls.controls, master_seed, ctrl.iteration_index, u_init)
        new_controls = ControlSequence._adopt(u_new, cfg.dt)  # views of a fresh output block
        norms.setflags(write=False)
        object.__setattr__(new_controls, "_shifted", (u_init, u_shift))
        return new_controls, UpdateDiagnostics(weights=None, min_cost=mc, effective_sample_size=ess,
                                               per_step_update_norm=norms, _ctx=ctx, _handle=handle, _z=z)
    out = ctx.iteration(x0, ctrl.nominal_controls.controls, master_seed, ctrl.iteration_index,
                        eps_c=eps_arg, jump=jump_arg, mapping=mapping, want_costs=return_rollouts,
                        want_weights=True, trace=return_rollouts, u_init=u_init,
                        stash_weights=not return_rollouts)
    dt = cfg.dt
    new_controls = ControlSequence(out.u_new, dt)
    object.__setattr__(new_controls, "_shifted", (u_init, out.u_shift))
    diagnostics = UpdateDiagnostics(
        weights=out.weights,
        min_cost=float(out.diag.min_cost),
        effective_sample_size=float(out.diag.ess),
        per_step_update_norm=out.norms,
        _ctx=ctx if out.stash else None,
        _handle=out.stash,
        _z=float(out.diag.normaliser),
    )
    if not return_rollouts:
        return new_controls, diagnostics
    if noise is None:
        eps_d, ind, eps_j, eps_c = ctx.sample_noise(master_seed, ctrl.iteration_index)
    rollouts: List[RolloutResult] = []
    for k in range(K):
        d = int(out.diverged[k])
        rollouts.append(RolloutResult(
            StateTrajectory(out.states[k], dt),
            NoiseRealization(eps_d[k], ind[k], eps_j[k], eps_c[k]),
            float(out.costs[k]),
            d if d >= 0 else None,
        ))
    return new_controls, diagnostics, rollouts
