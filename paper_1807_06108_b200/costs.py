"""Cost plugins, mirroring jump_mppi.costs
(/root/reference/pkg/src/jump_mppi/costs.py).

As with the dynamics, a cost is a parameter description of a device cost
(csrc/systems.cuh); the modified running cost
    q~ = q + 1/2 u'Ru + lambda u'eps/sqrt(dt) + 1/2 lambda (1-1/c) eps'eps/dt
(costs.py:80-111, control-channel form) is evaluated inside the rollout kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np


class CostModelError(RuntimeError):
    pass


@dataclass(frozen=True)
class CartpoleStateCost:
    """q = w_pos x^2 + w_vel xdot^2 + w_angle (1+cos th)^2 + w_avel thdot^2 (costs.py:149-168)."""

    w_pos: float = 2.5
    w_vel: float = 1.0
    w_angle: float = 50.0
    w_avel: float = 1.0


@dataclass(frozen=True)
class QuadrotorStateCost:
    """q = w_pos|p-p*|^2 + w_vel|v|^2 + w_att(roll^2+pitch^2) + w_rate|w|^2 (costs.py:171-190)."""

    target: Tuple[float, float, float]
    w_pos: float = 4.0
    w_vel: float = 1.0
    w_att: float = 10.0
    w_rate: float = 1.0


@dataclass(frozen=True)
class DiagQuadraticCost:
    """q = sum_i w_i (x_i - x*_i)^2.

    Covers tests/conftest.py:43-49 (quadratic_q: w = 1, x* = 0), the zero cost
    (w = 0) and the BASELINE cartpole cost diag(1, 0.1, 10, 0.1) on the error
    to upright x* = (0, 0, pi, 0) (angle error unwrapped).
    """

    weights: Tuple[float, ...]
    target: Optional[Tuple[float, ...]] = None


@dataclass(frozen=True)
class ScaledTerminalCost:
    """phi(x) = scale * q(x) (costs.py:193-201)."""

    running: object
    scale: float = 10.0


@dataclass(frozen=True)
class CostModel:
    """State cost, terminal cost, R, lambda, c (costs.py:28-56).

    `terminal_cost` is a ScaledTerminalCost, or the same cost object as
    `state_cost` (scale 1).  Only the control-channel form of the modified
    cost (control_channel=True, calB = bb = I) has a kernel.
    """

    state_cost: object
    terminal_cost: object
    control_cost_matrix: np.ndarray
    lambda_: float
    c: float
    control_channel: bool = True
    cal_b: Optional[np.ndarray] = None
    bb_term: Optional[np.ndarray] = None

    def __post_init__(self):
        r = np.atleast_2d(np.asarray(self.control_cost_matrix, dtype=float))
        object.__setattr__(self, "control_cost_matrix", r)


def control_cost_matrix_from_dynamics(model, x, t: float, lambda_: float) -> np.ndarray:
    """R = lambda G' (B B')^+ G at one state (costs.py:59-77); the pseudo-inverse
    keeps a rank-deficient diffusion consistent.  Host-side utility."""
    g = np.asarray(model.control_matrix(x, t), dtype=float)
    b = np.asarray(model.diffusion_matrix(x, t), dtype=float)
    try:
        sig_pinv = np.linalg.pinv(b @ b.T, hermitian=True)
    except np.linalg.LinAlgError as exc:
        raise CostModelError("control cost undefined for this dynamics") from exc
    r = lambda_ * (g.T @ sig_pinv @ g)
    if not np.all(np.isfinite(r)):
        raise CostModelError("control cost undefined for this dynamics")
    return r


def quadratic_cost_model(n: int, lambda_=1.0, c=1.0, m=1, r=1.0) -> CostModel:
    """tests/conftest.py:62-69: q = phi = x'x, R = r I."""
    q = DiagQuadraticCost(tuple([1.0] * n))
    return CostModel(q, q, r * np.eye(m), lambda_, c)


def zero_cost_model(n: int, lambda_=1.0, c=1.0, m=1) -> CostModel:
    """tests/conftest.py:52-59: q = phi = 0, R = 0."""
    q = DiagQuadraticCost(tuple([0.0] * n))
    return CostModel(q, q, np.zeros((m, m)), lambda_, c)
