"""Dynamics plugins, mirroring jump_mppi.dynamics
(/root/reference/pkg/src/jump_mppi/dynamics.py).

The reference's DynamicsModel carries numpy callables f, G, B, H.  Here a model
is a *description* the device kernels are compiled for (csrc/systems.cuh): the
physical parameter object (CartpoleModel / QuadrotorModel / IntegratorModel),
control limits and the noise routing.  Evaluation happens only on the GPU,
inside mppi_iteration / run_trial; there is no numpy path.

Noise routing:
  jump_channel="control"  B = H = G (the reference's cartpole_dynamics /
                          quadrotor_dynamics, dynamics.py:274-283, :399-409)
  jump_channel="state"    B = G, H = constant selector on `jump_rows`
                          (theta-dot for the cartpole, the linear velocities
                          for the quadrotor: the BASELINE configs; SURVEY
                          Appendix A), jump_scale_mode "unit" = O(1) increment.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np


class StateDivergedError(RuntimeError):
    """Non-finite state (dynamics.py:29-33)."""

    def __init__(self, step_index=None):
        self.step_index = step_index
        at = "" if step_index is None else f" at step {step_index}"
        super().__init__(f"state diverged{at}")


@dataclass(frozen=True)
class CartpoleModel:
    """Cart with a point-mass pole, theta = pi upright (dynamics.py:194-203)."""

    cart_mass: float = 1.0
    pole_mass: float = 0.1
    pole_half_length: float = 0.5
    gravity: float = 9.81

    def __post_init__(self):
        if min(self.cart_mass, self.pole_mass, self.pole_half_length, self.gravity) <= 0:
            raise ValueError("cartpole parameters must be positive")

    def control_matrix(self, x, t=0.0) -> np.ndarray:
        """G(x) (4, 1) of dynamics.py:221-228, host-side (the kernels inline it)."""
        th = float(np.asarray(x, float)[2])
        den = self.cart_mass + self.pole_mass * np.sin(th) ** 2
        g = np.zeros((4, 1))
        g[1, 0] = 1.0 / den
        g[3, 0] = -np.cos(th) / (self.pole_half_length * den)
        return g


@dataclass(frozen=True)
class QuadrotorModel:
    """12-state Euler-angle rigid body (dynamics.py:296-305)."""

    mass: float = 1.0
    arm_length: float = 0.2
    inertia_diag: Tuple[float, float, float] = (0.01, 0.01, 0.02)
    gravity: float = 9.81

    def control_matrix(self, x, t=0.0) -> np.ndarray:
        """G(x) (12, 4) of dynamics.py:331-347, host-side: thrust along the body z axis
        into the linear accelerations, torques through the inverse inertia."""
        x = np.asarray(x, float)
        (sr, cr), (sp, cp), (sy, cy) = ((np.sin(a), np.cos(a)) for a in x[6:9])
        g = np.zeros((12, 4))
        g[3:6, 0] = np.array([cr * sp * cy + sr * sy, cr * sp * sy - sr * cy, cr * cp]) / self.mass
        g[9:12, 1:4] = np.diag(1.0 / np.asarray(self.inertia_diag, float))
        return g

    def __post_init__(self):
        if self.mass <= 0 or self.arm_length <= 0 or min(self.inertia_diag) <= 0:
            raise ValueError("quadrotor parameters must be positive")

    def hover_control(self) -> np.ndarray:
        return np.array([self.mass * self.gravity, 0.0, 0.0, 0.0])


@dataclass(frozen=True)
class IntegratorModel:
    """dx = u dt + eps sqrt(dt) with G = B = H = I (tests/conftest.py:19-30)."""

    dim: int = 1

    def __post_init__(self):
        if self.dim not in (1, 2):
            raise ValueError("the device integrator is compiled for dim 1 or 2")


@dataclass(frozen=True, eq=False)
class LinearModel:
    """A generic linear plant dx = (A x + G u) dt + G (eps sqrt(dt) + jumps): the
    reference's DynamicsModel with drift A @ x and constant G = B = H
    (noise_through_controls=True).  Device kernels exist for (n, m) in
    LINEAR_SHAPES."""

    A: np.ndarray
    G: np.ndarray

    def __post_init__(self):
        A = np.array(self.A, dtype=float, copy=True)
        G = np.array(self.G, dtype=float, copy=True)
        if G.ndim == 1:
            G = G[:, None]
        if A.ndim != 2 or A.shape[0] != A.shape[1] or G.shape[0] != A.shape[0]:
            raise ValueError("A must be n x n and G n x m")
        if (A.shape[0], G.shape[1]) not in LINEAR_SHAPES:
            raise NotImplementedError(f"linear plugin kernels exist for (n, m) in {sorted(LINEAR_SHAPES)}")
        A.setflags(write=False)
        G.setflags(write=False)
        object.__setattr__(self, "A", A)
        object.__setattr__(self, "G", G)

    def drift(self, x, t=0.0) -> np.ndarray:
        return np.asarray(x, float) @ self.A.T

    def control_matrix(self, x, t=0.0) -> np.ndarray:
        return self.G.copy()


LINEAR_SHAPES = frozenset({(2, 1), (4, 1), (4, 2), (6, 3)})


@dataclass(frozen=True)
class DynamicsModel:
    """Device-evaluable control-affine jump-diffusion model (dynamics.py:45-65)."""

    state_dim: int
    control_dim: int
    plant: object
    control_limits: Optional[Tuple[np.ndarray, np.ndarray]] = None
    noise_through_controls: bool = True
    jump_channel: str = "control"
    jump_rows: Tuple[int, ...] = ()
    jump_scale_mode: str = "sqrt_dt"

    def __post_init__(self):
        if self.jump_channel not in ("control", "state"):
            raise ValueError("jump_channel must be 'control' or 'state'")
        if self.jump_scale_mode not in ("sqrt_dt", "unit"):
            raise ValueError("jump_scale_mode must be 'sqrt_dt' or 'unit'")
        if self.jump_channel == "control" and self.jump_scale_mode != "sqrt_dt":
            raise ValueError("control-channel jumps use the sqrt(dt) scaling (controller.py:143)")

    @property
    def jump_dim(self) -> int:
        return self.control_dim if self.jump_channel == "control" else len(self.jump_rows)

    def control_matrix(self, x, t=0.0) -> np.ndarray:
        """G(x), host-side (utilities such as control_cost_matrix_from_dynamics)."""
        cm = getattr(self.plant, "control_matrix", None)
        return np.eye(self.state_dim, self.control_dim) if cm is None else cm(x, t)

    def diffusion_matrix(self, x, t=0.0) -> np.ndarray:
        """B(x): the diffusion enters through the control channel (B = G) in every model here."""
        return self.control_matrix(x, t)

    def clamp(self, u: np.ndarray) -> np.ndarray:
        """np.clip to control_limits (dynamics.py:61-65); a host helper for callers."""
        if self.control_limits is None:
            return u
        lo, hi = self.control_limits
        return np.clip(u, lo, hi)


def _limits(control_limits, m):
    if control_limits is None:
        return None
    lo, hi = control_limits
    lo = np.broadcast_to(np.atleast_1d(np.asarray(lo, float)), (m,)).copy()
    hi = np.broadcast_to(np.atleast_1d(np.asarray(hi, float)), (m,)).copy()
    return lo, hi


def cartpole_dynamics(
    params: Optional[CartpoleModel] = None,
    control_limits=None,
    jump_channel: str = "control",
    jump_scale_mode: str = "sqrt_dt",
) -> DynamicsModel:
    """Cartpole (dynamics.py:264-284).  jump_channel="state" puts the jump on
    theta-dot (BASELINE configs 0/1)."""
    return DynamicsModel(
        state_dim=4,
        control_dim=1,
        plant=params or CartpoleModel(),
        control_limits=_limits(control_limits, 1),
        noise_through_controls=jump_channel == "control",
        jump_channel=jump_channel,
        jump_rows=(3,) if jump_channel == "state" else (),
        jump_scale_mode=jump_scale_mode,
    )


def quadrotor_dynamics(
    params: Optional[QuadrotorModel] = None,
    control_limits=None,
    jump_channel: str = "control",
    jump_scale_mode: str = "sqrt_dt",
) -> DynamicsModel:
    """Quadrotor (dynamics.py:389-409).  jump_channel="state" puts 3-axis
    gusts on the linear velocities (BASELINE configs 2/3)."""
    return DynamicsModel(
        state_dim=12,
        control_dim=4,
        plant=params or QuadrotorModel(),
        control_limits=_limits(control_limits, 4),
        noise_through_controls=jump_channel == "control",
        jump_channel=jump_channel,
        jump_rows=(3, 4, 5) if jump_channel == "state" else (),
        jump_scale_mode=jump_scale_mode,
    )


def integrator_dynamics(dim: int = 1, control_limits=None) -> DynamicsModel:
    """The conftest scalar integrator (tests/conftest.py:19-30), dim in {1, 2}."""
    return DynamicsModel(
        state_dim=dim,
        control_dim=dim,
        plant=IntegratorModel(dim),
        control_limits=_limits(control_limits, dim),
    )


def linear_dynamics(A, G, control_limits=None) -> DynamicsModel:
    """The generic linear plugin: f(x) = A x, constant G = B = H."""
    plant = LinearModel(A, G)
    n, m = plant.A.shape[0], plant.G.shape[1]
    return DynamicsModel(state_dim=n, control_dim=m, plant=plant, control_limits=_limits(control_limits, m))
