"""Noise streams, mirroring jump_mppi.noise
(/root/reference/pkg/src/jump_mppi/noise.py).

`sample_noise_batch` draws one iteration's noise table on the GPU with the
same Philox stream the rollout kernel consumes (csrc/philox.cuh), so a
(master_seed, stream_id) pair names the same draws everywhere.  The values are
not numpy's (the reference never pins RNG values); the sampling
distribution and draw-order contract are the reference's:
  eps_d ~ N(0, c Sigma_D); indicator = U < nu dt (zero-one law);
  marks ~ N(mark_mean, Sigma_J) only at jump events; eps_c = eps_d + eps_j
  for control-channel jumps (eps_d for state-space jumps).
With MppiConfig.jump_process="poisson" the indicator becomes the Poisson(nu dt)
arrival count n of the step and eps_j the sum of its n marks.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine
from .costs import CostModel, DiagQuadraticCost
from .dynamics import QuadrotorModel, integrator_dynamics, quadrotor_dynamics
from .errors import NoiseError  # noqa: F401

# Stream ids below 2**62 belong to controller iterations (noise.py:31); the
# device plant uses its own counter slot (philox.cuh slot 3).
PLANT_STREAM_ID = 1 << 62


@dataclass(frozen=True)
class RngStream:
    """(master_seed, stream_id) handle (noise.py:38-51)."""

    master_seed: int
    stream_id: int

    def __post_init__(self):
        if self.master_seed < 0 or self.stream_id < 0:
            raise ValueError("master_seed and stream_id must be nonnegative")


def _noise_model(cfg, model):
    if model is not None:
        return model
    m = cfg.control_dim
    if m in (1, 2):
        return integrator_dynamics(m)
    if m == 4:
        return quadrotor_dynamics(QuadrotorModel())
    raise NotImplementedError(f"no device noise sampler for control_dim {m} without a model")


def sample_noise_batch(stream: RngStream, cfg, n_rollouts: int, model=None, precision=None):
    """(eps_d, indicators, eps_j, eps_combined) with shapes (M,N,m), (M,N),
    (M,N,q), (M,N,m) drawn on the device (noise.py:129-161)."""
    mdl = _noise_model(cfg, model)
    n = mdl.state_dim
    q = DiagQuadraticCost(tuple([0.0] * n))
    cm = CostModel(q, q, np.zeros((cfg.control_dim, cfg.control_dim)), 1.0, 1.0)
    ctx = engine.get_context(mdl, cm, cfg, samples=n_rollouts, precision=precision)
    return ctx.sample_noise(stream.master_seed, stream.stream_id)
