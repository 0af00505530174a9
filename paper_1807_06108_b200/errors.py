"""Exceptions of the controller boundary, named as in the reference
(controller.py:31 ControllerError, noise.py:34-35 NoiseError,
dynamics.py:29-33 StateDivergedError, types.py:23-28 ConfigError)."""

from .dynamics import StateDivergedError  # noqa: F401
from .types import ConfigError  # noqa: F401


class ControllerError(RuntimeError):
    """e.g. "no viable rollout" when every sampled cost is non-finite."""


class NoiseError(RuntimeError):
    """Covariance factorisation failure."""


class DeviceError(RuntimeError):
    """CUDA runtime failure inside libjmppi.so (no reference analogue)."""
