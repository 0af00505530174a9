"""Construction of (Task, MppiConfig) pairs: the BASELINE.json configs and the
reference's experiment configs (jump_mppi.experiment.build_task /
build_mppi_config, /root/reference/pkg/src/jump_mppi/experiment.py:252-358).

BASELINE configs (SURVEY 8(d), Appendix A conventions):
  * "sigma = 10 N" force noise: eps enters as G eps sqrt(dt), so
    Sigma_D = sigma^2 dt (force perturbation eps/sqrt(dt) has std sigma); c = 1.
  * jumps: Bernoulli(nu dt) (zero-one law), state-space (theta-dot / linear
    velocities), marks N(mu, s^2), O(1) increment (jump_scale_mode="unit"),
    excluded from the update (eps_combined = eps_d).
  * cartpole cost: diag(1, .1, 10, .1) on x - (0, 0, pi, 0), R = 0.01,
    terminal 10 q, lambda = 1.
  * quadrotor cost: QuadrotorStateCost(target (4,4,2), 10/1/5/0.1), R = 0.01 I.
`mode="control"` gives the reference-expressible twin of each config
(control-channel jumps with zero-mean marks, the reference's own cost
family): same shapes and per-state-step work, runnable through the
reference's batched mppi_iteration (the CPU baseline arm).
"""

from __future__ import annotations

import copy
from typing import Dict, Optional, Tuple

import numpy as np

from .costs import CartpoleStateCost, CostModel, DiagQuadraticCost, QuadrotorStateCost, ScaledTerminalCost
from .dynamics import CartpoleModel, QuadrotorModel, cartpole_dynamics, quadrotor_dynamics
from .harness import Task
from .types import MppiConfig, validate_config

# ---------------------------------------------------------------- BASELINE.json configs
BASELINE_SHAPES = {
    0: dict(system="cartpole", K=1024, T=100, closed_loop_steps=0),
    1: dict(system="cartpole", K=65536, T=100, closed_loop_steps=500),
    2: dict(system="quadrotor", K=8192, T=150, closed_loop_steps=0),
    3: dict(system="quadrotor", K=1 << 20, T=200, closed_loop_steps=200),
}


def _cartpole(K: int, T: int, mode: str, steps: int) -> Tuple[Task, MppiConfig]:
    dt, sigma, nu = 0.02, 10.0, 0.5
    params = CartpoleModel(cart_mass=1.0, pole_mass=0.1, pole_half_length=0.5, gravity=9.81)
    x0 = np.array([0.0, 0.0, np.pi, 0.0])
    if mode == "state":
        model = cartpole_dynamics(params, jump_channel="state", jump_scale_mode="unit")
        running = DiagQuadraticCost((1.0, 0.1, 10.0, 0.1), (0.0, 0.0, np.pi, 0.0))
        cfg = MppiConfig(lambda_=1.0, c=1.0, sigma_d=sigma * sigma * dt, sigma_j=0.5 ** 2, nu=nu, dt=dt,
                         horizon_n=T, samples_m=K, u_init=[0.0], mark_mean=[1.0], jump_dim=1)
    else:
        model = cartpole_dynamics(params)
        running = CartpoleStateCost(w_pos=1.0, w_vel=0.1, w_angle=10.0, w_avel=0.1)
        cfg = MppiConfig(lambda_=1.0, c=1.0, sigma_d=sigma * sigma * dt, sigma_j=sigma * sigma * dt, nu=nu,
                         dt=dt, horizon_n=T, samples_m=K, u_init=[0.0])
    cost = CostModel(running, ScaledTerminalCost(running, 10.0), 0.01 * np.eye(1), 1.0, 1.0)
    task = Task("cartpole", model, cost, x0, steps, None,
                ("cart_pos", "cart_vel", "pole_angle", "pole_avel"), ("force",))
    return task, validate_config(cfg)


def _quadrotor(K: int, T: int, mode: str, steps: int) -> Tuple[Task, MppiConfig]:
    dt, nu = 0.01, 1.0
    sig = np.array([2.0, 0.1, 0.1, 0.1])
    params = QuadrotorModel(mass=1.0, arm_length=0.2, inertia_diag=(0.0082, 0.0082, 0.0149), gravity=9.81)
    running = QuadrotorStateCost(target=(4.0, 4.0, 2.0), w_pos=10.0, w_vel=1.0, w_att=5.0, w_rate=0.1)
    u_init = [9.81, 0.0, 0.0, 0.0]
    if mode == "state":
        model = quadrotor_dynamics(params, jump_channel="state", jump_scale_mode="unit")
        cfg = MppiConfig(lambda_=1.0, c=1.0, sigma_d=np.diag(sig ** 2) * dt, sigma_j=np.eye(3), nu=nu, dt=dt,
                         horizon_n=T, samples_m=K, u_init=u_init, mark_mean=np.zeros(3), jump_dim=3)
    else:
        model = quadrotor_dynamics(params)
        cfg = MppiConfig(lambda_=1.0, c=1.0, sigma_d=np.diag(sig ** 2) * dt, sigma_j=np.diag(sig ** 2) * dt,
                         nu=nu, dt=dt, horizon_n=T, samples_m=K, u_init=u_init)
    cost = CostModel(running, ScaledTerminalCost(running, 10.0), 0.01 * np.eye(4), 1.0, 1.0)
    names = ("px", "py", "pz", "vx", "vy", "vz", "roll", "pitch", "yaw", "wx", "wy", "wz")
    task = Task("quadrotor", model, cost, np.zeros(12), steps, None, names,
                ("thrust", "tau_x", "tau_y", "tau_z"))
    return task, validate_config(cfg)


def baseline_config(index: int, mode: str = "state", K: Optional[int] = None, T: Optional[int] = None,
                    steps: Optional[int] = None) -> Tuple[Task, MppiConfig]:
    """(Task, MppiConfig) of BASELINE.json configs[index] (0..3).

    mode="state": the config as BASELINE states it; mode="control": its
    reference-expressible twin.  K / T / steps override the shape (the
    throughput sweep, config 4, is baseline_config(0 or 2, K=..., T=...)).
    """
    if index not in BASELINE_SHAPES:
        raise ValueError("BASELINE configs 0..3 (config 4 is a sweep over 0/2 shapes)")
    if mode not in ("state", "control"):
        raise ValueError("mode must be 'state' or 'control'")
    s = BASELINE_SHAPES[index]
    KK = s["K"] if K is None else int(K)
    TT = s["T"] if T is None else int(T)
    st = s["closed_loop_steps"] if steps is None else int(steps)
    if s["system"] == "cartpole":
        return _cartpole(KK, TT, mode, st)
    return _quadrotor(KK, TT, mode, st)


# ---------------------------------------------------------------- reference experiment configs
# Task defaults of the reference (experiment.py:41-116): its desk-scale calibration.
CARTPOLE_DEFAULTS: Dict = {
    "task": "cartpole", "duration_seconds": 10.0,
    "physical": {"cart_mass": 1.0, "pole_mass": 0.1, "pole_half_length": 0.5, "gravity": 9.81},
    "cost": {"w_pos": 2.5, "w_vel": 1.0, "w_angle": 50.0, "w_avel": 1.0, "terminal_scale": 10.0,
             "control_weight": 1.0},
    "mppi": {"lambda": 5.0, "c": 1.25, "sigma_d": 0.25, "sigma_j": 2.0, "nu": 0.25, "dt": 0.02,
             "horizon": 50, "samples": 1000, "u_init": [0.0]},
    "control_limits": [[-30.0], [30.0]],
    "diffusion_channel_scale": [1.0],
    "jump_channel_scale": [2.0],
}
QUADROTOR_DEFAULTS: Dict = {
    "task": "quadrotor", "duration_seconds": 8.0,
    "physical": {"mass": 1.0, "arm_length": 0.2, "inertia": [0.01, 0.01, 0.02], "gravity": 9.81,
                 "target": [4.0, 4.0, 2.0]},
    "cost": {"w_pos": 4.0, "w_vel": 1.0, "w_att": 10.0, "w_rate": 1.0, "terminal_scale": 10.0,
             "control_weight": 0.1},
    "mppi": {"lambda": 40.0, "c": 1.5, "sigma_d": 1.0, "sigma_j": 20.0, "nu": 0.2, "dt": 0.02,
             "horizon": 50, "samples": 1000, "u_init": [9.81, 0.0, 0.0, 0.0]},
    "control_limits": [[0.0, -1.0, -1.0, -1.0], [25.0, 1.0, 1.0, 1.0]],
    "diffusion_channel_scale": [1.0, 0.03, 0.03, 0.03],
    "jump_channel_scale": [1.0, 0.03, 0.03, 0.03],
}


# run-level keys of both tasks (experiment.py:43-46, :76, :81-84, :115)
_RUN_DEFAULTS = {"cartpole": {"trials": 40}, "quadrotor": {"trials": 25}}
_RUN_COMMON: Dict = {"base_seed": 2024, "out_dir": "results", "variants": "both",
                     "sweep": {"nu": None, "sigma_j": None, "samples": None}}


class ExperimentConfigError(ValueError):
    """A config file that does not resolve (experiment.py:33)."""


def _defaults(task) -> Dict:
    base = {"cartpole": CARTPOLE_DEFAULTS, "quadrotor": QUADROTOR_DEFAULTS}.get(task)
    if base is None:
        raise ExperimentConfigError(f"unknown task {task!r}; expected one of ['cartpole', 'quadrotor']")
    return _merge(_merge(base, _RUN_COMMON), _RUN_DEFAULTS[task])


def _unknown_keys(given: Dict, allowed: Dict, path: str = ""):
    for k, v in given.items():
        where = f"{path}.{k}" if path else k
        if k not in allowed:
            raise ExperimentConfigError(f"unknown key '{where}'")
        if isinstance(v, dict) and isinstance(allowed[k], dict):
            _unknown_keys(v, allowed[k], where)


def config_from_dict(raw: Dict) -> Dict:
    """A raw mapping (a parsed pkg/configs/*.yaml) resolved against the task
    defaults, unknown keys fatal (experiment.py:161-214).  Returns the resolved
    mapping build_task / build_mppi_config / sweep_cells accept."""
    if not isinstance(raw, dict):
        raise ExperimentConfigError("config must be a mapping")
    d = _defaults(raw.get("task"))
    _unknown_keys(raw, d)
    out = _merge(d, raw)
    if out["variants"] not in ("old", "new", "both"):
        raise ExperimentConfigError(f"variants must be old|new|both, got {out['variants']!r}")
    return out


def load_config(path: str) -> Dict:
    """Parse a YAML experiment config (pkg/configs/*.yaml; experiment.py:217-226)."""
    import yaml

    with open(path) as fh:
        try:
            raw = yaml.safe_load(fh)
        except yaml.YAMLError as exc:
            raise ExperimentConfigError(f"config parse error: {exc}") from exc
    return config_from_dict(raw or {})


def sweep_cells(exp) -> list:
    """(nu, sigma_j, samples_m) cells, one factor at a time around the base point
    (experiment.py:229-243)."""
    e = resolve(exp)
    mp = e["mppi"]
    sw = e.get("sweep") or {}
    base_nu, base_sj = float(mp["nu"]), float(mp["sigma_j"])
    if isinstance(exp, dict):
        nus = [float(v) for v in (sw.get("nu") or [base_nu])]
        sjs = [float(v) for v in (sw.get("sigma_j") or [base_sj])]
        sams = [int(v) for v in (sw.get("samples") or [int(mp["samples"])])]
    else:  # a reference ExperimentConfig
        nus, sjs, sams = list(exp.sweep_nu), list(exp.sweep_sigma_j), list(exp.sweep_samples)
    cells = []
    for c in [(base_nu, s) for s in sjs] + [(v, base_sj) for v in nus if v != base_nu]:
        if c not in cells:
            cells.append(c)
    return [(nu, s, m) for nu, s in cells for m in sams]


def _merge(base: Dict, over: Dict) -> Dict:
    out = copy.deepcopy(base)
    for k, v in over.items():
        out[k] = _merge(out[k], v) if isinstance(v, dict) and isinstance(out.get(k), dict) else v
    return out


def _field(cfg, name):
    return cfg[name] if isinstance(cfg, dict) else getattr(cfg, name)


def resolve(raw) -> Dict:
    """A reference ExperimentConfig (or a raw mapping with the same keys) ->
    plain dict with task defaults merged in."""
    if isinstance(raw, dict):
        return _merge(_defaults(raw.get("task")), raw)
    return {k: _field(raw, k) for k in ("task", "duration_seconds", "physical", "cost", "mppi",
                                         "control_limits", "diffusion_channel_scale",
                                         "jump_channel_scale")}


def channel_covariance(label: float, scale) -> np.ndarray:
    """Sigma = label * diag(scale)^2 (experiment.py:246-249)."""
    s = np.asarray(scale, dtype=float)
    return label * np.diag(s * s)


def build_mppi_config(exp, nu=None, sigma_j=None, samples_m=None, jump_sampling_enabled=True) -> MppiConfig:
    """experiment.py:252-276."""
    e = resolve(exp)
    mp = e["mppi"]
    return validate_config(MppiConfig(
        lambda_=float(mp["lambda"]), c=float(mp["c"]),
        sigma_d=channel_covariance(float(mp["sigma_d"]), e["diffusion_channel_scale"]),
        sigma_j=channel_covariance(float(mp["sigma_j"] if sigma_j is None else sigma_j), e["jump_channel_scale"]),
        nu=float(mp["nu"] if nu is None else nu), dt=float(mp["dt"]), horizon_n=int(mp["horizon"]),
        samples_m=int(mp["samples"] if samples_m is None else samples_m),
        u_init=np.asarray(mp["u_init"], dtype=float), jump_sampling_enabled=jump_sampling_enabled))


def build_task(exp) -> Task:
    """experiment.py:279-358 (success predicates are evaluated by the caller)."""
    e = resolve(exp)
    dt = float(e["mppi"]["dt"])
    steps = int(round(float(e["duration_seconds"]) / dt))
    cc, lam, c = e["cost"], float(e["mppi"]["lambda"]), float(e["mppi"]["c"])
    phys, lim = e["physical"], e["control_limits"]
    if e["task"] == "cartpole":
        model = cartpole_dynamics(CartpoleModel(float(phys["cart_mass"]), float(phys["pole_mass"]),
                                                float(phys["pole_half_length"]), float(phys["gravity"])), lim)
        running = CartpoleStateCost(float(cc["w_pos"]), float(cc["w_vel"]), float(cc["w_angle"]),
                                    float(cc["w_avel"]))
        cost = CostModel(running, ScaledTerminalCost(running, float(cc["terminal_scale"])),
                         float(cc["control_weight"]) * np.eye(1), lam, c)
        return Task("cartpole", model, cost, np.zeros(4), steps, None,
                    ("cart_pos", "cart_vel", "pole_angle", "pole_avel"), ("force",))
    target = tuple(float(v) for v in phys["target"])
    model = quadrotor_dynamics(QuadrotorModel(float(phys["mass"]), float(phys["arm_length"]),
                                              tuple(float(v) for v in phys["inertia"]),
                                              float(phys["gravity"])), lim)
    running = QuadrotorStateCost(target, float(cc["w_pos"]), float(cc["w_vel"]), float(cc["w_att"]),
                                 float(cc["w_rate"]))
    cost = CostModel(running, ScaledTerminalCost(running, float(cc["terminal_scale"])),
                     float(cc["control_weight"]) * np.eye(4), lam, c)
    return Task("quadrotor", model, cost, np.zeros(12), steps, None,
                ("px", "py", "pz", "vx", "vy", "vz", "roll", "pitch", "yaw", "wx", "wy", "wz"),
                ("thrust", "tau_x", "tau_y", "tau_z"))
