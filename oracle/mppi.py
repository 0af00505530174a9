"""Vectorised numpy restatement of one MPC iteration of the reference.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows /root/reference/pkg/src/jump_mppi (abbreviated jm/):
  sample_noise_batch_ref  jm/noise.py:129-161 (same numpy calls, same order)
  cartpole_fg             jm/dynamics.py:231-249
  quadrotor_fg            jm/dynamics.py:349-383
  step                    jm/dynamics.py:87-135 (general path :130-135, fused
                          B=H=G path :115-129)
  state costs             jm/costs.py:149-201
  modified_cost           jm/costs.py:80-111 (control-channel branch)
  mppi_iteration_oracle   jm/controller.py:103-181
  compute_weights         jm/controller.py:62-71
Generic over the compute dtype (float64: the reference; float32: the
"straightforward fp32 evaluation" the fp32 parity gate is defined against,
SURVEY 8(c)) and over the jump channel (control channel as in the reference;
state-space selector H for the BASELINE configs, whose
reference-side anchor is the per-rollout path, see gen_golden.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np


class OracleNoViable(RuntimeError):
    pass


@dataclass
class Spec:
    model: str                 # "cartpole" | "quadrotor" | "integrator" | "linear" (params = A, G flattened)
    n: int
    m: int
    params: Tuple[float, ...]  # cartpole: mc, mp, l, g; quadrotor: mass, arm, ixx, iyy, izz, g
    limits: Optional[Tuple[np.ndarray, np.ndarray]]
    jump_channel: str          # "control" | "state"
    jump_rows: Tuple[int, ...]
    jump_scale: str            # "sqrt_dt" | "unit"
    cost: str                  # "cartpole_swingup" | "quadrotor_hover" | "diag"
    weights: Tuple[float, ...]
    target: Tuple[float, ...]
    terminal_scale: float
    R: np.ndarray
    cost_lambda: float
    cost_c: float
    lam: float
    c: float
    sigma_d: np.ndarray
    sigma_j: np.ndarray
    nu: float
    dt: float
    T: int
    K: int
    jump_enabled: bool = True
    mark_mean: np.ndarray = field(default_factory=lambda: np.zeros(1))
    cal_b: Optional[np.ndarray] = None   # CostModel.control_channel == False (jm/costs.py:50-54)
    bb_term: Optional[np.ndarray] = None

    @property
    def q(self) -> int:
        return self.m if self.jump_channel == "control" else len(self.jump_rows)


def _plant(model):
    plant = getattr(model, "plant", None)
    if plant is None:
        plant = getattr(getattr(model, "fused_drift_control", None), "__self__", None)
    return plant


def spec_from_plugins(model, cost_model, cfg) -> Spec:
    """Duck-typed: works with the reference's plugin objects and this repo's."""
    plant = _plant(model)
    name = type(plant).__name__
    if name == "CartpoleModel":
        kind, params = "cartpole", (plant.cart_mass, plant.pole_mass, plant.pole_half_length, plant.gravity)
    elif name == "QuadrotorModel":
        kind = "quadrotor"
        params = (plant.mass, plant.arm_length) + tuple(plant.inertia_diag) + (plant.gravity,)
    elif name == "IntegratorModel":
        kind, params = "integrator", ()
    elif name == "LinearModel":
        kind = "linear"
        params = tuple(np.asarray(plant.A, float).ravel()) + tuple(np.asarray(plant.G, float).ravel())
    else:
        raise TypeError(f"oracle has no model {name}")
    sc = cost_model.state_cost
    cname = type(sc).__name__
    n, m = int(model.state_dim), int(model.control_dim)
    if cname == "CartpoleStateCost":
        cost, w, tgt = "cartpole_swingup", (sc.w_pos, sc.w_vel, sc.w_angle, sc.w_avel), ()
    elif cname == "QuadrotorStateCost":
        cost, w, tgt = "quadrotor_hover", (sc.w_pos, sc.w_vel, sc.w_att, sc.w_rate), tuple(sc.target)
    elif cname == "DiagQuadraticCost":
        cost, w = "diag", tuple(sc.weights)
        tgt = tuple(sc.target) if sc.target is not None else (0.0,) * n
    else:
        raise TypeError(f"oracle has no cost {cname}")
    tc = cost_model.terminal_cost
    scale = float(tc.scale) if type(tc).__name__ == "ScaledTerminalCost" else 1.0
    lim = getattr(model, "control_limits", None)
    if lim is not None:
        lim = (np.broadcast_to(np.asarray(lim[0], float), (m,)).copy(),
               np.broadcast_to(np.asarray(lim[1], float), (m,)).copy())
    channel = getattr(model, "jump_channel", "control")
    rows = tuple(getattr(model, "jump_rows", ()))
    q = m if channel == "control" else len(rows)
    mm = getattr(cfg, "mark_mean", None)
    mm = np.zeros(q) if mm is None else np.atleast_1d(np.asarray(mm, float))
    return Spec(kind, n, m, tuple(float(p) for p in params), lim, channel, rows,
                getattr(model, "jump_scale_mode", "sqrt_dt"), cost, tuple(float(v) for v in w),
                tuple(float(v) for v in tgt), scale, np.atleast_2d(np.asarray(cost_model.control_cost_matrix, float)),
                float(cost_model.lambda_), float(cost_model.c), float(cfg.lambda_), float(cfg.c),
                np.asarray(cfg.sigma_d, float), np.asarray(cfg.sigma_j, float), float(cfg.nu),
                float(cfg.dt), int(cfg.horizon_n), int(cfg.samples_m),
                bool(getattr(cfg, "jump_sampling_enabled", True)), mm, *_general_channel(cost_model))


def _general_channel(cost_model):
    """(cal_b, bb_term) when the cost model is not control-channel (jm/costs.py:50-54), else (None, None)."""
    if getattr(cost_model, "control_channel", True):
        return None, None
    cb, bb = getattr(cost_model, "cal_b", None), getattr(cost_model, "bb_term", None)
    return (None if cb is None else np.atleast_2d(np.asarray(cb, float)),
            None if bb is None else np.atleast_2d(np.asarray(bb, float)))


# ---------------------------------------------------------------- noise (jm/noise.py:129-161)
def sample_noise_batch_ref(seed: int, stream_id: int, spec: Spec, K: Optional[int] = None):
    """The reference's batch sampler, reproduced call for call with numpy's
    Philox(key=[seed, stream_id]) (jm/noise.py:49-51).  For the state-space
    jump channel the marks are q-dimensional with mean mark_mean and
    eps_combined = eps_d."""
    K = spec.K if K is None else K
    T, m, q = spec.T, spec.m, spec.q
    gen = np.random.Generator(np.random.Philox(key=np.array([seed, stream_id], dtype=np.uint64)))
    ld = np.linalg.cholesky(np.asarray(spec.c * spec.sigma_d, dtype=float))
    z = gen.standard_normal((K, T, m))
    eps_d = z * ld[0, 0] if m == 1 else z @ ld.T
    eps_j = np.zeros((K, T, q))
    if spec.jump_enabled:
        if not spec.nu * spec.dt < 0.1:
            raise ValueError(f"zero-one jump law violated (nu*dt = {spec.nu * spec.dt:g})")
        lj = np.linalg.cholesky(np.asarray(spec.sigma_j, dtype=float))
        ind = (gen.random((K, T)) < spec.nu * spec.dt).astype(np.int64)
        rows, cols = np.nonzero(ind)
        if rows.size:
            zj = gen.standard_normal((rows.size, q))
            marks = zj * lj[0, 0] if q == 1 else zj @ lj.T
            if spec.jump_channel == "state":
                marks = marks + spec.mark_mean
            eps_j[rows, cols] = marks
        eps_c = eps_d.copy()
        if spec.jump_channel == "control":
            eps_c[rows, cols] += eps_j[rows, cols]
    else:
        ind = np.zeros((K, T), dtype=np.int64)
        eps_c = eps_d.copy()
    return eps_d, ind, eps_j, eps_c


# ---------------------------------------------------------------- dynamics
def cartpole_fg(x, params, dt_type):
    mc, mp, l, g = (dt_type(p) for p in params)
    xdot, th, thdot = x[..., 1], x[..., 2], x[..., 3]
    s, co = np.sin(th), np.cos(th)
    denom = mc + mp * s * s
    xdd = mp * s * (g * co + l * thdot * thdot) / denom
    thdd = -(xdd * co + g * s) / l
    f = np.empty_like(x)
    f[..., 0] = xdot
    f[..., 1] = xdd
    f[..., 2] = thdot
    f[..., 3] = thdd
    G = np.zeros(x.shape[:-1] + (4, 1), dtype=x.dtype)
    G[..., 1, 0] = dt_type(1.0) / denom
    G[..., 3, 0] = -co / (l * denom)
    return f, G


def quadrotor_fg(x, params, dt_type):
    mass, _arm, ixx, iyy, izz, g = (dt_type(p) for p in params)
    v = x[..., 3:6]
    roll, pitch, yaw = x[..., 6], x[..., 7], x[..., 8]
    wx, wy, wz = x[..., 9], x[..., 10], x[..., 11]
    sr, cr = np.sin(roll), np.cos(roll)
    sp, cp = np.sin(pitch), np.cos(pitch)
    sy, cy = np.sin(yaw), np.cos(yaw)
    floor = dt_type(1e-6)
    cp_safe = np.where(np.abs(cp) < floor, np.copysign(floor, cp), cp)
    tp = sp / cp_safe
    f = np.zeros_like(x)
    f[..., 0:3] = v
    f[..., 5] = -g
    f[..., 6] = wx + sr * tp * wy + cr * tp * wz
    f[..., 7] = cr * wy - sr * wz
    f[..., 8] = (sr * wy + cr * wz) / cp_safe
    f[..., 9] = (iyy - izz) * wy * wz / ixx
    f[..., 10] = (izz - ixx) * wx * wz / iyy
    f[..., 11] = (ixx - iyy) * wx * wy / izz
    G = np.zeros(x.shape[:-1] + (12, 4), dtype=x.dtype)
    inv_m = dt_type(1.0) / mass
    G[..., 3, 0] = (cr * sp * cy + sr * sy) * inv_m
    G[..., 4, 0] = (cr * sp * sy - sr * cy) * inv_m
    G[..., 5, 0] = (cr * cp) * inv_m
    G[..., 9, 1] = dt_type(1.0) / ixx
    G[..., 10, 2] = dt_type(1.0) / iyy
    G[..., 11, 3] = dt_type(1.0) / izz
    return f, G


def integrator_fg(x, dt_type):
    n = x.shape[-1]
    G = np.zeros(x.shape[:-1] + (n, n), dtype=x.dtype)
    idx = np.arange(n)
    G[..., idx, idx] = dt_type(1.0)
    return np.zeros_like(x), G


def linear_fg(x, spec: Spec, dt_type):
    """A generic linear DynamicsModel: drift A @ x, constant G (= B = H)."""
    n, m = spec.n, spec.m
    p = np.asarray(spec.params, dtype=dt_type)
    A, G = p[: n * n].reshape(n, n), p[n * n: n * n + n * m].reshape(n, m)
    return x @ A.T, np.broadcast_to(G, x.shape[:-1] + (n, m)).astype(x.dtype)


def drift_control(spec: Spec, x, dt_type):
    if spec.model == "cartpole":
        return cartpole_fg(x, spec.params, dt_type)
    if spec.model == "quadrotor":
        return quadrotor_fg(x, spec.params, dt_type)
    if spec.model == "linear":
        return linear_fg(x, spec, dt_type)
    return integrator_fg(x, dt_type)


def clamp(spec: Spec, u):
    if spec.limits is None:
        return u
    lo, hi = spec.limits
    return np.clip(u, lo.astype(u.dtype), hi.astype(u.dtype))


def _matvec(mat, vec):
    # jm/dynamics.py:36-42
    if mat.shape[-1] == 1:
        return mat[..., 0] * vec[..., 0, None]
    return (mat @ vec[..., None])[..., 0]


def step_batch(spec: Spec, x, u, eps_d_row, jump_row, flag, dt, dt_type):
    """One Euler step for all samples (jm/dynamics.py:87-135).

    control channel: jump_row = eps_j (already masked), flag = 1.0 as the
    batched controller passes it (jm/controller.py:143).
    state channel:   jump_row = marks (q), flag = indicator per sample, H =
    selector on spec.jump_rows, scale 1 ("unit") or sqrt(dt)."""
    u = clamp(spec, u)
    f, g = drift_control(spec, x, dt_type)
    sqrt_dt = np.sqrt(dt_type(dt))
    dtt = dt_type(dt)
    if spec.jump_channel == "control":
        jump_scale = sqrt_dt
        if g.shape[-1] > 1:  # fused B = H = G path, jm/dynamics.py:115-129
            rhs = np.empty(eps_d_row.shape + (3,), dtype=x.dtype)
            rhs[..., 0] = u
            rhs[..., 1] = eps_d_row
            rhs[..., 2] = jump_row
            prod = g @ rhs
            out = f + prod[..., 0]
            out *= dtt
            out += x
            out += prod[..., 1] * sqrt_dt
            out += flag * prod[..., 2] * jump_scale
            return out
        return x + (f + _matvec(g, u)) * dtt + _matvec(g, eps_d_row) * sqrt_dt + flag * _matvec(g, jump_row) * jump_scale
    jump_scale = dt_type(1.0) if spec.jump_scale == "unit" else sqrt_dt
    hj = np.zeros_like(x)
    for i, r in enumerate(spec.jump_rows):
        hj[..., r] = jump_row[..., i]
    fl = np.asarray(flag, dtype=x.dtype)
    if fl.ndim:
        fl = fl[..., None]
    return x + (f + _matvec(g, u)) * dtt + _matvec(g, eps_d_row) * sqrt_dt + fl * hj * jump_scale


# ---------------------------------------------------------------- costs
def state_cost(spec: Spec, x, dt_type):
    w = [dt_type(v) for v in spec.weights]
    if spec.cost == "cartpole_swingup":  # jm/costs.py:161-168
        return (w[0] * x[..., 0] ** 2 + w[1] * x[..., 1] ** 2
                + w[2] * (dt_type(1.0) + np.cos(x[..., 2])) ** 2 + w[3] * x[..., 3] ** 2)
    if spec.cost == "quadrotor_hover":  # jm/costs.py:181-190
        tgt = np.asarray(spec.target, dtype=x.dtype)
        pe = x[..., 0:3] - tgt
        return (w[0] * np.einsum("...i,...i->...", pe, pe)
                + w[1] * np.einsum("...i,...i->...", x[..., 3:6], x[..., 3:6])
                + w[2] * (x[..., 6] ** 2 + x[..., 7] ** 2)
                + w[3] * np.einsum("...i,...i->...", x[..., 9:12], x[..., 9:12]))
    tgt = np.asarray(spec.target, dtype=x.dtype)
    e = x - tgt
    return np.einsum("...i,i,...i->...", e, np.asarray(w, dtype=x.dtype), e)


def modified_cost(spec: Spec, q, u, eps, dt, dt_type):
    """jm/costs.py:80-124: control-channel branch (u one shared row, :95-111) or,
    with cal_b / bb_term, the general branch (:112-124)."""
    lam, c = dt_type(spec.cost_lambda), dt_type(spec.cost_c)
    R = spec.R.astype(dt_type)
    if spec.cal_b is not None or spec.bb_term is not None:
        u_ru = np.einsum("...i,ij,...j->...", u, R, u)
        mapped = eps if spec.cal_b is None else np.einsum("ij,...j->...i", spec.cal_b.astype(dt_type), eps)
        cross = np.einsum("...i,...i->...", u, mapped)
        if spec.bb_term is None:
            quad = np.einsum("...i,...i->...", eps, eps)
        else:
            quad = np.einsum("...i,ij,...j->...", eps, spec.bb_term.astype(dt_type), eps)
        dtt = dt_type(dt)
        return (q + dt_type(0.5) * u_ru + lam * cross / np.sqrt(dtt)
                + dt_type(0.5) * lam * (dt_type(1.0) - dt_type(1.0) / c) * quad / dtt)
    if u.shape[0] == 1:
        u_ru = u[0] * R[0, 0] * u[0]
        cross = u[0] * eps[..., 0]
        quad = eps[..., 0] * eps[..., 0]
    else:
        u_ru = u @ R @ u
        cross = eps @ u
        quad = np.einsum("...i,...i->...", eps, eps)
    dtt = dt_type(dt)
    return (q + dt_type(0.5) * u_ru + lam * cross / np.sqrt(dtt)
            + dt_type(0.5) * lam * (dt_type(1.0) - dt_type(1.0) / c) * quad / dtt)


# ---------------------------------------------------------------- weights / update
def compute_weights(costs, lam, dt_type=np.float64):
    """jm/controller.py:62-71."""
    costs = np.asarray(costs, dtype=dt_type)
    finite = np.isfinite(costs)
    if not finite.any():
        raise OracleNoViable("no viable rollout")
    w = np.zeros(costs.shape, dtype=dt_type)
    shifted = costs[finite] - costs[finite].min()
    w[finite] = np.exp(-shifted / dt_type(lam))
    return w / w.sum()


def mppi_iteration_oracle(spec: Spec, x0, u_nom, noise, dtype=np.float64, mapping=None, trace=False):
    """jm/controller.py:103-181 on fed noise (eps_d, ind, eps_j, eps_c)."""
    dt_type = np.dtype(dtype).type
    eps_d, ind, eps_j, eps_c = noise
    K, T, m = eps_c.shape
    eps_d_t = np.ascontiguousarray(np.swapaxes(eps_d, 0, 1), dtype=dtype)
    eps_j_t = np.ascontiguousarray(np.swapaxes(eps_j, 0, 1), dtype=dtype)
    eps_c_t = np.ascontiguousarray(np.swapaxes(eps_c, 0, 1), dtype=dtype)
    # the reference's flag is the indicator; with Poisson counts (device sampler
    # extension) eps_j already holds the sum of the step's marks, so n -> 1
    ind_t = np.ascontiguousarray(np.swapaxes(np.minimum(ind, 1), 0, 1))
    u_nom = np.asarray(u_nom, dtype=dtype).reshape(T, m)
    u_eff = clamp(spec, u_nom)
    xs = np.repeat(np.asarray(x0, dtype=dtype)[None, :], K, axis=0)
    costs = np.zeros(K, dtype=dtype)
    dead = np.zeros(K, dtype=bool)
    dstep = np.full(K, -1, dtype=np.int64)
    states = np.empty((K, T + 1, spec.n), dtype=dtype) if trace else None
    if trace:
        states[:, 0] = xs
    dt = spec.dt
    zero = dt_type(0.0)
    with np.errstate(all="ignore"):
        for j in range(T):
            q = state_cost(spec, xs, dt_type)
            qt = modified_cost(spec, q, u_eff[j], eps_c_t[j], dt, dt_type)
            costs = costs + np.where(dead, zero, qt * dt_type(dt))
            if spec.jump_channel == "control":
                x_new = step_batch(spec, xs, u_nom[j], eps_d_t[j], eps_j_t[j], dt_type(1.0), dt, dt_type)
            else:
                x_new = step_batch(spec, xs, u_nom[j], eps_d_t[j], eps_j_t[j], ind_t[j], dt, dt_type)
            bad = ~np.all(np.isfinite(x_new), axis=-1)
            newly = bad & ~dead
            if newly.any():
                costs[newly] = np.inf
                dstep[newly] = j
                dead |= newly
            if dead.any():
                x_new[dead] = xs[dead]
            xs = x_new
            if trace:
                states[:, j + 1] = xs
        costs = costs + np.where(dead, zero, dt_type(spec.terminal_scale) * state_cost(spec, xs, dt_type))
        weights = compute_weights(costs, spec.lam, dt_type)
        delta = np.einsum("m,mjk->jk", weights, eps_c.astype(dtype)) / np.sqrt(dt_type(dt))
    if mapping is not None:
        delta = delta @ np.asarray(mapping, dtype=dtype).T
    finite = np.isfinite(costs)
    out = {
        "u_new": (u_nom + delta).astype(np.float64),
        "delta": delta.astype(np.float64),
        "costs": costs.astype(np.float64),
        "weights": weights.astype(np.float64),
        "min_cost": float(costs[finite].min()),
        "ess": float(1.0 / np.sum(weights.astype(np.float64) ** 2)),
        "norms": np.linalg.norm(delta.astype(np.float64), axis=1),
        "diverged": dstep,
    }
    if trace:
        out["states"] = states.astype(np.float64)
    return out


def warm_start_shift(u, u_init):
    """jm/controller.py:96-100."""
    u = np.asarray(u, float)
    return np.vstack([u[1:], np.atleast_1d(np.asarray(u_init, float))[None, :]])


# ---------------------------------------------------------------- shard records (multi-GPU merge)
def partial_record(costs, eps_c, lam):
    """One shard's weighting record [rho, Z, sum w^2, n_finite, N[T*m]] relative
    to the shard's own minimum (the format libjmppi exchanges between ranks)."""
    costs = np.asarray(costs, float)
    fin = np.isfinite(costs)
    K, T, m = eps_c.shape
    rec = np.zeros(4 + T * m)
    if not fin.any():
        rec[0] = np.inf
        return rec
    rho = costs[fin].min()
    w = np.where(fin, np.exp(-(np.where(fin, costs, rho) - rho) / lam), 0.0)
    rec[0], rec[1], rec[2], rec[3] = rho, w.sum(), (w * w).sum(), fin.sum()
    rec[4:] = np.einsum("k,ktj->tj", w, eps_c).reshape(-1)
    return rec


def combine_records(records, lam, dt, u_nom):
    """Log-sum-exp merge of shard records in order; returns (u_new, rho, ess)."""
    records = np.asarray(records, float)
    rho = records[:, 0].min()
    if not np.isfinite(rho):
        raise OracleNoViable("no viable rollout")
    e = np.where(np.isfinite(records[:, 0]), np.exp(-(records[:, 0] - rho) / lam), 0.0)
    Z = (records[:, 1] * e).sum()
    W2 = (records[:, 2] * e * e).sum()
    N = (records[:, 4:] * e[:, None]).sum(axis=0)
    u_nom = np.asarray(u_nom, float)
    return u_nom + (N / (Z * np.sqrt(dt))).reshape(u_nom.shape), rho, Z * Z / W2
