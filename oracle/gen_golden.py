"""Generate tests/golden/*.npz by running the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  Run in the build container (it imports the
read-only reference from /root/reference/pkg/src; that tree does not exist on
the GPU box, so the vectors are committed):

    python -m oracle.gen_golden

Control-channel cases ("r_*") call the reference's batched
jump_mppi.mppi_iteration(..., return_rollouts=True) with its own sampler
(RngStream(seed, iteration)), except r_divergence, which injects a noise table
with non-finite entries through the reference's own sampler hook.
State-space-jump cases ("b_*", the BASELINE configs) run the reference's
per-rollout path -- jump_mppi.rollout + update_controls with a custom
DynamicsModel (constant H, noise_through_controls=False) and an explicit
NoiseRealization (marks / sqrt(dt) through the sqrt(dt) path = O(1) jumps,
eps_combined = eps_d) -- exactly as SURVEY 8(c) / Appendix A prescribe.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import jump_mppi  # noqa: F401

    return jump_mppi


def spec_json(model_kind, params, n, m, limits, jump_channel, jump_rows, jump_scale, cost, weights,
              target, terminal_scale, R, cost_lambda, cost_c, lam, c, sigma_d, sigma_j, nu, dt, T, K,
              jump_enabled=True, mark_mean=None, cal_b=None, bb_term=None):
    q = m if jump_channel == "control" else len(jump_rows)
    extra = {}
    if cal_b is not None or bb_term is not None:  # CostModel.control_channel == False (jm/costs.py:50-54)
        extra = dict(cal_b=np.atleast_2d(cal_b).astype(float).tolist(),
                     bb_term=np.atleast_2d(bb_term).astype(float).tolist())
    return dict(**extra,
        model=model_kind, params=list(map(float, params)), n=n, m=m,
        limits=None if limits is None else [list(map(float, np.atleast_1d(limits[0]))),
                                            list(map(float, np.atleast_1d(limits[1])))],
        jump_channel=jump_channel, jump_rows=list(jump_rows), jump_scale=jump_scale, cost=cost,
        weights=list(map(float, weights)), target=list(map(float, target)),
        terminal_scale=float(terminal_scale), R=np.atleast_2d(R).astype(float).tolist(),
        cost_lambda=float(cost_lambda), cost_c=float(cost_c), lam=float(lam), c=float(c),
        sigma_d=np.atleast_2d(sigma_d).astype(float).tolist(),
        sigma_j=np.atleast_2d(sigma_j).astype(float).tolist(), nu=float(nu), dt=float(dt), T=int(T),
        K=int(K), jump_enabled=bool(jump_enabled),
        mark_mean=list(map(float, np.zeros(q) if mark_mean is None else mark_mean)),
    )


def save(name, spec, x0, u_nom, seed, iteration, noise, out, mapping=None, keep_states=True):
    eps_d, ind, eps_j, _eps_c = noise  # eps_c = eps_d + eps_j (control) / eps_d (state): recomputed exactly
    OUT.mkdir(parents=True, exist_ok=True)
    arrays = dict(
        spec=np.array(json.dumps(spec)), x0=np.asarray(x0, float), u_nom=np.asarray(u_nom, float),
        seed=np.array(seed, dtype=np.uint64), iteration=np.array(iteration, dtype=np.uint64),
        eps_d=np.asarray(eps_d, float), ind=np.asarray(ind, np.int8), eps_j=np.asarray(eps_j, float),
        costs=np.asarray(out["costs"], float), weights=np.asarray(out["weights"], float),
        u_new=np.asarray(out["u_new"], float), min_cost=np.array(out["min_cost"]),
        ess=np.array(out["ess"]), norms=np.asarray(out["norms"], float),
        diverged=np.asarray(out["diverged"], np.int64),
        final_states=np.asarray(out["states"][:, -1], float),
    )
    if mapping is not None:
        arrays["mapping"] = np.asarray(mapping, float)
    if keep_states:
        arrays["states"] = np.asarray(out["states"], float)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"{name}: K={spec['K']} T={spec['T']} min_cost={out['min_cost']:.6g} ess={out['ess']:.4g}")


def run_batched(jm, ctrl, model, cost_model, x0, seed, mapping=None, noise_override=None):
    """Reference mppi_iteration; optionally inject a noise table through its sampler."""
    import jump_mppi.controller as jc

    orig = jc.sample_noise_batch
    if noise_override is not None:
        jc.sample_noise_batch = lambda stream, cfg, n: tuple(np.array(a) for a in noise_override)
    try:
        seq, diag, rollouts = jm.mppi_iteration(ctrl, model, cost_model, x0, master_seed=seed,
                                                mapping=mapping, return_rollouts=True)
    finally:
        jc.sample_noise_batch = orig
    noise = (np.stack([r.noise.eps_d for r in rollouts]), np.stack([r.noise.jump_indicator for r in rollouts]),
             np.stack([r.noise.eps_j for r in rollouts]), np.stack([r.noise.eps_combined for r in rollouts]))
    out = dict(costs=np.array([r.cost for r in rollouts]), weights=diag.weights, u_new=seq.controls,
               min_cost=diag.min_cost, ess=diag.effective_sample_size, norms=diag.per_step_update_norm,
               diverged=np.array([-1 if r.diverged_at is None else r.diverged_at for r in rollouts]),
               states=np.stack([r.trajectory.states for r in rollouts]))
    return noise, out


def integrator_model(jm):
    def zero_f(x, t=0.0):
        return np.zeros_like(np.asarray(x, dtype=float))

    def unit_g(x, t=0.0):
        x = np.asarray(x, dtype=float)
        out = np.zeros(x.shape[:-1] + (x.shape[-1], x.shape[-1]))
        idx = np.arange(x.shape[-1])
        out[..., idx, idx] = 1.0
        return out

    return jm.DynamicsModel(state_dim=1, control_dim=1, drift=zero_f, control_matrix=unit_g,
                            diffusion_matrix=unit_g, jump_matrix=unit_g, noise_through_controls=True)


def quad_cost(jm, lam, c, r):
    def q(x, t=0.0):
        x = np.asarray(x, dtype=float)
        return np.einsum("...i,...i->...", x, x)

    def phi(x):
        return q(x)

    return jm.CostModel(state_cost=q, terminal_cost=phi, control_cost_matrix=r * np.eye(1), lambda_=lam, c=c)


def gen_control_channel(jm):
    # --- scalar integrator cases (tests/test_controller.py:207-265 settings)
    model = integrator_model(jm)
    for name, kw, u0, x0, seed, cm_kw in [
        ("r_integrator", dict(lambda_=2.0, c=1.5, sigma_d=1.0, sigma_j=4.0, nu=0.25, dt=0.02, horizon_n=6,
                              samples_m=16, u_init=0.0), np.linspace(-1, 1, 6)[:, None], 0.3, 55,
         dict(lam=2.0, c=1.5, r=1.0)),
        ("r_integrator_m2n1", dict(lambda_=1.5, c=2.0, sigma_d=1.0, sigma_j=4.0, nu=0.25, dt=0.04, horizon_n=1,
                                   samples_m=2, u_init=0.0), np.array([[0.6]]), 0.2, 7,
         dict(lam=1.5, c=2.0, r=1.0)),
        ("r_integrator_big", dict(lambda_=1.0, c=1.5, sigma_d=1.0, sigma_j=4.0, nu=2.0, dt=0.02, horizon_n=40,
                                  samples_m=512, u_init=0.0), np.zeros((40, 1)), 0.5, 17,
         dict(lam=1.0, c=1.5, r=1.0)),
    ]:
        cfg = jm.MppiConfig(**kw)
        cm = quad_cost(jm, **cm_kw)
        ctrl = jm.ControllerState(jm.ControlSequence(u0, cfg.dt), 0, cfg)
        noise, out = run_batched(jm, ctrl, model, cm, np.array([x0]), seed)
        spec = spec_json("integrator", (), 1, 1, None, "control", (), "sqrt_dt", "diag", (1.0,), (0.0,), 1.0,
                         cm.control_cost_matrix, cm.lambda_, cm.c, cfg.lambda_, cfg.c, cfg.sigma_d, cfg.sigma_j,
                         cfg.nu, cfg.dt, cfg.horizon_n, cfg.samples_m, cfg.jump_sampling_enabled)
        save(name, spec, [x0], u0, seed, 0, noise, out)

    # --- divergence: non-finite noise entries kill samples 3 and 7; a huge one
    # overflows sample 11's cost without a non-finite state
    cfg = jm.MppiConfig(lambda_=1.0, c=1.0, sigma_d=1.0, sigma_j=1.0, nu=0.0, dt=0.02, horizon_n=8,
                        samples_m=16, u_init=0.0, jump_sampling_enabled=False)
    rng = np.random.default_rng(99)
    eps_d = rng.standard_normal((16, 8, 1))
    eps_d[3, 2, 0] = np.inf
    eps_d[7, 5, 0] = -np.inf
    eps_d[11, 1, 0] = 1e200
    noise_in = (eps_d, np.zeros((16, 8), np.int64), np.zeros((16, 8, 1)), eps_d.copy())
    cm = quad_cost(jm, 1.0, 1.0, 1.0)
    ctrl = jm.initial_controller_state(cfg)
    noise, out = run_batched(jm, ctrl, model, cm, np.array([0.1]), 5, noise_override=noise_in)
    spec = spec_json("integrator", (), 1, 1, None, "control", (), "sqrt_dt", "diag", (1.0,), (0.0,), 1.0,
                     cm.control_cost_matrix, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.0, 0.02, 8, 16, False)
    save("r_divergence", spec, [0.1], np.zeros((8, 1)), 5, 0, noise, out)

    # --- reference tasks (experiment.py defaults)
    for task_name, K, T, x0, seed, it, mapping, enabled in [
        ("cartpole", 64, 50, np.zeros(4), 2024, 3, None, True),
        ("cartpole", 64, 50, np.array([0.2, -0.1, 2.5, 0.3]), 2025, 0, None, False),
        ("quadrotor", 64, 50, np.zeros(12), 11, 1, None, True),
        ("quadrotor", 32, 40, np.array([0.1, -0.2, 0.5, 0, 0, 0, 0.05, -0.03, 0.2, 0, 0, 0]), 12, 4,
         np.array([[0, 1, 0, 0], [1, 0, 0, 0], [0, 0, 0.5, 0], [0, 0, 0, 2.0]]), True),
    ]:
        ecfg = jm.config_from_dict({"task": task_name})
        task = jm.build_task(ecfg)
        cfg = jm.build_mppi_config(ecfg, samples_m=K, jump_sampling_enabled=enabled)
        cfg = jm.MppiConfig(cfg.lambda_, cfg.c, cfg.sigma_d, cfg.sigma_j, cfg.nu, cfg.dt, T, K, cfg.u_init,
                            cfg.jump_sampling_enabled)
        rng = np.random.default_rng(seed)
        u_nom = np.tile(cfg.u_init, (T, 1)) + rng.normal(scale=0.5, size=(T, cfg.control_dim)) * (
            np.array([5.0]) if task_name == "cartpole" else np.array([1.0, 0.02, 0.02, 0.02]))
        ctrl = jm.ControllerState(jm.ControlSequence(u_nom, cfg.dt), it, cfg)
        noise, out = run_batched(jm, ctrl, task.model, task.cost_model, x0, seed, mapping=mapping)
        fd = task.model.fused_drift_control.__self__
        sc = task.cost_model.state_cost
        if task_name == "cartpole":
            params = (fd.cart_mass, fd.pole_mass, fd.pole_half_length, fd.gravity)
            cw, tgt, ck = (sc.w_pos, sc.w_vel, sc.w_angle, sc.w_avel), (), "cartpole_swingup"
        else:
            params = (fd.mass, fd.arm_length) + tuple(fd.inertia_diag) + (fd.gravity,)
            cw, tgt, ck = (sc.w_pos, sc.w_vel, sc.w_att, sc.w_rate), tuple(sc.target), "quadrotor_hover"
        spec = spec_json(task_name, params, task.model.state_dim, task.model.control_dim, task.model.control_limits,
                         "control", (), "sqrt_dt", ck, cw, tgt, task.cost_model.terminal_cost.scale,
                         task.cost_model.control_cost_matrix, task.cost_model.lambda_, task.cost_model.c,
                         cfg.lambda_, cfg.c, cfg.sigma_d, cfg.sigma_j, cfg.nu, cfg.dt, T, K,
                         cfg.jump_sampling_enabled)
        tag = ("map" if mapping is not None else ("old" if not enabled else "task"))
        save(f"r_{task_name}_{tag}", spec, x0, u_nom, seed, it, noise, out, mapping=mapping,
             keep_states=task_name == "cartpole")

    # --- BASELINE twins (control channel, upright cartpole lambda=1: the fp32-sensitive case)
    dt = 0.02
    params = jm.CartpoleModel(1.0, 0.1, 0.5, 9.81)
    model = jm.cartpole_dynamics(params)
    running = jm.CartpoleStateCost(w_pos=1.0, w_vel=0.1, w_angle=10.0, w_avel=0.1)
    cm = jm.CostModel(running, jm.ScaledTerminalCost(running, 10.0), 0.01 * np.eye(1), 1.0, 1.0)
    for T, K, name in [(100, 128, "r_cartpole_twin_T100"), (25, 128, "r_cartpole_twin_T25")]:
        cfg = jm.MppiConfig(1.0, 1.0, 100.0 * dt, 100.0 * dt, 0.5, dt, T, K, np.zeros(1))
        ctrl = jm.initial_controller_state(cfg)
        x0 = np.array([0.0, 0.0, np.pi, 0.0])
        noise, out = run_batched(jm, ctrl, model, cm, x0, 0)
        spec = spec_json("cartpole", (1.0, 0.1, 0.5, 9.81), 4, 1, None, "control", (), "sqrt_dt",
                         "cartpole_swingup", (1.0, 0.1, 10.0, 0.1), (), 10.0, 0.01 * np.eye(1), 1.0, 1.0,
                         1.0, 1.0, cfg.sigma_d, cfg.sigma_j, 0.5, dt, T, K)
        save(name, spec, x0, np.zeros((T, 1)), 0, 0, noise, out, keep_states=False)

    dt = 0.01
    qp = jm.QuadrotorModel(1.0, 0.2, (0.0082, 0.0082, 0.0149), 9.81)
    model = jm.quadrotor_dynamics(qp)
    running = jm.QuadrotorStateCost((4.0, 4.0, 2.0), 10.0, 1.0, 5.0, 0.1)
    cm = jm.CostModel(running, jm.ScaledTerminalCost(running, 10.0), 0.01 * np.eye(4), 1.0, 1.0)
    sd = np.diag(np.array([2.0, 0.1, 0.1, 0.1]) ** 2) * dt
    T, K = 150, 64
    cfg = jm.MppiConfig(1.0, 1.0, sd, sd, 1.0, dt, T, K, np.array([9.81, 0, 0, 0]))
    ctrl = jm.initial_controller_state(cfg)
    noise, out = run_batched(jm, ctrl, model, cm, np.zeros(12), 1)
    spec = spec_json("quadrotor", (1.0, 0.2, 0.0082, 0.0082, 0.0149, 9.81), 12, 4, None, "control", (),
                     "sqrt_dt", "quadrotor_hover", (10.0, 1.0, 5.0, 0.1), (4.0, 4.0, 2.0), 10.0, 0.01 * np.eye(4),
                     1.0, 1.0, 1.0, 1.0, sd, sd, 1.0, dt, T, K)
    save("r_quadrotor_twin", spec, np.zeros(12), np.tile([9.81, 0, 0, 0], (T, 1)), 1, 0, noise, out,
         keep_states=False)


def gen_general_channel(jm):
    """CostModel(control_channel=False, cal_b, bb_term): the general modified running cost
    (jm/costs.py:112-124) through the reference's batched mppi_iteration."""
    for task_name, K, T, seed, cal_b, bb in [
        ("cartpole", 96, 40, 31, np.array([[0.7]]), np.array([[1.4]])),
        ("quadrotor", 48, 30, 32,
         np.array([[1.0, 0.2, 0.0, 0.0], [0.0, 0.8, 0.1, 0.0], [0.0, 0.0, 1.2, 0.3], [0.1, 0.0, 0.0, 0.9]]),
         np.array([[2.0, 0.3, 0.0, 0.1], [0.3, 1.5, 0.2, 0.0], [0.0, 0.2, 1.0, 0.1], [0.1, 0.0, 0.1, 0.7]])),
    ]:
        ecfg = jm.config_from_dict({"task": task_name})
        task = jm.build_task(ecfg)
        cfg = jm.build_mppi_config(ecfg, samples_m=K)
        cfg = jm.MppiConfig(cfg.lambda_, cfg.c, cfg.sigma_d, cfg.sigma_j, cfg.nu, cfg.dt, T, K, cfg.u_init,
                            cfg.jump_sampling_enabled)
        tcm = task.cost_model
        cm = jm.CostModel(tcm.state_cost, tcm.terminal_cost, tcm.control_cost_matrix, tcm.lambda_, tcm.c,
                          control_channel=False, cal_b=cal_b, bb_term=bb)
        rng = np.random.default_rng(seed)
        u_nom = np.tile(cfg.u_init, (T, 1)) + rng.normal(scale=0.5, size=(T, cfg.control_dim)) * (
            np.array([5.0]) if task_name == "cartpole" else np.array([1.0, 0.02, 0.02, 0.02]))
        x0 = np.zeros(task.model.state_dim)
        ctrl = jm.ControllerState(jm.ControlSequence(u_nom, cfg.dt), 2, cfg)
        noise, out = run_batched(jm, ctrl, task.model, cm, x0, seed)
        fd = task.model.fused_drift_control.__self__
        sc = tcm.state_cost
        if task_name == "cartpole":
            params = (fd.cart_mass, fd.pole_mass, fd.pole_half_length, fd.gravity)
            cw, tgt, ck = (sc.w_pos, sc.w_vel, sc.w_angle, sc.w_avel), (), "cartpole_swingup"
        else:
            params = (fd.mass, fd.arm_length) + tuple(fd.inertia_diag) + (fd.gravity,)
            cw, tgt, ck = (sc.w_pos, sc.w_vel, sc.w_att, sc.w_rate), tuple(sc.target), "quadrotor_hover"
        spec = spec_json(task_name, params, task.model.state_dim, task.model.control_dim, task.model.control_limits,
                         "control", (), "sqrt_dt", ck, cw, tgt, tcm.terminal_cost.scale, tcm.control_cost_matrix,
                         tcm.lambda_, tcm.c, cfg.lambda_, cfg.c, cfg.sigma_d, cfg.sigma_j, cfg.nu, cfg.dt, T, K,
                         cfg.jump_sampling_enabled, cal_b=cal_b, bb_term=bb)
        save(f"r_{task_name}_general", spec, x0, u_nom, seed, 2, noise, out, keep_states=False)


def gen_linear(jm):
    """A generic linear plugin (f = A x, constant G = B = H) through the reference's
    batched mppi_iteration, with a diagonal quadratic cost."""
    cases = [
        ("r_linear_2x1", np.array([[0.0, 1.0], [-2.0, -0.3]]), np.array([[0.0], [1.0]]), 64, 30, 41),
        ("r_linear_4x2", np.array([[0, 1, 0, 0], [-1.5, -0.2, 0.4, 0], [0, 0, 0, 1], [0.3, 0, -0.8, -0.1]], float),
         np.array([[0, 0], [1.0, 0.2], [0, 0], [-0.1, 0.7]]), 48, 25, 42),
        ("r_linear_6x3", np.kron(np.eye(3), np.array([[0.0, 1.0], [-1.0, -0.4]])) + 0.05 * np.ones((6, 6)),
         np.kron(np.eye(3), np.array([[0.0], [1.0]])), 32, 20, 43),
    ]
    for name, A, G, K, T, seed in cases:
        n, m = G.shape

        def drift(x, t=0.0, A=A):
            return np.asarray(x, dtype=float) @ A.T

        def gmat(x, t=0.0, G=G):
            x = np.asarray(x, dtype=float)
            return np.broadcast_to(G, x.shape[:-1] + G.shape).copy()

        model = jm.DynamicsModel(state_dim=n, control_dim=m, drift=drift, control_matrix=gmat,
                                 diffusion_matrix=gmat, jump_matrix=gmat, noise_through_controls=True)
        w = np.linspace(1.0, 2.0, n)

        def q(x, t=0.0, w=w):
            x = np.asarray(x, dtype=float)
            return np.einsum("...i,i,...i->...", x, w, x)

        def phi(x, w=w):
            return 4.0 * q(x)

        R = 0.1 * np.eye(m)
        cm = jm.CostModel(state_cost=q, terminal_cost=phi, control_cost_matrix=R, lambda_=1.5, c=1.2)
        sd = 0.5 * np.eye(m)
        cfg = jm.MppiConfig(2.0, 1.2, sd, 2.0 * np.eye(m), 1.0, 0.05, T, K, np.zeros(m))
        rng = np.random.default_rng(seed)
        u_nom = 0.3 * rng.standard_normal((T, m))
        x0 = rng.standard_normal(n)
        ctrl = jm.ControllerState(jm.ControlSequence(u_nom, cfg.dt), 1, cfg)
        noise, out = run_batched(jm, ctrl, model, cm, x0, seed)
        spec = spec_json("linear", tuple(A.ravel()) + tuple(G.ravel()), n, m, None, "control", (), "sqrt_dt",
                         "diag", tuple(w), (0.0,) * n, 4.0, R, 1.5, 1.2, cfg.lambda_, cfg.c, cfg.sigma_d,
                         cfg.sigma_j, cfg.nu, cfg.dt, T, K, cfg.jump_sampling_enabled)
        save(name, spec, x0, u_nom, seed, 1, noise, out, keep_states=False)


def gen_state_jumps(jm):
    """BASELINE configs 0 and 2 (state-space jumps) via the reference per-rollout path."""
    from oracle import mppi as om

    cases = []
    # cfg0: cartpole, theta-dot jumps N(1, .5^2), O(1)
    dt = 0.02
    cp = jm.CartpoleModel(1.0, 0.1, 0.5, 9.81)
    H = np.zeros((4, 1))
    H[3, 0] = 1.0
    wq = np.array([1.0, 0.1, 10.0, 0.1])
    xs = np.array([0.0, 0.0, np.pi, 0.0])
    cases.append(dict(name="b_cartpole", kind="cartpole", plant=cp, H=H, n=4, m=1, q=1, rows=(3,),
                      params=(1.0, 0.1, 0.5, 9.81), cost="diag", w=wq, tgt=xs, R=0.01 * np.eye(1),
                      sigma_d=np.array([[100.0 * dt]]), sigma_j=np.array([[0.25]]), mark_mean=np.array([1.0]),
                      nu=0.5, dt=dt, T=100, K=64, x0=xs, u_init=np.zeros(1), seed=0))
    # cfg2: quadrotor gusts on v, N(0, I3), O(1)
    dt = 0.01
    qp = jm.QuadrotorModel(1.0, 0.2, (0.0082, 0.0082, 0.0149), 9.81)
    H = np.zeros((12, 3))
    H[3, 0] = H[4, 1] = H[5, 2] = 1.0
    cases.append(dict(name="b_quadrotor", kind="quadrotor", plant=qp, H=H, n=12, m=4, q=3, rows=(3, 4, 5),
                      params=(1.0, 0.2, 0.0082, 0.0082, 0.0149, 9.81), cost="quadrotor_hover",
                      w=np.array([10.0, 1.0, 5.0, 0.1]), tgt=np.array([4.0, 4.0, 2.0]), R=0.01 * np.eye(4),
                      sigma_d=np.diag(np.array([2.0, 0.1, 0.1, 0.1]) ** 2) * dt, sigma_j=np.eye(3),
                      mark_mean=np.zeros(3), nu=1.0, dt=dt, T=150, K=32, x0=np.zeros(12),
                      u_init=np.array([9.81, 0, 0, 0]), seed=2))
    for cs in cases:
        n, m, q, T, K, dt = cs["n"], cs["m"], cs["q"], cs["T"], cs["K"], cs["dt"]
        plant, Hc = cs["plant"], cs["H"]
        model = jm.DynamicsModel(state_dim=n, control_dim=m, drift=plant.drift,
                                 control_matrix=plant.control_matrix, diffusion_matrix=plant.control_matrix,
                                 jump_matrix=lambda x, t=0.0, Hc=Hc: Hc, noise_through_controls=False)
        if cs["cost"] == "diag":
            w, tgt = cs["w"], cs["tgt"]

            def running(x, t=0.0, w=w, tgt=tgt):
                e = np.asarray(x, dtype=float) - tgt
                return np.einsum("...i,i,...i->...", e, w, e)

            spec_cost = ("diag", tuple(w), tuple(tgt))
        else:
            running = jm.QuadrotorStateCost(tuple(cs["tgt"]), *cs["w"])
            spec_cost = ("quadrotor_hover", tuple(cs["w"]), tuple(cs["tgt"]))
        cm = jm.CostModel(running, jm.ScaledTerminalCost(running, 10.0), cs["R"], 1.0, 1.0)
        cfg = jm.MppiConfig(1.0, 1.0, cs["sigma_d"], np.eye(m), cs["nu"], dt, T, K, cs["u_init"])
        spec = spec_json(cs["kind"], cs["params"], n, m, None, "state", cs["rows"], "unit", spec_cost[0],
                         spec_cost[1], spec_cost[2], 10.0, cs["R"], 1.0, 1.0, 1.0, 1.0, cs["sigma_d"],
                         cs["sigma_j"], cs["nu"], dt, T, K, True, cs["mark_mean"])
        ospec = om.Spec(cs["kind"], n, m, tuple(cs["params"]), None, "state", cs["rows"], "unit", spec_cost[0],
                        spec_cost[1], spec_cost[2], 10.0, cs["R"], 1.0, 1.0, 1.0, 1.0, cs["sigma_d"],
                        cs["sigma_j"], cs["nu"], dt, T, K, True, cs["mark_mean"])
        eps_d, ind, marks, eps_c = om.sample_noise_batch_ref(cs["seed"], 0, ospec)
        u_nom = np.tile(cs["u_init"], (T, 1))
        ctrl = jm.ControllerState(jm.ControlSequence(u_nom, dt), 0, cfg)
        sq = math.sqrt(dt)
        rollouts = []
        for k in range(K):
            nr = jm.NoiseRealization(eps_d[k], ind[k], marks[k] / sq, eps_d[k])
            rollouts.append(jm.rollout(model, cs["x0"], ctrl.nominal_controls, nr, cm))
        seq = jm.update_controls(ctrl, rollouts)
        costs = np.array([r.cost for r in rollouts])
        weights = jm.compute_weights(costs, 1.0)
        delta = seq.controls - u_nom
        finite = np.isfinite(costs)
        out = dict(costs=costs, weights=weights, u_new=seq.controls, min_cost=float(costs[finite].min()),
                   ess=float(1.0 / np.sum(weights ** 2)), norms=np.linalg.norm(delta, axis=1),
                   diverged=np.array([-1 if r.diverged_at is None else r.diverged_at for r in rollouts]),
                   states=np.stack([r.trajectory.states for r in rollouts]))
        save(cs["name"], spec, cs["x0"], u_nom, cs["seed"], 0, (eps_d, ind, marks, eps_c), out,
             keep_states=cs["kind"] == "cartpole")


def gen_edge_branches(jm):
    """Branches the other cases never reach."""
    model = integrator_model(jm)
    # --- divergence with values float32 can hold: +-inf kills samples 3 and 7 (a non-finite
    # state); 1e17 drives sample 11's cost to ~1e33 with a finite state in float32 AND float64
    # (r_divergence's 1e200 is a float64-only value)
    cfg = jm.MppiConfig(lambda_=1.0, c=1.0, sigma_d=1.0, sigma_j=1.0, nu=0.0, dt=0.02, horizon_n=8,
                        samples_m=16, u_init=0.0, jump_sampling_enabled=False)
    rng = np.random.default_rng(101)
    eps_d = rng.standard_normal((16, 8, 1))
    eps_d[3, 2, 0] = np.inf
    eps_d[7, 5, 0] = -np.inf
    eps_d[11, 1, 0] = 1e17
    noise_in = (eps_d, np.zeros((16, 8), np.int64), np.zeros((16, 8, 1)), eps_d.copy())
    cm = quad_cost(jm, 1.0, 1.0, 1.0)
    ctrl = jm.initial_controller_state(cfg)
    noise, out = run_batched(jm, ctrl, model, cm, np.array([0.1]), 5, noise_override=noise_in)
    spec = spec_json("integrator", (), 1, 1, None, "control", (), "sqrt_dt", "diag", (1.0,), (0.0,), 1.0,
                     cm.control_cost_matrix, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.0, 0.02, 8, 16, False)
    save("r_divergence_f32", spec, [0.1], np.zeros((8, 1)), 5, 0, noise, out)

    # --- quadrotor cos-pitch floor (jm/dynamics.py:293, :361-363): pitch = pi/2 - 4e-7 gives
    # cos = +4e-7 < 1e-6 -> +1e-6; a slow pitch rate (4e-7 rad per step) carries the pitch across
    # pi/2 (cos < 0 -> -1e-6) and out of the band after four steps; torque noise of 1e-6 keeps
    # yaw-dot = q / cos(pitch) at O(10) rad/s there, so the costs stay comparable (ESS > 1)
    ecfg = jm.config_from_dict({"task": "quadrotor"})
    task = jm.build_task(ecfg)
    cfg = jm.build_mppi_config(ecfg, samples_m=32, jump_sampling_enabled=True)
    T, K = 12, 32
    sd = np.diag(np.array([0.5, 1e-6, 1e-6, 1e-6]) ** 2)
    cfg = jm.MppiConfig(50.0, cfg.c, sd, sd, cfg.nu, cfg.dt, T, K, cfg.u_init, cfg.jump_sampling_enabled)
    x0 = np.zeros(12)
    x0[7] = np.pi / 2 - 4e-7
    x0[9:12] = (1e-7, 2e-5, -1e-7)  # pitch-dot = cos(roll) wy: +4e-7 per step at dt = 0.02
    u_nom = np.tile(cfg.u_init, (T, 1))
    ctrl = jm.ControllerState(jm.ControlSequence(u_nom, cfg.dt), 2, cfg)
    noise, out = run_batched(jm, ctrl, task.model, task.cost_model, x0, 31)
    pitch = out["states"][:, :, 7]
    cp = np.cos(pitch[:, :-1])
    print(f"  pitch-floor: |cos| < 1e-6 on {np.mean(np.abs(cp) < 1e-6):.2f} of the state-steps, "
          f"{np.mean((np.abs(cp) < 1e-6) & (cp < 0)):.2f} with cos < 0")
    fd = task.model.fused_drift_control.__self__
    sc = task.cost_model.state_cost
    params = (fd.mass, fd.arm_length) + tuple(fd.inertia_diag) + (fd.gravity,)
    spec = spec_json("quadrotor", params, 12, 4, task.model.control_limits, "control", (), "sqrt_dt",
                     "quadrotor_hover", (sc.w_pos, sc.w_vel, sc.w_att, sc.w_rate), tuple(sc.target),
                     task.cost_model.terminal_cost.scale, task.cost_model.control_cost_matrix,
                     task.cost_model.lambda_, task.cost_model.c, cfg.lambda_, cfg.c, cfg.sigma_d, cfg.sigma_j,
                     cfg.nu, cfg.dt, T, K, cfg.jump_sampling_enabled)
    save("r_quadrotor_pitch_floor", spec, x0, u_nom, 31, 2, noise, out, keep_states=True)


def main():
    jm = _ref()
    only = sys.argv[1:]
    gens = dict(control=gen_control_channel, general=gen_general_channel, linear=gen_linear,
                state=gen_state_jumps, edge=gen_edge_branches)
    for name, fn in gens.items():
        if not only or name in only:
            fn(jm)


if __name__ == "__main__":
    main()
