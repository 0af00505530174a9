"""Ports of the reference's known-answer and statistical tests
(/root/reference/pkg/tests/test_controller.py, test_dynamics.py,
test_noise.py), run on the GPU through the drop-in API."""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import pytest

import paper_1807_06108_b200 as jb
from conftest import load_golden, oracle_spec, plugins, rel_err
from oracle import mppi as om
from oracle import philox_stream as ps

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- weights (test_controller.py:27-74)
def test_weights_closed_forms(gpu_device):
    w = jb.compute_weights(np.full(5, 3.3), 2.0)
    assert np.allclose(w, 0.2) and abs(w.sum() - 1) <= 1e-12
    lam = 0.7
    w = jb.compute_weights(np.array([0.0, lam * math.log(2.0)]), lam)
    assert w[0] == pytest.approx(2 / 3, rel=1e-12) and w[1] == pytest.approx(1 / 3, rel=1e-12)
    c = np.array([0.0, 1.0, 2.0])
    assert np.allclose(jb.compute_weights(c, 1.0), np.exp(-c) / np.exp(-c).sum(), rtol=1e-14)
    w = jb.compute_weights(np.array([1e9, 1e9 + 1.0]), 1.0)
    assert np.isfinite(w).all() and w[0] > w[1]
    w = jb.compute_weights(np.array([1.0, np.inf, 2.0]), 1.0)
    assert w[1] == 0.0 and w.sum() == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(jb.ControllerError, match="no viable rollout"):
        jb.compute_weights(np.array([np.inf, np.inf]), 1.0)


def test_weights_randomized_invariance(gpu_device):
    rng = np.random.default_rng(123)
    for _ in range(50):
        costs = rng.normal(scale=rng.uniform(0.1, 50.0), size=rng.integers(2, 64))
        lam = rng.uniform(0.05, 20.0)
        w = jb.compute_weights(costs, lam)
        assert abs(w.sum() - 1.0) <= 1e-12
        assert np.max(np.abs(w - om.compute_weights(costs, lam))) <= 1e-14
        order = np.argsort(costs)
        assert np.all(np.diff(w[order]) <= 1e-15)


# ---------------------------------------------------------------- update / shift (test_controller.py:98-161)
def _stub(cost, eps, dt):
    eps = np.asarray(eps, float)
    n, m = eps.shape
    return jb.RolloutResult(jb.StateTrajectory(np.zeros((n + 1, 1)), dt),
                            jb.NoiseRealization(eps * 0, np.zeros(n, int), eps * 0, eps), cost)


def _ctrl(n=1, m=1, dt=0.04, samples=3, u0=None):
    cfg = jb.MppiConfig(lambda_=1.0, c=1.0, sigma_d=np.eye(m), sigma_j=np.eye(m), nu=0.0, dt=dt, horizon_n=n,
                        samples_m=samples, u_init=np.zeros(m))
    u = np.zeros((n, m)) if u0 is None else np.asarray(u0, float)
    return jb.ControllerState(jb.ControlSequence(u, dt), 0, cfg)


def test_update_hand_values(gpu_device):
    ctrl = _ctrl()
    seq = jb.update_controls(ctrl, [_stub(c, np.zeros((1, 1)), 0.04) for c in (1.0, 2.0, 3.0)])
    assert np.array_equal(seq.controls, ctrl.nominal_controls.controls)
    seq = jb.update_controls(_ctrl(samples=1, u0=[[0.7]]), [_stub(5.0, [[0.3]], 0.04)])
    assert seq.controls[0, 0] == pytest.approx(0.7 + 0.3 / math.sqrt(0.04), rel=1e-15)
    seq = jb.update_controls(_ctrl(), [_stub(2.0, [[0.1]], 0.04), _stub(2.0, [[-0.2]], 0.04),
                                       _stub(2.0, [[0.4]], 0.04)])
    assert seq.controls[0, 0] == pytest.approx(0.5, rel=1e-12)
    seq = jb.update_controls(_ctrl(m=2, dt=0.25, samples=1, u0=np.zeros((1, 2))), [_stub(1.0, [[1.0, 2.0]], 0.25)],
                             mapping=np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(seq.controls[0], np.array([2.0, 1.0]) / math.sqrt(0.25))
    with pytest.raises(jb.ControllerError, match="no viable rollout"):
        jb.update_controls(_ctrl(), [_stub(np.inf, np.zeros((1, 1)), 0.04) for _ in range(3)])


def test_warm_start_shift_semantics(gpu_device):
    seq = jb.ControlSequence(np.array([[1.0], [2.0], [3.0]]), 0.02)
    assert np.array_equal(jb.warm_start_shift(seq, np.array([9.0])).controls, [[2.0], [3.0], [9.0]])
    assert np.array_equal(jb.warm_start_shift(jb.ControlSequence(np.array([[5.0]]), 0.02), [1.5]).controls, [[1.5]])
    for _ in range(3):
        seq = jb.warm_start_shift(seq, np.array([0.25]))
    assert np.array_equal(seq.controls, np.full((3, 1), 0.25))


# ---------------------------------------------------------------- end-to-end known answers
def test_two_sample_scalar_oracle(gpu_device):
    """test_controller.py:230-265 with the device kernels (fed noise)."""
    g = load_golden("r_integrator_m2n1")
    s = g["spec"]
    model, cost, cfg = plugins(s)
    ctrl = jb.ControllerState(jb.ControlSequence(np.array([[0.6]]), 0.04), 0, cfg)
    x0 = np.array([0.2])
    seq, diag = jb.mppi_iteration(ctrl, model, cost, x0, 7, noise=g["noise"], precision="f64")
    dt, costs, eps_l = 0.04, [], []
    for k in range(2):
        eps = float(g["noise"][3][k, 0, 0])
        eps_l.append(eps)
        qt = x0[0] ** 2 + 0.5 * 0.6 * 0.6 + 1.5 * 0.6 * eps / math.sqrt(dt) + 0.5 * 1.5 * 0.5 * eps * eps / dt
        x1 = x0[0] + 0.6 * dt + eps * math.sqrt(dt)
        costs.append(qt * dt + x1 ** 2)
    raw = np.exp(-(np.array(costs) - min(costs)) / 1.5)
    w = raw / raw.sum()
    assert np.allclose(diag.weights, w, rtol=1e-12)
    assert seq.controls[0, 0] == pytest.approx(0.6 + (w * np.array(eps_l)).sum() / math.sqrt(dt), rel=1e-12)


def test_cartpole_three_step_script(gpu_device):
    """test_dynamics.py:166-213: 3-step cartpole rollout vs a math-module script."""
    dt = 0.02
    controls = np.array([[2.0], [-1.0], [0.5]])
    eps_d = np.array([[0.3], [-0.6], [0.1]])
    ind = np.array([0, 1, 0])
    eps_j = np.array([[0.0], [1.8], [0.0]])
    model = jb.cartpole_dynamics()
    q = jb.DiagQuadraticCost((1.0, 1.0, 1.0, 1.0))
    cm = jb.CostModel(q, q, 0.7 * np.eye(1), 2.0, 1.5)
    cfg = jb.MppiConfig(lambda_=2.0, c=1.5, sigma_d=1.0, sigma_j=1.0, nu=0.5, dt=dt, horizon_n=3, samples_m=1,
                        u_init=[0.0])
    ctrl = jb.ControllerState(jb.ControlSequence(controls, dt), 0, cfg)
    noise = (eps_d[None], ind[None], eps_j[None], (eps_d + eps_j)[None])
    x0 = np.array([0.1, 0.0, 0.4, -0.2])
    _, _, ro = jb.mppi_iteration(ctrl, model, cm, x0, 0, return_rollouts=True, noise=noise, precision="f64")
    mc, mp, l, g = 1.0, 0.1, 0.5, 9.81
    state, total = list(x0), 0.0
    for j in range(3):
        u = controls[j, 0]
        eps = eps_d[j, 0] + eps_j[j, 0]
        total += (sum(v * v for v in state) + 0.5 * 0.7 * u * u + 2.0 * u * eps / math.sqrt(dt)
                  + 0.5 * 2.0 * (1 - 1 / 1.5) * eps * eps / dt) * dt
        s, co = math.sin(state[2]), math.cos(state[2])
        denom = mc + mp * s * s
        xdd = (u + mp * s * (g * co + l * state[3] ** 2)) / denom
        thdd = -(xdd * co + g * s) / l
        fn = eps_d[j, 0] * math.sqrt(dt) + ind[j] * eps_j[j, 0] * math.sqrt(dt)
        state = [state[0] + state[1] * dt, state[1] + xdd * dt + fn / denom, state[2] + state[3] * dt,
                 state[3] + thdd * dt - co / (l * denom) * fn]
    total += sum(v * v for v in state)
    assert ro[0].cost == pytest.approx(total, rel=1e-12)
    assert np.allclose(ro[0].trajectory.states[-1], state, rtol=1e-12)


def test_upright_and_hover_equilibria(gpu_device):
    """test_dynamics.py:34-38, :138-145 via zero-noise rollouts."""
    for model, x0, u in [(jb.cartpole_dynamics(), np.array([0.0, 0.0, np.pi, 0.0]), [0.0]),
                         (jb.quadrotor_dynamics(), np.zeros(12), [9.81, 0, 0, 0])]:
        n, m = model.state_dim, model.control_dim
        cm = jb.zero_cost_model(n, m=m)
        cfg = jb.MppiConfig(1.0, 1.0, np.eye(m), np.eye(m), 0.0, 0.02, 50, 4, u)
        z = np.zeros((4, 50, m))
        _, _, ro = jb.mppi_iteration(jb.initial_controller_state(cfg), model, cm, x0, 0, return_rollouts=True,
                                     noise=(z, np.zeros((4, 50)), z, z), precision="f64")
        assert np.allclose(ro[0].trajectory.states, x0, atol=1e-12)


def test_all_diverged_raises(gpu_device):
    g = load_golden("r_divergence")
    s = g["spec"]
    model, cost, cfg = plugins(s)
    eps = np.full((16, 8, 1), np.inf)
    z = np.zeros((16, 8, 1))
    for prec in ("f32", "f64"):
        with pytest.raises(jb.ControllerError, match="no viable rollout"):
            jb.mppi_iteration(jb.initial_controller_state(cfg), model, cost, g["x0"], 0,
                              noise=(eps, np.zeros((16, 8)), z, eps), precision=prec)


def test_unsupported_plugins_raise(gpu_device):
    model = jb.cartpole_dynamics()
    cfg = jb.MppiConfig(1.0, 1.0, 1.0, 1.0, 0.1, 0.02, 10, 8, [0.0])
    bad_cost = jb.CostModel(lambda x, t=0.0: x, lambda x: x, np.eye(1), 1.0, 1.0)
    with pytest.raises(NotImplementedError):
        jb.mppi_iteration(jb.initial_controller_state(cfg), model, bad_cost, np.zeros(4), 0)
    with pytest.raises(ValueError, match="zero-one jump law"):
        cfg2 = jb.MppiConfig(1.0, 1.0, 1.0, 1.0, 10.0, 0.02, 10, 8, [0.0])
        jb.mppi_iteration(jb.initial_controller_state(cfg2), model, jb.quadratic_cost_model(4), np.zeros(4), 0)
    with pytest.raises(jb.NoiseError):
        cfg3 = jb.MppiConfig(1.0, 1.0, -1.0, 1.0, 0.1, 0.02, 10, 8, [0.0])
        jb.mppi_iteration(jb.initial_controller_state(cfg3), model, jb.quadratic_cost_model(4), np.zeros(4), 0)


# ---------------------------------------------------------------- statistics (G-stat)
def test_device_noise_moments(gpu_device):
    """test_noise.py:30-46, :60-66, :79-84 on the device stream."""
    sd = np.array([[2.0, 0.3], [0.3, 1.0]])
    cfg = jb.MppiConfig(1.0, 1.5, sd, 4.0 * np.eye(2), 0.5, 0.02, 200, 2000, np.zeros(2))
    ed, ind, ej, ec = jb.sample_noise_batch(jb.RngStream(3, 5), cfg, 2000, precision="f64")
    x = ed.reshape(-1, 2)
    n = x.shape[0]
    cov = np.cov(x.T)
    target = 1.5 * sd
    for (i, j) in [(0, 0), (1, 1), (0, 1)]:
        se = math.sqrt((target[i, j] ** 2 + target[i, i] * target[j, j]) / n)
        assert abs(cov[i, j] - target[i, j]) < 4 * se
    p = 0.5 * 0.02
    assert abs(ind.mean() - p) < 4 * math.sqrt(p * (1 - p) / ind.size)
    assert set(np.unique(ind)) <= {0, 1}
    marks = ej[ind == 1]
    assert np.all(ej[ind == 0] == 0.0)
    v = marks.var(axis=0)
    assert np.all(np.abs(v - 4.0) < 5 * 4.0 * math.sqrt(2.0 / marks.shape[0]))
    assert np.array_equal(ec, ed + ej)


def test_update_unbiased_at_zero_cost_sensitivity(gpu_device):
    """test_controller.py:268-288: q = phi = 0, u = 0, c = 1 -> E[update] = 0."""
    model = jb.integrator_dynamics(1)
    cm = jb.zero_cost_model(1)
    sigma_d, M, dt, reps = 1.0, 1000, 0.02, 200
    cfg = jb.MppiConfig(1.0, 1.0, sigma_d, 4.0, 0.0, dt, 3, M, [0.0])
    ctrl = jb.initial_controller_state(cfg)
    up = np.empty((reps, 3))
    for k in range(reps):
        seq, _ = jb.mppi_iteration(jb.ControllerState(ctrl.nominal_controls, k, cfg), model, cm, np.zeros(1), 31415)
        up[k] = seq.controls[:, 0]
    se = math.sqrt(sigma_d) / math.sqrt(M * dt) / math.sqrt(reps)
    assert np.all(np.abs(up.mean(axis=0)) < 3.5 * se)


def test_control_statistics_over_seeds_match_oracle(gpu_device):
    """G-stat: GPU (device Philox) vs oracle (numpy Philox) control-update mean
    per (t, j) agree within sampling error over 24 seeds."""
    g = load_golden("r_cartpole_twin_T25")
    s = g["spec"]
    model, cost, cfg = plugins(s, K=512)
    spec = oracle_spec(s)
    spec.K = 512
    ref, gpu = [], []
    for seed in range(24):
        seq, _ = jb.mppi_iteration(jb.initial_controller_state(cfg), model, cost, g["x0"], seed, precision="f64")
        gpu.append(seq.controls[:, 0])
        noise = om.sample_noise_batch_ref(seed, 0, spec)
        ref.append(om.mppi_iteration_oracle(spec, g["x0"], np.zeros((s["T"], 1)), noise)["u_new"][:, 0])
    gpu, ref = np.array(gpu), np.array(ref)
    se = np.sqrt(gpu.var(0, ddof=1) / len(gpu) + ref.var(0, ddof=1) / len(ref))
    z = np.abs(gpu.mean(0) - ref.mean(0)) / se
    assert np.mean(z < 3.0) >= 0.9 and z.max() < 5.0


# ---------------------------------------------------------------- closed loop
def test_closed_loop_matches_iteration_and_plant(gpu_device):
    task, cfg = jb.baseline_config(0, K=1024, T=50, steps=20)
    rec = jb.run_trial(task, cfg, seed=11, precision="f64")
    assert rec.states.shape == (21, 4) and rec.controls.shape == (20, 1)
    assert np.isfinite(rec.states).all() and not rec.diverged
    assert np.all(rec.wall_time_per_iteration > 0)
    rec2 = jb.run_trial(task, cfg, seed=11, precision="f64")
    assert np.array_equal(rec.states, rec2.states)  # deterministic
    # step 0: the loop's iteration equals a standalone mppi_iteration from x0
    seq, _ = jb.mppi_iteration(jb.initial_controller_state(cfg), task.model, task.cost_model, task.x0, 11,
                               precision="f64")
    assert rec.controls[0, 0] == seq.controls[0, 0]
    # plant step 0 with the emulated plant stream (Sigma_D, theta-dot jump with N(1, .25) mark)
    key = ps.stream_key(11, 0)
    w = ps.draw(key, ps.SLOT_PLANT, np.array([0, 1, 2], np.uint32), np.uint32(0))
    z0, _ = ps.box_muller(w[0][0], w[1][0])
    jump = int(w[0][1]) < ps.jump_threshold(cfg.nu * cfg.dt)
    mk = 1.0 + 0.5 * ps.box_muller(w[0][2], w[1][2])[0]
    spec = om.Spec("cartpole", 4, 1, (1.0, 0.1, 0.5, 9.81), None, "state", (3,), "unit", "diag", (1, .1, 10, .1),
                   (0, 0, np.pi, 0), 10.0, 0.01 * np.eye(1), 1.0, 1.0, 1.0, 1.0, cfg.sigma_d, cfg.sigma_j, cfg.nu,
                   cfg.dt, 50, 1)
    x1 = om.step_batch(spec, task.x0[None], rec.controls[0], np.array([[math.sqrt(cfg.sigma_d[0, 0]) * z0]]),
                       np.array([[mk]]), np.array([1.0 if jump else 0.0]), cfg.dt, np.float64)[0]
    assert np.allclose(rec.states[1], x1, rtol=1e-5, atol=1e-6)
    assert rec.jump_indicators[0] == int(jump)


def test_closed_loop_f32_runs_and_stays_finite(gpu_device):
    task, cfg = jb.baseline_config(2, K=2048, T=100, steps=30)
    rec = jb.run_trial(task, cfg, seed=3)
    assert np.isfinite(rec.states).all()
    assert rec.wall_time_per_iteration.shape == (30,)


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_sharded_loop_world1_matches_graph_loop(scaling, gpu_device):
    """The multi-GPU stage split (rollout+record, all_gather, merge/plant) over a
    one-rank NCCL group reproduces the single-GPU graph loop (weak: K per rank;
    strong: config 3's K/N split, the whole K at world 1)."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1807_06108_b200 import distributed as jd

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        task, cfg = jb.baseline_config(0, K=2048, T=60, steps=12)
        rec = jb.run_trial(task, cfg, seed=5, precision="f64")
        loop = jd.ShardedLoop.create(task, cfg, 0, 1, 0, precision="f64", scaling=scaling)
        assert loop.k_total == 2048 and loop.ctx.K == 2048
        loop.init(task.x0, cfg.u_init, 5, 64)
        for _ in range(12):
            loop.step()
        x, it, st, halted, status = loop.read()
        assert st == 12 and it == 12 and not halted
        assert np.allclose(x, rec.states[-1], rtol=1e-9, atol=1e-12)
    finally:
        dist.destroy_process_group()


def test_lazy_weights_match_eager_and_survive_later_iterations(gpu_device):
    task, cfg = jb.baseline_config(0, K=4096, T=40)
    c0 = jb.initial_controller_state(cfg)
    s0, d0 = jb.mppi_iteration(c0, task.model, task.cost_model, task.x0, 3)        # graph fast path, lazy
    c1 = jb.ControllerState(jb.warm_start_shift(s0, cfg.u_init), 1, cfg)
    s1, d1 = jb.mppi_iteration(c1, task.model, task.cost_model, task.x0, 3)
    _, e0, ro = jb.mppi_iteration(c0, task.model, task.cost_model, task.x0, 3, return_rollouts=True)  # eager
    assert np.array_equal(d0.weights, e0.weights)  # fetched after a later iteration ran
    assert d0.weights.sum() == pytest.approx(1.0, abs=1e-12)
    costs = np.array([r.cost for r in ro])
    assert np.allclose(d0.weights, jb.compute_weights(costs, cfg.lambda_), rtol=1e-6, atol=1e-300)
    assert not np.array_equal(d0.weights, d1.weights)
    # the GPU-precomputed shift equals the device shift kernel
    assert np.array_equal(jb.warm_start_shift(s1, cfg.u_init).controls,
                          jb.warm_start_shift(jb.ControlSequence(s1.controls, cfg.dt), cfg.u_init).controls)


def test_batched_trials_equal_single_trials(gpu_device):
    """run_batch (trial dimension on the GPU) == run_trial per seed, bit for bit, both variants."""
    import dataclasses

    task, cfg = jb.baseline_config(0, K=640, T=30, steps=25)
    out = jb.run_batch(task, cfg, n_trials=3, base_seed=7, config_id="b")
    for variant, (recs, summ) in out.items():
        vcfg = dataclasses.replace(cfg, jump_sampling_enabled=(variant == "new"))
        assert [r.seed for r in recs] == [jb.trial_seed(7, k) for k in range(3)]
        for r in recs:
            one = jb.run_trial(task, vcfg, r.seed)
            assert np.array_equal(r.states, one.states) and np.array_equal(r.controls, one.controls)
            assert np.array_equal(r.jump_indicators, one.jump_indicators)
            assert r.success == one.success and r.diverged == one.diverged
            assert r.config_id == f"b/{variant}"
        assert summ.mean_states.shape == recs[0].states.shape
    # the quadrotor (12 states, 4 controls, 3-axis gusts) through the same path
    qtask, qcfg = jb.baseline_config(2, K=512, T=20, steps=10)
    q = jb.run_batch(qtask, qcfg, n_trials=2, base_seed=3, variants=("new",))["new"][0]
    for r in q:
        one = jb.run_trial(qtask, qcfg, r.seed)
        assert np.array_equal(r.states, one.states) and np.array_equal(r.controls, one.controls)


def test_sharded_loop_world1_peer_memory_exchange(gpu_device):
    """The NCCL-free exchange (symmetric buffer, push kernel, device-side epoch
    wait) over a one-rank group reproduces the single-GPU graph loop."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1807_06108_b200 import distributed as jd

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        task, cfg = jb.baseline_config(0, K=2048, T=60, steps=12)
        rec = jb.run_trial(task, cfg, seed=5, precision="f64")
        loop = jd.ShardedLoop.create(task, cfg, 0, 1, 0, precision="f64", transport="p2p")
        loop.init(task.x0, cfg.u_init, 5, 64)
        for _ in range(12):
            loop.step()
        x, it, st, halted, status = loop.read()
        assert st == 12 and it == 12 and not halted
        assert np.allclose(x, rec.states[-1], rtol=1e-9, atol=1e-12)
        sts, cos, jus = loop.history(12)
        assert np.allclose(sts, rec.states, rtol=1e-9, atol=1e-12)
    finally:
        dist.destroy_process_group()


def test_sharded_loop_world1_two_level_exchange_matches_nccl(gpu_device):
    """The two-level peer-memory exchange (rank-local reduce kernel pushes one
    record per rank, the finalize waits on world x column-block flags) runs the
    NCCL transport's merge tree: bit-identical trajectories, cartpole (one
    column block) and quadrotor (T*m = 240: two column blocks, two flags)."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1807_06108_b200 import distributed as jd

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        for idx, K, T in ((0, 2048, 60), (2, 512, 60)):
            task, cfg = jb.baseline_config(idx, K=K, T=T, steps=10)
            hist = {}
            for transport, two in (("nccl", None), ("p2p", True)):
                loop = jd.ShardedLoop.create(task, cfg, 0, 1, 0, precision="f64", transport=transport)
                loop.two_level = two
                loop.init(task.x0, cfg.u_init, 7, 64)
                for _ in range(10):
                    loop.step()
                x, it, st, halted, status = loop.read()
                assert st == 10 and not halted, (transport, status)
                hist[transport] = [np.array(h) for h in loop.history(10)]
            for a, b in zip(hist["nccl"], hist["p2p"]):
                assert np.array_equal(a, b)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("idx,K,T,steps", [(0, 512, 30, 24), (2, 256, 20, 20)])
def test_closed_loop_multistep_matches_oracle_loop(idx, K, T, steps, gpu_device):
    """The device-resident loop (harness.py:131-150) step by step against an
    oracle loop: at every control step k the oracle iteration (the restatement
    of controller.py:103-181) runs from the loop's state on the device sampler's
    noise table for iteration k and the oracle's own warm-started nominal
    (controller.py:96-100), and must give the loop's applied control u0
    (harness.py:136); the loop's plant step must equal the oracle Euler step
    with the emulated plant stream (Sigma_D, not c Sigma_D; the jump drawn and
    the mark always drawn, harness.py:137-139)."""
    from paper_1807_06108_b200 import engine

    task, cfg = jb.baseline_config(idx, K=K, T=T, steps=steps)
    seed = 11
    rec = jb.run_trial(task, cfg, seed=seed, precision="f64")
    assert not rec.diverged
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision="f64")
    spec = om.spec_from_plugins(task.model, task.cost_model, cfg)
    m, q = spec.m, spec.q
    Lp = np.linalg.cholesky(np.asarray(cfg.sigma_d, float))
    Lj = np.linalg.cholesky(np.asarray(cfg.sigma_j, float))
    mu = np.asarray(cfg.mark_mean, float)
    key = ps.stream_key(seed, 0)
    jthr = ps.jump_threshold(cfg.nu * cfg.dt)
    u_nom = np.tile(np.asarray(cfg.u_init, float), (T, 1))
    for k in range(steps):
        x = rec.states[k]
        out = om.mppi_iteration_oracle(spec, x, u_nom, ctx.sample_noise(seed, k), np.float64)
        u0 = om.clamp(spec, out["u_new"][0])
        # (f64 both sides; the two nominal chains drift apart by rounding, amplified by the
        # upright cartpole's instability: ~3e-8 after 18 steps -- the single-iteration gate is 1e-9)
        assert rel_err(rec.controls[k], u0, floor=1e-6) <= 1e-6, k
        w = ps.draw(key, ps.SLOT_PLANT, np.array([3 * k, 3 * k + 1, 3 * k + 2], np.uint32), np.uint32(0))
        z = np.concatenate([ps.box_muller(w[0][0], w[1][0]), ps.box_muller(w[2][0], w[3][0])])
        zm = np.concatenate([ps.box_muller(w[0][2], w[1][2]), ps.box_muller(w[2][2], w[3][2])])
        jump = int(w[0][1]) < jthr
        assert rec.jump_indicators[k] == int(jump), k
        ed = Lp @ z[:m]
        mk = mu + Lj @ zm[:q]
        x1 = om.step_batch(spec, x[None], rec.controls[k], ed[None], mk[None], np.array([1.0 if jump else 0.0]),
                           cfg.dt, np.float64)[0]
        # (the device's Box-Muller runs on MUFU lg2/sqrt/sincos: plant normals to ~1e-6)
        assert np.allclose(rec.states[k + 1], x1, rtol=2e-5, atol=2e-6), k
        u_nom = om.warm_start_shift(out["u_new"], cfg.u_init)
