"""Poisson jump counts (MppiConfig.jump_process="poisson", BASELINE north star
"Poisson jump counts per step drawn with rate nu dt").

The reference samples jumps by the zero-one law (an indicator U < nu dt per
step, jm/noise.py:151); the Poisson process is this repo's extension: per
(sample, step) N ~ Poisson(nu dt) arrivals whose N(mark_mean, Sigma_J) marks
add up (compound Poisson).  The device realises it as jump events with
P(N >= 1) = 1 - exp(-nu dt) (the renewal clock of csrc/philox.cuh) carrying a
zero-truncated count from slot 4.  CPU tests pin the count tables and the
emulated sampler's statistics; GPU tests pin the device draws bit-exactly to
the emulation (oracle/philox_stream.py) and the iteration to the oracle.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import pytest

from conftest import load_golden, oracle_spec, plugins, rel_err
from oracle import mppi as om
from oracle import philox_stream as ps

G_DOUBLE = 1e-9


def _poisson_pmf(lam, k):
    return math.exp(-lam) * lam ** k / math.factorial(k)


@pytest.mark.parametrize("lam", [1e-4, 0.01, 0.05, 0.099])
def test_count_tables_match_poisson(lam):
    ev, pl = ps.count_tables(lam)
    p1 = -math.expm1(-lam)
    assert np.all(np.diff(ev) <= 0) and np.all(np.diff(pl) <= 0)
    assert pl[0] == math.ceil(p1 * 2 ** 24)
    # implied count probabilities (exact integers / 2^24) vs the pmf, to the table's 2^-24 quantum
    bounds = np.concatenate([[2 ** 24], ev, [0]])
    for k in range(1, 6):
        implied = (bounds[k - 1] - bounds[k]) / 2 ** 24
        assert abs(implied - _poisson_pmf(lam, k) / p1) <= 2.0 ** -23
    pb = np.concatenate([[2 ** 24], pl, [0]])
    for k in range(0, 6):
        implied = (pb[k] - pb[k + 1]) / 2 ** 24
        assert abs(implied - _poisson_pmf(lam, k)) <= 2.0 ** -23


def test_emulated_poisson_sampler_statistics():
    """Counts per step ~ Poisson(nu dt) (mean = variance = nu dt, P(N >= 2)),
    event steps from the renewal clock with p = 1 - exp(-nu dt)."""
    lam, K, T = 0.08, 4096, 120
    ev, _ = ps.count_tables(lam)
    jthr = ps.jump_threshold(ps.event_probability(lam, True))
    L = np.eye(1)
    _, ind, ej, _ = ps.device_noise(5, 2, K, T, 1, 1, L, L, [0.5], jthr, jump_channel="state", counts=ev)
    n = ind.size
    assert abs(ind.mean() - lam) < 4 * math.sqrt(lam / n)
    assert abs(ind.var() - lam) < 4 * math.sqrt((lam + 2 * lam ** 2) / n)
    p2 = 1 - math.exp(-lam) * (1 + lam)
    assert abs(np.mean(ind >= 2) - p2) < 4 * math.sqrt(p2 / n)
    assert ind.max() >= 2
    # the step's mark is the sum of its n marks: mean n mu, variance n
    for c in (1, 2):
        sel = ej[ind == c][:, 0]
        assert abs(sel.mean() - 0.5 * c) < 5 * math.sqrt(c / sel.size)
    assert np.all(ej[ind == 0] == 0.0)
    # one arrival per event when counts are off: the Bernoulli sampler's events
    jb_ = ps.jump_threshold(lam)
    b = ps.device_noise(5, 2, 64, T, 1, 1, L, L, [0.5], jb_, jump_channel="state")[1]
    assert set(np.unique(b)) <= {0, 1}


def test_config_jump_process_validation():
    import paper_1807_06108_b200 as jb

    cfg = jb.MppiConfig(1.0, 1.0, 1.0, 1.0, 0.5, 0.02, 10, 8, [0.0], jump_process="poisson")
    assert jb.validate_config(cfg) is cfg
    with pytest.raises(jb.ConfigError):
        jb.validate_config(jb.MppiConfig(1.0, 1.0, 1.0, 1.0, 0.5, 0.02, 10, 8, [0.0], jump_process="levy"))


# ---------------------------------------------------------------- GPU: device draws == emulation
def _poisson_cfg(name, K, T, nu_dt=0.09):
    g = load_golden(name)
    s = g["spec"]
    model, cost, cfg = plugins(s, K=K, T=T)
    cfg = dataclasses.replace(cfg, nu=nu_dt / cfg.dt, jump_process="poisson", jump_sampling_enabled=True)
    return g, s, model, cost, cfg


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["r_cartpole_task", "r_quadrotor_task", "b_cartpole", "b_quadrotor"])
def test_device_poisson_noise_matches_emulation(name, gpu_device):
    import paper_1807_06108_b200 as jb

    g, s, model, cost, cfg = _poisson_cfg(name, 300, 37)
    ed, ind, ej, ec = jb.sample_noise_batch(jb.RngStream(123, 9), cfg, 300, model=model, precision="f64")
    spec = oracle_spec(s)
    Ld = np.linalg.cholesky(cfg.c * np.asarray(cfg.sigma_d))
    Lj = np.linalg.cholesky(np.asarray(cfg.sigma_j))
    lam = cfg.nu * cfg.dt
    jthr = ps.jump_threshold(ps.event_probability(lam, True))
    e = ps.device_noise(123, 9, 300, 37, spec.m, spec.q, Ld, Lj, np.asarray(cfg.mark_mean), jthr,
                        jump_channel=spec.jump_channel, counts=ps.count_tables(lam)[0])
    assert np.array_equal(ind, e[1])  # event steps and counts: bit-exact integer path
    assert ind.max() >= 2             # multi-arrival steps occur at nu dt = 0.09
    for a, b in zip((ed, ej, ec), (e[0], e[2], e[3])):
        assert np.max(np.abs(a - b) / (1.0 + np.abs(b))) < 2e-5


@pytest.mark.gpu
def test_device_poisson_moments(gpu_device):
    import paper_1807_06108_b200 as jb

    lam = 0.06
    cfg = jb.MppiConfig(1.0, 1.0, 1.0, 4.0, lam / 0.02, 0.02, 200, 4000, [0.0], jump_process="poisson")
    _, ind, ej, _ = jb.sample_noise_batch(jb.RngStream(3, 5), cfg, 4000, precision="f64")
    n = ind.size
    assert abs(ind.mean() - lam) < 4 * math.sqrt(lam / n)
    assert abs(ind.var() - lam) < 4 * math.sqrt((lam + 2 * lam ** 2) / n)
    p2 = 1 - math.exp(-lam) * (1 + lam)
    assert abs(np.mean(ind >= 2) - p2) < 4 * math.sqrt(p2 / n)
    for c in (1, 2):  # control-channel marks N(0, 4): the sum of c has variance 4c
        sel = ej[ind == c][:, 0]
        assert abs(sel.var() - 4.0 * c) < 5 * 4.0 * c * math.sqrt(2.0 / sel.size)


@pytest.mark.gpu
@pytest.mark.parametrize("name,K", [("b_cartpole", 256), ("b_cartpole", 8192), ("r_cartpole_task", 2048),
                                    ("b_quadrotor", 1024), ("r_quadrotor_task", 8192),
                                    # (rollout_fast with the indexed mark staging: state and control-channel marks)
                                    ("b_quadrotor", 24000), ("r_quadrotor_task", 24000)])
def test_f64_poisson_iteration_matches_oracle(name, K, gpu_device):
    """The rollout kernels (warp-specialised and main, per K) consume exactly
    the Poisson noise sample_noise_batch exports."""
    import paper_1807_06108_b200 as jb

    g, s, model, cost, cfg = _poisson_cfg(name, K, None)
    ctrl = jb.ControllerState(jb.ControlSequence(g["u_nom"], s["dt"]), 5, cfg)
    seq, diag = jb.mppi_iteration(ctrl, model, cost, g["x0"], 77, precision="f64")
    noise = jb.sample_noise_batch(jb.RngStream(77, 5), cfg, K, model=model, precision="f64")
    assert noise[1].max() >= 2
    spec = dataclasses.replace(oracle_spec(s), K=K, nu=cfg.nu)
    out = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], noise, np.float64)
    assert rel_err(seq.controls, out["u_new"], floor=1e-9) <= G_DOUBLE
    assert diag.min_cost == pytest.approx(out["min_cost"], rel=G_DOUBLE)
    # fp32 kernel on the same draws: within the fp32 gate of the oracle's update
    seq32, _ = jb.mppi_iteration(ctrl, model, cost, g["x0"], 77)
    d = out["u_new"] - g["u_nom"]
    assert np.linalg.norm(seq32.controls - out["u_new"]) <= max(1e-3 * np.linalg.norm(d), 1e-9)


@pytest.mark.gpu
def test_closed_loop_plant_poisson_counts(gpu_device):
    """The plant's arrivals per control step are Poisson(nu dt) counts drawn
    from the plant stream (slot 3, block 3k+1) against the plant table."""
    import paper_1807_06108_b200 as jb

    task, cfg = jb.baseline_config(0, K=512, T=30, steps=400)
    cfg = dataclasses.replace(cfg, nu=0.09 / cfg.dt, jump_process="poisson")
    rec = jb.run_trial(task, cfg, seed=21, precision="f64")
    assert not rec.diverged
    key = ps.stream_key(21, 0)
    steps = np.arange(400, dtype=np.uint32)
    w = ps.draw(key, ps.SLOT_PLANT, 3 * steps + 1, np.uint32(0))
    u24 = (w[0] >> np.uint32(8)).astype(np.int64)
    _, pl = ps.count_tables(cfg.nu * cfg.dt)
    n = np.sum(u24[:, None] < pl[None, :], axis=1)
    assert np.array_equal(rec.jump_indicators, n)
    assert n.max() >= 2


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["b_cartpole", "b_quadrotor", "r_cartpole_task"])
def test_fed_poisson_noise_matches_oracle(name, gpu_device):
    """HBM (fed-noise) mode with a Poisson noise table: counts > 1 carry the
    summed marks in eps_j, the kernels apply them once (flag = count != 0)."""
    import paper_1807_06108_b200 as jb

    g, s, model, cost, cfg = _poisson_cfg(name, 512, None)
    noise = jb.sample_noise_batch(jb.RngStream(5, 3), cfg, 512, model=model, precision="f64")
    assert noise[1].max() >= 2
    ctrl = jb.ControllerState(jb.ControlSequence(g["u_nom"], s["dt"]), 3, cfg)
    seq, diag = jb.mppi_iteration(ctrl, model, cost, g["x0"], 5, noise=noise, precision="f64")
    spec = dataclasses.replace(oracle_spec(s), K=512, nu=cfg.nu)
    out = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], noise, np.float64)
    assert rel_err(seq.controls, out["u_new"], floor=1e-9) <= G_DOUBLE
    # and the fed table reproduces the in-kernel Philox iteration of the same stream
    seq_p, _ = jb.mppi_iteration(ctrl, model, cost, g["x0"], 5, precision="f64")
    assert rel_err(seq_p.controls, seq.controls, floor=1e-9) <= G_DOUBLE
