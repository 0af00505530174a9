"""Size-independent properties of the product kernels at BASELINE's FULL sizes.

The oracle finishes K = 2^20 x T = 200 quadrotor rollouts in hours, so at the
full shapes of BASELINE configs 1 and 3 the benchmarked fp32 Philox kernels
(`jm_kernel_name` asserted) are checked through properties the path offers:

  * normalisation: the weights sum to 1, ESS = 1 / sum w^2, min_cost = min S
    (controller.py:62-71, :163-169);
  * the sparse epilogue at full size: the update equals the weighted noise sum
    over the samples that carry weight, u_new - u_nom = sum_k w_k eps_k / sqrt(dt)
    (controller.py:74-78, :158-161), with those samples' noise regenerated
    independently through the device sampler at their GLOBAL sample indices,
    and their costs reproduced by the float64 oracle on that noise (G-float);
  * shard additivity: two half-size launches at sample offsets 0 and K/2 give
    records whose log-sum-exp merge is the full launch's (rho bit for bit, Z,
    sum w^2 and n_finite to reduction-order rounding) -- the noise does not
    depend on the launch shape;
  * determinism: a second run is bit-identical.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1807_06108_b200 as jb
from oracle import mppi as om
from paper_1807_06108_b200 import engine

pytestmark = pytest.mark.gpu

FULL = [
    ("cfg1", 1, 65536, 100, "rollout_fast/philox/single_wave/f32"),
    ("cfg3", 3, 1 << 20, 200, "rollout_fast/philox/multi_wave/f32"),
]


def _run(task, cfg, K, offset=0, seed=11, iteration=3):
    ctx = engine.get_context(task.model, task.cost_model, cfg, samples=K, precision="f32", sample_offset=offset)
    u_nom = np.tile(np.atleast_1d(np.asarray(cfg.u_init, float)), (cfg.horizon_n, 1))
    out = ctx.iteration(task.x0, u_nom, seed, iteration, want_costs=True, want_weights=True)
    return ctx, u_nom, out


@pytest.mark.parametrize("case,idx,K,T,variant", FULL)
def test_full_size_properties(case, idx, K, T, variant, gpu_device):
    task, cfg = jb.baseline_config(idx)
    assert cfg.samples_m == K and cfg.horizon_n == T
    ctx, u_nom, out = _run(task, cfg, K)
    assert ctx.kernel_name().startswith(variant), ctx.kernel_name()
    w, S = out.weights, out.costs
    fin = np.isfinite(S)
    assert fin.sum() == out.diag.n_finite and fin.mean() > 0.9
    # normalisation and diagnostics (fp64 sums over K samples)
    assert abs(w.sum() - 1.0) <= 1e-5  # (Z sums the rollout's fp32 exponentials)
    assert np.all(w >= 0.0) and np.all(w[~fin] == 0.0)
    assert out.diag.min_cost == S[fin].min()  # the same fp32 value, bit for bit
    assert out.diag.ess == pytest.approx(1.0 / np.sum(w * w), rel=1e-5)
    lam = cfg.lambda_
    heavy = np.flatnonzero(w > 1e-15)
    assert heavy.size >= 1
    # weights are exp(-(S - rho)/lambda) / Z on the kernel's own costs
    wref = np.exp(-(S[heavy] - out.diag.min_cost) / lam) / out.diag.normaliser
    assert np.allclose(w[heavy], wref, rtol=1e-5, atol=0)

    # the heavy samples' noise, regenerated one sample at a time at its global index
    dt, m = cfg.dt, cfg.control_dim
    order = heavy[np.argsort(-w[heavy])]
    ntop = int(min(256, 1 + np.searchsorted(np.cumsum(w[order]), w.sum() * (1.0 - 1e-8))))
    top = order[:ntop]
    eps = {}
    noises = []
    for k in top:
        c1 = engine.get_context(task.model, task.cost_model, cfg, samples=1, precision="f32", sample_offset=int(k))
        n = c1.sample_noise(11, 3)
        eps[int(k)] = n[3][0]
        noises.append(tuple(a[0] for a in n))
    acc = np.zeros((T, m))
    for k in top:
        acc += w[k] * eps[int(k)]
    du_ref = acc / np.sqrt(dt)
    du = out.u_new - u_nom
    rest = max(0.0, float(w.sum() - w[top].sum()))  # weight outside `top`; |eps| <= 5.65 std (Box-Muller grid)
    scale = np.abs(du_ref).max()
    std = float(np.sqrt(np.max(np.diag(np.atleast_2d(cfg.sigma_d)))))
    # the kernel's weights are fp32 exponentials (~2e-7 relative each)
    assert np.abs(du - du_ref).max() <= 2e-6 * scale + 8.0 * rest * std / np.sqrt(dt), (ntop, rest)

    # G-float on the heavy samples: the float64 oracle on the regenerated noise
    spec = om.spec_from_plugins(task.model, task.cost_model, cfg)
    stack = tuple(np.stack([n[i] for n in noises]) for i in range(4))
    ref = om.mppi_iteration_oracle(spec, task.x0, u_nom, stack)
    o32 = om.mppi_iteration_oracle(spec, task.x0, u_nom, stack, np.float32)
    rel = np.abs(S[top] - ref["costs"]) / np.abs(ref["costs"])
    rel32 = np.abs(o32["costs"] - ref["costs"]) / np.abs(ref["costs"])
    assert np.all(rel <= np.maximum(1e-4, 2.0 * rel32.max())), (rel.max(), rel32.max())

    # determinism
    _, _, again = _run(task, cfg, K)
    assert np.array_equal(again.u_new, out.u_new) and np.array_equal(again.costs, S)

    # shard additivity: halves at global offsets 0 and K/2
    halves = [_run(task, cfg, K // 2, offset=o)[2] for o in (0, K // 2)]
    assert np.array_equal(np.concatenate([h.costs for h in halves]), S)  # same noise, same arithmetic per sample
    rho = min(h.diag.min_cost for h in halves)
    assert rho == out.diag.min_cost
    z = sum(h.diag.normaliser * np.exp(-(h.diag.min_cost - rho) / lam) for h in halves)
    assert z == pytest.approx(out.diag.normaliser, rel=2e-6)  # (fp32 exponentials relative to each launch's own rho)
    assert sum(h.diag.n_finite for h in halves) == out.diag.n_finite
    # and the merged update: Z-weighted combination of the halves' updates
    zs = [h.diag.normaliser * np.exp(-(h.diag.min_cost - rho) / lam) for h in halves]
    du_merged = sum(zi * (h.u_new - u_nom) for zi, h in zip(zs, halves)) / z
    assert np.abs(du_merged - du).max() <= 2e-6 * scale


@pytest.mark.parametrize("idx,K,T,process", [(1, 65536, 100, "bernoulli"), (3, 32768, 200, "bernoulli"),
                                             (3, 80000, 30, "poisson"), (1, 160000, 40, "poisson")])
def test_philox_and_hbm_kernels_agree_on_the_same_noise(idx, K, T, process, gpu_device):
    """The two product kernels against each other at BASELINE shapes: the device sampler's table of
    stream (seed, iteration) -- the very draws the Philox kernel makes in registers -- fed to the
    HBM kernel in the fp32 wire format gives the same per-sample costs bit for bit (the same
    arithmetic per sample; with c = 1 the eps'eps term the fed-noise kernel forms is multiplied by
    an exact 0) and the same update to the fp32 exponentials' rounding."""
    import dataclasses

    task, cfg = jb.baseline_config(idx, K=K, T=T)
    if process == "poisson":  # compound-Poisson arrival counts, at a rate where multi-arrival steps occur
        cfg = dataclasses.replace(cfg, nu=0.09 / cfg.dt, jump_process="poisson")
    seed, it = 5, 2
    u_nom = np.tile(np.atleast_1d(np.asarray(cfg.u_init, float)), (T, 1))
    cp = engine.get_context(task.model, task.cost_model, cfg, precision="f32")
    a = cp.iteration(task.x0, u_nom, seed, it, want_costs=True, want_weights=False)
    eps_d, ind, eps_j, eps_c = cp.sample_noise(seed, it)
    ch = engine.get_context(task.model, task.cost_model, cfg, precision="f32", hbm=True)
    assert "/hbm/" in ch.kernel_name() and "/philox/" in cp.kernel_name()
    jump = (ind != 0).astype(float)[..., None] * eps_j
    b = ch.iteration(task.x0, u_nom, seed, it, eps_c=ch.step_major(eps_c, cp.M), jump=ch.step_major(jump, cp.Q),
                     want_costs=True, want_weights=False)
    assert np.array_equal(a.costs, b.costs)
    assert a.diag.min_cost == b.diag.min_cost and a.diag.n_finite == b.diag.n_finite
    scale = np.abs(a.u_new - u_nom).max()
    assert np.abs(a.u_new - b.u_new).max() <= 2e-6 * scale


def test_philox_and_hbm_kernels_agree_control_channel_jumps(gpu_device):
    """The same cross-check on the reference's own (control-channel) jump model at a multi-wave shape:
    the quadrotor task's marks ride on eps_combined (noise.py:156-157), q = m = 4 -- the packed kernel's
    indexed mark staging with the marks added to the noise instead of the state."""
    import dataclasses

    from conftest import load_golden, plugins

    g = load_golden("r_quadrotor_task")
    s = g["spec"]
    K, T = 80000, 50
    model, cost, cfg = plugins(s, K=K, T=T)
    cfg = dataclasses.replace(cfg, nu=0.08 / s["dt"])
    u_nom = np.resize(g["u_nom"], (T, s["m"]))
    cp = engine.get_context(model, cost, cfg, precision="f32")
    assert cp.kernel_name().startswith("rollout_fast/philox/multi_wave/f32/spt2"), cp.kernel_name()
    a = cp.iteration(g["x0"], u_nom, 3, 1, want_costs=True, want_weights=False)
    eps_d, ind, eps_j, eps_c = cp.sample_noise(3, 1)
    assert 0.05 < (ind != 0).mean() < 0.11
    ch = engine.get_context(model, cost, cfg, precision="f32", hbm=True)
    b = ch.iteration(g["x0"], u_nom, 3, 1, eps_c=ch.step_major(eps_c, cp.M), want_costs=True, want_weights=False)
    assert np.array_equal(a.costs, b.costs)
    scale = np.abs(a.u_new - u_nom).max()
    assert np.abs(a.u_new - b.u_new).max() <= 2e-6 * scale
