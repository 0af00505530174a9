"""f32 parity gate of the kernels the bench times (SURVEY 8(c) G-float, G-stat).

The golden-vector gate (test_gpu_parity.py) runs the fed-noise TRACE kernel at
small K.  Here the *non-trace* product kernels -- the ones `bench.py` launches
for BASELINE configs 0-3 (warp-specialised, single-wave, multi-wave, HBM) --
run at their BASELINE shapes; `jm_kernel_name` names the variant, asserted
below, and the context is the very one bench.py builds (same engine cache key).

G-float (per config): the kernel draws its noise in registers (Philox); the
same stream's table, exported by the device sampler (bit-identical draws, the
same fp32 Cholesky product), is fed to the oracle (oracle/mppi.py, the
restatement of jm/controller.py:103-181 pinned to the reference's golden
vectors) in float64 and float32:
  * per-sample cost rel err <= max(1e-4, 2 x the float32 restatement's own error)
    for every sample with weight > 1e-12, and <= 1e-4 for >= 98% of samples
    (or the restatement's own fraction);
  * normwise update error ||du_gpu - du_ref|| / ||du_ref|| <= max(1e-4, 2 x the
    float32 restatement's error).
G-stat: over 24 seeds, the f32 device-Philox control update and the float64
oracle on numpy-Philox noise (the reference's own sampler, jm/noise.py:129-161)
agree per (t, j) within sampling error -- the reference's own statistical
test style (tests/test_controller.py:268-288, tests/test_noise.py:30-66).
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import paper_1807_06108_b200 as jb
from conftest import normwise
from oracle import mppi as om
from paper_1807_06108_b200 import engine

pytestmark = pytest.mark.gpu

# (case, BASELINE config index, K, T, kernel variant the bench launches at this shape)
CASES = [
    ("cfg0", 0, 1024, 100, "rollout_kernel_ws/philox/ws/f32"),
    ("cfg1", 1, 65536, 100, "rollout_fast/philox/single_wave/f32"),
    ("cfg2", 2, 8192, 150, "rollout_kernel_ws/philox/ws/f32"),
    # cfg3's kernel (quadrotor, T=200) at a multi-wave K that the oracle finishes in ~1 min
    ("cfg3_multiwave", 3, 80000, 200, "rollout_fast/philox/multi_wave/f32"),
    ("cartpole_multiwave", 1, 200000, 100, "rollout_fast/philox/multi_wave/f32"),
]


def _report(case, **kv):
    path = os.environ.get("JM_GATE_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"case": case, **kv}) + "\n")


def _nominal(cfg, T):
    """The BASELINE nominal (u_init) plus a slow sinusoid on every input, small
    enough to keep the system in its operating regime (0.5 N on the cart, 0.01
    on the quadrotor's thrust and torques: larger torques tumble it, where fp32
    and fp64 trajectories part chaotically whatever the implementation)."""
    m = cfg.control_dim
    t = np.arange(T)[:, None]
    amp = 0.5 if m == 1 else 0.01
    return np.tile(np.asarray(cfg.u_init, float), (T, 1)) + amp * np.sin(0.07 * t + np.arange(m)[None, :])


def g_float(case, costs, u_new, spec, x0, u_nom, noise):
    ref = om.mppi_iteration_oracle(spec, x0, u_nom, noise, np.float64)
    o32 = om.mppi_iteration_oracle(spec, x0, u_nom, noise, np.float32)
    rc = ref["costs"]
    fin = np.isfinite(rc)
    rel = np.full(rc.shape, np.inf)
    ok = fin & np.isfinite(costs)
    rel[ok] = np.abs(costs[ok] - rc[ok]) / np.maximum(np.abs(rc[ok]), 1e-30)
    rel[~fin & ~np.isfinite(costs)] = 0.0
    heavy = ref["weights"] > 1e-12
    rel32 = np.abs(o32["costs"] - rc) / np.maximum(np.abs(rc), 1e-30)
    floor_heavy = float(np.nanmax(rel32[heavy & fin])) if (heavy & fin).any() else 0.0
    frac_ok, frac_ok32 = float(np.mean(rel <= 1e-4)), float(np.mean(rel32[fin] <= 1e-4))
    dref = ref["u_new"] - u_nom
    err_gpu = normwise(u_new - u_nom, dref)
    err_np32 = normwise(o32["u_new"] - u_nom, dref)
    _report(case, heavy_cost_err=float(rel[heavy].max()), heavy_cost_err_numpy_f32=floor_heavy,
            frac_cost_le_1e4=frac_ok, frac_cost_le_1e4_numpy_f32=frac_ok32, update_err=err_gpu,
            update_err_numpy_f32=err_np32, min_cost_ref=ref["min_cost"], ess_ref=ref["ess"], n_heavy=int(heavy.sum()))
    assert np.all(rel[heavy] <= max(1e-4, 2.0 * floor_heavy)), (
        f"{case}: heavy-sample cost error {rel[heavy].max():.3g} (numpy f32 {floor_heavy:.3g})")
    assert frac_ok >= min(0.98, frac_ok32 - 0.01), f"{case}: {frac_ok:.4f} of costs within 1e-4"
    assert err_gpu <= max(1e-4, 2.0 * err_np32), f"{case}: update error {err_gpu:.3g} (numpy f32 {err_np32:.3g})"
    ref["cost_tol"] = max(1e-4, 2.0 * floor_heavy)
    return ref


@pytest.mark.parametrize("case,idx,K,T,variant", CASES, ids=[c[0] for c in CASES])
def test_benchmarked_philox_kernel_f32_gate(case, idx, K, T, variant, gpu_device):
    task, cfg = jb.baseline_config(idx, K=K, T=T)
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision="f32")  # the bench's context
    assert ctx.kernel_name().startswith(variant), ctx.kernel_name()
    x0 = np.asarray(task.x0, float)  # the BASELINE start state (cartpole upright, quadrotor at the origin)
    u_nom = _nominal(cfg, T)
    seed, it = 11, 3
    out = ctx.iteration(x0, u_nom, seed, it, want_costs=True, want_weights=False)  # non-trace kernel
    noise = ctx.sample_noise(seed, it)  # the same stream's draws
    spec = om.spec_from_plugins(task.model, task.cost_model, cfg)
    ref = g_float(case, out.costs, out.u_new, spec, x0, u_nom, noise)
    assert out.diag.min_cost == pytest.approx(ref["min_cost"], rel=ref["cost_tol"])
    # the drop-in call (graph fast path, same kernel) returns the same update bit for bit
    seq, _ = jb.mppi_iteration(jb.ControllerState(jb.ControlSequence(u_nom, cfg.dt), it, cfg), task.model,
                               task.cost_model, x0, seed, precision="f32")
    assert np.array_equal(seq.controls, out.u_new)


HBM_CASES = [
    ("hbm_cartpole", 1, 300000, 100, "rollout_fast/hbm/multi_wave/f32"),
    ("hbm_quadrotor", 2, 20000, 150, "rollout_fast/hbm/single_wave/f32"),
]


@pytest.mark.parametrize("case,idx,K,T,variant", HBM_CASES, ids=[c[0] for c in HBM_CASES])
def test_benchmarked_hbm_kernel_f32_gate(case, idx, K, T, variant, gpu_device):
    """The noise-from-HBM non-trace kernel (bench --noise hbm) fed the device sampler's tensors."""
    task, cfg = jb.baseline_config(idx, K=K, T=T)
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision="f32", hbm=True)
    assert ctx.kernel_name().startswith(variant), ctx.kernel_name()
    philox = engine.get_context(task.model, task.cost_model, cfg, precision="f32")
    noise = philox.sample_noise(5, 1)
    eps_d, ind, eps_j, eps_c = noise
    x0 = np.asarray(task.x0, float)
    u_nom = _nominal(cfg, T)
    q = ctx.Q
    jump = (ind != 0).astype(float)[..., None] * eps_j
    out = ctx.iteration(x0, u_nom, 5, 1, eps_c=ctx.step_major(eps_c, cfg.control_dim), jump=ctx.step_major(jump, q),
                        want_costs=True, want_weights=False)
    spec = om.spec_from_plugins(task.model, task.cost_model, cfg)
    g_float(case, out.costs, out.u_new, spec, x0, u_nom, noise)
    # fed the same draws, the HBM kernel computes the Philox kernel's costs bit for bit:
    # the in-register normals (packed Box-Muller for sample pairs) equal the sampler's
    # scalar ones, and the sparse epilogue's regenerated eps equal the fed columns
    po = philox.iteration(x0, u_nom, 5, 1, want_costs=True, want_weights=False)
    if ctx.kernel_name().split("/")[-1] == philox.kernel_name().split("/")[-1]:  # same samples per thread
        assert np.array_equal(out.costs, po.costs)
        if philox.kernel_name().split("/")[2] == "single_wave" == ctx.kernel_name().split("/")[2]:
            assert np.array_equal(out.u_new, po.u_new)  # same tiles: the same records, merged alike
    else:  # one sample per thread vs packed pairs: the compiler contracts the scalar code its own way
        assert np.allclose(out.costs, po.costs, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("case,idx,K,T", [("cfg0", 0, 1024, 100), ("cfg2", 2, 8192, 150)])
def test_f32_control_statistics_over_seeds_match_oracle(case, idx, K, T, gpu_device):
    """G-stat at the BASELINE shapes in f32: device Philox vs numpy Philox over 24 seeds."""
    task, cfg = jb.baseline_config(idx, K=K, T=T)
    spec = om.spec_from_plugins(task.model, task.cost_model, cfg)
    u_nom = np.tile(np.asarray(cfg.u_init, float), (T, 1))
    gpu, ref = [], []
    for seed in range(24):
        seq, _ = jb.mppi_iteration(jb.initial_controller_state(cfg), task.model, task.cost_model, task.x0, seed,
                                   precision="f32")
        gpu.append(seq.controls - u_nom)
        noise = om.sample_noise_batch_ref(seed, 0, spec)
        ref.append(om.mppi_iteration_oracle(spec, task.x0, u_nom, noise)["u_new"] - u_nom)
    gpu, ref = np.array(gpu), np.array(ref)
    se = np.sqrt(gpu.var(0, ddof=1) / len(gpu) + ref.var(0, ddof=1) / len(ref))
    z = np.abs(gpu.mean(0) - ref.mean(0)) / np.maximum(se, 1e-300)
    _report(f"gstat_{case}", frac_z_lt_3=float(np.mean(z < 3.0)), z_max=float(z.max()))
    assert np.mean(z < 3.0) >= 0.9 and z.max() < 5.0
