"""Edge shapes and jump rates of the on-device (Philox) path against the oracle.

Each case runs one fp64 iteration on the GPU and the oracle (oracle/mppi.py,
restating jm/controller.py:103-181) fed the very noise table the device
sampler exports for the same (seed, iteration) -- so the cases pin the
rollout kernels' own noise consumption (jump clocks, cooperative jump
windows, warp-specialised and multi-wave launch shapes, ragged tiles, short
and long horizons) to the reference algorithm at the G-double tolerance.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

import paper_1807_06108_b200 as jb
from conftest import load_golden, oracle_spec, plugins, rel_err
from oracle import mppi as om

pytestmark = pytest.mark.gpu
G_DOUBLE = 1e-9


def _case(name, K, T, seed=11, iteration=3, **cfg_changes):
    g = load_golden(name)
    s = g["spec"]
    model, cost, cfg = plugins(s, K=K, T=T)
    if cfg_changes:
        cfg = dataclasses.replace(cfg, **cfg_changes)
    rng = np.random.default_rng(K * 1000 + T)
    u_nom = 0.3 * rng.standard_normal((T, s["m"]))
    ctrl = jb.ControllerState(jb.ControlSequence(u_nom, s["dt"]), iteration, cfg)
    seq, diag = jb.mppi_iteration(ctrl, model, cost, g["x0"], seed, precision="f64")
    noise = jb.sample_noise_batch(jb.RngStream(seed, iteration), cfg, K, model=model, precision="f64")
    out = om.mppi_iteration_oracle(oracle_spec(s), g["x0"], u_nom, noise, np.float64)
    return seq, diag, out, noise


def _check(seq, diag, out):
    assert rel_err(seq.controls, out["u_new"], floor=1e-9) <= G_DOUBLE
    assert np.allclose(diag.weights, out["weights"], rtol=1e-8, atol=1e-14)
    assert diag.min_cost == pytest.approx(out["min_cost"], rel=G_DOUBLE)


@pytest.mark.parametrize("name", ["b_cartpole", "r_cartpole_task", "b_quadrotor"])
def test_near_limit_jump_rate(name, gpu_device):
    """nu*dt just under the zero-one-law limit (0.1): ~75 events per warp and
    window, several cooperative generation rounds per window."""
    g = load_golden(name)
    dt = g["spec"]["dt"]
    seq, diag, out, noise = _case(name, 500, 60, nu=0.099 / dt, jump_sampling_enabled=True)
    assert noise[1].mean() == pytest.approx(0.099, abs=0.01)
    _check(seq, diag, out)


@pytest.mark.parametrize("name,K,T", [("b_cartpole", 64, 500), ("r_quadrotor_task", 40, 300)])
def test_long_horizon(name, K, T, gpu_device):
    _check(*_case(name, K, T)[:3])


@pytest.mark.parametrize("K,T", [(1, 1), (33, 3), (31, 5), (97, 9)])
def test_tiny_and_ragged_shapes(K, T, gpu_device):
    _check(*_case("b_cartpole", K, T)[:3])


def test_multi_wave_shape(gpu_device):
    """K > 148 x 512: 256-sample tiles, grid-strided, global eps slab."""
    _check(*_case("b_cartpole", 148 * 512 + 1000, 12)[:3])


def test_dropin_entry_equals_general_path(gpu_device):
    """jm_iteration_dropin (the Python API's fast path) vs jm_iteration_host's
    general path on the same (seed, iteration): identical kernels, identical bits."""
    from paper_1807_06108_b200 import engine

    g = load_golden("b_cartpole")
    s = g["spec"]
    model, cost, cfg = plugins(s, K=2000, T=50)
    ctx = engine.get_context(model, cost, cfg, precision="f32")
    u_nom = 0.2 * np.random.default_rng(5).standard_normal((50, 1))
    ui = np.zeros(1)
    u_new, norms, (mc, ess, z, nf), u_shift, h = ctx.iteration_dropin(g["x0"], u_nom, 7, 2, ui)
    ctx.stash_release(h)
    ref = ctx.iteration(g["x0"], u_nom, 7, 2, want_weights=True, u_init=ui)
    assert np.array_equal(u_new, ref.u_new) and np.array_equal(u_shift, ref.u_shift)
    assert np.array_equal(norms, ref.norms)
    assert (mc, ess, z, nf) == (ref.diag.min_cost, ref.diag.ess, ref.diag.normaliser, ref.diag.n_finite)


def test_noise_wire_file_replays_the_device_stream(gpu_device, tmp_path):
    """Device noise -> wire-format file -> fed (HBM-mode) iteration == the in-register Philox iteration."""
    from paper_1807_06108_b200 import io as jio

    g = load_golden("b_cartpole")
    s = g["spec"]
    model, cost, cfg = plugins(s, K=777, T=20)
    u_nom = 0.3 * np.random.default_rng(4).standard_normal((20, 1))
    ctrl = jb.ControllerState(jb.ControlSequence(u_nom, s["dt"]), 6, cfg)
    a, _ = jb.mppi_iteration(ctrl, model, cost, g["x0"], 21, precision="f64")
    noise = jb.sample_noise_batch(jb.RngStream(21, 6), cfg, 777, model=model, precision="f64")
    p = tmp_path / "noise.bin"
    jio.save_noise(str(p), noise, "state", seed=21, iteration=6)
    _, ec, jw = jio.load_noise(str(p))
    b, _ = jb.mppi_iteration(ctrl, model, cost, g["x0"], 21, noise=jio.from_wire(ec, jw), precision="f64")
    # the file holds fp32 values: agreement to fp32 resolution of the noise
    assert rel_err(b.controls, a.controls, floor=1e-3) <= 1e-5


def test_mark_table_overflow_path(gpu_device):
    """jump_window_idx's halve-and-redo path (csrc/rollout_fast.cuh): with JM_JW_NOCAP=1 the windows ignore
    the rate, a warp's window overflows its 255-entry mark table, and the results must not change --
    tests/_overflow_worker.py checks the fp64 kernel against the oracle and the packed fp32 kernel
    against the HBM kernel.  (A subprocess: the switch is read once per process.)"""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("JM_WS", "JM_SPT", "JM_NO_EPS_SMEM", "JM_JW")}
    env.update(JM_JW_NOCAP="1", PYTHONPATH=f"{root}{os.pathsep}{root / 'tests'}")  # (the default kernel choice)
    r = subprocess.run([sys.executable, str(root / "tests" / "_overflow_worker.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "overflow path ok" in r.stdout
