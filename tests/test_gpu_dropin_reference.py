"""The drop-in, proven with the reference's own objects.

baseline/_ref holds the unmodified reference package (jump_mppi, installed by
__graft_entry__.build(); it ships to the GPU box with the repo):

1. jump_mppi.experiment builds the cartpole and quadrotor tasks and configs
   from its own task defaults (config_from_dict + build_task /
   build_mppi_config, jm/experiment.py:161-215, :252-358);
2. paper_1807_06108_b200.mppi_iteration, called with the reference's
   ControllerState, DynamicsModel, CostModel and MppiConfig and fed the very
   noise table the reference draws (sample_noise_batch(RngStream(seed,
   iteration)), jm/controller.py:120-121), returns jump_mppi.mppi_iteration's
   update and diagnostics at the G-double tolerance (1e-9);
3. jump_mppi.harness.run_trial with its module-level mppi_iteration patched to
   ours (the INTEGRATION.md one-liner, jm/harness.py:21, :133) reproduces the
   unpatched trial's closed-loop trajectory, and runs end to end on our
   product path (device Philox, fp32).
"""

from __future__ import annotations

import dataclasses
import sys

import numpy as np
import pytest

import paper_1807_06108_b200 as jb
from conftest import ROOT, rel_err

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF / "jump_mppi" / "controller.py").exists():
        pytest.skip("baseline/_ref (the unmodified reference package) is not installed")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import jump_mppi

    assert str(REF) in jump_mppi.__file__
    return jump_mppi


def _task(ref, name, K, T):
    exp = ref.experiment.config_from_dict({"task": name, "mppi": {"samples": K, "horizon": T}})
    return ref.experiment.build_task(exp), ref.experiment.build_mppi_config(exp)


@pytest.mark.parametrize("name", ["cartpole", "quadrotor"])
def test_iteration_with_reference_objects_matches_reference(ref, name, gpu_device):
    task, cfg = _task(ref, name, K=512, T=50)
    ctrl0 = ref.controller.initial_controller_state(cfg)
    seed = 17
    x0 = np.asarray(task.x0, float)
    # a warm-started second iteration: a non-trivial nominal sequence, iteration index 1
    seq0, _ = ref.controller.mppi_iteration(ctrl0, task.model, task.cost_model, x0, master_seed=seed)
    ctrl = ref.controller.ControllerState(ref.controller.warm_start_shift(seq0, cfg.u_init), 1, cfg)
    seq_ref, diag_ref = ref.controller.mppi_iteration(ctrl, task.model, task.cost_model, x0, master_seed=seed)
    noise = ref.noise.sample_noise_batch(ref.noise.RngStream(seed, ctrl.iteration_index), cfg, cfg.samples_m)
    seq, diag = jb.mppi_iteration(ctrl, task.model, task.cost_model, x0, seed, noise=noise, precision="f64")
    assert rel_err(seq.controls, seq_ref.controls, floor=1e-9) <= 1e-9
    assert diag.min_cost == pytest.approx(diag_ref.min_cost, rel=1e-9)
    assert diag.effective_sample_size == pytest.approx(diag_ref.effective_sample_size, rel=1e-8)
    assert np.allclose(diag.weights, diag_ref.weights, rtol=1e-8, atol=1e-15)
    assert np.allclose(diag.per_step_update_norm, diag_ref.per_step_update_norm, rtol=1e-8, atol=1e-12)
    # the reference's own warm start of our sequence (controller.py:96-100) -- duck-typed value types
    sh = ref.controller.warm_start_shift(seq, cfg.u_init)
    assert np.array_equal(sh.controls[:-1], seq.controls[1:])
    # the product path (device Philox, fp32) on the same objects: a sane update of the same shape
    seq32, diag32 = jb.mppi_iteration(ctrl, task.model, task.cost_model, x0, seed)
    assert seq32.controls.shape == seq_ref.controls.shape and np.isfinite(seq32.controls).all()
    assert diag32.weights.sum() == pytest.approx(1.0, abs=1e-9)


def test_reference_run_trial_with_patched_mppi_iteration(ref, monkeypatch, gpu_device):
    task, cfg = _task(ref, "cartpole", K=256, T=30)
    task = dataclasses.replace(task, duration_steps=10)
    base = ref.harness.run_trial(task, cfg, seed=3)

    def ours_fed(ctrl, model, cost_model, x0, master_seed, mapping=None, return_rollouts=False):
        # our kernels on the reference's per-iteration noise table (f64): the trajectory must match
        c = ctrl.config
        noise = ref.noise.sample_noise_batch(ref.noise.RngStream(master_seed, ctrl.iteration_index), c, c.samples_m)
        return jb.mppi_iteration(ctrl, model, cost_model, x0, master_seed, mapping=mapping,
                                 return_rollouts=return_rollouts, noise=noise, precision="f64")

    monkeypatch.setattr(ref.harness, "mppi_iteration", ours_fed)
    rec = ref.harness.run_trial(task, cfg, seed=3)
    assert np.array_equal(rec.jump_indicators, base.jump_indicators)  # the plant's own stream
    assert np.allclose(rec.states, base.states, rtol=1e-8, atol=1e-10)
    assert np.allclose(rec.controls, base.controls, rtol=1e-8, atol=1e-10)
    # the INTEGRATION.md patch itself: the product path inside the reference's loop
    monkeypatch.setattr(ref.harness, "mppi_iteration", jb.mppi_iteration)
    rec2 = ref.harness.run_trial(task, cfg, seed=3)
    assert rec2.states.shape == base.states.shape and np.isfinite(rec2.states).all()
    assert np.array_equal(rec2.jump_indicators, base.jump_indicators)
