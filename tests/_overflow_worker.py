"""Worker of test_gpu_edges.test_mark_table_overflow_path (run with JM_JW_NOCAP=1 in the environment).

Quadrotor at nu dt = 0.09 with jump windows as long as shared memory allows: a warp's window holds
more (thread, step) events (32 x 0.09 x 100 = 288 expected) than its 255-entry mark table, so jump_window_idx halves the window and
redoes it from the saved clocks.  Checks (a) the fp64 Philox iteration of the single-wave kernel
against the oracle fed the device sampler's table of the same stream, (b) the packed fp32
multi-wave kernel's per-sample costs against the HBM kernel fed that table, bit for bit.
"""
import dataclasses
import sys

import numpy as np

import paper_1807_06108_b200 as jb
from oracle import mppi as om
from paper_1807_06108_b200 import engine


def main():
    task, cfg = jb.baseline_config(2, K=32768, T=100)
    cfg = dataclasses.replace(cfg, nu=0.09 / cfg.dt)
    u_nom = np.tile(np.atleast_1d(np.asarray(cfg.u_init, float)), (cfg.horizon_n, 1))
    # (a) fp64, single wave (one sample per thread)
    c64 = engine.get_context(task.model, task.cost_model, cfg, precision="f64")
    assert c64.kernel_name().startswith("rollout_fast/philox/single_wave/f64"), c64.kernel_name()
    out = c64.iteration(task.x0, u_nom, 7, 1, want_costs=True, want_weights=False)
    noise = c64.sample_noise(7, 1)
    assert 0.085 < (noise[1] != 0).mean() < 0.095
    spec = om.spec_from_plugins(task.model, task.cost_model, cfg)
    ref = om.mppi_iteration_oracle(spec, task.x0, u_nom, noise)
    fin = np.isfinite(ref["costs"])
    rel = np.abs(out.costs[fin] - ref["costs"][fin]) / np.abs(ref["costs"][fin])
    # (a handful of the 32768 samples tumble through |cos(pitch)| ~ 0 late in the horizon, where
    # q / cos(pitch) amplifies the last bit of either evaluation; they are the same samples at any
    # jump rate and window length)
    assert np.mean(rel <= 1e-9) >= 0.999 and rel.max() <= 1e-3, (np.mean(rel <= 1e-9), rel.max())
    assert np.abs(out.u_new - ref["u_new"]).max() <= 1e-9 * max(1.0, np.abs(ref["u_new"]).max())
    # (b) fp32 packed pairs, multi-wave, against the HBM kernel on the same table
    K2 = 80000
    task2, cfg2 = jb.baseline_config(2, K=K2, T=100)
    cfg2 = dataclasses.replace(cfg2, nu=0.09 / cfg2.dt)
    cp = engine.get_context(task2.model, task2.cost_model, cfg2, precision="f32")
    assert cp.kernel_name().startswith("rollout_fast/philox/multi_wave/f32/spt2"), cp.kernel_name()
    a = cp.iteration(task2.x0, u_nom, 9, 4, want_costs=True, want_weights=False)
    eps_d, ind, eps_j, eps_c = cp.sample_noise(9, 4)
    ch = engine.get_context(task2.model, task2.cost_model, cfg2, precision="f32", hbm=True)
    jump = (ind != 0).astype(float)[..., None] * eps_j
    b = ch.iteration(task2.x0, u_nom, 9, 4, eps_c=ch.step_major(eps_c, cp.M), jump=ch.step_major(jump, cp.Q),
                     want_costs=True, want_weights=False)
    assert np.array_equal(a.costs, b.costs)
    print("overflow path ok", float(rel.max()))


if __name__ == "__main__":
    sys.exit(main())
