"""Controller construction from experiment configs (jm/experiment.py:161-358).

The reference's own YAML files (pkg/configs/*.yaml) resolve through this
package's load_config / build_task / build_mppi_config / sweep_cells to the
same tasks, configs and sweep cells as through the reference's.  Runs where
/root/reference is mounted (the build container); skipped elsewhere.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg")
CONFIGS = sorted((REF / "configs").glob("*.yaml")) if REF.exists() else []

pytestmark = pytest.mark.skipif(not CONFIGS, reason="reference configs not mounted")


def _ref():
    src = str(REF / "src")
    if src not in sys.path:
        sys.path.insert(0, src)
    import jump_mppi.experiment as rexp

    return rexp


@pytest.mark.parametrize("path", CONFIGS, ids=lambda p: p.stem)
def test_yaml_configs_resolve_like_the_reference(path):
    import paper_1807_06108_b200 as jb

    rexp = _ref()
    ours, ref = jb.load_config(str(path)), rexp.load_config(str(path))
    assert jb.sweep_cells(ours) == rexp.sweep_cells(ref)
    assert jb.sweep_cells(ref) == rexp.sweep_cells(ref)  # a reference ExperimentConfig is accepted too
    for nu, sj, m in jb.sweep_cells(ours):
        a, b = jb.build_mppi_config(ours, nu=nu, sigma_j=sj, samples_m=m), rexp.build_mppi_config(ref, nu, sj, m)
        for f in ("lambda_", "c", "nu", "dt", "horizon_n", "samples_m", "jump_sampling_enabled"):
            assert getattr(a, f) == getattr(b, f), f
        for f in ("sigma_d", "sigma_j", "u_init"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
    ta, tb = jb.build_task(ours), rexp.build_task(ref)
    assert ta.name == tb.name and ta.duration_steps == tb.duration_steps
    assert ta.state_names == tb.state_names and ta.control_names == tb.control_names
    assert np.array_equal(ta.x0, tb.x0)
    lo_a, hi_a = ta.model.control_limits
    lo_b, hi_b = tb.model.control_limits
    assert np.array_equal(lo_a, lo_b) and np.array_equal(hi_a, hi_b)
    assert np.array_equal(ta.cost_model.control_cost_matrix, tb.cost_model.control_cost_matrix)
    assert ta.cost_model.lambda_ == tb.cost_model.lambda_ and ta.cost_model.c == tb.cost_model.c
    # model / cost parameters as the oracle reads them off either package's plugin objects
    from oracle import mppi as om

    cfg_b = rexp.build_mppi_config(ref)
    sa = om.spec_from_plugins(ta.model, ta.cost_model, jb.build_mppi_config(ours))
    sb = om.spec_from_plugins(tb.model, tb.cost_model, cfg_b)
    for f in ("model", "n", "m", "params", "jump_channel", "cost", "weights", "target", "terminal_scale",
              "cost_lambda", "cost_c"):
        assert getattr(sa, f) == getattr(sb, f), f
    assert np.array_equal(sa.R, sb.R)


def test_unknown_keys_and_tasks_are_fatal():
    import paper_1807_06108_b200 as jb

    with pytest.raises(jb.ExperimentConfigError):
        jb.config_from_dict({"task": "cartpole", "mppi": {"horizn": 10}})
    with pytest.raises(jb.ExperimentConfigError):
        jb.config_from_dict({"task": "pendulum"})
    with pytest.raises(jb.ExperimentConfigError):
        jb.config_from_dict({"task": "quadrotor", "variants": "newest"})
    e = jb.config_from_dict({"task": "quadrotor", "mppi": {"samples": 64}})
    assert jb.build_mppi_config(e).samples_m == 64
