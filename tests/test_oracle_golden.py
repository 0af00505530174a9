"""Pin the CPU oracle against vectors produced by the reference itself
(oracle/gen_golden.py) and against the Random123 Philox known answers.
CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_names, load_golden, oracle_spec, rel_err
from oracle import mppi as om
from oracle import philox_stream as ps

R_CASES = golden_names("r_")
B_CASES = golden_names("b_")


@pytest.mark.parametrize("name", R_CASES + B_CASES)
def test_oracle_reproduces_reference(name):
    g = load_golden(name)
    spec = oracle_spec(g["spec"])
    out = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], g["noise"], np.float64,
                                   mapping=g.get("mapping"), trace="states" in g)
    # control channel: same formulas in the same order as the batched reference;
    # state jumps: the reference per-rollout path scales marks/sqrt(dt)*sqrt(dt)
    # (a 1-ulp difference the unstable cartpole amplifies over T=100 steps)
    tol = 1e-12 if name.startswith("r_") else 1e-9
    assert rel_err(out["costs"], g["costs"]) <= tol
    assert np.allclose(out["weights"], g["weights"], rtol=tol, atol=1e-300, equal_nan=True)
    assert rel_err(out["u_new"], g["u_new"], floor=1e-12) <= tol
    assert out["min_cost"] == pytest.approx(float(g["min_cost"]), rel=tol)
    assert out["ess"] == pytest.approx(float(g["ess"]), rel=max(tol, 1e-12))
    assert np.allclose(out["norms"], g["norms"], rtol=max(tol, 1e-10), atol=1e-12, equal_nan=True)
    assert np.array_equal(out["diverged"], g["diverged"])
    if "states" in g:
        assert rel_err(out["states"], g["states"], floor=1e-9) <= max(tol, 1e-10)


@pytest.mark.parametrize("name", [n for n in R_CASES if not n.startswith("r_divergence")])
def test_sampler_restatement_is_bit_exact(name):
    g = load_golden(name)
    spec = oracle_spec(g["spec"])
    ed, ind, ej, ec = om.sample_noise_batch_ref(g["seed"], g["iteration"], spec)
    assert np.array_equal(ed, g["noise"][0])
    assert np.array_equal(ind, g["noise"][1])
    assert np.array_equal(ej, g["noise"][2])
    assert np.array_equal(ec, g["noise"][3])


def test_divergence_fixture_semantics():
    g = load_golden("r_divergence")
    assert g["diverged"][3] == 2 and g["diverged"][7] == 5
    assert g["weights"][3] == 0.0 and g["weights"][7] == 0.0
    # eps = 1e200: eps^2 overflows and 0 * inf = NaN in the c = 1 correction term
    # (costs.py:101,110) -- a non-finite cost with a finite state, weight 0
    assert np.isnan(g["costs"][11]) and g["diverged"][11] == -1 and g["weights"][11] == 0.0
    # the weighted noise sum multiplies the zero weights into the inf noise
    # entries (einsum, controller.py:78): NaN at those steps, as the reference does
    assert np.isnan(g["u_new"][[2, 5]]).all() and np.isfinite(np.delete(g["u_new"], [2, 5])).all()


KAT = [  # Random123 kat_vectors, philox4x32 10 rounds
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,expect", KAT)
def test_philox_known_answers(ctr, key, expect):
    out = ps.philox4x32_10(*ctr, *key)
    assert tuple(int(v) for v in out) == expect


def test_emulated_stream_contract():
    """nu = 0 / jumps disabled leave eps_d bit-identical (noise.py:114-115 contract);
    indicator frequency ~ nu dt; marks only at events."""
    L = np.array([[1.5]])
    a = ps.device_noise(7, 3, 256, 200, 1, 1, L, np.eye(1), [0.0], ps.jump_threshold(0.01))
    b = ps.device_noise(7, 3, 256, 200, 1, 1, L, np.eye(1), [0.0], 0)
    assert np.array_equal(a[0], b[0])
    p = a[1].mean()
    se = np.sqrt(0.01 * 0.99 / a[1].size)
    assert abs(p - 0.01) < 4 * se
    assert np.all(a[2][a[1] == 0] == 0.0) and np.all(a[2][a[1] == 1] != 0.0)
    # sample-offset shards reproduce the unsharded stream
    c = ps.device_noise(7, 3, 128, 200, 1, 1, L, np.eye(1), [0.0], ps.jump_threshold(0.01), sample_offset=128)
    assert np.array_equal(c[1], a[1][128:]) and np.allclose(c[0], a[0][128:])


def test_emulated_normals_moments():
    e = ps.device_noise(1, 0, 2048, 64, 4, 4, np.eye(4), np.eye(4), np.zeros(4), 0)[0].reshape(-1, 4)
    n = e.shape[0]
    cov = np.cov(e.T)
    assert np.all(np.abs(np.diag(cov) - 1.0) < 4 * np.sqrt(2.0 / n))
    off = cov[~np.eye(4, dtype=bool)]
    assert np.all(np.abs(off) < 4 * np.sqrt(1.0 / n))
    assert np.all(np.abs(e.mean(0)) < 4 / np.sqrt(n))


def test_f32_divergence_fixture_semantics():
    """r_divergence_f32: the same semantics with values float32 holds (the f32 kernels' divergence case)."""
    g = load_golden("r_divergence_f32")
    assert g["diverged"][3] == 2 and g["diverged"][7] == 5 and g["diverged"][11] == -1
    assert g["weights"][3] == 0.0 and g["weights"][7] == 0.0
    assert np.isfinite(g["costs"][11]) and g["costs"][11] > 1e30 and g["weights"][11] == 0.0
    assert np.float32(g["costs"][11]) < np.inf  # a finite float32 cost
    assert np.isnan(g["u_new"][[2, 5]]).all() and np.isfinite(np.delete(g["u_new"], [2, 5])).all()


def test_pitch_floor_fixture_reaches_both_signs():
    """r_quadrotor_pitch_floor drives |cos(pitch)| < 1e-6 with both signs (jm/dynamics.py:293, :361-363)."""
    g = load_golden("r_quadrotor_pitch_floor")
    cp = np.cos(g["states"][:, :-1, 7])
    band = np.abs(cp) < 1e-6
    assert band.mean() > 0.2 and (band & (cp > 0)).any() and (band & (cp < 0)).any()
    # the floor matters: without it the oracle's costs move far outside the parity tolerance
    spec = oracle_spec(g["spec"])
    out = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], g["noise"], np.float64)
    assert rel_err(out["costs"], g["costs"]) <= 1e-12
