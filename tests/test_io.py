"""Result files and the noise wire format (reference jump_mppi/io.py)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1807_06108_b200 import io as jio
from paper_1807_06108_b200.harness import TrialRecord


def _records(n=3, steps=5, nx=4, m=1):
    rng = np.random.default_rng(1)
    return [TrialRecord("c", k, rng.standard_normal((steps + 1, nx)), rng.standard_normal((steps, m)),
                        rng.integers(0, 2, steps), bool(k % 2), np.zeros(steps)) for k in range(n)]


def test_trajectory_csv_round_trip_and_layout(tmp_path):
    recs = _records()
    p = tmp_path / "traj.csv"
    jio.write_trajectory_csv(recs, str(p), ["x", "xd", "th", "thd"], ["F"], 0.02)
    head = p.read_text().splitlines()[0]
    assert head == "trial,step,t,x,xd,th,thd,F,jump_indicator"  # io.py:62-63 column order
    cols = jio.read_trajectory_csv(str(p))
    assert cols["trial"].size == 15
    got = np.stack([cols[c] for c in ("x", "xd", "th", "thd")], 1).reshape(3, 5, 4)
    assert np.array_equal(got, np.stack([r.states[:5] for r in recs]))  # 17 digits: exact
    assert np.array_equal(cols["t"][:5], np.arange(5) * 0.02)
    q = tmp_path / "traj2.csv"
    jio.write_trajectory_csv(recs, str(q), ["x", "xd", "th", "thd"], ["F"], 0.02)
    assert p.read_bytes() == q.read_bytes()  # deterministic bytes


def test_csv_bytes_equal_the_reference_writers(tmp_path):
    """tests/golden/csv/*.csv were written by the reference's own jm/io.py:47-84 (oracle/gen_golden_csv.py,
    run in the build container) from these seeded records: this package's writers give the same bytes."""
    from pathlib import Path

    from oracle.gen_golden_csv import SUMMARY, synthetic_records

    gold = Path(__file__).parent / "golden" / "csv"
    recs = [TrialRecord("c", k, s, c, j, ok, np.zeros(len(c))) for k, (s, c, j, ok) in enumerate(synthetic_records())]
    p = tmp_path / "trajectory.csv"
    jio.write_trajectory_csv(recs, str(p), ["x", "xd", "th", "thd"], ["F"], 0.02)
    assert p.read_bytes() == (gold / "trajectory.csv").read_bytes()
    q = tmp_path / "summary.csv"
    jio.write_summary_csv([jio.SummaryRow(*r) for r in SUMMARY], str(q))
    assert q.read_bytes() == (gold / "summary.csv").read_bytes()
    # and this package's readers parse the reference's files exactly
    cols = jio.read_trajectory_csv(str(gold / "trajectory.csv"))
    assert np.array_equal(cols["x"].reshape(3, 5), np.stack([r.states[:5, 0] for r in recs]))
    back = jio.read_summary_csv(str(gold / "summary.csv"))
    assert back[2]["seed"] == 2**40 + 1 and back[1]["total_variance"] == 1.0 / 3.0


def test_summary_csv_round_trip(tmp_path):
    rows = [jio.SummaryRow("cartpole", "new", 0.25, 2.0, 1000, 8, 0.875, 12.5, 3.25, 42),
            jio.SummaryRow("cartpole", "old", 0.25, 2.0, 1000, 8, 0.5, 1.0 / 3.0, 3.5, 42)]
    p = tmp_path / "s.csv"
    jio.write_summary_csv(rows, str(p))
    back = jio.read_summary_csv(str(p))
    assert back[1]["total_variance"] == 1.0 / 3.0 and back[0]["trials"] == 8 and back[0]["variant"] == "new"


@pytest.mark.parametrize("channel", ["control", "state"])
def test_noise_wire_format_round_trip(tmp_path, channel):
    rng = np.random.default_rng(2)
    K, T, m, q = 7, 5, 2, 3 if channel == "state" else 2
    eps_d = rng.standard_normal((K, T, m))
    ind = (rng.random((K, T)) < 0.3).astype(np.int64)
    eps_j = rng.standard_normal((K, T, q)) * ind[..., None]
    eps_c = eps_d + eps_j if channel == "control" else eps_d
    p = tmp_path / "noise.bin"
    jio.save_noise(str(p), (eps_d, ind, eps_j, eps_c), channel, seed=3)
    head, ec, jw = jio.load_noise(str(p))
    assert head["seed"] == 3 and ec.shape == (T, m, K) and ec.dtype == np.float32
    assert np.array_equal(ec, np.transpose(eps_c, (1, 2, 0)).astype(np.float32))
    if channel == "state":
        assert np.array_equal(jw, np.transpose(ind[..., None] * eps_j, (1, 2, 0)).astype(np.float32))
        d, i2, j2, c2 = jio.from_wire(ec, jw)
        assert np.array_equal(i2, ind) and np.allclose(j2, ind[..., None] * eps_j, atol=1e-6)
    else:
        assert jw is None


def test_control_cost_matrix_from_dynamics_matches_reference_formula():
    """costs.py:59-77 on this package's models: R = lambda G'(BB')^+ G with B = G."""
    import paper_1807_06108_b200 as jb

    cp = jb.cartpole_dynamics()
    x = np.array([0.1, -0.2, 2.9, 0.4])
    g = cp.control_matrix(x)
    # reference expressions (dynamics.py:221-228)
    den = 1.0 + 0.1 * np.sin(2.9) ** 2
    assert np.allclose(g[:, 0], [0.0, 1.0 / den, 0.0, -np.cos(2.9) / (0.5 * den)])
    r = jb.control_cost_matrix_from_dynamics(cp, x, 0.0, 2.5)
    assert r.shape == (1, 1) and r[0, 0] == pytest.approx(2.5)  # full column rank G: G'(GG')^+G = I
    q = jb.quadrotor_dynamics()
    xq = np.array([0, 0, 0, 0, 0, 0, 0.1, -0.2, 0.3, 0, 0, 0.0])
    rq = jb.control_cost_matrix_from_dynamics(q, xq, 0.0, 1.0)
    assert np.allclose(rq, np.eye(4), atol=1e-9)
