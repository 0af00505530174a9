"""Generate tests/golden/csv/*.csv with the REFERENCE's own writers (jm/io.py:47-84).

TEST INFRASTRUCTURE ONLY.  Run in the build container (imports the read-only
reference from /root/reference/pkg/src; the files are committed):

    python -m oracle.gen_golden_csv

The records are seeded synthetic trials (tests/test_io.py builds the same ones
from the same seed), including values whose shortest round-trip form needs all
17 digits, negative zeros and integers stored as floats.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "csv"


def synthetic_records(n=3, steps=5, nx=4, m=1):
    """(states, controls, jump_indicators, success) per trial -- shared with tests/test_io.py."""
    rng = np.random.default_rng(1)
    out = []
    for k in range(n):
        states = rng.standard_normal((steps + 1, nx))
        controls = rng.standard_normal((steps, m))
        jumps = rng.integers(0, 2, steps)
        states[0, 0] = 1.0 / 3.0
        states[1, 1] = -0.0
        states[2, 2] = 3.0
        states[3, 3] = 1e-310  # subnormal
        controls[0, 0] = 0.1 + 0.2
        out.append((states, controls, jumps, bool(k % 2)))
    return out


SUMMARY = [("cartpole", "new", 0.25, 2.0, 1000, 8, 0.875, 12.5, 3.25, 42),
           ("cartpole", "old", 0.25, 2.0, 1000, 8, 0.5, 1.0 / 3.0, 3.5, 42),
           ("quadrotor", "new", 1.0, 0.1, 8192, 16, 1.0, 2.5e-7, 0.0484, 2**40 + 1)]


def main():
    sys.path.insert(0, str(REF))
    from jump_mppi import io as rio
    from jump_mppi.harness import TrialRecord

    OUT.mkdir(parents=True, exist_ok=True)
    recs = [TrialRecord("c", k, s, c, j, ok, np.zeros(len(c))) for k, (s, c, j, ok) in enumerate(synthetic_records())]
    rio.write_trajectory_csv(recs, str(OUT / "trajectory.csv"), ["x", "xd", "th", "thd"], ["F"], 0.02)
    rio.write_summary_csv([rio.SummaryRow(*r) for r in SUMMARY], str(OUT / "summary.csv"))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
