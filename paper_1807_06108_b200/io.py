"""Result files and the noise wire format.

* CSV outputs with the reference's layout (jump_mppi/io.py): a summary table
  (io.py:18-59) and per-step trajectories (io.py:62-84), reals written with
  17 significant digits (exact IEEE-double round trip) in a fixed row order,
  so equal inputs give byte-identical files.  The trajectories come from the
  device-resident loop histories (run_trial / run_batch records).
* The noise wire format: the step-major fp32 tensors the HBM-mode rollout
  kernels read (eps_combined (T, m, K) and, for state-space jumps, the dense
  indicator x mark tensor (T, q, K)), stored as one file -- a JSON header line
  then the raw little-endian arrays -- so a noise table can be generated once
  (on the GPU or by the reference) and replayed through mppi_iteration(noise=...)
  or the HBM bench.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

SUMMARY_COLUMNS = ("task", "variant", "nu", "sigma_j", "samples_m", "trials",
                   "success_rate", "total_variance", "mean_iter_ms", "seed")


@dataclass(frozen=True)
class SummaryRow:
    """One row of the summary table (io.py:24-35)."""

    task: str
    variant: str
    nu: float
    sigma_j: float
    samples_m: int
    trials: int
    success_rate: float
    total_variance: float
    mean_iter_ms: float
    seed: int


def fmt(value) -> str:
    """Integers and booleans as integers, reals with 17 significant digits."""
    if isinstance(value, (bool, np.bool_, int, np.integer)):
        return str(int(value))
    return format(float(value), ".17g")


def write_summary_csv(rows: Sequence[SummaryRow], path: str) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(SUMMARY_COLUMNS)
        for r in rows:
            w.writerow([r.task, r.variant] + [fmt(getattr(r, c)) for c in SUMMARY_COLUMNS[2:]])


def read_summary_csv(path: str) -> List[Dict]:
    kinds = {"task": str, "variant": str, "samples_m": int, "trials": int, "seed": int}
    with open(path, "r", newline="") as fh:
        return [{k: kinds.get(k, float)(v) for k, v in row.items()} for row in csv.DictReader(fh)]


def trajectory_columns(state_names: Sequence[str], control_names: Sequence[str]) -> Tuple[str, ...]:
    return ("trial", "step", "t", *state_names, *control_names, "jump_indicator")


def write_trajectory_csv(records, path: str, state_names: Sequence[str], control_names: Sequence[str],
                         dt: float) -> None:
    """One row per executed control step: the state at the start of the step,
    the applied control and the plant's jump indicator (io.py:66-84)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(trajectory_columns(state_names, control_names))
        for trial, rec in enumerate(records):
            for k in range(rec.controls.shape[0]):
                w.writerow([str(trial), str(k), fmt(k * dt)] + [fmt(v) for v in rec.states[k]]
                           + [fmt(v) for v in rec.controls[k]] + [str(int(rec.jump_indicators[k]))])


def read_trajectory_csv(path: str) -> Dict[str, np.ndarray]:
    with open(path, "r", newline="") as fh:
        rows = list(csv.reader(fh))
    header, body = rows[0], rows[1:]
    data = np.array(body, dtype=float).reshape(len(body), len(header))
    return {name: data[:, i] for i, name in enumerate(header)}


# ---------------------------------------------------------------- noise wire format
_MAGIC = "jmppi-noise-v1"


def to_wire(noise, jump_channel: str = "control") -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """(eps_d, ind, eps_j, eps_c) sample-major (K, T, .) -> the step-major fp32
    tensors of the HBM kernels: eps_c (T, m, K) and, for state-space jumps,
    ind x mark (T, q, K)."""
    eps_d, ind, eps_j, eps_c = (np.asarray(a) for a in noise)
    ec = np.ascontiguousarray(np.transpose(np.asarray(eps_c, np.float64), (1, 2, 0)), dtype=np.float32)
    if jump_channel != "state":
        return ec, None
    jm = np.asarray(ind, np.float64)[..., None] * np.asarray(eps_j, np.float64)
    return ec, np.ascontiguousarray(np.transpose(jm, (1, 2, 0)), dtype=np.float32)


def save_noise(path: str, noise, jump_channel: str = "control", **meta) -> None:
    """Write a noise table in the wire format (JSON header line, then raw arrays)."""
    ec, jw = to_wire(noise, jump_channel)
    head = dict(format=_MAGIC, jump_channel=jump_channel, eps_shape=list(ec.shape),
                jump_shape=None if jw is None else list(jw.shape), dtype="<f4", **meta)
    with open(path, "wb") as fh:
        fh.write((json.dumps(head, sort_keys=True) + "\n").encode())
        fh.write(ec.astype("<f4").tobytes())
        if jw is not None:
            fh.write(jw.astype("<f4").tobytes())


def load_noise(path: str):
    """(header, eps_c (T, m, K), jump (T, q, K) or None) of a wire-format file."""
    with open(path, "rb") as fh:
        head = json.loads(fh.readline().decode())
        if head.get("format") != _MAGIC:
            raise ValueError(f"{path}: not a {_MAGIC} file")
        ec = np.frombuffer(fh.read(4 * int(np.prod(head["eps_shape"]))), dtype="<f4").reshape(head["eps_shape"])
        jw = None
        if head["jump_shape"] is not None:
            jw = np.frombuffer(fh.read(4 * int(np.prod(head["jump_shape"]))), dtype="<f4").reshape(head["jump_shape"])
    return head, ec, jw


def from_wire(eps_c_sm: np.ndarray, jump_sm: Optional[np.ndarray] = None):
    """Step-major wire tensors -> a (eps_d, ind, eps_j, eps_c) table for
    mppi_iteration(noise=...): the control-channel table carries eps_c only
    (eps_d = eps_c, no jumps); the state-jump table marks ind = (jump != 0)
    and eps_j = the jump rows (the indicator x mark product the kernels use)."""
    ec = np.transpose(np.asarray(eps_c_sm, np.float64), (2, 0, 1))
    K, T, _ = ec.shape
    if jump_sm is None:
        return ec.copy(), np.zeros((K, T), np.int64), np.zeros_like(ec), ec
    jm = np.transpose(np.asarray(jump_sm, np.float64), (2, 0, 1))
    ind = np.any(jm != 0.0, axis=2).astype(np.int64)
    return ec.copy(), ind, jm, ec
