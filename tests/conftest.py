"""Shared test helpers.

`-m "not gpu"` runs here (no GPU): oracle vs golden vectors, host logic, the
C-ABI library's exports.  `-m gpu` runs on a B200 through gpurun: parity of
the CUDA path against the oracle / golden vectors, through the C ABI.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libjmppi.so")
    config.addinivalue_line("markers", "slow: long-running")


def golden_names(prefix=""):
    return sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz"))


def load_golden(name):
    z = np.load(GOLDEN / f"{name}.npz")
    g = {k: z[k] for k in z.files}
    g["spec"] = json.loads(str(g["spec"]))
    s = g["spec"]
    eps_d, ind, eps_j = g["eps_d"], g["ind"].astype(np.int64), g["eps_j"]
    if s["jump_channel"] == "control":
        eps_c = np.where(ind[..., None] != 0, eps_d + eps_j, eps_d)
    else:
        eps_c = eps_d.copy()
    g["noise"] = (eps_d, ind, eps_j, eps_c)
    g["seed"] = int(g["seed"])
    g["iteration"] = int(g["iteration"])
    return g


def oracle_spec(s):
    from oracle.mppi import Spec

    lim = None if s["limits"] is None else (np.array(s["limits"][0]), np.array(s["limits"][1]))
    return Spec(s["model"], s["n"], s["m"], tuple(s["params"]), lim, s["jump_channel"], tuple(s["jump_rows"]),
                s["jump_scale"], s["cost"], tuple(s["weights"]), tuple(s["target"]), s["terminal_scale"],
                np.array(s["R"]), s["cost_lambda"], s["cost_c"], s["lam"], s["c"], np.array(s["sigma_d"]),
                np.array(s["sigma_j"]), s["nu"], s["dt"], s["T"], s["K"], s["jump_enabled"],
                np.array(s["mark_mean"]), *_general(s))


def _general(s):
    """(cal_b, bb_term) of a CostModel(control_channel=False) fixture, else (None, None)."""
    if "cal_b" not in s:
        return None, None
    return np.array(s["cal_b"]), np.array(s["bb_term"])


def plugins(s, K=None, T=None):
    """(model, cost_model, cfg) of this package for a golden spec."""
    import paper_1807_06108_b200 as jb

    lim = None if s["limits"] is None else (np.array(s["limits"][0]), np.array(s["limits"][1]))
    if s["model"] == "cartpole":
        model = jb.cartpole_dynamics(jb.CartpoleModel(*s["params"]), lim, jump_channel=s["jump_channel"],
                                     jump_scale_mode=s["jump_scale"])
    elif s["model"] == "quadrotor":
        p = s["params"]
        model = jb.quadrotor_dynamics(jb.QuadrotorModel(p[0], p[1], tuple(p[2:5]), p[5]), lim,
                                      jump_channel=s["jump_channel"], jump_scale_mode=s["jump_scale"])
    elif s["model"] == "linear":
        n, m = s["n"], s["m"]
        p = np.array(s["params"])
        model = jb.linear_dynamics(p[: n * n].reshape(n, n), p[n * n:].reshape(n, m), lim)
    else:
        model = jb.integrator_dynamics(s["n"], lim)
    if s["cost"] == "cartpole_swingup":
        running = jb.CartpoleStateCost(*s["weights"])
    elif s["cost"] == "quadrotor_hover":
        running = jb.QuadrotorStateCost(tuple(s["target"]), *s["weights"])
    else:
        running = jb.DiagQuadraticCost(tuple(s["weights"]), tuple(s["target"]) if s["target"] else None)
    term = jb.ScaledTerminalCost(running, s["terminal_scale"]) if s["terminal_scale"] != 1.0 else running
    cb, bb = _general(s)
    if cb is None:
        cost = jb.CostModel(running, term, np.array(s["R"]), s["cost_lambda"], s["cost_c"])
    else:
        cost = jb.CostModel(running, term, np.array(s["R"]), s["cost_lambda"], s["cost_c"], control_channel=False,
                            cal_b=cb, bb_term=bb)
    q = s["m"] if s["jump_channel"] == "control" else len(s["jump_rows"])
    cfg = jb.MppiConfig(lambda_=s["lam"], c=s["c"], sigma_d=np.array(s["sigma_d"]), sigma_j=np.array(s["sigma_j"]),
                        nu=s["nu"], dt=s["dt"], horizon_n=s["T"] if T is None else T,
                        samples_m=s["K"] if K is None else K, u_init=np.zeros(s["m"]),
                        jump_sampling_enabled=s["jump_enabled"], mark_mean=np.array(s["mark_mean"]), jump_dim=q)
    return model, cost, cfg


def rel_err(a, b, floor=1e-300):
    a, b = np.asarray(a, float), np.asarray(b, float)
    fin = np.isfinite(a) & np.isfinite(b)
    same_inf = ((~np.isfinite(a)) & (a == b)) | (np.isnan(a) & np.isnan(b))
    if not np.all(fin | same_inf):
        return np.inf
    if not fin.any():
        return 0.0
    d = np.abs(a[fin] - b[fin])
    return float(np.max(d / np.maximum(np.abs(b[fin]), floor)))


def normwise(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture
def gpu_device():
    import paper_1807_06108_b200._lib as L

    lib = L.load()
    import ctypes

    n = ctypes.c_int(0)
    rc = lib.jm_device_count(ctypes.byref(n))
    if rc != 0 or n.value < 1:
        pytest.fail("gpu test without a visible CUDA device (no CPU fallback exists)")
    return 0
