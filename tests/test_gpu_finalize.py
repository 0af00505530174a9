"""The finalize's record merge at multi-GPU record counts (world x grid records,
e.g. 8 x 147 = 1176 > 1024: the loop branch of the head pass), through
jm_finalize_dev, against a float64 numpy restatement of the merge
(online softmax over records: rho = min rho_b, e_b = exp(-(rho_b - rho)/lambda),
u_new = u_nom + sum_b e_b N_b / (sum_b e_b Z_b sqrt(dt)), controller.py:62-78,158-161)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest


def _merge_ref(rec, TM, lam, dt, u_nom):
    rho = np.min(rec[:, 0])
    e = np.where(np.isfinite(rec[:, 0]), np.exp(-(rec[:, 0] - rho) / lam), 0.0)
    Z = np.sum(e * rec[:, 1])
    N = e @ rec[:, 4:4 + TM]
    return u_nom + N / (Z * np.sqrt(dt)), rho, Z * Z / np.sum(e * e * rec[:, 2])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 3, 8, 20])
def test_finalize_merges_many_records(world, gpu_device):
    import torch

    import paper_1807_06108_b200 as jb
    from paper_1807_06108_b200 import engine

    task, cfg = jb.baseline_config(1, K=65536, T=100)
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision="f64")
    rs = C.c_int64()
    assert ctx.lib.jm_record_doubles(ctx.h, C.byref(rs)) == 0
    rs, TM = rs.value, cfg.horizon_n
    n = world * 147
    rng = np.random.default_rng(world)
    rec = np.zeros((n, rs))
    rec[:, 0] = 100.0 + 5.0 * rng.random(n)
    rec[rng.random(n) < 0.05, 0] = np.inf   # CTAs without a finite cost
    rec[:, 1] = 1.0 + rng.random(n)
    rec[:, 2] = 0.5 + rng.random(n)
    rec[:, 3] = 443.0
    rec[:, 4:4 + TM] = rng.standard_normal((n, TM))
    rec[~np.isfinite(rec[:, 0]), 1:] = 0.0
    u_nom = rng.standard_normal(TM)
    dev = torch.device("cuda")
    r_d = torch.tensor(rec, device=dev)
    un_d = torch.tensor(u_nom, device=dev)
    out_d = torch.zeros(TM, dtype=torch.float64, device=dev)
    diag_d = torch.zeros(4, dtype=torch.float64, device=dev)
    st_d = torch.zeros(1, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    rc = ctx.lib.jm_finalize_dev(ctx.h, C.c_void_p(r_d.data_ptr()), n, C.c_void_p(un_d.data_ptr()), None,
                                 C.c_void_p(out_d.data_ptr()), None, C.c_void_p(diag_d.data_ptr()),
                                 C.c_void_p(st_d.data_ptr()))
    assert rc == 0
    torch.cuda.synchronize()
    u_ref, rho_ref, ess_ref = _merge_ref(rec, TM, cfg.lambda_, cfg.dt, u_nom)
    u = out_d.cpu().numpy()
    assert np.max(np.abs(u - u_ref) / (1e-12 + np.abs(u_ref))) < 1e-10
    d = diag_d.cpu().numpy()
    assert d[0] == rho_ref
    assert abs(d[1] - ess_ref) / ess_ref < 1e-10
