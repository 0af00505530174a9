"""Multi-GPU host logic on CPU (gloo, world_size 2): shard ranges, the record
exchange in rank order and the log-sum-exp merge reproduce the unsharded
iteration.  The per-shard arithmetic here is the oracle's; on
GPUs the same exchange_records() feeds libjmppi's finalize kernel."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden, oracle_spec
from oracle import mppi as om
from oracle import philox_stream as ps
from paper_1807_06108_b200 import distributed as jd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_partition():
    for k, w in [(65536, 8), (1000, 3), (7, 4)]:
        spans = [jd.shard_strong(k, r, w) for r in range(w)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == k
        for (o0, c0), (o1, _) in zip(spans, spans[1:]):
            assert o0 + c0 == o1
    assert jd.shard(4096, 3) == (3 * 4096, 4096)


def test_record_merge_matches_unsharded_oracle():
    g = load_golden("b_cartpole")
    spec = oracle_spec(g["spec"])
    Ld = np.linalg.cholesky(spec.c * spec.sigma_d)
    Lj = np.linalg.cholesky(spec.sigma_j)
    jthr = ps.jump_threshold(spec.nu * spec.dt)
    full = ps.device_noise(1, 0, 96, spec.T, 1, 1, Ld, Lj, spec.mark_mean, jthr, jump_channel="state")
    spec.K = 96
    ref = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], full)
    recs = []
    for off, cnt in [(0, 40), (40, 56)]:
        part = tuple(a[off:off + cnt] for a in full)
        spec.K = cnt
        o = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], part)
        recs.append(om.partial_record(o["costs"], part[3], spec.lam))
    u_new, rho, ess = om.combine_records(recs, spec.lam, spec.dt, g["u_nom"])
    assert rho == ref["min_cost"]
    assert np.allclose(u_new, ref["u_new"], rtol=1e-12, atol=1e-12)
    assert ess == pytest.approx(ref["ess"], rel=1e-12)


def _run_world2(**extra):
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2", CUDA_VISIBLE_DEVICES="",
               **{k: str(v) for k, v in extra.items()})
    procs = [subprocess.Popen([sys.executable, str(ROOT / "tests" / "_dist_worker.py")],
                              env=dict(env, RANK=str(r), LOCAL_RANK=str(r)), stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=300)
        assert p.returncode == 0, e[-3000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    return outs


@pytest.mark.parametrize("case,scaling", [("b_cartpole", "weak"), ("r_quadrotor_task", "weak"),
                                          ("b_cartpole", "strong"), ("r_quadrotor_task", "strong")])
def test_gloo_world2_exchange(case, scaling):
    """Weak: 48 samples per rank.  Strong (BASELINE config 3's K/N split): 97
    samples in total, ragged 49 + 48."""
    if scaling == "weak":
        k_global = 2 * 48
        outs = _run_world2(JM_CASE=case, JM_K_LOCAL=48)
    else:
        k_global = 97
        outs = _run_world2(JM_CASE=case, JM_K_TOTAL=k_global)
        assert [(o["offset"], o["count"]) for o in outs] == [(0, 49), (49, 48)]
    # every rank merged the same records into the same update
    assert outs[0]["u_new"] == outs[1]["u_new"]
    # ... equal to one unsharded iteration over the k_global global samples
    g = load_golden(case)
    spec = oracle_spec(g["spec"])
    Ld = np.linalg.cholesky(spec.c * spec.sigma_d)
    Lj = np.linalg.cholesky(spec.sigma_j)
    jthr = ps.jump_threshold(spec.nu * spec.dt) if spec.jump_enabled else 0
    full = ps.device_noise(7, 3, k_global, spec.T, spec.m, spec.q, Ld, Lj, spec.mark_mean, jthr,
                           jump_channel=spec.jump_channel)
    spec.K = k_global
    ref = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], full)
    assert np.allclose(np.array(outs[0]["u_new"]), ref["u_new"], rtol=1e-11, atol=1e-11)
    assert outs[0]["rho"] == pytest.approx(ref["min_cost"], rel=1e-13)


def test_gloo_world2_transport_agreement():
    """A rank whose peer-buffer setup failed pulls every rank onto the NCCL path."""
    outs = _run_world2(JM_AGREE=1)
    assert [o["agree"] for o in outs] == [False, False]
    assert [o["all_ok"] for o in outs] == [True, True]


def test_shard_for():
    assert jd.shard_for("weak", 100, 2, 4) == (200, 100)
    assert jd.shard_for("strong", 10, 3, 4) == (8, 2)
    with pytest.raises(ValueError):
        jd.shard_for("linear", 10, 0, 2)


def test_two_level_exchange_policy():
    """p2p exchange form: flat below 6 ranks, rank-local reduce from 6 (DESIGN 7b
    measurements), JM_P2P_TWO_LEVEL forcing either, anything else rejected."""
    from paper_1807_06108_b200 import distributed as jd

    assert [jd.use_two_level(w, {}) for w in (1, 2, 4, 5, 6, 8)] == [False] * 4 + [True] * 2
    assert jd.use_two_level(8, {"JM_P2P_TWO_LEVEL": "0"}) is False
    assert jd.use_two_level(1, {"JM_P2P_TWO_LEVEL": "1"}) is True
    with pytest.raises(ValueError):
        jd.use_two_level(2, {"JM_P2P_TWO_LEVEL": "yes"})
