"""How many samples carry a non-negligible weight relative to their tile's minimum?

Runs a closed loop through the drop-in API (plant stepped on the host with the
oracle's Euler step) and, at each control step, reads the per-sample costs of
the non-trace Philox kernel; reports per tile (the rollout's CTA tile) the
fraction of samples with (S_k - min_tile S) / lambda <= 55 (weight >= e^-55
relative to the tile minimum) -- the samples a sparse epilogue must revisit.
"""
import sys, json
import numpy as np
sys.path.insert(0, ".")
import paper_1807_06108_b200 as jb
from paper_1807_06108_b200 import engine
from oracle import mppi as om

def run(idx, K, T, steps, tile, thr=55.0):
    task, cfg = jb.baseline_config(idx, K=K, T=T)
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision="f32")
    spec = om.spec_from_plugins(task.model, task.cost_model, cfg)
    rng = np.random.default_rng(0)
    x = np.array(task.x0, float)
    u = np.tile(cfg.u_init, (T, 1)).astype(float)
    out = []
    for k in range(steps):
        o = ctx.iteration(x, u, 0, k, want_costs=True, want_weights=False)
        S = o.costs
        St = S[: (K // tile) * tile].reshape(-1, tile)
        rel = (St - St.min(axis=1, keepdims=True)) / cfg.lambda_
        frac_tile = float(np.mean(rel <= thr))
        relg = (S - S.min()) / cfg.lambda_
        frac_glob = float(np.mean(relg <= thr))
        out.append((k, frac_tile, frac_glob, float(np.median(S)), float(S.min())))
        u_new = o.u_new
        ed = rng.standard_normal(cfg.control_dim) @ np.linalg.cholesky(np.asarray(cfg.sigma_d)).T
        x = om.step_batch(spec, x[None], u_new[0], ed[None], np.zeros((1, spec.q)), np.zeros(1), cfg.dt, np.float64)[0]
        u = np.vstack([u_new[1:], np.atleast_2d(cfg.u_init)])
    return out

for name, idx, K, T, tile in (("cfg1", 1, 65536, 100, 448), ("cfg3-1/8", 3, 1 << 17, 200, 256), ("cfg2", 2, 8192, 150, 128)):
    res = run(idx, K, T, 40, tile)
    print(name, json.dumps([(k, round(a, 4), round(b, 5), round(m, 1), round(s, 1)) for k, a, b, m, s in res[::4]]))
