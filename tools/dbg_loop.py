import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1807_06108_b200 as jb
from paper_1807_06108_b200 import engine
task, cfg = jb.baseline_config(0, K=1024, T=50, steps=20)
for prec in ("f64", "f32"):
    seq, _ = jb.mppi_iteration(jb.initial_controller_state(cfg), task.model, task.cost_model, task.x0, 11, precision=prec)
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision=prec)
    o = ctx.iteration(task.x0, np.tile(cfg.u_init, (50, 1)), 11, 0, want_costs=True, want_weights=False)
    rec = jb.run_trial(task, cfg, seed=11, precision=prec)
    print(prec, ctx.kernel_name(), "dropin", seq.controls[:3, 0], "host", o.u_new[:3, 0], "loop", rec.controls[:3, 0])
