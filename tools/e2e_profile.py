"""Where the drop-in call spends its time (host side).  GPU box only."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1807_06108_b200 as jb  # noqa: E402

task, cfg = jb.baseline_config(1)
ctrl = jb.initial_controller_state(cfg)
x0 = np.asarray(task.x0, float)


def loop(n):
    global ctrl
    for _ in range(n):
        seq, diag = jb.mppi_iteration(ctrl, task.model, task.cost_model, x0, 0)
        ctrl = jb.ControllerState(jb.warm_start_shift(seq, cfg.u_init), ctrl.iteration_index + 1, cfg)


loop(5)
t0 = time.perf_counter()
loop(50)
print("ms/step", (time.perf_counter() - t0) / 50 * 1e3)
pr = cProfile.Profile()
pr.enable()
loop(50)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
