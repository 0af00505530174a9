"""Split the drop-in call time: raw C call vs the Python API.  GPU box only."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1807_06108_b200 as jb  # noqa: E402
from paper_1807_06108_b200 import _lib as L  # noqa: E402
from paper_1807_06108_b200 import engine  # noqa: E402

task, cfg = jb.baseline_config(1)
ctrl = jb.initial_controller_state(cfg)
x0 = np.asarray(task.x0, float)
ctx = engine.get_context(task.model, task.cost_model, cfg)
u = np.ascontiguousarray(ctrl.nominal_controls.controls)
ui = np.ascontiguousarray(cfg.u_init)
un, no, us = np.empty(100), np.empty(100), np.empty(100)
d = L.Diag()
h = C.c_uint64()


def raw(n, stash=True, shift=True):
    for i in range(n):
        rc = ctx.lib.jm_iteration_host(ctx.h, L.dptr(x0), L.dptr(u), 0, i, None, None, None, L.dptr(un), None, None,
                                       L.dptr(no), None, None, C.byref(d), L.dptr(ui) if shift else None,
                                       L.dptr(us) if shift else None, C.byref(h) if stash else None)
        assert rc == 0
        if stash:
            ctx.lib.jm_stash_release(ctx.h, h)


def api(n):
    c = ctrl
    for _ in range(n):
        seq, diag = jb.mppi_iteration(c, task.model, task.cost_model, x0, 0)
        c = jb.ControllerState(jb.warm_start_shift(seq, cfg.u_init), c.iteration_index + 1, cfg)


for name, f in [("raw C call (stash+shift)", lambda n: raw(n)), ("raw C call (no stash/shift)", lambda n: raw(n, False, False)),
                ("python API", api)]:
    f(5)
    t0 = time.perf_counter()
    f(100)
    print(f"{name:32s} {(time.perf_counter() - t0) * 1e4:.1f} us/iter")
