"""Device timeline of closed-loop control steps (%globaltimer stamps, kernels.cuh kTl*).

    JM_TIMELINE=1 python tools/timeline.py [cfg1|cfg3|cfg0] [steps]

Prints, averaged over the steps after a warm-up, each stamp relative to the
rollout kernel's entry: where a control step's time goes between the two
kernels (grid-dependency waits, prologue, horizon, epilogue, finalize, plant).
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("JM_TIMELINE", "1")
import paper_1807_06108_b200 as jb  # noqa: E402
from paper_1807_06108_b200 import _lib as L  # noqa: E402
from paper_1807_06108_b200 import engine  # noqa: E402

NAMES = ["roll_entry", "roll_wait", "roll_horizon", "horizon_end_min", "horizon_end_max", "roll_end_max",
         "fin_entry", "fin_wait", "fin_merged", "fin_end"]


def main(wl="cfg1", steps=40):
    idx = {"cfg0": 0, "cfg1": 1, "cfg2": 2, "cfg3": 3}[wl]
    task, cfg = jb.baseline_config(idx)
    ctx = engine.get_context(task.model, task.cost_model, cfg, precision="f32")
    lib, h = ctx.lib, ctx.h
    x0 = np.ascontiguousarray(task.x0, float)
    ui = np.ascontiguousarray(cfg.u_init, float)
    ctx.check(lib.jm_loop_init(h, L.dptr(x0), L.dptr(ui), C.c_uint64(0), C.c_uint64(0), steps))
    for _ in range(steps):
        ctx.check(lib.jm_loop_step(h))
    tl = np.zeros(steps * 12, dtype=np.uint64)
    ctx.check(lib.jm_loop_timeline(h, steps, tl.ctypes.data_as(C.POINTER(C.c_uint64))))
    raw = tl.reshape(steps, 12)[:, 10:12].copy()
    tl = tl.reshape(steps, 12).astype(np.float64)
    tl[:, 3] = (2.0 ** 64 - 1) - tl[:, 3]  # stored as ~t (atomicMax of the complement)
    w = tl[steps // 4:]
    base = w[:, 0:1]
    rel = (w[:, :10] - base) / 1e3
    period = np.diff(w[:, 0]) / 1e3
    print(f"{wl}: K={cfg.samples_m} T={cfg.horizon_n}; step period {period.mean():.2f} us (rollout entry to entry)")
    for i, n in enumerate(NAMES[:10]):
        print(f"  {n:16s} {rel[:, i].mean():8.2f} us  (sd {rel[:, i].std():.2f})")
    if os.environ.get("JM_TL_PROBE"):
        r = raw[steps // 4:]
        hi = lambda v: (v >> np.uint64(32)).astype(float).mean()
        lo = lambda v: (v & np.uint64(0xffffffff)).astype(float).mean()
        print(f"  probe cycles: loads+warpmin {hi(r[:, 0]):.0f} barrier+min {lo(r[:, 0]):.0f} "
              f"exp+sums {hi(r[:, 1]):.0f} update {lo(r[:, 1]):.0f}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg1", int(sys.argv[2]) if len(sys.argv) > 2 else 40)
