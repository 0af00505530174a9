"""Time jm_finalize_dev on synthetic records: nrec = world x 147 (cfg1 grid), world 1..8."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1807_06108_b200 as jb
from paper_1807_06108_b200 import engine
task, cfg = jb.baseline_config(1)
ctx = engine.get_context(task.model, task.cost_model, cfg)
lib = ctx.lib
rs = C.c_int64(); lib.jm_record_doubles(ctx.h, C.byref(rs)); rs = rs.value
TM = cfg.horizon_n
dev = torch.device('cuda')
unom = torch.zeros(TM, dtype=torch.float64, device=dev)
unew = torch.zeros(TM, dtype=torch.float64, device=dev)
torch.cuda.set_stream(torch.cuda.Stream())
for world in (1, 2, 4, 8):
    n = world * 147
    rec = torch.zeros((n, rs), dtype=torch.float64, device=dev)
    g = torch.Generator(device='cpu').manual_seed(0)
    rec[:, 0] = torch.rand(n, generator=g, dtype=torch.float64).to(dev) * 5 + 100
    rec[:, 1] = 1.0 + torch.rand(n, generator=g, dtype=torch.float64).to(dev)
    rec[:, 2] = 0.5
    rec[:, 3] = 443.0
    rec[:, 4:4 + TM] = torch.randn((n, TM), generator=g, dtype=torch.float64).to(dev)
    stream = ctypes_stream = torch.cuda.current_stream().cuda_stream
    lib.jm_set_stream(ctx.h, C.c_void_p(stream))
    for _ in range(5):
        lib.jm_finalize_dev(ctx.h, C.c_void_p(rec.data_ptr()), n, C.c_void_p(unom.data_ptr()), None,
                            C.c_void_p(unew.data_ptr()), None, None, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        lib.jm_finalize_dev(ctx.h, C.c_void_p(rec.data_ptr()), n, C.c_void_p(unom.data_ptr()), None,
                            C.c_void_p(unew.data_ptr()), None, None, None)
    e1.record(); torch.cuda.synchronize()
    print(f"world {world}: nrec {n}: finalize {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")

# Two-level alternative (DESIGN 7b item 3): each rank first reduces its own 147 CTA
# records into one (jm_reduce_dev, the NCCL transport's reduce step), then merges
# `world` records.  Critical path per step = reduce(147) + finalize(world).
ctx.iteration(np.zeros(ctx.N), np.zeros(TM), 1, 0)  # populate this context's CTA records
rec1 = torch.zeros(rs, dtype=torch.float64, device=dev)


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


lib.jm_set_stream(ctx.h, C.c_void_p(torch.cuda.current_stream().cuda_stream))
t_red = timed(lambda: lib.jm_reduce_dev(ctx.h, C.c_void_p(rec1.data_ptr())))
for world in (1, 2, 4, 8):
    recw = rec1.repeat(world, 1).contiguous()
    t_fin = timed(lambda: lib.jm_finalize_dev(ctx.h, C.c_void_p(recw.data_ptr()), world, C.c_void_p(unom.data_ptr()),
                                              None, C.c_void_p(unew.data_ptr()), None, None, None))
    t_both = timed(lambda: (lib.jm_reduce_dev(ctx.h, C.c_void_p(rec1.data_ptr())),
                            lib.jm_finalize_dev(ctx.h, C.c_void_p(recw.data_ptr()), world, C.c_void_p(unom.data_ptr()),
                                                None, C.c_void_p(unew.data_ptr()), None, None, None)))
    print(f"world {world}: two-level: reduce(147) {t_red:.1f} us + finalize({world}) {t_fin:.1f} us; "
          f"back to back {t_both:.1f} us")
