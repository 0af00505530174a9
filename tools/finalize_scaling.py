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
