"""A/B helper: median time of one interface-preconditioner application (de_precond_apply_device) on a config,
and (DE_PREC_TIMERS=1) the per-phase durations of the cooperative kernel. Usage: python tools/prec_ab.py c5 [reps]"""
import os, sys, ctypes as C, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synthetic import make_config
from paper_1501_06211_b200 import binding as B
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = make_config(name)
S = B.Solver.from_problem(p, device=0)
S.factor()
nG = S.stats().n_Gamma
g = torch.Generator(device="cuda").manual_seed(0)
r = torch.randn(nG, dtype=torch.float64, device="cuda", generator=g); z = torch.empty_like(r)
ts = []
for rep in range(reps + 3):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); B.de_precond_apply_device(S.ctx, r.data_ptr(), z.data_ptr()); e1.record(); torch.cuda.synchronize()
    if rep >= 3:
        ts.append(e0.elapsed_time(e1))
print(f"{name} precond ms median {statistics.median(ts):.4f} min {min(ts):.4f} env "
      f"{ {k: v for k, v in os.environ.items() if k.startswith('DE_')} } zsum {float(z.sum()):.12e}")
if os.environ.get("DE_PREC_TIMERS"):
    L = B.lib()
    L.de_debug_prec_timers.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    t = (C.c_ulonglong * (200 + 8192))()
    L.de_debug_prec_timers(S.ctx, t, 200 + 8192)
    st = [x for x in list(t)[:100] if x]
    print("phases us:", " ".join(f"{(b - a) / 1e3:.1f}" for a, b in zip(st, st[1:])), "total", (st[-1] - st[0]) / 1e3)
    e = list(t)[180:186]
    if all(e):
        print("last elimination, cross phase (block 0) us: t_C", (e[1] - e[0]) / 1e3, "gemv", (e[2] - e[1]) / 1e3,
              "syncthreads", (e[3] - e[2]) / 1e3, "sums+fold", (e[4] - e[3]) / 1e3, "grid.sync", (e[5] - e[4]) / 1e3)
S.close()
