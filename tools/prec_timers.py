"""Diagnostic: per-phase time of the cooperative preconditioner on config c (DE_PREC_TIMERS=1)."""
import os, sys, ctypes as C
os.environ["DE_PREC_TIMERS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synthetic import make_config
from paper_1501_06211_b200 import binding as B
if os.environ.get("AB_LIB"):   # A/B experiments: load another build of libde.so
    B.LIB_PATH = os.environ["AB_LIB"]
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = make_config(name)
S = B.Solver.from_problem(p, device=0)
S.factor()
L = B.lib()
L.de_debug_prec_timers.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
nG = S.stats().n_Gamma
r = torch.randn(nG, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for rep in range(3):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); B.de_precond_apply_device(S.ctx, r.data_ptr(), z.data_ptr()); e1.record(); torch.cuda.synchronize()
    print("precond ms", e0.elapsed_time(e1))
t = (C.c_ulonglong * (200 + 8192))()
L.de_debug_prec_timers(S.ctx, t, 200 + 8192)
print("ritz_warp us", (t[101] - t[100]) / 1e3, "setup", (t[103]-t[102])/1e3, "jacobi", (t[104]-t[103])/1e3, "sweeps", t[106], "final", (t[105]-t[104])/1e3)
for nm, b0 in (("A", 120), ("B", 130)):
    print(f"phase{nm} j=5: rows", (t[b0+1]-t[b0])/1e3, "partials", (t[b0+2]-t[b0+1])/1e3, "sync", (t[b0+3]-t[b0+2])/1e3, "totals", (t[b0+4]-t[b0+3])/1e3)
print("phaseA per-warp row cycles (blocks 0-3):", list(t)[140:172])
print("E2 (step 5): tC", (t[181]-t[180])/1e3, "gemv", (t[182]-t[181])/1e3, "syncthreads", (t[183]-t[182])/1e3, "sums", (t[184]-t[183])/1e3, "grid.sync", (t[185]-t[184])/1e3)
print("phaseC j=5: rows", (t[111]-t[110])/1e3, "partials", (t[112]-t[111])/1e3, "sync", (t[113]-t[112])/1e3, "totals", (t[114]-t[113])/1e3)
ts = [x for x in list(t)[:100] if x]
d = np.diff(np.array(ts, dtype=np.float64)) / 1e3
print("phases", len(d), "total us", d.sum())
print(" ".join(f"{x:.1f}" for x in d))

f0 = np.array(list(t)[200:200 + 4096], dtype=np.float64); f1 = np.array(list(t)[200 + 4096:200 + 8192], dtype=np.float64)
f0 = f0[f0 > 0]; f1 = f1[f1 > 0]
print("face mode0 warp cycles: n", len(f0), "mean", f0.mean(), "max", f0.max(), "p50", np.median(f0))
if len(f1): print("face mode1 warp cycles: n", len(f1), "mean", f1.mean(), "max", f1.max(), "p50", np.median(f1))
f1all = np.array(list(t)[200 + 4096:200 + 4096 + 2368], dtype=np.float64)
slow = np.argsort(-f1all)[:12]
print("slowest mode1 warps (gw, cycles, block, warp):", [(int(g), int(f1all[g]), int(g) // 8, int(g) % 8) for g in slow])
f0all = np.array(list(t)[200:200 + 2368], dtype=np.float64)
print("their mode0 cycles:", [int(f0all[g]) for g in slow])
