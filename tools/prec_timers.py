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
# consumer phase (Lanczos step 5; phase C with the fold, else phase A) per block: start and arrival at its barrier (globaltimer ns)
st = np.array(list(t)[200 + 4096 + 1024:200 + 4096 + 1024 + 512], dtype=np.float64)
ar = np.array(list(t)[200 + 4096 + 1536:200 + 4096 + 1536 + 512], dtype=np.float64)
nbk = int((st > 0).sum())
if nbk:
    st, ar = st[:nbk], ar[:nbk]
    t0 = st.min()
    print("phaseA blocks", nbk, "start spread us", (st.max() - t0) / 1e3, "arrival min/p50/max us", (ar.min() - t0) / 1e3,
          (np.median(ar) - t0) / 1e3, (ar.max() - t0) / 1e3)
    late = np.argsort(-(ar - t0))[:12]
    print("latest arrivals (block, start us, arrive us):", [(int(b), round((st[b] - t0) / 1e3, 2), round((ar[b] - t0) / 1e3, 2)) for b in late])
    dur = (ar - st) / 1e3
    print("A duration by component (even/odd blocks): mean", dur[0::2].mean(), dur[1::2].mean(), "max", dur[0::2].max(), dur[1::2].max())
    early = np.argsort(st - t0)[-8:]
    print("latest starts:", [(int(b), round((st[b] - t0) / 1e3, 2)) for b in early])
sm = np.array(list(t)[200 + 4096 + 2048:200 + 4096 + 2048 + 512], dtype=np.int64)[:nbk]
if nbk:
    d = (ar - t0) / 1e3
    bysm = {}
    for b in range(nbk):
        bysm.setdefault(int(sm[b]), []).append(d[b])
    slow = sorted(bysm.items(), key=lambda kv: -max(kv[1]))[:10]
    print("slowest SMs (smid: arrivals us):", [(k, [round(x, 1) for x in v]) for k, v in slow])
    print("latest blocks' SMs:", [(int(b), int(sm[b])) for b in late])
    s_ids = np.array(sorted(bysm)); mx = np.array([max(bysm[k]) for k in s_ids])
    print("mean arrival by SM range 0-73 / 74-147:", mx[s_ids < 74].mean(), mx[s_ids >= 74].mean())
