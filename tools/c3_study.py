"""Diagnostic (R15 / SURVEY Q15): config 3 at full size -- interface PCG progress with and without the
coefficient-weighted trace norm (R19) at several iteration budgets: true relative residual, normwise backward
error ||f - K u|| / (||K||_1 ||u|| + ||f||) and forward difference against the oracle's direct solve."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synthetic import make_config
from paper_1501_06211_b200 import binding as B
from oracle.fem import free_system
from oracle.direct import direct_solve

p = make_config("c3")
K, f, free = free_system(p)
nK = abs(K).sum(axis=0).max()
u_ref = direct_solve(p)
bwd = lambda u: float(np.linalg.norm(f - K @ u[free]) / (nK * np.linalg.norm(u[free]) + np.linalg.norm(f)))
rows = []
budgets = [int(b) for b in (sys.argv[1:] or ["2000", "5000", "20000"])]
for weighted in (0, 1):
    for mi in budgets:
        S = B.Solver.from_problem(p, device=0, max_iter=mi, weighted_trace=weighted)
        S.factor()
        t = time.perf_counter()
        u, its, rel, st = S.solve(p.rhs, p.rtol, allow_noconv=True)
        dt = time.perf_counter() - t
        s = S.stats()
        row = dict(weighted=weighted, budget=mi, iterations=its, status=int(st), relres=rel,
                   relres_recursive=s.relres_recursive, backward_error=bwd(u),
                   forward_diff=float(np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref)), seconds=dt)
        print(json.dumps(row), flush=True)
        rows.append(row)
        S.close()
print("oracle direct: backward error", bwd(u_ref), "||u_ref||", float(np.linalg.norm(u_ref)))
