"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): c1 and a scaled c2 through every
launch path -- factor, interface PCG with the cooperative preconditioner (fold path), the multi-kernel
preconditioner, the explicit and implicit Schur applies, FGMRES, the topology-optimisation step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synthetic import make_config
from paper_1501_06211_b200 import binding as B

for name, kw in (("c1", {}), ("c2", dict(nel=(64, 32), sub=(16, 16))), ("c4", dict(nel=(12, 6, 6), sub=(6, 6, 6)))):
    p = make_config(name, **kw)
    for opts in (dict(), dict(prec_kernels=1), dict(schur_mode=1), dict(outer=1, restart=20)):
        S = B.Solver.from_problem(p, device=0, **opts)
        S.factor()
        u, its, rel, st = S.solve(p.rhs, p.rtol, allow_noconv=True)
        print(name, opts, "its", its, "relres %.2e" % rel, "status", st, flush=True)
        if not opts:
            rho, c, lam = S.oc_step(u, p.nelem)
            print("  oc step compliance %.6e" % c)
        S.close()
print("sanitize workload done")
