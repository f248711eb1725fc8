"""Diagnostic: one full-size solve, timings, residual floor estimate (not part of the product)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synthetic import make_config
from paper_1501_06211_b200 import binding as B
if os.environ.get("AB_LIB"):   # A/B experiments: load another build of libde.so
    B.LIB_PATH = os.environ["AB_LIB"]
from oracle.fem import element_stiffness, simp_modulus, element_dofs, true_relres

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = int(v)
p = make_config(name)
t = time.time(); S = B.Solver.from_problem(p, device=0, **kw); print("setup s", time.time() - t, flush=True)
for rep in range(2):
    t = time.time(); S.factor(); print("factor s", time.time() - t, "ms_factor", S.stats().ms_factor, flush=True)
    t = time.time(); u, its, rel, st = S.solve(p.rhs, p.rtol, allow_noconv=True); dt = time.time() - t
    s = S.stats()
    print(f"solve s {dt:.3f} its {its} relres_true {rel:.3e} rec {s.relres_recursive:.3e} refines {s.restarts} "
          f"ms_pcg {s.ms_pcg:.1f} ms/it {s.ms_pcg/max(its,1):.3f} launches/it {s.launches_per_iter} status {st}", flush=True)
print("oracle true_relres", true_relres(p, u))
KE = np.abs(element_stiffness(p.dim, p.nu)); E = simp_modulus(p.density, p.E0, p.Emin, p.p)
ed = element_dofs(p.dim, p.nel); ue = np.abs(u)[ed]; fe = (ue @ KE.T) * E[:, None]
out = np.zeros_like(u); np.add.at(out, ed.ravel(), fe.ravel())
free = p.fixed == 0
print("eps*|| |K||u| ||/||f||", 1.1e-16 * np.linalg.norm(out[free]) / np.linalg.norm(p.rhs[free]), "max|u|", np.abs(u).max())
