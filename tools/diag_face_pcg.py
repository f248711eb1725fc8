"""Diagnostic: GPU inner_mode 0 (face-PCG inner solves) against the oracle's mode F at three inner tolerances:
inner iteration counts and the relative difference of z on the same input."""
import numpy as np, torch, sys
sys.path.insert(0, '.')
from synthetic import make_config
from oracle.topology import build_topology
from oracle.precond import build_components, apply_precond
from paper_1501_06211_b200 import binding as B
for name, nel, sub in [("c2", (64, 32), (16, 16)), ("c2", (100, 36), (20, 12)), ("c4", (16, 8, 8), (4, 4, 4))]:
    p = make_config(name, nel=nel, sub=sub); topo = build_topology(p)
    for tol in (1e-3, 1e-6, 1e-12):
        comps = build_components(p, topo)
        for cd in comps: cd.inner_tol = tol; cd.inner_its = []
        S = B.Solver.from_problem(p, device=0, inner_mode=0, inner_tol=tol); S.factor()
        rng = np.random.default_rng(17)
        for rep in range(2):
            r = rng.normal(size=topo.n_G)
            for cd in comps: cd.inner_its = []
            ref = apply_precond(comps, r, "lanczos", 0.5, 10, "F")
            n0 = S.stats().inner_iterations
            dr = torch.tensor(r, dtype=torch.float64, device="cuda"); dz = torch.empty_like(dr)
            B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr())
            z = dz.cpu().numpy()
            print(name, nel, tol, rep, "its", S.stats().inner_iterations - n0, sum(sum(cd.inner_its) for cd in comps), [cd.inner_its for cd in comps][0][:9], "rel", np.linalg.norm(z-ref)/np.linalg.norm(ref))
        S.close()
