import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from synthetic import paper_problem, make_config
from oracle.topology import build_topology
from paper_1501_06211_b200 import binding as B
def z_of(p, r, nofold):
    if nofold: os.environ['DE_NO_FOLD'] = '1'
    S = B.Solver.from_problem(p, device=0)
    os.environ.pop('DE_NO_FOLD', None)
    S.factor()
    dr = torch.tensor(r, device='cuda'); dz = torch.empty_like(dr)
    B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr()); z = dz.cpu().numpy(); S.close(); return z
for p in [paper_problem(32, 16), paper_problem(16, 4), make_config("c2", nel=(64, 32), sub=(16, 16))]:
    nG = build_topology(p).n_G
    rng = np.random.default_rng(1)
    for kind in ("rand", "xonly", "smallcomp"):
        r = rng.normal(size=nG)
        if kind == "xonly": r[1::2] = 0.0   # (dof parity is not the component map, but makes components unequal)
        if kind == "smallcomp": r[1::2] *= 1e-9
        z1 = z_of(p, r, False); z2 = z_of(p, r, True)
        print(p.name, kind, np.linalg.norm(z1 - z2) / np.linalg.norm(z2))
