"""Full-system flexible GMRES with the block-triangular preconditioner on the GPU (NEXT(4))
against the oracle's FGMRES (tests/test_oracle_fgmres.py pins it)."""
import numpy as np
import pytest
import torch

from synthetic import make_config, paper_problem
from oracle.solver import DDOracle, monolithic_solve

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gpu(p, rtol, **kw):
    from paper_1501_06211_b200 import binding as B
    S = B.Solver.from_problem(p, device=0, outer=1, **kw)
    try:
        S.factor()
        u, its, rel, st = S.solve(p.rhs, rtol)
        return u, its, rel
    finally:
        S.close()


@pytest.mark.parametrize("inv_h,n", [(16, 4), (16, 16), (32, 16)])
def test_fgmres_matches_oracle(inv_h, n):
    p = paper_problem(inv_h, n)
    for mode, kw in (("lanczos", {}), ("identity", dict(inner_mode=3))):
        u, its, rel = _gpu(p, 1e-8, **kw)
        r = DDOracle(p, mode=mode).solve_fgmres(rtol=1e-8, maxit=5000)
        # Arnoldi by CGS2 on the GPU, MGS in the oracle: equal in exact arithmetic
        assert abs(its - r.iterations) <= max(2, int(0.03 * r.iterations)), (mode, its, r.iterations)
        uref = monolithic_solve(p)
        free = p.fixed == 0
        assert rel <= 1e-8
        assert np.linalg.norm((u - uref)[free]) <= 1e-6 * np.linalg.norm(uref[free]), mode


def test_fgmres_c1_to_1e10():
    p = make_config("c1")
    u, its, rel = _gpu(p, 1e-10)
    uref = monolithic_solve(p)
    assert rel <= 1e-10 and np.linalg.norm(u - uref) <= 1e-8 * np.linalg.norm(uref)
