"""Paper-mode reproduction: the test problem of PAPER.md:187 and the qualitative claims
of Table 1: with the interface preconditioner H_theta the iteration count does not grow with
the mesh parameter, without it (S~ = I) it grows ~log-like, and it grows with the number of subdomains.

Differences from the paper, by design (R18): interface PCG (the BASELINE method) instead of GMRES on the
full system, so counts are compared as trends, not values; traction extent/direction and the subdomain layout
are readings."""
import numpy as np
import pytest
import torch

from synthetic import paper_problem
from oracle.solver import DDOracle, monolithic_solve


# ----------------------------------------------------------------------------------------------- host / oracle
def test_paper_problem_loads_and_clamp():
    """Resultants of the consistent nodal loads: body force 0.75 over the area 2, traction 1 over the edge 1."""
    for inv_h, n in ((8, 4), (16, 16), (32, 64)):
        p = paper_problem(inv_h, n)
        assert p.nel == (2 * inv_h, inv_h) and p.h == 1.0 / inv_h
        assert np.isclose(p.rhs[1::2].sum(), -0.75 * 2.0, rtol=0, atol=1e-12)
        assert np.isclose(p.rhs[0::2].sum(), -1.0, rtol=0, atol=1e-12)
        nx, ny = p.nel
        fixed = p.fixed.reshape(ny + 1, nx + 1, 2)
        assert fixed[:, nx, :].all() and fixed.sum() == 2 * (ny + 1)
        assert tuple(a // b for a, b in zip(p.nel, p.sub)) == (int(n ** 0.5),) * 2
        assert np.all(p.density == 1.0) and p.p == 1.0 and p.Emin == 0.0


def _its(p, mode, theta=0.5):
    o = DDOracle(p, mode=mode, theta=theta)
    return o.solve(rtol=p.rtol, maxit=5000, max_refine=0).its_pass1


def test_oracle_table1_trends_small():
    """Oracle pinned against Table 1's claims at small h: H_theta iterations nearly flat under h-refinement,
    S~ = I iterations growing by a roughly constant factor per halving (the paper: 28 -> 41 -> 59, x1.45)."""
    for n in (4, 16):
        h_its = [_its(paper_problem(ih, n), "lanczos") for ih in (8, 16, 32)]
        i_its = [_its(paper_problem(ih, n), "identity") for ih in (8, 16, 32)]
        assert max(h_its) <= 1.25 * min(h_its), (n, h_its)
        assert all(b >= 1.3 * a for a, b in zip(i_its, i_its[1:])), (n, i_its)
        assert all(a < b for a, b in zip(h_its, i_its)), (n, h_its, i_its)
    assert _its(paper_problem(16, 16), "lanczos") > _its(paper_problem(16, 4), "lanczos")


# ----------------------------------------------------------------------------------------------- GPU
gpu = pytest.mark.gpu


def _gpu_solve(p, **kw):
    from paper_1501_06211_b200 import binding as B
    S = B.Solver.from_problem(p, device=0, **kw)
    try:
        S.factor()
        u, its, rel, st = S.solve(p.rhs, p.rtol, allow_noconv=False)
        return u, its, S.stats().iterations_pass1
    finally:
        S.close()


@gpu
@pytest.mark.parametrize("inv_h,n", [(16, 4), (32, 16)])
def test_paper_mode_gpu_matches_oracle(inv_h, n):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = paper_problem(inv_h, n)
    for mode, kw in (("lanczos", {}), ("identity", dict(inner_mode=3))):
        u, its, its1 = _gpu_solve(p, **kw)
        o = DDOracle(p, mode=mode)
        r = o.solve(rtol=p.rtol, maxit=5000, max_refine=0)
        assert abs(its1 - r.its_pass1) <= max(1, int(0.05 * r.its_pass1)), (mode, its1, r.its_pass1)
        uref = monolithic_solve(p)
        free = p.fixed == 0
        assert np.linalg.norm((u - uref)[free]) <= 1e-4 * np.linalg.norm(uref[free]), mode


@gpu
def test_paper_table1_trends_gpu():
    """Table 1 sizes (h = 1/32, 1/64, 1/128; N = 4, 16, 64) on the GPU path: H_theta nearly flat in h, S~ = I
    growing like the paper's column, H_theta growing with N."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    its = {}
    for n in (4, 16, 64):
        for ih in (32, 64, 128):
            p = paper_problem(ih, n)
            its[("H", n, ih)] = _gpu_solve(p)[2]
            its[("I", n, ih)] = _gpu_solve(p, inner_mode=3)[2]
    for n in (4, 16, 64):
        h = [its[("H", n, ih)] for ih in (32, 64, 128)]
        i = [its[("I", n, ih)] for ih in (32, 64, 128)]
        # measured (round 1): H 28/29/37, 58/74/74, 97/98/109; I 72/102/144, 117/165/235, 171/245/350. The
        # unpreconditioned count doubles over the 4x refinement (the paper: x2.0-2.1); H_theta grows far less
        # (k = 10 Lanczos vectors on a spectrum that widens like 1/h^2)
        assert max(h) <= 1.4 * min(h), (n, h)
        assert i[-1] >= 1.8 * i[0] and all(b >= 1.25 * a for a, b in zip(i, i[1:])), (n, i)
        assert all(3 * a < 2 * b for a, b in zip(h, i)), (n, h, i)
    for ih in (32, 64, 128):
        assert its[("H", 4, ih)] < its[("H", 16, ih)] < its[("H", 64, ih)], ih
