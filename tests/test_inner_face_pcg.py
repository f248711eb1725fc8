"""inner_mode 0 (SURVEY.md §8(a) C5 mode F, R10): inverse Lanczos whose K-solves are SPEC's face-
preconditioned PCG (tol 1e-3, x0 = 0, cap 1000) instead of the exact
elimination. The oracle's mode F (oracle/precond.py K_solve_face_pcg, pinned against mode X at a tight inner
tolerance in tests/test_oracle_trace_precond.py) is the reference; the GPU path runs the inner PCG in one
cooperative kernel per solve (k_face_pcg)."""
import numpy as np
import pytest
import torch

from synthetic import make_config
from oracle.topology import build_topology
from oracle.precond import build_components, apply_precond
from oracle.solver import DDOracle, monolithic_solve


def test_inner_mode0_argument_checks():
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    for bad in (dict(inner_tol=0.0), dict(inner_max_iter=0), dict(lanczos_k=0)):
        with pytest.raises(B.DEError) as ei:
            B.Solver.from_problem(p, host_only=1, inner_mode=0, **bad)
        assert ei.value.status == B.DE_EINVAL, bad
    S = B.Solver.from_problem(p, host_only=1, inner_mode=0)   # defaults: tol 1e-3, cap 1000
    S.close()


gpu = pytest.mark.gpu
CASES = [("c2", (64, 32), (16, 16)), ("c2", (100, 36), (20, 12)), ("c4", (16, 8, 8), (4, 4, 4))]


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_06211_b200 import binding as B
    return B


@gpu
@pytest.mark.parametrize("name,nel,sub", CASES)
def test_face_pcg_preconditioner_matches_oracle(name, nel, sub):
    """Same input r on both sides: the inner PCG takes the same number of iterations (the stopping test at 1e-3
    is far from the rounding differences of the two summation orders) and z agrees to 1e-6: with the inner
    solves stopped early, every Lanczos vector is a Krylov polynomial whose coefficients come from rounded dot
    products, and in 2D the face-preconditioned system has few distinct eigenvalues, so the stopped iterate lies
    in PCG's finite-termination phase where rounding is amplified (measured: 2.4e-7 on the 100x36 case at tol
    1e-3, 1e-12 on the same case at tol 1e-6, 1e-14 in 3D; tools/diag_face_pcg.py)."""
    B = _gpu()
    p = make_config(name, nel=nel, sub=sub)
    topo = build_topology(p)
    comps = build_components(p, topo)
    S = B.Solver.from_problem(p, device=0, inner_mode=0)
    try:
        S.factor()
        rng = np.random.default_rng(17)
        for rep in range(2):
            r = rng.normal(size=topo.n_G)
            for cd in comps:
                cd.inner_its = []
            ref = apply_precond(comps, r, "lanczos", 0.5, 10, "F")
            its_ref = sum(sum(cd.inner_its) for cd in comps)
            n0 = S.stats().inner_iterations
            dr = torch.tensor(r, dtype=torch.float64, device="cuda")
            dz = torch.empty_like(dr)
            B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr())
            z = dz.cpu().numpy()
            its = S.stats().inner_iterations - n0
            assert its == its_ref, (rep, its, its_ref)
            assert np.linalg.norm(z - ref) <= 1e-6 * np.linalg.norm(ref), rep
    finally:
        S.close()


@gpu
def test_face_pcg_tight_tolerance_equals_exact_inner():
    """At inner tol 1e-13 the face-PCG inner solve reaches the exact elimination (mode X) result: the two GPU
    inner modes then give the same preconditioner (the limit that defines mode X, R10)."""
    B = _gpu()
    p = make_config("c2", nel=(64, 32), sub=(16, 16))
    topo = build_topology(p)
    r = np.random.default_rng(3).normal(size=topo.n_G)
    dr = torch.tensor(r, dtype=torch.float64, device="cuda")
    out = []
    for kw in (dict(inner_mode=0, inner_tol=1e-13), dict(inner_mode=1)):
        S = B.Solver.from_problem(p, device=0, **kw)
        try:
            S.factor()
            dz = torch.empty_like(dr)
            B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr())
            out.append(dz.cpu().numpy())
        finally:
            S.close()
    assert np.linalg.norm(out[0] - out[1]) <= 1e-8 * np.linalg.norm(out[1])


@gpu
@pytest.mark.parametrize("name,nel,sub", CASES[:1] + CASES[2:])
def test_face_pcg_solve_matches_oracle(name, nel, sub):
    B = _gpu()
    p = make_config(name, nel=nel, sub=sub)
    S = B.Solver.from_problem(p, device=0, inner_mode=0)
    try:
        S.factor()
        u, its, rel, st = S.solve(p.rhs, 1e-10)
        its1 = S.stats().iterations_pass1
    finally:
        S.close()
    o = DDOracle(p, inner="F").solve(rtol=1e-10, maxit=3000, max_refine=0)
    assert abs(its1 - o.its_pass1) <= max(2, int(0.05 * o.its_pass1)), (its1, o.its_pass1)
    uref = monolithic_solve(p)
    free = p.fixed == 0
    assert np.linalg.norm((u - uref)[free]) <= 1e-7 * np.linalg.norm(uref[free])
