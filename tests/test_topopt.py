"""Topology-optimisation design update (R20): compliance
sensitivities and one optimality-criteria step, oracle (oracle/topopt.py) pinned, then the GPU path
(de_sensitivities_device / de_oc_update_device / de_oc_step) against it.

Pins of the oracle, each independent of its formulas:
  * energy identity: sum_e E_e u_e^T KE0 u_e = f.u for the assembled solve (a wrong KE, gather or modulus fails);
  * the sensitivity equals the central finite difference of the compliance f.u(rho) computed by re-solving
    (the adjoint claim dc/drho_e = -u^T dK/drho_e u; a dropped factor p or a sign fails);
  * a uniform sensitivity field maps a uniform design onto the uniform design rho = V;
  * on a random field: the volume constraint holds to the bisection tolerance, the move limit and the bounds
    hold, and every element strictly inside its bounds satisfies the OC fixed point rho' = rho (g/lambda)^eta."""
import numpy as np
import pytest
import torch

from synthetic import make_config
from oracle.solver import monolithic_solve
from oracle.topopt import compliance, sensitivities, oc_update, element_energies
from oracle.fem import element_stiffness, element_dofs, simp_modulus

EPS = np.finfo(np.float64).eps


def _energy_error_bounds(p, u):
    """Forward-error bound of u_e^T KE0 u_e evaluated in any summation order: two nested length-nke dot
    products, so |computed - exact| <= 2 nke eps |u_e|^T |KE0| |u_e| (Higham's gamma_n, first order); the
    rigid-body part of u_e cancels only in exact arithmetic (large |u_e|, small energy at a cantilever tip), so
    the bound is relative to |u_e|^T|KE0||u_e|, not to the energy. Two independent evaluations differ by at most
    twice that; returned per element for dc and summed (weighted by E, plus the n_elem-term sum) for c."""
    KE = element_stiffness(p.dim, p.nu, 1.0, p.h)
    ue = np.abs(u[element_dofs(p.dim, p.nel)])
    mag = np.einsum("ei,ij,ej->e", ue, np.abs(KE), ue)
    nke = KE.shape[0]
    per = 2.0 * 2 * nke * EPS * mag
    scale = p.p * p.density ** (p.p - 1.0) * (p.E0 - p.Emin)
    E = simp_modulus(p.density, p.E0, p.Emin, p.p)
    return per * scale, float(np.sum(E * per)) + p.nelem * EPS * float(np.sum(E * mag))


def _small(dim=2):
    if dim == 2:
        return make_config("c2", nel=(24, 12), sub=(8, 6))
    return make_config("c4", nel=(8, 4, 4), sub=(4, 4, 4))


@pytest.mark.parametrize("dim", [2, 3])
def test_energy_identity(dim):
    p = _small(dim)
    u = monolithic_solve(p)
    c = compliance(p, u)
    fu = float(p.rhs[p.fixed == 0] @ u[p.fixed == 0])
    assert abs(c - fu) <= 1e-10 * abs(fu)
    assert np.all(element_energies(p, u) >= -1e-14 * abs(fu))


@pytest.mark.parametrize("dim", [2, 3])
def test_sensitivity_matches_finite_difference(dim):
    p = _small(dim)
    u = monolithic_solve(p)
    dc = sensitivities(p, u)
    rng = np.random.default_rng(11)
    for e in rng.choice(p.nelem, 4, replace=False):
        d = 1e-5 * p.density[e]
        cs = []
        for sgn in (1, -1):
            rho = p.density.copy()
            rho[e] += sgn * d
            q = p.with_density(rho)
            cs.append(float(q.rhs[q.fixed == 0] @ monolithic_solve(q)[q.fixed == 0]))
        fd = (cs[0] - cs[1]) / (2 * d)
        assert abs(fd - dc[e]) <= 1e-5 * abs(dc[e]) + 1e-12 * abs(dc).max(), (e, fd, dc[e])
    assert np.all(dc <= 0)


def test_uniform_sensitivity_gives_uniform_design():
    rho = np.full(500, 0.6)
    new, lam = oc_update(rho, np.full(500, -2.0), volfrac=0.5, move=0.2)
    assert np.allclose(new, 0.5, rtol=0, atol=1e-10)
    assert np.isclose(lam, 2.0 * (0.6 / 0.5) ** 2, rtol=1e-9)     # 0.6 sqrt(2/lam) = 0.5


def test_oc_update_constraint_bounds_fixed_point():
    rng = np.random.default_rng(5)
    n = 4000
    rho = rng.uniform(0.05, 1.0, n)
    dc = -rng.lognormal(0.0, 2.0, n)
    dc[::97] = 0.0                                  # zero sensitivity: the lower bound
    V, move, rmin = 0.4, 0.15, 1e-3
    new, lam = oc_update(rho, dc, V, move=move, rho_min=rmin)
    assert abs(new.sum() - V * n) <= 1e-8 * V * n
    lo, hi = np.maximum(rmin, rho - move), np.minimum(1.0, rho + move)
    assert np.all(new >= lo) and np.all(new <= hi)
    inner = (new > lo + 1e-12) & (new < hi - 1e-12)
    assert inner.sum() > n // 10
    ref = rho[inner] * np.sqrt(-dc[inner] / lam)
    assert np.allclose(new[inner], ref, rtol=1e-13, atol=0)
    assert np.all(new[dc == 0] == lo[dc == 0])


def test_oc_params_rejected_before_device():
    from paper_1501_06211_b200 import binding as B
    p = _small(2)
    S = B.Solver.from_problem(p, host_only=1)
    try:
        for bad in (dict(volfrac=0.0), dict(move=-1.0), dict(rho_min=1.0), dict(eta=0.0), dict(maxit=0)):
            with pytest.raises(B.DEError) as ei:
                S.oc_step(np.zeros(p.ndof), p.nelem, **bad)
            assert ei.value.status == B.DE_EINVAL, bad
    finally:
        S.close()


# ----------------------------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name,nel,sub", [("c2", (64, 32), (16, 16)), ("c2", (100, 36), (20, 12)),
                                          ("c4", (24, 12, 12), (6, 6, 6))])
def test_gpu_sensitivities_and_oc_match_oracle(name, nel, sub):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_06211_b200 import binding as B
    p = make_config(name, nel=nel, sub=sub)
    S = B.Solver.from_problem(p, device=0)
    try:
        S.factor()
        u, *_ = S.solve(p.rhs, 1e-10)
        du = torch.tensor(u, device="cuda")
        ddc = torch.empty(p.nelem, dtype=torch.float64, device="cuda")
        c = B.de_sensitivities_device(S.ctx, du.data_ptr(), ddc.data_ptr())
        dc = ddc.cpu().numpy()
        ref = sensitivities(p, u)
        b_dc, b_c = _energy_error_bounds(p, u)
        assert np.all(np.abs(dc - ref) <= b_dc)
        assert abs(c - compliance(p, u)) <= b_c
        prm = B.de_default_oc_params(volfrac=0.45, move=0.2)
        drho = torch.empty(p.nelem, dtype=torch.float64, device="cuda")
        lam = B.de_oc_update_device(S.ctx, ddc.data_ptr(), prm, drho.data_ptr())
        new_ref, lam_ref = oc_update(p.density, dc, 0.45, move=0.2)   # same dc on both sides
        assert abs(lam - lam_ref) <= 1e-10 * lam_ref
        assert np.abs(drho.cpu().numpy() - new_ref).max() <= 1e-9
        # the context now holds the new design: factor + solve must reproduce the oracle solve for it
        S.factor()
        u2, *_ = S.solve(p.rhs, 1e-10)
        q = p.with_density(drho.cpu().numpy())
        uref = monolithic_solve(q)
        free = q.fixed == 0
        assert np.linalg.norm((u2 - uref)[free]) <= 1e-7 * np.linalg.norm(uref[free])
    finally:
        S.close()


@pytest.mark.gpu
def test_gpu_topopt_loop_matches_oracle_loop():
    """Three design iterations (solve -> sensitivities -> OC -> factor) through the host-buffer call
    de_oc_step, against the same loop on the oracle (monolithic solve + oracle OC). The GPU step is checked
    against the oracle evaluated at the GPU's own u (parity of the step), the trajectories against each other
    with a tolerance set by the solve accuracy (u differs from the direct solve by ~1e-8 relative)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_06211_b200 import binding as B
    p = make_config("c2", nel=(64, 32), sub=(16, 16)).with_density(np.full(64 * 32, 0.5))
    S = B.Solver.from_problem(p, device=0)
    q = p
    dens = p.density.copy()
    try:
        for it in range(3):
            S.factor()
            u, *_ = S.solve(p.rhs, 1e-11)
            rho, c, lam = S.oc_step(u, p.nelem, volfrac=0.5)
            g = p.with_density(dens)
            _, b_c = _energy_error_bounds(g, u)
            assert abs(c - compliance(g, u)) <= b_c, it
            rg, lg = oc_update(dens, sensitivities(g, u), 0.5)
            assert abs(lam - lg) <= 1e-10 * lg and np.abs(rho - rg).max() <= 1e-9, it
            assert abs(rho.sum() - 0.5 * p.nelem) <= 1e-8 * p.nelem
            uq = monolithic_solve(q)
            cq = compliance(q, uq)
            rq, _ = oc_update(q.density, sensitivities(q, uq), 0.5)
            assert abs(c - cq) <= 1e-6 * cq, (it, c, cq)
            assert np.abs(rho - rq).max() <= 1e-5, it
            q = q.with_density(rq)
            dens = rho
    finally:
        S.close()
