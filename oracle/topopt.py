"""ORACLE (test infrastructure only) — one optimality-criteria (OC) design update.

Paper: PAPER.md:283-306 (the topology-optimisation application: minimum compliance with a volume constraint,
densities updated between the finite element solves). The paper does not state its OC constants; reading R20
(DESIGN.md): the standard optimality-criteria update for minimum compliance,
    dc_e = -p rho_e^(p-1) (E0 - Emin) u_e^T KE0 u_e          (compliance sensitivity, modified SIMP)
    B_e(lambda) = -dc_e / lambda                               (dv_e = 1: unit element volumes)
    rho_e' = clip(rho_e * B_e^eta, max(rho_min, rho_e - move), min(1, rho_e + move))
with lambda found by bisection so that sum rho_e' = V * n_elem; eta = 1/2. VTS is p = 1, Emin = 0.

Pins (tests/test_topopt.py): compliance f.u = sum_e E_e u_e^T KE0 u_e (energy identity); a uniform sensitivity
field returns the uniform design rho = V; the volume constraint holds to the bisection tolerance; the update
respects the move limit and the bounds.
"""
from __future__ import annotations

import numpy as np

from .fem import element_stiffness, simp_modulus, element_dofs


def element_energies(prob, u):
    """u_e^T KE0 u_e per element (unit-modulus element stiffness)."""
    KE = element_stiffness(prob.dim, prob.nu, 1.0, prob.h)
    ue = u[element_dofs(prob.dim, prob.nel)]
    return np.einsum("ei,ij,ej->e", ue, KE, ue)


def compliance(prob, u):
    E = simp_modulus(prob.density, prob.E0, prob.Emin, prob.p)
    return float(np.sum(E * element_energies(prob, u)))


def sensitivities(prob, u):
    rho = prob.density
    return -prob.p * rho ** (prob.p - 1.0) * (prob.E0 - prob.Emin) * element_energies(prob, u)


def oc_update(rho, dc, volfrac, move=0.2, rho_min=1e-3, eta=0.5, tol=1e-12, maxit=200):
    """Bisection on lambda in [0, lmax] until (l2 - l1) <= tol (l1 + l2) (at most maxit halvings)."""
    n = rho.size
    target = volfrac * n
    lo_b = np.maximum(rho_min, rho - move)
    hi_b = np.minimum(1.0, rho + move)
    g = np.maximum(-dc, 0.0)
    l1, l2 = 0.0, max(float(g.max()), 1e-300) * 1e9
    for _ in range(maxit):
        lm = 0.5 * (l1 + l2)
        new = np.clip(rho * (g / lm) ** eta, lo_b, hi_b)
        if new.sum() > target:
            l1 = lm
        else:
            l2 = lm
        if l2 - l1 <= tol * (l1 + l2):
            break
    lm = 0.5 * (l1 + l2)
    return np.clip(rho * (g / lm) ** eta, lo_b, hi_b), lm
