"""ORACLE (test infrastructure only) — end-to-end reference solves.

monolithic_solve: the plain definition of the result — u solves K(rho) u = f
on the free dofs (Eq.(4)), by SuperLU.
dd_solve: the method step by step in the paper's order (PAPER.md:137-146
Eq.(7)): interior factorisations -> condensed rhs -> interface PCG with
H^_theta -> back-substitution.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np
import scipy.sparse.linalg as spla

from dataclasses import replace

from .fem import free_system, true_relres, apply_K
from .topology import build_topology
from .dd import (subdomain_blocks, factor_subdomains, schur_apply, condensed_rhs, back_substitute, solve_II,
                 dense_schur)
from .precond import build_components, apply_precond
from .krylov import pcg, fgmres


def monolithic_solve(prob):
    K, f, free = free_system(prob)
    u = np.zeros(prob.ndof)
    if len(free):
        u[free] = spla.splu(K.tocsc()).solve(f)
    return u


@dataclass
class DDResult:
    u: np.ndarray
    iterations: int
    converged: bool
    relres: float
    uG: np.ndarray
    history: list = field(default_factory=list)
    its_pass1: int = 0


class DDOracle:
    """Setup/factor/solve split mirroring de_setup / de_factor / de_solve."""

    def __init__(self, prob, mode="lanczos", theta=0.5, k=10, inner="X", beta="FR", weighted=False):
        self.prob = prob
        self.topo = build_topology(prob)
        self.weighted = weighted
        self.comps = build_components(prob, self.topo, weighted) if mode != "identity" else []
        self.mode, self.theta, self.k, self.inner, self.beta = mode, theta, k, inner, beta
        self.blocks = None
        self.uG_prev = None

    def factor(self, prob=None):
        if prob is not None:
            self.prob = prob
            if self.weighted and self.mode != "identity":   # R19: the weighted norm follows the densities
                self.comps = build_components(self.prob, self.topo, True)
        self.blocks = factor_subdomains(subdomain_blocks(self.prob, self.topo))

    def S(self, x):
        return schur_apply(self.blocks, self.topo.n_G, x)

    def P(self, r):
        return apply_precond(self.comps, r, self.mode, self.theta, self.k, self.inner)

    def _dd_solve(self, rhs, tol_abs, maxit, x0):
        """One pass of Eq. (7) for the load vector `rhs`."""
        prob = replace(self.prob, rhs=rhs)
        g = condensed_rhs(prob, self.topo, self.blocks)
        uG, its, conv, hist = pcg(self.S, g, self.P, tol_abs, maxit, x0=x0, beta=self.beta)
        return back_substitute(prob, self.topo, self.blocks, uG), its, conv, hist

    def P_full(self, v, exact_S=None):
        """P~^-1 v on a full dof vector: z_Gamma = S~^-1 v_Gamma, then
        z_I = K_II^-1 (v_I - K_IGamma z_Gamma) per subdomain; Dirichlet entries 0."""
        topo = self.topo
        vG = v[topo.gamma_dofs]
        zG = np.linalg.solve(exact_S, vG) if exact_S is not None else self.P(vG)
        z = np.zeros_like(v)
        z[topo.gamma_dofs] = zG
        for b in self.blocks:
            if len(b.I):
                z[b.I] = solve_II(b, v[b.I] - b.AIG @ zG[b.R])
        return z

    def solve_fgmres(self, rtol=None, maxit=2000, restart=30, exact_S=False):
        """The paper's formulation (NEXT(4)): right-preconditioned flexible GMRES on the
        full system K u = f over the free dofs with P~ = [[K_II, K_IGamma], [0, S~]], S~ = H_theta (or the exact
        Schur complement when exact_S). Stop: ||f - K u|| <= rtol ||f_free|| (the estimate, then the true
        residual at each restart). Returns DDResult."""
        prob = self.prob
        rtol = prob.rtol if rtol is None else rtol
        if self.blocks is None:
            self.factor()
        free = prob.fixed == 0
        Sd = dense_schur(self.blocks, self.topo.n_G) if exact_S else None

        def A(u):
            out = apply_K(prob, u)
            out[~free] = 0.0
            return out

        b = np.where(free, prob.rhs, 0.0)
        nf = np.linalg.norm(b)
        u, its, conv, hist = fgmres(A, b, lambda v: self.P_full(v, Sd), rtol * nf, maxit, restart)
        return DDResult(u=u, iterations=its, converged=conv, relres=true_relres(prob, u),
                        uG=u[self.topo.gamma_dofs], history=hist, its_pass1=its)

    def solve(self, rtol=None, maxit=20000, warm=False, max_refine=3):
        """Interface PCG to ||r_Gamma|| <= rtol ||f_free|| (recursive residual), then iterative
        refinement on the full system while the true ||f - K u|| > rtol ||f|| (R11):
        u += DD-solve(f - K u) with the interface tolerance 0.5 rtol ||f||, at most max_refine times,
        and only while each round at least halves the residual."""
        prob = self.prob
        rtol = prob.rtol if rtol is None else rtol
        if self.blocks is None:
            self.factor()
        free = prob.fixed == 0
        nf = np.linalg.norm(prob.rhs[free])
        if nf == 0:
            return DDResult(np.zeros(prob.ndof), 0, True, 0.0, np.zeros(self.topo.n_G))
        x0 = self.uG_prev if (warm and self.uG_prev is not None) else None
        u, its, conv, hist = self._dd_solve(prob.rhs, rtol * nf, maxit, x0)
        its1 = its
        relres = true_relres(prob, u)
        prev = np.inf
        for _ in range(max_refine):
            # stop when converged, or when a round no longer halves the residual (FP64 floor)
            if relres <= rtol or not conv or its >= maxit or not relres < 0.5 * prev:
                break
            prev = relres
            res = np.where(free, prob.rhs - apply_K(prob, u), 0.0)
            du, k, conv, h2 = self._dd_solve(res, 0.5 * rtol * nf, maxit - its, None)
            u = u + du
            its += k
            hist += h2
            relres = true_relres(prob, u)
        uG = u[self.topo.gamma_dofs]
        self.uG_prev = uG
        return DDResult(u, its, conv and relres <= rtol, relres, uG, hist, its1)
