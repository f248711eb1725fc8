"""ORACLE (test infrastructure only) — non-overlapping DD algebra.

Paper: Eqs.(4)-(5) (block system, K_II = (+)_i K_IiIi),
PAPER.md:126-146 Eqs.(6)-(7) (three-step Schur solve:
  K_IiIi u1_Ii = f_Ii;  S u_Gamma = f_Gamma - sum_i K_GammaIi u1_Ii;
  K_IiIi u2_Ii = -K_IiGamma u_Gamma;  u = (u1_I,0) + (u2_I,u_Gamma)),
PAPER.md:103-107 (S = sum_i S_i, subassembled Steklov-Poincare operator).
Discrete S = sum_i R_i^T (A_GG,i - A_GI,i A_II,i^-1 A_IG,i) R_i where the
A blocks are assembled from subdomain i's elements only.

Pins (tests/test_oracle_dd_krylov.py): assembled sum_i R_i^T S_i R_i equals the dense
Schur complement K_GG - K_GI K_II^-1 K_IG of the monolithic matrix (an
independent formula); S_i symmetric PSD; kernel of a floating S_i = rigid
modes restricted to Gamma_i; DD solve with a dense exact interface solve
equals the monolithic SuperLU solve to 1e-12 on tiny grids.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np
import scipy.sparse as sp
import scipy.linalg as sla

from .fem import element_stiffness, simp_modulus, element_dofs


@dataclass
class SubBlocks:
    I: np.ndarray       # interior dofs (global ids, ascending)
    G: np.ndarray       # Gamma dofs touched (global ids, ascending)
    R: np.ndarray       # positions of G in the global Gamma list
    AII: sp.csr_matrix
    AIG: sp.csr_matrix
    AGG: sp.csr_matrix
    band: int = 0       # half bandwidth of AII (local lexicographic order)
    chol: np.ndarray = None   # lower band Cholesky factor (scipy cholesky_banded layout)


def subdomain_blocks(prob, topo, only=None):
    """A_II,i, A_IG,i, A_GG,i from subdomain i's elements only.
    `only`: optional list of subdomain ids (sampled checks at full size)."""
    KE = element_stiffness(prob.dim, prob.nu, 1.0, prob.h)
    E_e = simp_modulus(prob.density, prob.E0, prob.Emin, prob.p)
    edofs = element_dofs(prob.dim, prob.nel)
    ndof = prob.ndof
    order = np.argsort(topo.elem_sub, kind="stable")
    eb = np.searchsorted(topo.elem_sub[order], np.arange(topo.nsub + 1))
    m = edofs.shape[1]
    out = []
    for s in (range(topo.nsub) if only is None else only):
        els = order[eb[s]:eb[s + 1]]
        ed = edofs[els]
        loc, inv = np.unique(ed, return_inverse=True)
        inv = inv.reshape(ed.shape)
        rows = np.repeat(inv, m, axis=1).ravel()
        cols = np.tile(inv, (1, m)).ravel()
        vals = (E_e[els][:, None, None] * KE[None]).ravel()
        Ks = sp.coo_matrix((vals, (rows, cols)), shape=(len(loc), len(loc))).tocsr()
        I = topo.interior[s]
        G = topo.gamma_local[s]
        li = np.searchsorted(loc, I)
        lg = np.searchsorted(loc, G)
        out.append(SubBlocks(I, G, topo.R[s], Ks[li][:, li].tocsr(), Ks[li][:, lg].tocsr(),
                             Ks[lg][:, lg].tocsr()))
    return out


def half_bandwidth(A: sp.csr_matrix) -> int:
    C = A.tocoo()
    return int(np.max(np.abs(C.row - C.col))) if C.nnz else 0


def factor_subdomains(blocks):
    """Banded Cholesky A_II,i = L L^T in local lexicographic order (PAPER.md:271:
    'sparse matrix inversion (O(k^2 n), k is the bandwidth)')."""
    for b in blocks:
        n = b.AII.shape[0]
        if n == 0:
            b.band, b.chol = 0, np.zeros((1, 0))
            continue
        kb = half_bandwidth(b.AII)
        ab = np.zeros((kb + 1, n))
        C = b.AII.tocoo()
        low = C.row >= C.col
        ab[C.row[low] - C.col[low], C.col[low]] = C.data[low]
        b.band = kb
        b.chol = sla.cholesky_banded(ab, lower=True)
    return blocks


def solve_II(b: SubBlocks, rhs):
    if b.AII.shape[0] == 0:
        return np.zeros_like(rhs)
    return sla.cho_solve_banded((b.chol, True), rhs)


def local_schur_apply(b: SubBlocks, x):
    """S_i x = A_GG x - A_GI A_II^-1 A_IG x."""
    return b.AGG @ x - b.AIG.T @ solve_II(b, b.AIG @ x)


def schur_apply(blocks, n_G, p):
    """q = sum_i R_i^T S_i R_i p (implicit, through interior Dirichlet solves)."""
    q = np.zeros(n_G)
    for b in blocks:
        np.add.at(q, b.R, local_schur_apply(b, p[b.R]))
    return q


def dense_local_schur(b: SubBlocks):
    AGG = b.AGG.toarray()
    if b.AII.shape[0] == 0:
        return AGG
    X = solve_II(b, b.AIG.toarray())
    return AGG - b.AIG.T.toarray() @ X


def dense_schur(blocks, n_G):
    S = np.zeros((n_G, n_G))
    for b in blocks:
        S[np.ix_(b.R, b.R)] += dense_local_schur(b)
    return S


def condensed_rhs(prob, topo, blocks):
    """g = f_Gamma - sum_i K_GammaIi K_IiIi^-1 f_Ii  (Eq.(7) row 2)."""
    f = prob.rhs
    g = f[topo.gamma_dofs].copy()
    for b in blocks:
        if len(b.I):
            np.add.at(g, b.R, -(b.AIG.T @ solve_II(b, f[b.I])))
    return g


def back_substitute(prob, topo, blocks, uG):
    """u_Ii = K_IiIi^-1 (f_Ii - K_IiGamma u_Gamma) (PAPER.md:141,143 rows 1+3 combined,
    PAPER.md:136 u = (u1_I,0)+(u2_I,u_Gamma)); u = 0 at Dirichlet dofs."""
    u = np.zeros(prob.ndof)
    u[topo.gamma_dofs] = uG
    for b in blocks:
        if len(b.I):
            u[b.I] = solve_II(b, prob.rhs[b.I] - b.AIG @ uG[b.R])
    return u
