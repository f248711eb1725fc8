"""ORACLE (test infrastructure only) — a plain sparse direct solve of K(rho) u = f for the meshes SuperLU
cannot factor (scipy's SuperLU stops with "Not enough memory" on config 5, 4.2 M dofs, and on config 4).

What it computes: the plain definition of the result, u = K_ff^-1 f_f on the free dofs (PAPER.md:112-114,
Eq. (4)), by a textbook multifrontal Cholesky factorisation K = L L^T in a geometric
nested-dissection order (George 1973): the node grid is bisected recursively along its longest axis by a
one-node-thick separator plane (Q1 elements couple nodes at most one grid step apart, so the plane splits
the two halves), children are ordered before their separator, and each tree node's frontal matrix
  F_t = [[K_PP, K_PU], [K_UP, 0]] + extend-add of the children's update matrices
(P = the tree node's own dofs, U = the not-yet-eliminated dofs its subtree couples to) is partially
factored: L_PP = chol(F_PP), L_UP = F_UP L_PP^-T, update F_UU - L_UP L_UP^T to the parent. Forward and
backward substitution walk the same tree. Library primitives: numpy.linalg.cholesky, scipy triangular solves.
Nothing is reordered or approximated beyond the elimination order, so the result is the exact solve up to
rounding.

refine_dd: iterative refinement with the residual computed in extended precision (numpy longdouble, 64-bit
mantissa on x86-64): u is carried as an unevaluated sum hi + lo, so fl(hi + lo) is the solution rounded to
FP64 (the quantity whose residual is the FP64 floor of the final-residual gate, R17).

Pinned by (tests/test_oracle_direct.py): equality with SuperLU (`monolithic_solve`) on 2D and 3D grids
SuperLU can factor, including Dirichlet rollers and SIMP contrast; a dense numpy solve on a tiny grid; the
patch test (linear fields) through this solver.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import os

from threadpoolctl import ThreadpoolController

from .fem import free_system, element_stiffness, simp_modulus, element_dofs


# ---------------------------------------------------------------- nested-dissection tree (node level)

def nd_tree(nn, leaf=64):
    """Post-ordered tree of the node grid nn = (nodes per axis): list of (node_ids, child_indices).
    A box with more than `leaf` nodes is split along its longest axis at the middle node plane."""
    dim = len(nn)
    out = []

    def box_nodes(lo, hi):
        grids = np.meshgrid(*[np.arange(l, h) for l, h in zip(reversed(lo), reversed(hi))], indexing="ij")
        idx = [g.ravel() for g in reversed(grids)]
        node = idx[0].astype(np.int64)
        stride = nn[0]
        for d in range(1, dim):
            node = node + idx[d].astype(np.int64) * stride
            stride *= nn[d]
        return node

    def rec(lo, hi):
        sizes = [h - l for l, h in zip(lo, hi)]
        if min(sizes) <= 0:
            return None
        if int(np.prod(sizes)) <= leaf or max(sizes) < 3:
            out.append((box_nodes(lo, hi), []))
            return len(out) - 1
        a = int(np.argmax(sizes))
        mid = (lo[a] + hi[a]) // 2
        h1 = list(hi); h1[a] = mid
        l2 = list(lo); l2[a] = mid + 1
        kids = [k for k in (rec(lo, tuple(h1)), rec(tuple(l2), hi)) if k is not None]
        ls = list(lo); ls[a] = mid
        hs = list(hi); hs[a] = mid + 1
        out.append((box_nodes(tuple(ls), tuple(hs)), kids))
        return len(out) - 1

    rec(tuple(0 for _ in nn), tuple(nn))
    return out


# ---------------------------------------------------------------- multifrontal Cholesky

class NDCholesky:
    """K = L L^T of an SPD matrix over the free dofs, elimination order from nd_tree."""

    def __init__(self, K: sp.csr_matrix, dim: int, nn, free: np.ndarray, leaf: int = 64):
        ndof = dim * int(np.prod(nn))
        red = -np.ones(ndof, dtype=np.int64)          # global dof -> free-system index
        red[free] = np.arange(len(free))
        tree = nd_tree(tuple(nn), leaf)
        piv = []
        for nodes, _ in tree:
            d = (dim * nodes[:, None] + np.arange(dim)[None, :]).ravel()
            d = red[d]
            piv.append(d[d >= 0])
        order = np.concatenate(piv)
        assert len(order) == K.shape[0] and len(np.unique(order)) == len(order)
        pos = np.empty(len(order), dtype=np.int64)
        pos[order] = np.arange(len(order))
        K = K.tocsr()
        self.fronts = []
        upd = {}
        last = 0
        where = -np.ones(K.shape[0], dtype=np.int64)   # dof -> column of the current front
        # OpenBLAS threads only pay on large fronts (measured: 8 threads on the small ones are 13x slower)
        ctl = ThreadpoolController()
        with ctl.limit(limits=1, user_api="blas"):
            for t, (nodes, kids) in enumerate(tree):
                P = piv[t]
                last += len(P)
                sub = K[P]
                cand = [sub.indices.astype(np.int64)] + [upd[k][0] for k in kids]
                cand = np.unique(np.concatenate(cand))
                U = cand[pos[cand] >= last]            # not yet eliminated (pos of the subtree < last)
                idx = np.concatenate([P, U])
                m, n = len(P), len(idx)
                where[idx] = np.arange(n)
                F = np.zeros((n, n))
                rows = np.repeat(np.arange(m), np.diff(sub.indptr))
                cols = where[sub.indices]
                keep = cols >= 0                       # entries to eliminated dofs were taken by the children
                F[rows[keep], cols[keep]] = sub.data[keep]
                F[m:, :m] = F[:m, m:].T
                for k in kids:
                    Uk, Mk = upd.pop(k)
                    loc = where[Uk]
                    F[np.ix_(loc, loc)] += Mk
                where[idx] = -1
                if m:
                    if n >= 1024:
                        with ctl.limit(limits=os.cpu_count() or 1, user_api="blas"):
                            Lpp, Lup, Mt = self._partial(F, m)
                    else:
                        Lpp, Lup, Mt = self._partial(F, m)
                else:
                    Lpp, Lup, Mt = np.zeros((0, 0)), np.zeros((len(U), 0)), F[m:, m:]
                self.fronts.append((P, U, Lpp, np.ascontiguousarray(Lup)))
                upd[t] = (U, Mt)
        self.n = K.shape[0]
        self._ctl = ctl

    @staticmethod
    def _partial(F, m):
        Lpp = np.linalg.cholesky(F[:m, :m])            # raises LinAlgError if not SPD
        Lup = sla.solve_triangular(Lpp, F[:m, m:], lower=True, check_finite=False).T
        return Lpp, Lup, F[m:, m:] - Lup @ Lup.T

    def solve(self, b: np.ndarray) -> np.ndarray:
        with self._ctl.limit(limits=1, user_api="blas"):
            return self._solve(b)

    def _solve(self, b: np.ndarray) -> np.ndarray:
        y = np.array(b, dtype=np.float64, copy=True)
        for P, U, Lpp, Lup in self.fronts:             # forward: L y = b
            if len(P):
                yp = sla.solve_triangular(Lpp, y[P], lower=True, check_finite=False)
                y[P] = yp
                if len(U):
                    y[U] -= Lup @ yp
        x = y
        for P, U, Lpp, Lup in reversed(self.fronts):   # backward: L^T x = y
            if len(P):
                r = x[P] - (Lup.T @ x[U] if len(U) else 0.0)
                x[P] = sla.solve_triangular(Lpp, r, lower=True, trans="T", check_finite=False)
        return x


def direct_solve(prob, leaf: int = 64):
    """u (full dof vector, 0 at Dirichlet dofs) = K_ff^-1 f_f by the nested-dissection Cholesky."""
    K, f, free = free_system(prob)
    u = np.zeros(prob.ndof)
    if len(free):
        ch = NDCholesky(K, prob.dim, prob.nnodes_axis, free, leaf)
        u[free] = ch.solve(f)
    return u


# ---------------------------------------------------------------- extended-precision residual + refinement

def apply_K_ext(prob, u_hi, u_lo=None):
    """K (u_hi + u_lo) over all dofs in numpy longdouble (element-by-element, PAPER.md:286 / Eq. (4))."""
    KE = element_stiffness(prob.dim, prob.nu, 1.0, prob.h).astype(np.longdouble)
    E_e = simp_modulus(prob.density, prob.E0, prob.Emin, prob.p).astype(np.longdouble)
    edofs = element_dofs(prob.dim, prob.nel)
    u = np.asarray(u_hi, dtype=np.longdouble)
    if u_lo is not None:
        u = u + np.asarray(u_lo, dtype=np.longdouble)
    out = np.zeros(prob.ndof, dtype=np.longdouble)
    m = edofs.shape[1]
    for a in range(m):                                 # out[edofs[:, a]] += E_e * sum_b KE[a, b] u[edofs[:, b]]
        acc = np.zeros(edofs.shape[0], dtype=np.longdouble)
        for b in range(m):
            acc += KE[a, b] * u[edofs[:, b]]
        np.add.at(out, edofs[:, a], E_e * acc)
    return out


def residual_ext(prob, u_hi, u_lo=None):
    """(f - K u) on the free dofs in longdouble (0 at Dirichlet dofs)."""
    r = np.asarray(prob.rhs, dtype=np.longdouble) - apply_K_ext(prob, u_hi, u_lo)
    r[prob.fixed != 0] = 0
    return r


def relres_ext(prob, u_hi, u_lo=None) -> float:
    """||f - K u||_2 / ||f_free||_2 with the residual in longdouble (R17 floor measurement)."""
    r = residual_ext(prob, u_hi, u_lo)
    nf = np.linalg.norm(prob.rhs[prob.fixed == 0])
    return float(np.sqrt(np.sum(r * r)) / nf)


def refine_dd(prob, rounds: int = 3, leaf: int = 64, solver: NDCholesky | None = None):
    """u_ref as hi + lo: the direct solve, then `rounds` refinement steps with longdouble residuals.
    Returns (u_hi, u_lo, history of relres of fl(hi + lo))."""
    K, f, free = free_system(prob)
    ch = solver or NDCholesky(K, prob.dim, prob.nnodes_axis, free, leaf)
    hi = np.zeros(prob.ndof)
    hi[free] = ch.solve(f)
    lo = np.zeros(prob.ndof)
    hist = [relres_ext(prob, hi)]
    for _ in range(rounds):
        r = residual_ext(prob, hi, lo)
        d = np.zeros(prob.ndof)
        d[free] = ch.solve(np.asarray(r[free], dtype=np.float64))
        s = np.asarray(hi, dtype=np.longdouble) + np.asarray(lo, dtype=np.longdouble) + d
        hi = np.asarray(s, dtype=np.float64)
        lo = np.asarray(s - hi, dtype=np.float64)
        hist.append(relres_ext(prob, hi))
    return hi, lo, hist
