"""ORACLE (test infrastructure only) — interface preconditioner S~ = H^_theta.

Paper: Eq.(8) H_theta = M + M(M^-1 L)^(1-theta);
PAPER.md:173-175 H~_theta = M(M^-1 L)^(1-theta); Eq.(9)
H^_theta = (+)_{1..d} H~_theta (component-wise); PAPER.md:181,191 (fractional
powers by generalised eigendecomposition for small problems; inverse Lanczos
"delivered the most promising results"); PAPER.md:235-237,273 (inner PCG on
the interface Laplacian preconditioned by L restricted to faces with the
cross points removed, tol 1e-3).  SPEC.md:374-413 fixes the interface used
here (seed M^-1 v, k = 10, explicit Rayleigh-Ritz, Jacobi at cross points).

Readings: R7 singular components use H_theta (f(l) = 1/(1+l^(1-theta)))
with (L+M)^-1 M as the Lanczos operator; R9 Lanczos details (CGS2 in the
M-inner product, breakdown threshold 1e-12, zero input -> zero output);
R10 inner modes: 'X' exact solve of K_c (the tol->0 limit of 'F'),
'F' face-preconditioned PCG (tol 1e-3, x0 = 0, cap 1000).

Pins (tests/test_oracle_trace_precond.py): SPEC.md:260 scalar example (M=[2], L=[8],
theta=1/2 -> H~v = 4, H~^-1 v = 0.25); theta = 1 gives M^-1 v; a pencil
eigenvector input returns lambda^(theta-1) times itself; k = n inverse Lanczos
equals the dense fractional inverse (1e-8) for theta in {1/4,1/2,3/4};
block diagonality; single-face topology makes the face preconditioner exact.
Inverse Lanczos at k < n is "parity unpinned" beyond these properties.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .topology import component_skeletons
from .trace import component_trace_matrices


class Breakdown(RuntimeError):
    pass


def frac_weight(lam, theta, singular):
    """Spectral function of the (inverse) preconditioner: lambda^(theta-1) for
    H~_theta^-1; 1/(1+lambda^(1-theta)) for H_theta^-1 (Eq.(8))."""
    lam = np.asarray(lam, dtype=np.float64)
    if singular:
        return 1.0 / (1.0 + np.maximum(lam, 0.0) ** (1.0 - theta))
    return lam ** (theta - 1.0)


def dense_fractional(M, L, theta, v, sign=-1, singular=False):
    """Dense H~_theta^{sign} v via L Phi = M Phi Lambda, Phi^T M Phi = I
    (PAPER.md:181)."""
    Md = M.toarray() if sp.issparse(M) else np.asarray(M, dtype=float)
    Ld = L.toarray() if sp.issparse(L) else np.asarray(L, dtype=float)
    lam, Phi = sla.eigh(Ld, Md)
    if sign < 0:
        return Phi @ (frac_weight(lam, theta, singular) * (Phi.T @ v))
    w = (1.0 + np.maximum(lam, 0) ** (1 - theta)) if singular else lam ** (1.0 - theta)
    return Md @ (Phi @ (w * (Phi.T @ (Md @ v))))


def pcg_plain(apply_A, b, apply_P, tol, maxit):
    """Textbook PCG (used for the inner face-preconditioned solve, mode F)."""
    x = np.zeros_like(b)
    r = b.copy()
    nb = np.linalg.norm(b)
    if nb == 0:
        return x, 0
    z = apply_P(r)
    p = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        q = apply_A(p)
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        if np.linalg.norm(r) <= tol * nb:
            return x, it
        z = apply_P(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return x, maxit


@dataclass
class ComponentData:
    skel: object
    M: sp.csr_matrix
    L: sp.csr_matrix
    singular: bool
    K: sp.csr_matrix            # L (or L + M when singular)
    _Klu: object = None
    _Mlu: object = None
    _face_lu: list = None
    _cross_diag: np.ndarray = None

    def M_solve(self, b):
        if self._Mlu is None:
            self._Mlu = spla.splu(self.M.tocsc())
        return self._Mlu.solve(b)

    def K_solve_exact(self, b):
        if self._Klu is None:
            self._Klu = spla.splu(self.K.tocsc())
        return self._Klu.solve(b)

    def face_precond(self, r):
        """K restricted to each face (cross points removed) inverted
        exactly; Jacobi (diag K) at cross points."""
        if self._face_lu is None:
            self._face_lu = []
            for f in self.skel.faces:
                Kf = self.K[f][:, f].toarray()
                self._face_lu.append(sla.cho_factor(Kf, lower=True))
            self._cross_diag = self.K.diagonal()[self.skel.cross]
        z = np.zeros_like(r)
        for f, lu in zip(self.skel.faces, self._face_lu):
            z[f] = sla.cho_solve(lu, r[f])
        z[self.skel.cross] = r[self.skel.cross] / self._cross_diag
        return z

    inner_tol = 1e-3          # SPEC.md:411 ("relatively coarse tolerance for PCG of 1e-3")
    inner_maxit = 1000

    def K_solve_face_pcg(self, b):
        x, its = pcg_plain(lambda v: self.K @ v, b, self.face_precond, self.inner_tol, self.inner_maxit)
        self.inner_its.append(its)
        return x


def build_components(prob, topo, weighted=False):
    comps = []
    for skel in component_skeletons(prob, topo):
        M, L, singular = component_trace_matrices(prob, skel, weighted)
        K = (L + M).tocsr() if singular else L
        cd = ComponentData(skel, M, L, singular, K)
        cd.inner_its = []
        comps.append(cd)
    return comps


def inverse_lanczos(cd: ComponentData, r, k, theta, inner="X", breakdown_tol=1e-12):
    """z ~= H~_theta^-1 r by k-step inverse Lanczos (
    DESIGN.md R9):
      s = M^-1 r;  q1 = s/||s||_M
      q_{j+1} ~ K^-1 M q_j, orthogonalised twice (classical GS, M-inner product)
      A_k = W^T L W, B_k = W^T M W;  (Theta, Y) = eig(A_k, B_k), Y^T B_k Y = I
      z = W Y f(Theta) Y^T W^T r."""
    if not np.any(r):
        return np.zeros_like(r)
    M, L = cd.M, cd.L
    solve = cd.K_solve_exact if inner == "X" else cd.K_solve_face_pcg
    s = cd.M_solve(r)
    W = [s / np.sqrt(s @ (M @ s))]
    for _ in range(1, k):
        w = solve(M @ W[-1])
        nb = np.sqrt(w @ (M @ w))
        Wm = np.stack(W, axis=1)
        for _pass in range(2):
            h = Wm.T @ (M @ w)
            w = w - Wm @ h
        na = np.sqrt(max(w @ (M @ w), 0.0))
        if not (na > breakdown_tol * nb):
            break
        W.append(w / na)
    Wm = np.stack(W, axis=1)
    A = Wm.T @ (L @ Wm)
    B = Wm.T @ (M @ Wm)
    A = 0.5 * (A + A.T)
    B = 0.5 * (B + B.T)
    th, Y = sla.eigh(A, B)
    if not cd.singular and np.any(th <= 0):
        raise Breakdown("non-positive Ritz value")
    return Wm @ (Y @ (frac_weight(th, theta, cd.singular) * (Y.T @ (Wm.T @ r))))


def apply_precond(comps, r, mode="lanczos", theta=0.5, k=10, inner="X"):
    """Component-wise z = H^_theta^-1 r (Eq.(9)); mode in
    {'identity', 'dense', 'lanczos'}."""
    if mode == "identity":
        return r.copy()
    z = np.zeros_like(r)
    for cd in comps:
        rc = r[cd.skel.gidx]
        if mode == "dense":
            zc = dense_fractional(cd.M, cd.L, theta, rc, -1, cd.singular) if len(rc) else rc
        else:
            zc = inverse_lanczos(cd, rc, k, theta, inner) if len(rc) else rc
        z[cd.skel.gidx] = zc
    return z
