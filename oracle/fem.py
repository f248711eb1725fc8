"""ORACLE (test infrastructure only) — Q1 finite elements for isotropic
linear elasticity with SIMP-weighted Young's modulus.

Paper: Eq.(1) (BVP), :42-45 (linearised strain), :48-55
(Hooke's law sigma = 2 mu eps + lambda tr(eps) I, Lame constants), :286
Eq.(10) (K(rho) = sum_i rho_i K_i; here the SIMP reading of DESIGN.md R1:
E_e = Emin + rho_e^p (E0 - Emin)), :112-114 Eq.(4) (assembled system).

Pins (tests/test_oracle_fem.py): Lame closed forms; the classic closed-form
entries of the 2D plane-stress Q1 stiffness; rigid-body null spaces (3 in 2D,
6 in 3D); patch test (linear fields reproduced exactly); symmetry; SIMP(p=1,
Emin=0) linearity; load sums.
"""
from __future__ import annotations

import itertools
import numpy as np
import scipy.sparse as sp


# ---------------------------------------------------------------- material

def lame(E: float, nu: float):
    """mu = E/(2(1+nu)), lambda_hat = nu E/((1+nu)(1-2nu))."""
    mu = E / (2.0 * (1.0 + nu))
    lam = nu * E / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return mu, lam


def plane_stress_lambda(E: float, nu: float):
    """2D plane stress reduction lambda* = 2 mu lambda/(lambda + 2 mu) (R2)."""
    mu, lam = lame(E, nu)
    return 2.0 * mu * lam / (lam + 2.0 * mu)


def constitutive(dim: int, E: float, nu: float) -> np.ndarray:
    """Voigt form of sigma = 2 mu eps + lambda tr(eps) I, with
    engineering shear strains gamma = 2 eps_ij.  2D: plane stress."""
    mu, lam = lame(E, nu)
    if dim == 2:
        lam = plane_stress_lambda(E, nu)
    n = 3 if dim == 2 else 6
    D = np.zeros((n, n))
    D[:dim, :dim] = lam
    D[np.arange(dim), np.arange(dim)] += 2.0 * mu
    D[np.arange(dim, n), np.arange(dim, n)] = mu
    return D


# ---------------------------------------------------------------- element

def local_nodes(dim: int):
    """Element-local node offsets, lexicographic (x fastest): a -> (ax, ay[, az])."""
    return [tuple(reversed(t)) for t in itertools.product((0, 1), repeat=dim)]


def _shape_grad(dim, xi, h):
    """Gradients (w.r.t. physical x) of the 2^d trilinear shape functions of
    the element [0,h]^d at reference point xi in [0,1]^d."""
    offs = local_nodes(dim)
    G = np.zeros((len(offs), dim))
    for a, o in enumerate(offs):
        for d in range(dim):
            g = 1.0
            for e in range(dim):
                if e == d:
                    g *= (1.0 if o[e] else -1.0)
                else:
                    g *= (xi[e] if o[e] else 1.0 - xi[e])
            G[a, d] = g / h
    return G


def strain_displacement(dim, G):
    """B matrix: eps_voigt = B u_e, u_e = (u_x, u_y[, u_z]) per local node (component fastest).
    PAPER.md:44 eps_ij = (du_i/dx_j + du_j/dx_i)/2; shear rows hold gamma = 2 eps_ij."""
    nn = G.shape[0]
    n = 3 if dim == 2 else 6
    B = np.zeros((n, dim * nn))
    shear = [(0, 1)] if dim == 2 else [(0, 1), (1, 2), (0, 2)]
    for a in range(nn):
        for d in range(dim):
            B[d, dim * a + d] = G[a, d]
        for s, (i, j) in enumerate(shear):
            B[dim + s, dim * a + i] = G[a, j]
            B[dim + s, dim * a + j] = G[a, i]
    return B


def element_stiffness(dim: int, nu: float, E: float = 1.0, h: float = 1.0) -> np.ndarray:
    """KE = int_{[0,h]^d} B^T D B dV by 2^d-point Gauss quadrature (exact for Q1)."""
    D = constitutive(dim, E, nu)
    g = 0.5 / np.sqrt(3.0)
    pts = (0.5 - g, 0.5 + g)
    w = h ** dim / 2 ** dim
    K = np.zeros((dim * 2 ** dim, dim * 2 ** dim))
    for xi in itertools.product(pts, repeat=dim):
        B = strain_displacement(dim, _shape_grad(dim, xi, h))
        K += w * B.T @ D @ B
    return 0.5 * (K + K.T)


def simp_modulus(rho, E0, Emin, p):
    """Modified SIMP (R1): E_e = Emin + rho_e^p (E0 - Emin)."""
    rho = np.asarray(rho, dtype=np.float64)
    return Emin + rho ** p * (E0 - Emin)


# ---------------------------------------------------------------- mesh maps

def element_dofs(dim: int, nel) -> np.ndarray:
    """[nelem, dim*2^dim] global dof ids of every element, local order of local_nodes()."""
    nel = tuple(nel)
    nn = [n + 1 for n in nel]
    grids = np.meshgrid(*[np.arange(n) for n in reversed(nel)], indexing="ij")
    e_idx = [g.ravel() for g in reversed(grids)]       # ex, ey[, ez], x fastest
    out = []
    for o in local_nodes(dim):
        node = np.zeros_like(e_idx[0])
        stride = 1
        for d in range(dim):
            node = node + (e_idx[d] + o[d]) * stride
            stride *= nn[d]
        for c in range(dim):
            out.append(dim * node + c)
    return np.stack(out, axis=1)


def node_coords(dim: int, nel, h=1.0) -> np.ndarray:
    nn = [n + 1 for n in nel]
    grids = np.meshgrid(*[np.arange(n) for n in reversed(nn)], indexing="ij")
    return np.stack([g.ravel() for g in reversed(grids)], axis=1).astype(np.float64) * h


# ---------------------------------------------------------------- assembly

def assemble_global(dim, nel, E_e, KE) -> sp.csr_matrix:
    """Monolithic K = sum_e E_e KE over all dofs (no BCs), PAPER.md:112-114 / :286."""
    edofs = element_dofs(dim, nel)
    ne, m = edofs.shape
    rows = np.repeat(edofs, m, axis=1).ravel()
    cols = np.tile(edofs, (1, m)).ravel()
    vals = (E_e[:, None, None] * KE[None, :, :]).ravel()
    ndof = dim * int(np.prod([n + 1 for n in nel]))
    return sp.coo_matrix((vals, (rows, cols)), shape=(ndof, ndof)).tocsr()


def free_system(prob):
    """(K_ff, f_f, free_idx): Dirichlet rows/columns eliminated (homogeneous)."""
    KE = element_stiffness(prob.dim, prob.nu, 1.0, prob.h)
    E_e = simp_modulus(prob.density, prob.E0, prob.Emin, prob.p)
    K = assemble_global(prob.dim, prob.nel, E_e, KE)
    free = np.flatnonzero(prob.fixed == 0)
    return K[free][:, free].tocsr(), prob.rhs[free].copy(), free


def apply_K(prob, u):
    """Matrix-free K u over all dofs (used for residual checks)."""
    KE = element_stiffness(prob.dim, prob.nu, 1.0, prob.h)
    E_e = simp_modulus(prob.density, prob.E0, prob.Emin, prob.p)
    edofs = element_dofs(prob.dim, prob.nel)
    ue = u[edofs]
    fe = (ue @ KE.T) * E_e[:, None]
    out = np.zeros_like(u)
    np.add.at(out, edofs.ravel(), fe.ravel())
    return out


def true_relres(prob, u):
    """||f - K u||_2 / ||f||_2 over free dofs (SURVEY.md §8(b) final_relres)."""
    free = prob.fixed == 0
    r = (prob.rhs - apply_K(prob, u))[free]
    nf = np.linalg.norm(prob.rhs[free])
    return float(np.linalg.norm(r) / nf) if nf > 0 else float(np.linalg.norm(r))
