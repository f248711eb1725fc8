"""ORACLE (test infrastructure only) — interface trace mass M and Laplacian L.

Paper: PAPER.md:167-172 ("M and L denote the mass and Laplacian matrices
respectively assembled on the interface Gamma"), Eq.(9)
(applied component-wise).  Readings: R6 trace elements are the
element facets (edges in 2D, faces in 3D) whose two adjacent elements lie in
different subdomains; linear (2D) / bilinear (3D) facet elements; Dirichlet
rows/columns of component c eliminated; no coefficient weighting by default.
NEXT(3) / R19 (weighted=True): every facet element is scaled by the mean modulus
(E_a + E_b)/2 of its two adjacent elements (SIMP moduli of the current densities),
the coefficient-weighted trace norm of SURVEY.md §8(f); pinned by uniform density
(weighted = E x unweighted, preconditioner / E) and by one face between two uniform
subdomains (weight (E_a + E_b)/2), tests/test_weighted_trace.py.  R7: a
component whose skeleton has a connected piece without Dirichlet contact is
"singular" (L_c has constants in its kernel).

Pins (tests/test_oracle_trace_precond.py): SPEC.md:179 worked example (single face,
one interior node, h=1/2 -> M=[1/3], L=[4]); L row sums vanish away from
Dirichlet; the 1D pencil eigenvalues (6/h^2)(1-cos phi_j)/(2+cos phi_j);
M sums to the total facet measure (1^T M 1 = |Gamma_c| incl. eliminated part); the 3D
facet matrices by the tensor-product pencil of one square interface with a Dirichlet rim
(eigenvalues alpha_i + alpha_j of the 1D pencil, mass eigenvalues mu_i mu_j).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .topology import element_subdomain
from .fem import element_dofs, local_nodes


def facet_matrices(dim: int, h: float):
    """Mass and Laplacian of one Q1 facet element of dimension dim-1, nodes in
    lexicographic order of the facet's own axes (first axis fastest).
    1D: m = h/6 [[2,1],[1,2]], k = 1/h [[1,-1],[-1,1]]; 2D facet: tensor products."""
    m = h / 6.0 * np.array([[2.0, 1.0], [1.0, 2.0]])
    k = 1.0 / h * np.array([[1.0, -1.0], [-1.0, 1.0]])
    if dim == 2:
        return m, k
    M = np.kron(m, m)
    L = np.kron(k, m) + np.kron(m, k)
    return M, L


def trace_facets(prob, with_elements=False):
    """Node ids [nf, 2^(d-1)] of every facet shared by two elements of different
    subdomains (facet-local lexicographic node order); with_elements: also the two
    adjacent element ids [nf, 2]."""
    dim, nel = prob.dim, tuple(prob.nel)
    esub = element_subdomain(dim, nel, prob.sub)
    enodes = element_dofs(dim, nel)[:, ::dim] // dim
    offs = local_nodes(dim)
    coords = np.stack(np.unravel_index(np.arange(np.prod(nel)), tuple(reversed(nel))), 1)[:, ::-1]
    out, els = [], []
    for a in range(dim):
        stride = int(np.prod(nel[:a]))
        has_nb = coords[:, a] < nel[a] - 1
        e = np.flatnonzero(has_nb)
        e = e[esub[e] != esub[e + stride]]
        cols = [i for i, o in enumerate(offs) if o[a] == 1]   # lexicographic in remaining axes
        out.append(enodes[e][:, cols])
        els.append(np.stack([e, e + stride], axis=1))
    F = np.concatenate(out, axis=0) if out else np.zeros((0, 2 ** (dim - 1)), dtype=np.int64)
    if with_elements:
        return F, (np.concatenate(els, axis=0) if els else np.zeros((0, 2), dtype=np.int64))
    return F


def component_trace_matrices(prob, skel, weighted=False):
    """(M_c, L_c, singular_c) as CSR over positions in skel.nodes; weighted: facet elements scaled by the
    mean SIMP modulus of their two adjacent elements (R19)."""
    from .fem import simp_modulus
    dim = prob.dim
    Mf, Lf = facet_matrices(dim, prob.h)
    F, FE = trace_facets(prob, with_elements=True)
    nn = prob.nnodes
    m = F.shape[1]
    rows = np.repeat(F, m, axis=1).ravel()
    cols = np.tile(F, (1, m)).ravel()
    w = np.ones(len(F))
    if weighted:
        E = simp_modulus(prob.density, prob.E0, prob.Emin, prob.p)
        w = 0.5 * (E[FE[:, 0]] + E[FE[:, 1]])
    Mfull = sp.coo_matrix(((w[:, None] * Mf.ravel()[None, :]).ravel(), (rows, cols)), shape=(nn, nn)).tocsr()
    Lfull = sp.coo_matrix(((w[:, None] * Lf.ravel()[None, :]).ravel(), (rows, cols)), shape=(nn, nn)).tocsr()
    tn = np.unique(F)
    fixed_c = prob.fixed[dim * tn + skel.c] != 0
    keep = tn[~fixed_c]
    if not np.array_equal(np.sort(keep), np.sort(skel.nodes)):
        raise AssertionError("trace nodes != Gamma_c nodes")
    idx = skel.nodes
    M = Mfull[idx][:, idx].tocsr()
    L = Lfull[idx][:, idx].tocsr()
    # singularity (R7): a connected piece of the trace graph with no Dirichlet node
    pattern = sp.coo_matrix((np.ones(len(rows)), (rows, cols)), shape=(nn, nn)).tocsr()
    ncomp, lab = connected_components(pattern[tn][:, tn], directed=False)
    has_d = np.zeros(ncomp, dtype=bool)
    has_d[lab[fixed_c]] = True
    singular = bool((~has_d).any())
    return M, L, singular
