"""ORACLE (test infrastructure only) — decomposition topology.

Paper: PAPER.md:56 ("N nonoverlapping subdomains Omega_i ... Gamma_i :=
dOmega_i minus dOmega ... I := closure(Omega) minus Gamma the set of interior
nodes"), Eqs.(4)-(5) (interior-first ordering, K_II block
diagonal over subdomains), PAPER.md:237 ("with the cross points removed").
Readings: R4 canonical numbering, R5 per-DOF classification
(Dirichlet wins), R8 faces/cross points (wirebasket in 3D).

Everything here is computed from the plain definitions by scanning
element->node incidences ("a node is on Gamma iff it touches elements of >= 2
subdomains").  Pins (tests/test_oracle_topology.py): closed-form counts
(faces px(py-1)+py(px-1), cross points (px-1)(py-1), n_Gamma formulas),
an independent coordinate formula for the subdomain count of a node,
SPEC.md:80-82 worked example (n_Gamma = 6), bijection of the numbering.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np

from .fem import element_dofs

I_CLS, G_CLS, D_CLS = 0, 1, 2


def element_subdomain(dim, nel, sub) -> np.ndarray:
    """Subdomain id s = sx + px*(sy + py*sz) of every element (x-fastest elements)."""
    nel = tuple(nel)
    ps = [n // s for n, s in zip(nel, sub)]
    grids = np.meshgrid(*[np.arange(n) for n in reversed(nel)], indexing="ij")
    e_idx = [g.ravel() for g in reversed(grids)]
    s = np.zeros_like(e_idx[0])
    stride = 1
    for d in range(dim):
        s = s + (e_idx[d] // sub[d]) * stride
        stride *= ps[d]
    return s


@dataclass
class Topology:
    dim: int
    nel: tuple
    sub: tuple
    nsub: int
    nnodes: int
    node_nsub: np.ndarray      # number of distinct subdomains touching each node
    node_pair: np.ndarray      # [nnodes, 2] (min, max) subdomain ids (valid if node_nsub == 2)
    cls: np.ndarray            # int8[ndof] 0=I 1=Gamma 2=D
    dof_sub: np.ndarray        # int32[ndof] subdomain of interior dofs, -1 otherwise
    reduced: np.ndarray        # int32[ndof] canonical index (interior by (s,dof), then Gamma by dof); -1 for D
    n_I: int
    n_G: int
    gamma_dofs: np.ndarray     # Gamma dofs ascending (global Gamma index = position)
    interior: list             # per subdomain: its interior dofs, ascending
    gamma_local: list          # per subdomain: Gamma dofs touched by its elements, ascending
    R: list                    # per subdomain: positions of gamma_local in gamma_dofs
    elem_sub: np.ndarray


def build_topology(prob) -> Topology:
    dim, nel, sub = prob.dim, tuple(prob.nel), tuple(prob.sub)
    for n, s in zip(nel, sub):
        if s <= 0 or n % s:
            raise ValueError("partition does not divide the mesh")
    nnodes = int(np.prod([n + 1 for n in nel]))
    ndof = dim * nnodes
    esub = element_subdomain(dim, nel, sub)
    nsub = int(np.prod([n // s for n, s in zip(nel, sub)]))
    enodes = element_dofs(dim, nel)[:, ::dim] // dim          # [ne, 2^d] node ids
    # distinct (node, subdomain) incidences
    pairs = np.unique(np.stack([enodes.ravel(), np.repeat(esub, enodes.shape[1])], 1), axis=0)
    node_nsub = np.bincount(pairs[:, 0], minlength=nnodes)
    first = np.searchsorted(pairs[:, 0], np.arange(nnodes))
    node_pair = np.full((nnodes, 2), -1, dtype=np.int64)
    has2 = node_nsub >= 2
    node_pair[:, 0] = pairs[first, 1]
    node_pair[has2, 1] = pairs[first[has2] + 1, 1]

    node_of = np.arange(ndof) // dim
    cls = np.full(ndof, I_CLS, dtype=np.int8)
    cls[node_nsub[node_of] >= 2] = G_CLS
    fixed = np.asarray(prob.fixed) != 0
    cls[fixed] = D_CLS
    dof_sub = np.where(cls == I_CLS, node_pair[node_of, 0], -1).astype(np.int32)

    idof = np.flatnonzero(cls == I_CLS)
    order = idof[np.argsort(dof_sub[idof], kind="stable")]      # by (s, dof)
    bnd = np.searchsorted(dof_sub[order], np.arange(nsub + 1))
    interior = [order[bnd[s]:bnd[s + 1]] for s in range(nsub)]
    gamma_dofs = np.flatnonzero(cls == G_CLS)
    n_I = int(sum(len(a) for a in interior))
    n_G = len(gamma_dofs)
    reduced = np.full(ndof, -1, dtype=np.int32)
    pos = 0
    for a in interior:
        reduced[a] = np.arange(pos, pos + len(a))
        pos += len(a)
    reduced[gamma_dofs] = np.arange(n_I, n_I + n_G)

    # Gamma dofs touched by each subdomain's elements
    gpos = np.full(ndof, -1, dtype=np.int64)
    gpos[gamma_dofs] = np.arange(n_G)
    gamma_local, R = [], []
    psort = pairs[np.argsort(pairs[:, 1], kind="stable")]
    pb = np.searchsorted(psort[:, 1], np.arange(nsub + 1))
    for s in range(nsub):
        nodes = np.unique(psort[pb[s]:pb[s + 1], 0])
        dofs = (dim * nodes[:, None] + np.arange(dim)[None, :]).ravel()
        dofs = np.sort(dofs[cls[dofs] == G_CLS])
        gamma_local.append(dofs)
        R.append(gpos[dofs])
    return Topology(dim, nel, sub, nsub, nnodes, node_nsub, node_pair, cls, dof_sub,
                    reduced, n_I, n_G, gamma_dofs, interior, gamma_local, R, esub)


@dataclass
class ComponentSkeleton:
    """Interface skeleton of one displacement component c (R6/R8)."""
    c: int
    nodes: np.ndarray          # Gamma_c nodes ascending (their c-dof is Gamma)
    gidx: np.ndarray           # global Gamma index of each node's c-dof
    faces: list                # list of arrays of positions into `nodes` (ascending node id), one per face
    face_keys: list            # (s_a, s_b) per face
    cross: np.ndarray          # positions into `nodes` of cross points (>= 3 subdomains)


def component_skeletons(prob, topo: Topology):
    out = []
    gpos = {int(d): i for i, d in enumerate(topo.gamma_dofs)}
    for c in range(prob.dim):
        dofs = topo.gamma_dofs[topo.gamma_dofs % prob.dim == c]
        nodes = dofs // prob.dim
        gidx = np.array([gpos[int(d)] for d in dofs], dtype=np.int64)
        ns = topo.node_nsub[nodes]
        cross = np.flatnonzero(ns >= 3)
        keys = {}
        for k in np.flatnonzero(ns == 2):
            key = (int(topo.node_pair[nodes[k], 0]), int(topo.node_pair[nodes[k], 1]))
            keys.setdefault(key, []).append(k)
        face_keys = sorted(keys)
        faces = [np.array(keys[k], dtype=np.int64) for k in face_keys]
        out.append(ComponentSkeleton(c, nodes, gidx, faces, face_keys, cross))
    return out
