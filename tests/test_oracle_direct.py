"""Oracle pins for oracle/direct.py (the nested-dissection multifrontal Cholesky used for u_ref where SuperLU
cannot factor: configs 4 and 5). Pinned against things other than itself: SuperLU (a library routine) on
grids it can factor, a dense numpy solve on a tiny grid, the patch test, and the tree's separator property."""
import numpy as np
import pytest

from synthetic import make_config
from oracle import fem
from oracle.direct import nd_tree, NDCholesky, direct_solve, refine_dd, relres_ext
from oracle.solver import monolithic_solve


@pytest.mark.parametrize("nn,leaf", [((9, 5), 4), ((33, 17), 16), ((7, 5, 4), 8)])
def test_nd_tree_partitions_and_separates(nn, leaf):
    tree = nd_tree(nn, leaf)
    allnodes = np.concatenate([t[0] for t in tree])
    assert np.array_equal(np.sort(allnodes), np.arange(int(np.prod(nn))))   # a partition of the nodes
    # post-order and separation: every node of a tree node couples (grid distance <= 1 per axis) only to nodes
    # of its own subtree or of its ancestors -- the property the multifrontal elimination needs
    owner = np.empty(int(np.prod(nn)), dtype=np.int64)
    for t, (nodes, _) in enumerate(tree):
        owner[nodes] = t
    parent = {k: t for t, (_, kids) in enumerate(tree) for k in kids}
    def ancestors(t):
        out = set()
        while t in parent:
            t = parent[t]
            out.add(t)
        return out
    sub = {}
    for t, (_, kids) in enumerate(tree):
        assert all(k < t for k in kids)
        sub[t] = {t}.union(*[sub[k] for k in kids]) if kids else {t}
    grid = owner.reshape(tuple(reversed(nn)))
    dim = len(nn)
    for t, (nodes, _) in enumerate(tree):
        ok = sub[t] | ancestors(t)
        c = np.stack(np.unravel_index(nodes, tuple(reversed(nn))), 1)
        for off in np.ndindex(*(3,) * dim):
            o = np.array(off) - 1
            nb = c + o
            inb = np.all((nb >= 0) & (nb < np.array(tuple(reversed(nn)))), axis=1)
            for q in grid[tuple(nb[inb].T)]:
                assert int(q) in ok


def test_dense_equals_direct_tiny():
    p = make_config("c1", nel=(6, 4), sub=(3, 2))
    K, f, free = fem.free_system(p)
    ud = np.linalg.solve(K.toarray(), f)
    u = direct_solve(p, leaf=4)
    np.testing.assert_allclose(u[free], ud, rtol=1e-12, atol=1e-14 * np.abs(ud).max())


@pytest.mark.parametrize("name,kw", [("c2", dict(nel=(64, 32), sub=(16, 16))),
                                     ("c3", dict(nel=(64, 32), sub=(16, 16))),      # rollers + contrast
                                     ("c4", dict(nel=(12, 6, 6), sub=(6, 6, 6))),
                                     ("c1", {})])
def test_direct_equals_superlu(name, kw):
    p = make_config(name, **kw)
    u_slu = monolithic_solve(p)
    u = direct_solve(p, leaf=32)
    if name == "c3":   # FP64-ill-posed recipe (R15): compare backward errors, both at rounding level
        K, f, free = fem.free_system(p)
        for v in (u, u_slu):
            r = f - K @ v[free]
            assert np.linalg.norm(r) / (np.linalg.norm(K.data, 1) * np.linalg.norm(v) + np.linalg.norm(f)) < 1e-13
        return
    assert np.linalg.norm(u - u_slu) / np.linalg.norm(u_slu) < 1e-11
    assert relres_ext(p, u) < 1e-11


def test_patch_test_through_direct_solver():
    """Linear displacement field prescribed on the whole boundary: interior exact."""
    p = make_config("c2", nel=(12, 8), sub=(4, 4))
    p = p.with_density(np.full(p.nelem, 0.7))     # the patch test needs a uniform material
    nx, ny = p.nel
    X = fem.node_coords(2, p.nel)
    ulin = np.zeros(p.ndof)
    ulin[0::2] = 1e-3 * (0.3 + 0.7 * X[:, 0] - 0.2 * X[:, 1])
    ulin[1::2] = 1e-3 * (-0.1 + 0.4 * X[:, 0] + 0.9 * X[:, 1])
    bnd = (X[:, 0] == 0) | (X[:, 0] == nx) | (X[:, 1] == 0) | (X[:, 1] == ny)
    fixed = np.repeat(bnd, 2).astype(np.uint8)
    # rhs = -K_fb u_b on the free dofs (homogeneous-Dirichlet form of the inhomogeneous problem)
    from dataclasses import replace
    Kfull = fem.assemble_global(2, p.nel, fem.simp_modulus(p.density, p.E0, p.Emin, p.p),
                                fem.element_stiffness(2, p.nu, 1.0, p.h))
    ub = np.where(fixed == 1, ulin, 0.0)
    rhs = -(Kfull @ ub)
    q = replace(p, fixed=fixed, rhs=np.where(fixed == 1, 0.0, rhs))
    u = direct_solve(q, leaf=8) + ub
    assert np.abs(u - ulin).max() <= 1e-12 * np.abs(ulin).max()


def test_refinement_reaches_rounding_floor():
    p = make_config("c2", nel=(64, 32), sub=(16, 16))
    hi, lo, hist = refine_dd(p, rounds=2, leaf=32)
    u_slu = monolithic_solve(p)
    assert np.linalg.norm(hi - u_slu) / np.linalg.norm(hi) < 1e-11
    assert hist[-1] <= hist[0] and hist[-1] < 1e-11
