"""Bit-exact DOF map and skeleton of the C++ host setup (libde, host_only context, no GPU)
against the oracle's topology (R4/R5/R8)."""
import numpy as np
import pytest

from synthetic import make_config
from oracle.topology import build_topology, component_skeletons

CASES = [("c1", {}), ("c2", {}), ("c3", dict(nel=(128, 64), sub=(32, 32))),
         ("c4", dict(nel=(12, 6, 6), sub=(3, 3, 3))), ("c2", dict(nel=(40, 24), sub=(8, 6)))]


def _host_ctx(p):
    from paper_1501_06211_b200 import binding as B
    opt = B.de_default_options(host_only=1)
    return B.de_setup(p.dim, p.nel, p.h, p.fixed, p.density, p.E0, p.Emin, p.p, p.nu, p.sub, opt)


@pytest.mark.parametrize("name,kw", CASES)
def test_dofmap_bit_exact(name, kw):
    from paper_1501_06211_b200 import binding as B
    p = make_config(name, **kw)
    T = build_topology(p)
    ctx = _host_ctx(p)
    try:
        cls, sub, red, nI, nG = B.de_get_dofmap(ctx)
        np.testing.assert_array_equal(cls, T.cls)
        np.testing.assert_array_equal(sub, T.dof_sub)
        np.testing.assert_array_equal(red, T.reduced)
        assert (nI, nG) == (T.n_I, T.n_G)
        for sk in component_skeletons(p, T):
            nodes, face = B.de_get_skeleton(ctx, sk.c)
            np.testing.assert_array_equal(nodes, sk.nodes)
            exp = np.full(len(sk.nodes), -1)
            for fid, f in enumerate(sk.faces):
                exp[f] = fid
            np.testing.assert_array_equal(face, exp)
        s = B.de_get_stats(ctx)
        assert s.n_free == T.n_I + T.n_G
    finally:
        B.de_destroy(ctx)


def test_host_only_refuses_factor():
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    ctx = _host_ctx(p)
    try:
        with pytest.raises(B.DEError) as ei:
            B.de_factor(ctx)
        assert ei.value.status == B.DE_ESTATE
    finally:
        B.de_destroy(ctx)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_dofmap_bit_exact_full_size(name):
    from paper_1501_06211_b200 import binding as B
    p = make_config(name)
    T = build_topology(p)
    ctx = _host_ctx(p)
    try:
        cls, sub, red, nI, nG = B.de_get_dofmap(ctx)
        np.testing.assert_array_equal(cls, T.cls)
        np.testing.assert_array_equal(sub, T.dof_sub)
        np.testing.assert_array_equal(red, T.reduced)
    finally:
        B.de_destroy(ctx)
