"""Oracle pins: decomposition topology (CPU only)."""
import json
import os

import numpy as np
import pytest

from synthetic import make_config, Problem
from oracle.topology import build_topology, component_skeletons, I_CLS, G_CLS, D_CLS

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def _nsub_formula(prob):
    """Independent coordinate formula: along each axis a node at index i touches
    2 subdomain slabs iff 0 < i < n and i % s == 0; the count multiplies over axes."""
    nn = [n + 1 for n in prob.nel]
    idx = np.unravel_index(np.arange(int(np.prod(nn))), tuple(reversed(nn)))[::-1]
    cnt = np.ones(len(idx[0]), dtype=int)
    for d in range(prob.dim):
        i = idx[d]
        cnt *= np.where((i > 0) & (i < prob.nel[d]) & (i % prob.sub[d] == 0), 2, 1)
    return cnt


def _brute_classes(prob):
    """Brute-force element scan in pure Python (small meshes)."""
    dim = prob.dim
    nn = [n + 1 for n in prob.nel]
    subs = {}
    for e in np.ndindex(*reversed(prob.nel)):
        e = e[::-1]
        s = 0
        stride = 1
        for d in range(dim):
            s += (e[d] // prob.sub[d]) * stride
            stride *= prob.nel[d] // prob.sub[d]
        for o in np.ndindex(*([2] * dim)):
            node = 0
            st = 1
            for d in range(dim):
                node += (e[d] + o[d]) * st
                st *= nn[d]
            subs.setdefault(node, set()).add(s)
    cls = np.zeros(prob.ndof, dtype=np.int8)
    for node, ss in subs.items():
        for c in range(dim):
            dof = dim * node + c
            cls[dof] = D_CLS if prob.fixed[dof] else (G_CLS if len(ss) >= 2 else I_CLS)
    return cls


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", dict(nel=(16, 8), sub=(4, 4))),
                                     ("c3", dict(nel=(16, 8), sub=(4, 4))),
                                     ("c4", dict(nel=(6, 4, 4), sub=(2, 2, 2)))])
def test_classification_vs_bruteforce_and_formula(name, kw):
    p = make_config(name, **kw)
    T = build_topology(p)
    np.testing.assert_array_equal(T.node_nsub, _nsub_formula(p))
    np.testing.assert_array_equal(T.cls, _brute_classes(p))


def test_spec_classify_example():
    pin = PINS["spec_classify_example"]
    nel, sub = tuple(pin["nel"]), tuple(pin["sub"])
    nn = (nel[0] + 1) * (nel[1] + 1)
    fixed = np.zeros(2 * nn, dtype=np.uint8)
    for j in range(nel[1] + 1):
        node = nel[0] + (nel[0] + 1) * j
        fixed[2 * node:2 * node + 2] = 1
    p = Problem("spec", 2, nel, sub, fixed, np.ones(8), np.zeros(2 * nn))
    assert build_topology(p).n_G == pin["n_gamma"]


@pytest.mark.parametrize("px,py,faces,cross", PINS["partition_counts"]["cases"])
def test_face_and_cross_counts(px, py, faces, cross):
    p = make_config("c2", nel=(4 * px, 4 * py), sub=(4, 4))
    T = build_topology(p)
    for sk in component_skeletons(p, T):
        assert len(sk.faces) == faces
        assert len(sk.cross) == cross


def test_numbering_is_canonical_bijection():
    p = make_config("c3", nel=(16, 8), sub=(4, 4))
    T = build_topology(p)
    free = np.flatnonzero(T.cls != D_CLS)
    assert sorted(T.reduced[free]) == list(range(len(free)))
    assert np.all(T.reduced[T.cls == D_CLS] == -1)
    # interior first, grouped by subdomain, ascending dof inside; then Gamma by dof
    order = np.argsort(T.reduced[free])
    seq = free[order]
    keys = [(0, T.dof_sub[d], d) if T.cls[d] == I_CLS else (1, 0, d) for d in seq]
    assert keys == sorted(keys)
    # per-DOF classification at the roller line (R5): node (0, 4) x-dof D, y-dof Gamma
    node = 0 + 17 * 4
    assert T.cls[2 * node] == D_CLS and T.cls[2 * node + 1] == G_CLS


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_appendix_a_counts_small(name):
    pin = PINS["appendix_a"][name]
    p = make_config(name)
    T = build_topology(p)
    assert T.n_I + T.n_G == pin["n_free"]
    assert T.n_G == pin["n_gamma"]
    sk = component_skeletons(p, T)
    assert len(sk[0].faces) == pin["faces"] and len(sk[0].cross) == pin["cross"]
    nI = [len(a) for a in T.interior]
    nG = [len(r) for r in T.R]
    assert [min(nI), max(nI)] == pin["nI"] and [min(nG), max(nG)] == pin["nGi"]
    assert sum(nG) == pin["sum_nGi"]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_appendix_a_counts_large(name):
    pin = PINS["appendix_a"][name]
    p = make_config(name)
    T = build_topology(p)
    assert T.n_I + T.n_G == pin["n_free"]
    assert T.n_G == pin["n_gamma"]
    sk = component_skeletons(p, T)
    if name == "c3":
        assert (len(sk[0].nodes), len(sk[1].nodes)) == (pin["n_gamma_x"], pin["n_gamma_y"])
    if "cross" in pin:
        assert len(sk[-1].cross) == pin["cross"] and len(sk[-1].faces) == pin["faces"]
    if "wirebasket" in pin:
        assert len(sk[0].cross) == pin["wirebasket"] and len(sk[0].faces) == pin["faces"]
    if "sum_nGi" in pin:
        assert sum(len(r) for r in T.R) == pin["sum_nGi"]
