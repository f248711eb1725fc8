"""Oracle pins: trace matrices and the interface preconditioner (CPU only)."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from synthetic import make_config, Problem
from oracle.topology import build_topology, component_skeletons
from oracle.trace import component_trace_matrices, facet_matrices
from oracle.precond import (build_components, dense_fractional, inverse_lanczos,
                            apply_precond, pcg_plain, ComponentData)

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def _single_line(k, h):
    """Mesh 2 x (k+1) elements split into 2x1 subdomains: one vertical interface line
    with k+2 nodes; its two end nodes are Dirichlet (all components)."""
    nel, sub = (2, k + 1), (1, k + 1)
    nn = 3 * (k + 2)
    fixed = np.zeros(2 * nn, dtype=np.uint8)
    for j in (0, k + 1):
        node = 1 + 3 * j
        fixed[2 * node:2 * node + 2] = 1
    return Problem("line", 2, nel, sub, fixed, np.ones(2 * (k + 1)), np.zeros(2 * nn), h=h)


def test_spec_single_face_trace():
    pin = PINS["single_face_trace"]
    p = _single_line(1, pin["h"])
    T = build_topology(p)
    for sk in component_skeletons(p, T):
        M, L, sing = component_trace_matrices(p, sk)
        assert M.shape == (1, 1) and not sing
        assert M[0, 0] == pytest.approx(pin["M"], rel=1e-15)
        assert L[0, 0] == pytest.approx(pin["L"], rel=1e-15)


def test_pencil_closed_form():
    pin = PINS["pencil_1d_k5_h025"]
    p = _single_line(5, 0.25)
    T = build_topology(p)
    sk = component_skeletons(p, T)[0]
    M, L, _ = component_trace_matrices(p, sk)
    np.testing.assert_allclose(sla.eigh(L.toarray(), M.toarray(), eigvals_only=True),
                               pin["values"], rtol=1e-12)


def _single_plane(N, h):
    """3D mesh 2 x N x N elements split into 2 x 1 x 1 subdomains: one interface plane x = h with (N+1)^2
    nodes; its rim (y or z at the boundary) is Dirichlet in every component."""
    nel, sub = (2, N, N), (1, N, N)
    nx, ny, nz = 3, N + 1, N + 1
    fixed = np.zeros(3 * nx * ny * nz, dtype=np.uint8)
    for k in range(nz):
        for j in range(ny):
            if j in (0, N) or k in (0, N):
                for i in range(nx):
                    node = i + nx * (j + ny * k)
                    fixed[3 * node:3 * node + 3] = 1
    return Problem("plane", 3, nel, sub, fixed, np.ones(2 * N * N), np.zeros(3 * nx * ny * nz), h=h)


@pytest.mark.parametrize("N,h", [(5, 0.25), (7, 1.0)])
def test_3d_facet_trace_tensor_pencil(N, h):
    """3D trace elements (bilinear quads, R6) pinned by the tensor-product closed form: on one square interface
    with a Dirichlet rim, L = K1 (x) M1 + M1 (x) K1 and M = M1 (x) M1 for the 1D pencil (K1, M1) of the interior
    nodes, so the eigenvalues of (L, M) are alpha_i + alpha_j with alpha_j = (6/h^2)(1-cos(j pi/N))/(2+cos(j pi/N))
    (the 1D closed form of SPEC.md:196 / pencil_1d_k5_h025). A single Kronecker term, a wrong facet mass or
    stiffness scale (3D scales as h^0 for L and h^2 for M) all break it."""
    p = _single_plane(N, h)
    T = build_topology(p)
    phi = np.arange(1, N) * np.pi / N
    alpha = 6.0 / h ** 2 * (1 - np.cos(phi)) / (2 + np.cos(phi))
    expect = np.sort((alpha[:, None] + alpha[None, :]).ravel())
    for sk in component_skeletons(p, T):
        M, L, sing = component_trace_matrices(p, sk)
        assert M.shape == ((N - 1) ** 2,) * 2 and not sing
        np.testing.assert_allclose(np.sort(sla.eigh(L.toarray(), M.toarray(), eigvals_only=True)), expect,
                                   rtol=1e-11)
        # the mass alone: eigenvalues mu_i mu_j of M1 (x) M1, M1 = tridiag(h/6, 4h/6, h/6) -> (h/3)(2 + cos phi)
        mu = h / 3.0 * (2 + np.cos(phi))
        np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(M.toarray())),
                                   np.sort((mu[:, None] * mu[None, :]).ravel()), rtol=1e-12)


@pytest.mark.parametrize("name,kw", [("c2", dict(nel=(16, 8), sub=(4, 4))),
                                     ("c4", dict(nel=(6, 4, 4), sub=(2, 2, 2)))])
def test_trace_row_sums_and_measure(name, kw):
    p = make_config(name, **kw)
    T = build_topology(p)
    for sk in component_skeletons(p, T):
        M, L, sing = component_trace_matrices(p, sk)
        assert abs(M - M.T).max() < 1e-15 and abs(L - L.T).max() < 1e-15
        # nodes whose trace neighbours are all Gamma_c nodes: L row sum is 0
        Mf, Lf = facet_matrices(p.dim, p.h)
        assert abs(Lf.sum(axis=1)).max() < 1e-15
        assert Mf.sum() == pytest.approx(p.h ** (p.dim - 1), rel=1e-15)
        rs = np.asarray(L.sum(axis=1)).ravel()
        assert np.sum(np.abs(rs) < 1e-14) > 0.5 * len(rs)
        assert np.all(np.linalg.eigvalsh(L.toarray()) > 0)   # clamped at x=0: L_c SPD
        assert not sing


def test_singular_component_detected():
    """Config-3 recipe: u_y is never Dirichlet on the skeleton (R7)."""
    p = make_config("c3", nel=(16, 8), sub=(4, 4))
    comps = build_components(p, build_topology(p))
    assert [c.singular for c in comps] == [False, True]
    ev = np.linalg.eigvalsh(comps[1].L.toarray())
    assert abs(ev[0]) < 1e-12 and ev[1] > 1e-6


def test_scalar_fractional_example():
    pin = PINS["scalar_fractional"]
    M, L, v = np.array([[pin["M"]]]), np.array([[pin["L"]]]), np.array([pin["v"]])
    assert dense_fractional(M, L, pin["theta"], v, +1)[0] == pytest.approx(pin["H_v"], rel=1e-15)
    assert dense_fractional(M, L, pin["theta"], v, -1)[0] == pytest.approx(pin["Hinv_v"], rel=1e-15)


def _small_comp():
    p = make_config("c2", nel=(12, 8), sub=(4, 4))
    T = build_topology(p)
    return build_components(p, T)


@pytest.mark.parametrize("theta", [0.0, 0.25, 0.5, 0.75, 1.0])
def test_dense_fractional_roundtrip_and_theta1(theta):
    cd = _small_comp()[0]
    v = np.random.default_rng(0).normal(size=cd.M.shape[0])
    z = dense_fractional(cd.M, cd.L, theta, v, -1)
    np.testing.assert_allclose(dense_fractional(cd.M, cd.L, theta, z, +1), v, rtol=1e-9, atol=1e-10)
    if theta == 1.0:
        np.testing.assert_allclose(z, np.linalg.solve(cd.M.toarray(), v), rtol=1e-10)
    if theta == 0.0:
        np.testing.assert_allclose(dense_fractional(cd.M, cd.L, theta, v, +1), cd.L @ v, rtol=1e-10, atol=1e-12)


def test_eigenvector_input():
    cd = _small_comp()[0]
    lam, Phi = sla.eigh(cd.L.toarray(), cd.M.toarray())
    j = 3
    v = cd.M @ Phi[:, j]                   # H~^-1 (M phi) = lambda^(theta-1) phi
    for theta in (0.25, 0.5):
        z = dense_fractional(cd.M, cd.L, theta, v, -1)
        np.testing.assert_allclose(z, lam[j] ** (theta - 1) * Phi[:, j], rtol=1e-9, atol=1e-12)
        zl = inverse_lanczos(cd, v, 10, theta)   # exact eigen-input: breakdown at k=1, exact answer
        np.testing.assert_allclose(zl, lam[j] ** (theta - 1) * Phi[:, j], rtol=1e-8, atol=1e-11)


@pytest.mark.parametrize("theta", [0.25, 0.5, 0.75])
def test_lanczos_full_k_equals_dense(theta):
    for cd in _small_comp():
        n = cd.M.shape[0]
        v = np.random.default_rng(1).normal(size=n)
        z = inverse_lanczos(cd, v, n, theta)
        zd = dense_fractional(cd.M, cd.L, theta, v, -1)
        assert np.linalg.norm(z - zd) <= 1e-8 * np.linalg.norm(zd)


def test_lanczos_theta1_gives_mass_solve():
    cd = _small_comp()[0]
    v = np.random.default_rng(2).normal(size=cd.M.shape[0])
    z = inverse_lanczos(cd, v, 4, 1.0)
    np.testing.assert_allclose(z, np.linalg.solve(cd.M.toarray(), v), rtol=1e-10, atol=1e-12)


def test_singular_component_full_norm_lanczos_equals_dense():
    p = make_config("c3", nel=(12, 8), sub=(4, 4))
    cd = build_components(p, build_topology(p))[1]
    assert cd.singular
    n = cd.M.shape[0]
    v = np.random.default_rng(3).normal(size=n)
    z = inverse_lanczos(cd, v, n, 0.5)
    # H_theta = M + M (M^-1 L)^(1-theta): check by applying it densely
    lam, Phi = sla.eigh(cd.L.toarray(), cd.M.toarray())
    Md = cd.M.toarray()
    H = Md @ Phi @ np.diag(1 + np.maximum(lam, 0) ** 0.5) @ Phi.T @ Md
    np.testing.assert_allclose(H @ z, v, rtol=1e-7, atol=1e-8 * np.abs(v).max())


def test_block_diagonal_and_zero_input():
    comps = _small_comp()
    nG = sum(len(c.skel.gidx) for c in comps)
    r = np.random.default_rng(4).normal(size=nG)
    r[comps[1].skel.gidx] = 0.0
    z = apply_precond(comps, r, "lanczos")
    assert np.all(z[comps[1].skel.gidx] == 0.0)
    z1 = apply_precond(comps, np.where(np.isin(np.arange(nG), comps[0].skel.gidx), r, 0), "lanczos")
    np.testing.assert_allclose(z1, z, rtol=0, atol=0)


def test_face_preconditioner_exact_for_single_face():
    p = _single_line(6, 1.0)
    cd = build_components(p, build_topology(p))[0]
    assert len(cd.skel.faces) == 1 and len(cd.skel.cross) == 0
    b = np.random.default_rng(5).normal(size=cd.K.shape[0])
    x, its = pcg_plain(lambda v: cd.K @ v, b, cd.face_precond, 1e-12, 50)
    assert its == 1
    np.testing.assert_allclose(cd.K @ x, b, rtol=1e-12, atol=1e-12)


def test_inner_modes_agree_when_F_is_tight():
    """Mode X (exact) is the tol -> 0 limit of mode F (R10)."""
    cd = _small_comp()[0]
    v = np.random.default_rng(6).normal(size=cd.M.shape[0])
    zx = inverse_lanczos(cd, v, 6, 0.5, inner="X")
    cd.inner_tol = 1e-14
    zf = inverse_lanczos(cd, v, 6, 0.5, inner="F")
    assert max(cd.inner_its) > 1
    np.testing.assert_allclose(zf, zx, rtol=1e-9, atol=1e-12 * np.abs(zx).max())
