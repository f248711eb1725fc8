"""Oracle pins: DD algebra, interface CG and the end-to-end DD = monolithic equivalence (CPU only)."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from synthetic import make_config
from oracle import fem
from oracle.topology import build_topology
from oracle.dd import (subdomain_blocks, factor_subdomains, dense_schur, dense_local_schur,
                       schur_apply, condensed_rhs, back_substitute)
from oracle.krylov import pcg
from oracle.solver import DDOracle, monolithic_solve

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def _setup(name, **kw):
    p = make_config(name, **kw)
    T = build_topology(p)
    B = factor_subdomains(subdomain_blocks(p, T))
    return p, T, B


def _monolithic_blocks(p, T):
    """K in the canonical (interior-first) numbering, from the monolithic assembly."""
    K, f, free = fem.free_system(p)
    perm = np.argsort(T.reduced[free])
    K = K[perm][:, perm].toarray()
    f = f[perm]
    n_I = T.n_I
    return K[:n_I, :n_I], K[:n_I, n_I:], K[n_I:, n_I:], f[:n_I], f[n_I:]


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c3", dict(nel=(16, 8), sub=(4, 4))),
                                     ("c4", dict(nel=(4, 4, 2), sub=(2, 2, 1)))])
def test_assembled_schur_equals_monolithic_schur(name, kw):
    p, T, B = _setup(name, **kw)
    KII, KIG, KGG, fI, fG = _monolithic_blocks(p, T)
    S_mono = KGG - KIG.T @ np.linalg.solve(KII, KIG)
    S = dense_schur(B, T.n_G)
    assert np.abs(S - S_mono).max() <= 1e-10 * np.abs(S_mono).max()
    x = np.random.default_rng(0).normal(size=T.n_G)
    np.testing.assert_allclose(schur_apply(B, T.n_G, x), S_mono @ x, rtol=1e-9,
                               atol=1e-11 * np.abs(S_mono @ x).max())
    g = condensed_rhs(p, T, B)
    np.testing.assert_allclose(g, fG - KIG.T @ np.linalg.solve(KII, fI), atol=1e-12 * max(1, np.abs(fG).max()))
    # K_II block diagonal in this numbering
    off = 0
    for b in B:
        n = len(b.I)
        KII[off:off + n, off:off + n] = 0
        off += n
    assert np.abs(KII).max() == 0


def test_local_schur_spd_and_floating_kernel():
    p, T, B = _setup("c1")
    X = fem.node_coords(2, p.nel)
    for s, b in enumerate(B):
        Si = dense_local_schur(b)
        assert np.abs(Si - Si.T).max() <= 1e-12 * np.abs(Si).max()
        ev = np.linalg.eigvalsh(0.5 * (Si + Si.T))
        assert ev[0] >= -1e-12 * ev[-1]
        nodes = b.G // 2
        touches_d = bool(np.any(p.fixed[np.concatenate([b.I, b.G])]))   # local Dirichlet contact
        sx = s % 2
        if sx == 1:   # right subdomains do not touch the clamped edge: floating
            xy = X[nodes]
            comp = b.G % 2
            modes = [np.where(comp == 0, 1.0, 0.0), np.where(comp == 1, 1.0, 0.0),
                     np.where(comp == 0, -xy[:, 1], xy[:, 0])]
            R = np.stack(modes, 1)
            assert np.linalg.norm(Si @ R) <= 1e-12 * np.linalg.norm(Si) * np.linalg.norm(R)
            assert np.sum(ev < 1e-12 * ev[-1]) == 3
        else:
            assert ev[0] > 1e-10 * ev[-1]


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", dict(nel=(32, 16), sub=(8, 8))),
                                     ("c4", dict(nel=(6, 4, 4), sub=(2, 2, 2)))])
def test_dd_dense_interface_equals_monolithic(name, kw):
    """North star pin: DD with an exact dense interface solve equals the monolithic solve."""
    p, T, B = _setup(name, **kw)
    S = dense_schur(B, T.n_G)
    uG = np.linalg.solve(S, condensed_rhs(p, T, B))
    u = back_substitute(p, T, B, uG)
    u_ref = monolithic_solve(p)
    assert np.linalg.norm(u - u_ref) <= 1e-12 * np.linalg.norm(u_ref)
    assert np.all(u[p.fixed != 0] == 0)


def test_pcg_pins():
    # A = I -> 1 iteration
    b = np.random.default_rng(0).normal(size=7)
    _, its, conv, _ = pcg(lambda v: v, b, lambda v: v, 1e-10, 100)
    assert its == 1 and conv
    # preconditioner = A^-1 -> 1 iteration
    A = np.diag(np.arange(1.0, 8.0)) + 0.1
    _, its, _, _ = pcg(lambda v: A @ v, b, lambda v: np.linalg.solve(A, v), 1e-10, 100)
    assert its == 1
    # 1D Laplacian n=10, Jacobi: <= 10 iterations
    L = 2 * np.eye(10) - np.eye(10, k=1) - np.eye(10, k=-1)
    b = np.random.default_rng(1).normal(size=10)
    x, its, conv, _ = pcg(lambda v: L @ v, b, lambda v: v / 2, 1e-10 * np.linalg.norm(b), 100)
    assert its <= 10 and conv
    np.testing.assert_allclose(x, np.linalg.solve(L, b), rtol=1e-9)
    # SPEC.md:241 worked example through the same machinery
    pin = PINS["tridiag_solve"]
    L4 = 2 * np.eye(4) - np.eye(4, k=1) - np.eye(4, k=-1)
    x, _, _, _ = pcg(lambda v: L4 @ v, np.array(pin["b"], float), lambda v: v, 1e-14, 10)
    np.testing.assert_allclose(x, pin["x"], rtol=1e-12)


@pytest.mark.parametrize("n", [5, 20, 50])
def test_pcg_finite_termination(n):
    rng = np.random.default_rng(n)
    Q = np.linalg.qr(rng.normal(size=(n, n)))[0]
    A = Q @ np.diag(np.linspace(1, 10, n)) @ Q.T
    b = rng.normal(size=n)
    _, its, conv, _ = pcg(lambda v: A @ v, b, lambda v: v, 1e-10 * np.linalg.norm(b), 10 * n)
    assert conv and its <= n


def test_exact_schur_preconditioner_one_iteration():
    """S~ = S -> the Schur-system Krylov method converges in 1 iteration."""
    p, T, B = _setup("c1")
    S = dense_schur(B, T.n_G)
    g = condensed_rhs(p, T, B)
    _, its, conv, _ = pcg(lambda v: S @ v, g, lambda v: np.linalg.solve(S, v), 1e-10 * np.linalg.norm(p.rhs), 10)
    assert its == 1 and conv


@pytest.mark.parametrize("name,kw,mode", [
    ("c1", {}, "identity"), ("c1", {}, "lanczos"), ("c1", {}, "dense"),
    ("c2", dict(nel=(64, 32), sub=(16, 16)), "lanczos"),
    ("c4", dict(nel=(12, 6, 6), sub=(3, 3, 3)), "lanczos"),
])
def test_dd_pcg_equals_monolithic(name, kw, mode):
    p = make_config(name, **kw)
    o = DDOracle(p, mode=mode)
    r = o.solve()
    u_ref = monolithic_solve(p)
    assert r.converged
    assert np.linalg.norm(r.u - u_ref) <= 1e-8 * np.linalg.norm(u_ref)
    assert r.relres <= 1e-10


def test_zero_rhs():
    p = make_config("c1")
    p.rhs[:] = 0
    r = DDOracle(p).solve()
    assert r.iterations == 0 and not np.any(r.u)
