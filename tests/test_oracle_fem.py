"""Oracle pins: material law, Q1 element, assembly (CPU only)."""
import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from synthetic import make_config
from oracle import fem

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def test_lame_closed_forms():
    mu, lam = fem.lame(1.0, 0.3)
    assert mu == pytest.approx(PINS["lame_E1_nu03"]["mu"], rel=1e-15)
    assert lam == pytest.approx(PINS["lame_E1_nu03"]["lambda_hat"], rel=1e-15)
    assert fem.lame(2.6, 0.3)[0] == pytest.approx(1.0, rel=1e-15)
    assert fem.lame(1.0, 0.0) == (0.5, 0.0)
    # plane stress reduction vs the independent form nu E/(1-nu^2)
    assert fem.plane_stress_lambda(1.0, 0.3) == pytest.approx(
        PINS["plane_stress_lambda_E1_nu03"]["value"], rel=1e-14)


def test_q1_2d_matches_published_closed_form():
    pin = PINS["q1_2d_ke_k_vector"]
    nu = pin["nu"]
    k = np.array([1 / 2 - nu / 6, 1 / 8 + nu / 8, -1 / 4 - nu / 12, -1 / 8 + 3 * nu / 8,
                  -1 / 4 + nu / 12, -1 / 8 - nu / 8, nu / 6, 1 / 8 - 3 * nu / 8]) / (1 - nu ** 2)
    KT = k[np.array(pin["index"]) - 1]
    K = fem.element_stiffness(2, nu)
    # oracle local order is lexicographic (0,0),(1,0),(0,1),(1,1); closed form is CCW
    ccw = [0, 1, 3, 2]
    d = np.array([[2 * a, 2 * a + 1] for a in ccw]).ravel()
    np.testing.assert_allclose(K[np.ix_(d, d)], KT, atol=1e-15)
    np.testing.assert_allclose(np.linalg.eigvalsh(K), PINS["q1_2d_ke_eigs_nu03"]["values"], atol=1e-14)


def test_q1_2d_scales_with_E_not_h():
    K1 = fem.element_stiffness(2, 0.3, 1.0, 1.0)
    np.testing.assert_allclose(fem.element_stiffness(2, 0.3, 3.0, 0.25), 3.0 * K1, rtol=1e-14)


def test_q1_3d_invariants():
    pin = PINS["q1_3d_ke_nu03"]
    K = fem.element_stiffness(3, 0.3)
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12) == pin["n_zero"]
    assert ev[6] == pytest.approx(pin["smallest_nonzero"], rel=1e-10)
    np.testing.assert_allclose(np.diag(K), pin["diag"], rtol=1e-10)
    assert np.trace(K) == pytest.approx(pin["trace"], rel=1e-12)
    # 3D stiffness scales with h (length^(d-2))
    np.testing.assert_allclose(fem.element_stiffness(3, 0.3, 1.0, 2.0), 2.0 * K, rtol=1e-14)


@pytest.mark.parametrize("dim", [2, 3])
def test_rigid_modes_in_element_kernel(dim):
    K = fem.element_stiffness(dim, 0.3)
    X = np.array(fem.local_nodes(dim), dtype=float)
    modes = []
    for c in range(dim):
        t = np.zeros((len(X), dim))
        t[:, c] = 1
        modes.append(t.ravel())
    pairs = [(0, 1)] if dim == 2 else [(0, 1), (1, 2), (0, 2)]
    for a, b in pairs:
        r = np.zeros((len(X), dim))
        r[:, a] = -X[:, b]
        r[:, b] = X[:, a]
        modes.append(r.ravel())
    for m in modes:
        assert np.abs(K @ m).max() < 1e-14


def test_simp_law():
    assert fem.simp_modulus(1.0, 1.0, 1e-9, 3.0) == 1.0
    assert fem.simp_modulus(0.5, 1.0, 0.0, 3.0) == 0.125
    assert fem.simp_modulus(0.0, 2.0, 1e-9, 3.0) == 1e-9


def test_density_linearity_p1_emin0():
    """with p=1, Emin=0 the stiffness is linear in rho (the paper's VTS K(rho)=sum rho_i K_i)."""
    p = make_config("c2", nel=(8, 4), sub=(4, 2))
    KE = fem.element_stiffness(2, 0.3)
    rng = np.random.default_rng(0)
    r1, r2 = rng.uniform(0.1, 1, 32), rng.uniform(0.1, 1, 32)
    K = lambda r: fem.assemble_global(2, p.nel, fem.simp_modulus(r, 1.0, 0.0, 1.0), KE)
    assert abs(K(r1) + K(r2) - K(r1 + r2)).max() < 1e-14


@pytest.mark.parametrize("dim", [2, 3])
def test_patch_test(dim):
    """a linear displacement field prescribed on the boundary is reproduced
    exactly in the interior (uniform material)."""
    nel = (5, 4) if dim == 2 else (3, 3, 2)
    KE = fem.element_stiffness(dim, 0.3)
    K = fem.assemble_global(dim, nel, np.ones(int(np.prod(nel))), KE).tocsr()
    X = fem.node_coords(dim, nel)
    rng = np.random.default_rng(1)
    A, b = rng.normal(size=(dim, dim)), rng.normal(size=dim)
    u_ex = (X @ A.T + b).ravel()
    on_bnd = np.zeros(len(X), dtype=bool)
    for d in range(dim):
        on_bnd |= (X[:, d] == 0) | (X[:, d] == nel[d])
    bd = np.repeat(on_bnd, dim)
    fr = ~bd
    u = u_ex.copy()
    u[fr] = spla.spsolve(K[fr][:, fr].tocsc(), -K[fr][:, bd] @ u_ex[bd])
    assert np.abs(u - u_ex).max() < 1e-12


def test_assembled_symmetry_and_load_sums():
    p = make_config("c2", nel=(16, 8), sub=(8, 4))
    K, f, free = fem.free_system(p)
    assert abs(K - K.T).max() < 1e-14 * abs(K).max()
    assert p.rhs[1::2].sum() == pytest.approx(-1.0, abs=1e-14)
    p4 = make_config("c4", nel=(4, 2, 2), sub=(2, 1, 1))
    assert p4.rhs[1::3].sum() == pytest.approx(-1.0, abs=1e-14)


def test_matrix_free_equals_assembled():
    p = make_config("c4", nel=(4, 2, 2), sub=(2, 1, 1))
    KE = fem.element_stiffness(3, 0.3)
    K = fem.assemble_global(3, p.nel, fem.simp_modulus(p.density, 1, 1e-9, 3), KE)
    u = np.random.default_rng(3).normal(size=p.ndof)
    np.testing.assert_allclose(fem.apply_K(p, u), K @ u, rtol=1e-12, atol=1e-14)
