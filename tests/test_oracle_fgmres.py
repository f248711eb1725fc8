"""Pins of the oracle's full-system flexible GMRES (NEXT(4))."""
import numpy as np
import scipy.sparse as sp

from synthetic import make_config, paper_problem
from oracle.krylov import fgmres
from oracle.solver import DDOracle, monolithic_solve


def test_fgmres_minimises_the_residual_over_the_krylov_space():
    """With P = I, iteration k's residual estimate equals min ||b - A x|| over x in K_k(A, b) (brute force:
    least squares on the explicit Krylov basis)."""
    rng = np.random.default_rng(0)
    n = 12
    A = rng.normal(size=(n, n)) + 4 * np.eye(n)
    b = rng.normal(size=n)
    _, its, conv, hist = fgmres(lambda x: A @ x, b, lambda v: v, 0.0, 8, restart=8)
    Kb = np.stack([np.linalg.matrix_power(A, j) @ b for j in range(8)], axis=1)
    for k in range(1, 9):
        Q, _ = np.linalg.qr(Kb[:, :k])
        y, *_ = np.linalg.lstsq(A @ Q, b, rcond=None)
        best = np.linalg.norm(b - A @ Q @ y)
        assert abs(hist[k] - best) <= 1e-10 * np.linalg.norm(b), (k, hist[k], best)


def test_exact_schur_converges_in_two_iterations():
    """the minimum polynomial of K P^-1 is (lambda - 1)^d, d = 2 blocks -> at most 2 GMRES
    iterations with the exact Steklov-Poincare operator S~ = S."""
    p = make_config("c1")
    r = DDOracle(p).solve_fgmres(rtol=1e-10, exact_S=True)
    assert r.converged and r.iterations <= 2, r.iterations
    assert r.relres <= 1e-10


def test_fgmres_with_h_theta_matches_monolithic():
    p = paper_problem(16, 4)
    r = DDOracle(p).solve_fgmres(rtol=1e-8)
    uref = monolithic_solve(p)
    free = p.fixed == 0
    assert r.converged
    assert np.linalg.norm((r.u - uref)[free]) <= 1e-6 * np.linalg.norm(uref[free])
