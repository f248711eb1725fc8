"""ORACLE (test infrastructure only) — outer interface PCG.

Paper: PAPER.md:142 (interface equation S u_Gamma = g)
("conjugate gradient as a suitable alternative, coupled with an appropriate
preconditioning strategy (PCG)"); BASELINE.json metric "interface-PCG"
(rtol 1e-10).  SPEC.md:312-326 for the contract.  Readings (R11):
Fletcher-Reeves beta by default (Polak-Ribiere flexible variant optional);
stop when ||r||_2 <= rtol * ||f_free||_2 on the recursive residual, then
recompute the true residual g - S x and restart from it if it fails the test
(residual replacement).  Iterations = S applications inside the loop.

Pins (tests/test_oracle_dd_krylov.py): A = I -> 1 iteration; preconditioner =
A^-1 -> 1 iteration; finite termination <= n at 1e-10 for n <= 50; 1D
Laplacian n=10 with Jacobi <= 10 iterations.
"""
from __future__ import annotations

import numpy as np


class NotSPD(RuntimeError):
    pass


def pcg(apply_A, b, apply_P, tol_abs, maxit, x0=None, beta="FR", max_restarts=5):
    """Returns (x, iterations, converged, history)."""
    x = np.zeros_like(b) if x0 is None else x0.astype(np.float64).copy()
    r = b - apply_A(x) if x0 is not None and np.any(x0) else b.copy()
    its = 0
    hist = [float(np.linalg.norm(r))]
    restarts = 0
    while True:
        if np.linalg.norm(r) <= tol_abs:
            return x, its, True, hist
        z = apply_P(r)
        p = z.copy()
        rz = r @ z
        while its < maxit:
            q = apply_A(p)
            pq = p @ q
            if not pq > 0:
                raise NotSPD("p^T S p <= 0")
            a = rz / pq
            x = x + a * p
            r_old = r
            r = r - a * q
            its += 1
            hist.append(float(np.linalg.norm(r)))
            if hist[-1] <= tol_abs:
                break
            z_new = apply_P(r)
            if beta == "FR":
                rz_new = r @ z_new
                bta = rz_new / rz
            else:
                rz_new = r @ z_new
                bta = (z_new @ (r - r_old)) / rz
            p = z_new + bta * p
            rz = rz_new
        # residual replacement check
        r = b - apply_A(x)
        if np.linalg.norm(r) <= tol_abs or its >= maxit or restarts >= max_restarts:
            return x, its, bool(np.linalg.norm(r) <= tol_abs), hist
        restarts += 1
