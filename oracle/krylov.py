"""ORACLE (test infrastructure only) — outer interface PCG.

Paper: PAPER.md:142 (interface equation S u_Gamma = g)
("conjugate gradient as a suitable alternative, coupled with an appropriate
preconditioning strategy (PCG)"); BASELINE.json metric "interface-PCG"
(rtol 1e-10).  SPEC.md:312-326 for the contract.  Readings (R11):
Fletcher-Reeves beta by default (Polak-Ribiere flexible variant optional);
stop when ||r||_2 <= tol_abs on the recursive residual.  Iterations = S
applications inside the loop.  (The end-of-solve accuracy check is iterative
refinement on the full system, oracle/solver.py.)

Pins (tests/test_oracle_dd_krylov.py): A = I -> 1 iteration; preconditioner =
A^-1 -> 1 iteration; finite termination <= n at 1e-10 for n <= 50; 1D
Laplacian n=10 with Jacobi <= 10 iterations.
"""
from __future__ import annotations

import numpy as np


class NotSPD(RuntimeError):
    pass


def pcg(apply_A, b, apply_P, tol_abs, maxit, x0=None, beta="FR"):
    """Returns (x, iterations, converged, history)."""
    x = np.zeros_like(b) if x0 is None else x0.astype(np.float64).copy()
    r = b - apply_A(x) if x0 is not None and np.any(x0) else b.copy()
    its = 0
    hist = [float(np.linalg.norm(r))]
    if hist[0] <= tol_abs:
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
            return x, its, True, hist
        z_new = apply_P(r)
        rz_new = r @ z_new
        bta = rz_new / rz if beta == "FR" else (z_new @ (r - r_old)) / rz
        p = z_new + bta * p
        rz = rz_new
    return x, its, False, hist
