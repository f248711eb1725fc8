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

fgmres (NEXT(4), the paper's own outer solver): pinned in tests/test_oracle_fgmres.py by the
minimum-polynomial claim (exact S~ = S gives at most 2 iterations) and by brute-force
least squares over the Krylov space on a tiny system (the residual of GMRES is the minimum there).
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


def fgmres(apply_A, b, apply_P, tol_abs, maxit, restart=30, x0=None):
    """Right-preconditioned flexible GMRES(m) (GMRES on K P~^-1 u~ = f, "flexible GMRES
    [Saad93] to account for the changing nature of the preconditioner"). Arnoldi by modified Gram-Schmidt on
    v_j, z_j = P(v_j) kept for the update x = x0 + Z y; Givens rotations give the residual estimate |g_{j+1}|;
    stop when it is <= tol_abs (then the true residual is recomputed at the restart). Returns
    (x, iterations, converged, history of the estimate)."""
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else x0.astype(np.float64).copy()
    its = 0
    hist = []
    while True:
        r = b - apply_A(x)
        beta = float(np.linalg.norm(r))
        hist.append(beta)
        if beta <= tol_abs:
            return x, its, True, hist
        if its >= maxit:
            return x, its, False, hist
        m = min(restart, maxit - its)
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            Z[j] = apply_P(V[j])
            w = apply_A(Z[j])
            for i in range(j + 1):
                H[i, j] = w @ V[i]
                w = w - H[i, j] * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            if H[j + 1, j] > 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                       # previous rotations on column j
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            rho = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j], sn[j] = H[j, j] / rho, H[j + 1, j] / rho
            H[j, j], H[j + 1, j] = rho, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            k = j + 1
            hist.append(abs(g[j + 1]))
            if abs(g[j + 1]) <= tol_abs or its >= maxit:
                break
        y = np.linalg.solve(np.triu(H[:k, :k]), g[:k])
        x = x + Z[:k].T @ y
