"""Writes tests/golden/fullsize_<case>.npz: the ORACLE's reference answers at the BASELINE sizes, sampled.

Calls only oracle/ and synthetic/ (never the CUDA path). For each case the plain definition u_ref = K_ff^-1 f_f
(Eq. (4)) by oracle.direct (nested-dissection Cholesky + extended-precision refinement, u_ref =
hi + lo) is computed once here, because it takes minutes per case on a host (c4: a 3D factorisation of 0.7 M dofs;
c5: 4.2 M dofs, three density states) -- too long for the GPU test run. Stored per case:
  idx        16,384 seeded sample positions among the free dofs (sorted)
  u_hi,u_lo  u_ref at idx (hi + lo)
  norm_u     ||fl(u_ref)||_2 over all dofs
  floor      relres of fl(u_ref) in extended precision: the FP64 floor of the final-residual gate (R17)
  hist       refinement history of that relres
  sha        sha256 of the density and rhs bytes the case was generated from (the GPU test checks its inputs match)
  backward   (c3 only) normwise backward error of the direct solve, SURVEY Q15
Usage: python tools/make_fullsize_goldens.py [c2 c4 c5_t0 c5_t24 c5_t49 c3]
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synthetic import make_config, density_sequence_step  # noqa: E402
from oracle.direct import refine_dd, direct_solve  # noqa: E402
from oracle.fem import free_system  # noqa: E402

NSAMPLE = 16384


def input_sha(p):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(p.density, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(p.rhs, dtype=np.float64).tobytes())
    return h.hexdigest()


def sample_idx(p, seed=1234):
    free = np.flatnonzero(np.asarray(p.fixed) == 0)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(free, size=min(NSAMPLE, len(free)), replace=False))


def problem(case):
    if case.startswith("c5_t"):
        t_end = int(case[4:])
        p = make_config("c5")
        rho = p.density.copy()
        for t in range(1, t_end + 1):
            rho = density_sequence_step(rho, t)
        return p.with_density(rho)
    return make_config(case)


def main(cases):
    out = os.path.join(ROOT, "tests", "golden")
    for case in cases:
        t0 = time.time()
        p = problem(case)
        idx = sample_idx(p)
        extra = {}
        if case == "c3":   # FP64-ill-posed (R15): the direct solve and its normwise backward error
            K, f, free = free_system(p)
            hi = direct_solve(p)
            lo = np.zeros_like(hi)
            r = f - K @ hi[free]
            extra["backward"] = np.linalg.norm(r) / (abs(K).sum(axis=0).max() * np.linalg.norm(hi[free]) + np.linalg.norm(f))
            hist = [np.linalg.norm(r) / np.linalg.norm(f)]
        else:
            hi, lo, hist = refine_dd(p, rounds=2)
        np.savez(os.path.join(out, f"fullsize_{case}.npz"), idx=idx, u_hi=hi[idx], u_lo=lo[idx],
                 norm_u=np.linalg.norm(hi), floor=hist[-1], hist=np.asarray(hist), sha=input_sha(p), **extra)
        print(f"{case}: ndof {p.ndof}, ||u_ref|| {np.linalg.norm(hi):.6e}, floor {hist[-1]:.4e}, hist {hist}, "
              f"{extra} {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c4", "c5_t0", "c5_t24", "c5_t49", "c3"])
