"""Diagnostic: per-iteration time of the c5 bench step split into Schur apply, preconditioner and the rest
(PCG vector kernels, gathers, graph/launch gaps, host polling), for a few check_every values."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synthetic import make_config, density_sequence_step
from paper_1501_06211_b200 import binding as B
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = make_config(name)
for ce in [int(x) for x in (sys.argv[2:] or ["8", "32"])]:
    S = B.Solver.from_problem(p, device=0, warm_start=1, check_every=ce)
    d_rhs = torch.tensor(p.rhs, dtype=torch.float64, device="cuda"); d_u = torch.empty_like(d_rhs)
    rho = p.density.copy()
    rows = []
    for t in range(6):
        if t:
            rho = density_sequence_step(rho, t)
            S.update_densities(rho)
        S.factor()
        prof = t >= 4
        B.de_set_profiling(S.ctx, prof)
        its, rel, _ = B.de_solve_device(S.ctx, d_rhs.data_ptr(), p.rtol, d_u.data_ptr())
        st = S.stats()
        if t >= 2:
            rows.append((its, st.ms_pcg, st.iterations_pass1, st.restarts, prof))
        if prof:
            k_ms, k_n = B.de_get_kernel_time(S.ctx); p_ms, p_n = B.de_get_prec_time(S.ctx)
    B.de_set_profiling(S.ctx, False)
    plain = [r for r in rows if not r[4]]
    its = sum(r[0] for r in plain); ms = sum(r[1] for r in plain)
    print(f"{name} check_every={ce}: {its / len(plain):.0f} its/solve, {ms / its * 1e3:.1f} us/iteration (ms_pcg incl. "
          f"condense/refinement/backsub, profiling off), schur {k_ms * 1e3:.1f} us, prec {p_ms * 1e3:.1f} us, other "
          f"{ms / its * 1e3 - (k_ms + p_ms) * 1e3:.1f} us; passes {[r[2:4] for r in rows]}")
    S.close()
