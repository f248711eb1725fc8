"""Inner modes side by side on the GPU (R10): outer iterations, time per
outer iteration and inner face-PCG iterations per K-solve for mode X (exact elimination, inner_mode 1) and
mode F (SPEC's face-preconditioned PCG, tol 1e-3, inner_mode 0) on BASELINE configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synthetic import make_config  # noqa: E402
from paper_1501_06211_b200 import binding as B  # noqa: E402

rows = []
for name in sys.argv[1:] or ["c2", "c4", "c5"]:
    p = make_config(name)
    for mode in ((1,) if os.environ.get("ONLY_X") else (1, 0)):
        S = B.Solver.from_problem(p, device=0, inner_mode=mode)
        try:
            S.factor()
            S.solve(p.rhs, 1e-10, allow_noconv=True)          # warm-up (graph capture, allocations)
            n0 = S.stats().inner_iterations
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            u, its, rel, st = S.solve(p.rhs, 1e-10, allow_noconv=True)
            dt = time.perf_counter() - t0
            s = S.stats()
            k_solves = max(1, s.iterations * 9)
            rows.append(f"| {name} | {'X' if mode == 1 else 'F'} | {s.iterations_pass1} | {rel:.2e} | "
                        f"{1e3 * dt / max(1, s.iterations):.3f} | "
                        f"{(s.inner_iterations - n0) / k_solves:.1f} |" if mode == 0 else
                        f"| {name} | X | {s.iterations_pass1} | {rel:.2e} | {1e3 * dt / max(1, s.iterations):.3f} | exact |")
        finally:
            S.close()
print("| config | inner | outer iterations | true relres | ms / outer iteration | inner its per K-solve |")
print("|---|---|---|---|---|---|")
print("\n".join(rows))
