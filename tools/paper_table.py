"""Table 1 of the paper re-run on the GPU path: interface-PCG iteration counts for the test
problem of PAPER.md:187 (synthetic.paper_problem) with S~ = I, S~ = H_theta (theta 0.5) and S~ = H_OPT
(theta 0.5 / 0.6 / 0.7 for N = 4 / 16 / 64), rtol 1e-6. The paper's own counts (full-system GMRES) are printed
beside them for the trend comparison; R18 lists why the values differ."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synthetic import paper_problem  # noqa: E402
from paper_1501_06211_b200 import binding as B  # noqa: E402

PAPER = {  # (column, N, 1/h) -> GMRES iterations, Table 1
    "I": {4: (28, 41, 59), 16: (47, 66, 93), 64: (68, 96, 137)},
    "H": {4: (12, 12, 12), 16: (18, 19, 19), 64: (27, 27, 27)},
    "OPT": {4: (12, 12, 12), 16: (17, 18, 19), 64: (22, 23, 24)},
}
THETA_OPT = {4: 0.5, 16: 0.6, 64: 0.7}
HS = (32, 64, 128)
NS = (4, 16, 64)


def its(p, **kw):
    S = B.Solver.from_problem(p, device=0, **kw)
    try:
        S.factor()
        S.solve(p.rhs, p.rtol, allow_noconv=False)
        return S.stats().iterations_pass1
    finally:
        S.close()


def table(title, note, res):
    out = [f"## {title}", "", note, "",
           "| 1/h | I: N=4 | 16 | 64 | H_0.5: N=4 | 16 | 64 | H_OPT (0.5/0.6/0.7): N=4 | 16 | 64 |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for k, ih in enumerate(HS):
        cells = []
        for col in ("I", "H", "OPT"):
            for n in NS:
                cells.append(f"{res[(col, n, ih)]} / {PAPER[col][n][k]}")
        out.append(f"| {ih} | " + " | ".join(cells) + " |")
    return out


def main():
    t0 = time.time()
    out = ["# Table 1 re-run (PAPER.md:201-232) on the B200 path", "",
           "The paper's test problem (`synthetic.paper_problem`, DESIGN.md R18), k = 10 Lanczos vectors, exact inner",
           "solves, tolerance 1e-6; cell = ours / paper (paper: GMRES on the full system).", ""]
    for outer, title, note in (
            (1, "Full-system FGMRES with P~ = [[K_II, K_IG], [0, S~]] (the paper's solver, NEXT(4))",
             "Right-preconditioned flexible GMRES(31) on K u = f (PAPER.md:153-181)."),
            (0, "Interface PCG (the BASELINE method)", "PCG on S u_Gamma = g, rtol 1e-6 on ||f||.")):
        res = {}
        kw0 = dict(outer=1, restart=31) if outer else {}
        for n in NS:
            for ih in HS:
                p = paper_problem(ih, n)
                res[("I", n, ih)] = its(p, inner_mode=3, **kw0)
                res[("H", n, ih)] = its(p, theta=0.5, **kw0)
                res[("OPT", n, ih)] = its(p, theta=THETA_OPT[n], **kw0)
        out += table(title, note, res) + [""]
    out += [f"wall time {time.time() - t0:.1f} s"]
    print("\n".join(out))


if __name__ == "__main__":
    main()
