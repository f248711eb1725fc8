"""Error paths and reproducibility of the C-ABI on the GPU (include/de.h error contracts; SPEC.md:238 non-SPD,
:298 non-convergence returns the last iterate, :316 p^T S p <= 0, :387 Ritz breakdown)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synthetic import make_config  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_06211_b200.build import build
    build()
    torch.cuda.set_device(0)


def _solver(p, **kw):
    from paper_1501_06211_b200 import binding as B
    return B.Solver.from_problem(p, device=0, **kw)


def _interface_elements(p):
    """Element mask: elements with a node on a subdomain interface line (2D)."""
    nx, ny = p.nel
    sx, sy = p.sub
    ex, ey = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    on_x = ((ex % sx == 0) & (ex > 0)) | (((ex + 1) % sx == 0) & (ex + 1 < nx))
    on_y = ((ey % sy == 0) & (ey > 0)) | (((ey + 1) % sy == 0) & (ey + 1 < ny))
    return (on_x | on_y).ravel()


def test_enoconv_returns_last_iterate():
    from paper_1501_06211_b200 import binding as B
    p = make_config("c2", nel=(64, 32), sub=(16, 16))
    S = _solver(p, max_iter=3)
    try:
        S.factor()
        with pytest.raises(B.DEError) as ei:
            S.solve(p.rhs, 1e-10)
        assert ei.value.status == B.DE_ENOCONV
        u, its, rel, st = S.solve(p.rhs, 1e-10, allow_noconv=True)
        assert st == B.DE_ENOCONV and its == 3 and np.all(np.isfinite(u)) and np.isfinite(rel)
        assert u[p.fixed == 1].max() == 0 and u[p.fixed == 1].min() == 0
        # the returned u is the third PCG iterate (back-substituted): the oracle's after the same 3 iterations
        from oracle.solver import DDOracle
        ro = DDOracle(p).solve(maxit=3)
        assert ro.iterations == 3
        assert np.linalg.norm(u - ro.u) <= 1e-9 * np.linalg.norm(ro.u)
    finally:
        S.close()


def test_enotspd_names_the_subdomain():
    """Zero stiffness (Emin = 0, rho^p underflows to 0) on every element of subdomain 3: A_II,3 is singular."""
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    nx, ny = p.nel
    ex, ey = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    rho = np.where(((ex >= 16) & (ey >= 8)).ravel(), 1e-120, 0.5)
    q = p.with_density(rho)
    q.Emin = 0.0
    S = _solver(q)
    try:
        with pytest.raises(B.DEError) as ei:
            S.factor()
        assert ei.value.status == B.DE_ENOTSPD
        assert "subdomain 3" in str(ei.value)
        with pytest.raises(B.DEError) as ei:
            S.solve(p.rhs, 1e-10)
        assert ei.value.status == B.DE_ESTATE
    finally:
        S.close()


def test_ebreakdown_when_schur_complement_vanishes():
    """Zero stiffness on every element touching an interface line, the outer boundary clamped: the interior blocks
    stay SPD (each subdomain's stiff core touches the clamped boundary) but K_GG = K_GI = 0, so S = 0 and
    p^T S p = 0 at the first iteration."""
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    rho = np.where(_interface_elements(p), 1e-120, 0.5)
    q = p.with_density(rho)
    q.Emin = 0.0
    nx, ny = p.nel                                            # clamp the whole outer boundary so every
    X, Y = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), indexing="xy")   # subdomain's stiff core is anchored
    bnd = ((X == 0) | (X == nx) | (Y == 0) | (Y == ny)).ravel()
    q.fixed = np.repeat(bnd, 2).astype(np.uint8)
    f = np.zeros(p.ndof)
    f[2 * (16 + 33 * 8) + 1] = -1.0                           # the cross point (16, 8)
    S = _solver(q)
    try:
        S.factor()
        with pytest.raises(B.DEError) as ei:
            S.solve(f, 1e-10)
        assert ei.value.status == B.DE_EBREAKDOWN
    finally:
        S.close()


def test_einval_nonfinite_rhs():
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    S = _solver(p)
    try:
        S.factor()
        f = p.rhs.copy()
        f[np.flatnonzero(p.fixed == 0)[5]] = np.nan
        with pytest.raises(B.DEError) as ei:
            S.solve(f, 1e-10)
        assert ei.value.status == B.DE_EINVAL
    finally:
        S.close()


@pytest.mark.parametrize("name,kw", [("c2", dict(nel=(128, 64), sub=(32, 32))),
                                     ("c4", dict(nel=(24, 12, 12), sub=(6, 6, 6)))])
def test_bitwise_reproducible(name, kw):
    """every reduction is fixed-order, so two solves (two contexts, and the same context twice)
    give bitwise identical u and identical iteration counts."""
    p = make_config(name, **kw)
    outs = []
    for rep in range(2):
        S = _solver(p)
        try:
            S.factor()
            for _ in range(2):
                u, its, rel, _ = S.solve(p.rhs, p.rtol)
                outs.append((u.copy(), its, rel))
        finally:
            S.close()
    for u, its, rel in outs[1:]:
        assert its == outs[0][1] and rel == outs[0][2]
        assert np.array_equal(u, outs[0][0])
