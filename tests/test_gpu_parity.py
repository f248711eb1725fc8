"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded inputs.

Tolerances: integer/index data bit-exact; assembled blocks 1e-13 relative to the
block's max entry (same products, different summation order); factor 1e-11; Schur apply 1e-11
(norm-wise, relative); preconditioner 1e-9 (ten Lanczos steps with different reduction orders);
solutions: the BASELINE gates, ||u - u_ref|| <= 1e-8 ||u_ref|| and true relres <= 1e-10.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synthetic import make_config, density_sequence_step  # noqa: E402
from oracle.topology import build_topology  # noqa: E402
from oracle.dd import subdomain_blocks, factor_subdomains, schur_apply, half_bandwidth  # noqa: E402
from oracle.precond import build_components, apply_precond  # noqa: E402
from oracle.solver import monolithic_solve, DDOracle  # noqa: E402
from oracle.fem import true_relres  # noqa: E402

SMALL = [("c1", {}), ("c2", dict(nel=(64, 32), sub=(16, 16))), ("c2", dict(nel=(40, 24), sub=(8, 6))),
         ("c3", dict(nel=(64, 32), sub=(16, 16))), ("c4", dict(nel=(12, 6, 6), sub=(3, 3, 3))),
         ("c4", dict(nel=(12, 12, 6), sub=(6, 6, 6)))]


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


def _ids(c):
    return [f"{n}-{'x'.join(map(str, k.get('nel', ())))}" for n, k in c]


@pytest.mark.parametrize("name,kw", SMALL, ids=_ids(SMALL))
def test_bands_match_oracle(name, kw):
    from paper_1501_06211_b200 import binding as B
    p = make_config(name, **kw)
    T = build_topology(p)
    blocks = factor_subdomains(subdomain_blocks(p, T))
    S = _solver(p)
    try:
        for sl in sorted({0, T.nsub // 2, T.nsub - 1}):
            A = B.de_get_assembled_band(S.ctx, sl)
            b = blocks[sl]
            n, kb = b.AII.shape[0], half_bandwidth(b.AII)
            assert A.shape[0] == n
            C = b.AII.tocoo()
            ref = np.zeros_like(A)
            low = C.row >= C.col
            ref[C.col[low], C.row[low] - C.col[low]] = C.data[low]
            scale = np.abs(ref).max()
            assert np.abs(A - ref).max() <= 1e-13 * scale
            assert np.all(A[:, kb + 1:] == 0)
        S.factor()
        for sl in sorted({0, T.nsub // 2, T.nsub - 1}):
            L = B.de_get_factor_band(S.ctx, sl)
            b = blocks[sl]
            kb = b.band
            ref = b.chol.T          # scipy lower band: chol[k, j] = L[j+k, j]
            # backward error of the GPU factor (independent of the summation order): Cholesky gives
            # |L L^T - A| <= (b+2) eps |L||L^T| elementwise (Higham, Thm 10.3); checked normwise with a x4 margin
            n = L.shape[0]
            Ld = np.zeros((n, n))
            for k in range(kb + 1):
                idx = np.arange(n - k)
                Ld[idx + k, idx] = L[:n - k, k]
            Ad = b.AII.toarray()
            bound = 4 * (kb + 2) * np.finfo(float).eps * (np.abs(Ld) @ np.abs(Ld).T).max()
            assert np.abs(Ld @ Ld.T - Ad).max() <= bound
            # forward agreement with scipy's factor: each side has the backward error above, so they differ by
            # about kappa * (b+2) eps; 1e-9 covers the high-contrast c3 instance (densities 1e-3 .. 1)
            assert np.abs(L[:, :kb + 1] - ref).max() <= 1e-9 * np.abs(ref).max()
            assert np.all(L[:, kb + 1:] == 0)
    finally:
        S.close()


@pytest.mark.parametrize("name,kw", SMALL, ids=_ids(SMALL))
def test_schur_apply_matches_oracle(name, kw):
    from paper_1501_06211_b200 import binding as B
    p = make_config(name, **kw)
    T = build_topology(p)
    blocks = factor_subdomains(subdomain_blocks(p, T))
    for mode in (1, 2):     # 1: implicit (interior solves each apply), 2: explicit local S_s (NEXT(1))
        S = _solver(p, schur_mode=mode)
        try:
            S.factor()
            assert S.stats().schur_explicit == (1 if mode == 2 else 0)
            rng = np.random.default_rng(11)
            for trial in range(2):
                x = rng.normal(size=T.n_G)
                ref = schur_apply(blocks, T.n_G, x)
                dx = torch.tensor(x, dtype=torch.float64, device="cuda")
                dq = torch.empty_like(dx)
                B.de_schur_apply_device(S.ctx, dx.data_ptr(), dq.data_ptr())
                q = dq.cpu().numpy()
                assert np.linalg.norm(q - ref) <= 1e-11 * np.linalg.norm(ref), mode
                assert np.abs(q - ref).max() <= 1e-11 * np.abs(ref).max(), mode          # element-wise
        finally:
            S.close()


@pytest.mark.parametrize("name,kw", SMALL, ids=_ids(SMALL))
def test_preconditioner_matches_oracle(name, kw):
    from paper_1501_06211_b200 import binding as B
    p = make_config(name, **kw)
    T = build_topology(p)
    comps = build_components(p, T)
    for impl in (0, 1):     # 0: persistent cooperative kernel, 1: one kernel per phase
        _check_precond(p, T, comps, impl)


def _check_precond(p, T, comps, impl):
    from paper_1501_06211_b200 import binding as B
    S = _solver(p, prec_kernels=impl)
    try:
        rng = np.random.default_rng(12)
        for trial in range(2):
            r = rng.normal(size=T.n_G)
            if trial == 1:                      # zero component input -> zero output (R9)
                r[comps[0].skel.gidx] = 0.0
            ref = apply_precond(comps, r, "lanczos", 0.5, 10, "X")
            dr = torch.tensor(r, dtype=torch.float64, device="cuda")
            dz = torch.empty_like(dr)
            B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr())
            z = dz.cpu().numpy()
            assert np.linalg.norm(z - ref) <= 1e-9 * np.linalg.norm(ref), (impl, np.linalg.norm(z - ref) / np.linalg.norm(ref))
            for cd in comps:                                   # element-wise, per component (the norm is componentwise)
                g = cd.skel.gidx
                if np.abs(ref[g]).max() > 0:
                    assert np.abs(z[g] - ref[g]).max() <= 1e-9 * np.abs(ref[g]).max(), impl
            if trial == 1:
                assert np.all(z[comps[0].skel.gidx] == 0.0)
    finally:
        S.close()


@pytest.mark.parametrize("k,theta", [(4, 0.5), (12, 0.25), (16, 0.5)])
@pytest.mark.parametrize("name,kw", [SMALL[2], SMALL[4]], ids=_ids([SMALL[2], SMALL[4]]))
def test_preconditioner_lanczos_k_theta(name, kw, k, theta):
    """Basis sizes on both sides of the cooperative kernel's compile-time bound (10) and theta != 1/2
    (SPEC.md:374-413), cooperative kernel vs oracle O8."""
    from paper_1501_06211_b200 import binding as B
    p = make_config(name, **kw)
    T = build_topology(p)
    comps = build_components(p, T)
    S = _solver(p, lanczos_k=k, theta=theta)
    try:
        r = np.random.default_rng(13).normal(size=T.n_G)
        ref = apply_precond(comps, r, "lanczos", theta, k, "X")
        dr = torch.tensor(r, dtype=torch.float64, device="cuda")
        dz = torch.empty_like(dr)
        B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr())
        z = dz.cpu().numpy()
        assert np.linalg.norm(z - ref) <= 1e-9 * np.linalg.norm(ref), np.linalg.norm(z - ref) / np.linalg.norm(ref)
    finally:
        S.close()


WELL_POSED = [c for c in SMALL if c[0] != "c3"] + [("c2", {}), ("c4", dict(nel=(24, 12, 12), sub=(6, 6, 6)))]


@pytest.mark.parametrize("name,kw", WELL_POSED, ids=_ids(WELL_POSED))
def test_solve_matches_monolithic(name, kw):
    p = make_config(name, **kw)
    u_ref = monolithic_solve(p)
    S = _solver(p)
    try:
        S.factor()
        u, its, relres, _ = S.solve(p.rhs, p.rtol)
        err = np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref)
        assert err <= 1e-8, err
        assert relres <= 1e-10
        assert true_relres(p, u) <= 1e-10            # independent residual (oracle's K)
        assert np.all(u[p.fixed != 0] == 0.0)
        o = DDOracle(p)
        ro = o.solve()
        # same algorithm, different rounding: PCG iteration counts (before refinement) within 5 %
        its1 = S.stats().iterations_pass1
        assert abs(its1 - ro.its_pass1) <= max(2, 0.05 * ro.its_pass1), (its1, ro.its_pass1, its, ro.iterations)
    finally:
        S.close()


def test_identity_preconditioner_and_flexible_beta():
    p = make_config("c2", nel=(64, 32), sub=(16, 16))
    u_ref = monolithic_solve(p)
    for kw in (dict(inner_mode=3), dict(beta_variant=1), dict(use_graph=0, check_every=3), dict(prec_kernels=1),
               dict(schur_mode=1), dict(schur_mode=2)):
        S = _solver(p, **kw)
        try:
            S.factor()
            u, its, relres, _ = S.solve(p.rhs, p.rtol)
            assert np.linalg.norm(u - u_ref) <= 1e-8 * np.linalg.norm(u_ref), kw
            assert relres <= 1e-10
        finally:
            S.close()


def test_ill_posed_c3_iterates_match_oracle():
    """R15: config 3 cannot reach 1e-10 in FP64; compare the iterates at a fixed budget."""
    p = make_config("c3", nel=(64, 32), sub=(16, 16))
    S = _solver(p, max_iter=20)
    try:
        S.factor()
        u, its, relres, st = S.solve(p.rhs, p.rtol, allow_noconv=True)
        assert its == 20
        o = DDOracle(p)
        ro = o.solve(maxit=20)
        assert ro.iterations == 20
        assert np.linalg.norm(u - ro.u) <= 1e-6 * np.linalg.norm(ro.u)
    finally:
        S.close()


def test_zero_rhs_and_state_errors():
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    S = _solver(p)
    try:
        with pytest.raises(B.DEError) as ei:
            S.solve(p.rhs, 1e-10)
        assert ei.value.status == B.DE_ESTATE
        S.factor()
        u, its, relres, _ = S.solve(np.zeros_like(p.rhs), 1e-10)
        assert its == 0 and not np.any(u)
    finally:
        S.close()


def test_config5_sequence_warm_start():
    """C7: densities evolve, refactor each step, warm-started PCG (scaled-down config-5 recipe)."""
    p = make_config("c5", nel=(128, 64), sub=(32, 32))
    S = _solver(p, warm_start=1)
    rho = p.density.copy()
    try:
        its_all = []
        for t in range(4):
            if t > 0:
                rho = density_sequence_step(rho, t)
                S.update_densities(rho)
            S.factor()
            pt = p.with_density(rho)
            u, its, relres, _ = S.solve(p.rhs, p.rtol)
            its_all.append(its)
            u_ref = monolithic_solve(pt)
            assert np.linalg.norm(u - u_ref) <= 1e-8 * np.linalg.norm(u_ref)
            assert relres <= 1e-10
        assert max(its_all[1:]) < its_all[0]
    finally:
        S.close()


def test_c3_full_size_budgeted_iterates_match_oracle():
    """R15 at the BASELINE size: config 3 is FP64-ill-posed, so the gate is agreement of the GPU
    and oracle interface iterates after the same fixed budget (same algorithm, same inputs)."""
    p = make_config("c3")
    S = _solver(p, max_iter=6)
    try:
        S.factor()
        u, its, relres, st = S.solve(p.rhs, p.rtol, allow_noconv=True)
        assert its == 6
        o = DDOracle(p)
        ro = o.solve(maxit=6)
        uG = u[o.topo.gamma_dofs]
        assert np.linalg.norm(uG - ro.uG) <= 1e-6 * np.linalg.norm(ro.uG)
    finally:
        S.close()
