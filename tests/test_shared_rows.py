"""A shared cross-point inverse S_C^-1 (identical components: HElim::sc_shared) can be applied for ALL components by
the block that loads a row (default for three components, the 3D wirebasket; env DE_SHR=1 forces it in 2D, where it
measured slower). Same arithmetic per row, other reduction layout: checked against the default per-component path on
identical inputs, including a zero component (basis sizes differ between components) -- DESIGN.md §6."""
import os

import numpy as np
import pytest

from synthetic import make_config
from oracle.topology import build_topology
from oracle.precond import build_components


def _z(p, rs, shr):
    import torch
    from paper_1501_06211_b200 import binding as B
    if shr:
        os.environ["DE_SHR"] = "1"
    try:
        S = B.Solver.from_problem(p, device=0)
    finally:
        os.environ.pop("DE_SHR", None)
    try:
        S.factor()
        out = []
        for r in rs:
            dr = torch.tensor(r, dtype=torch.float64, device="cuda")
            dz = torch.empty_like(dr)
            B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr())
            out.append(dz.cpu().numpy())
        u, its, rel, st = S.solve(p.rhs, 1e-10)
        return out, its
    finally:
        S.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw", [("c2", dict(nel=(64, 32), sub=(16, 16))), ("c2", {}), ("c5", dict(nel=(256, 160), sub=(32, 32)))],
                         ids=["c2-64x32", "c2", "c5-8x5"])
def test_shared_rows_equal_per_component_rows(name, kw):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = make_config(name, **kw)
    T = build_topology(p)
    comps = build_components(p, T)
    rng = np.random.default_rng(41)
    r0 = rng.normal(size=T.n_G)
    r1 = r0.copy()
    r1[comps[0].skel.gidx] = 0.0           # zero component input -> zero output (R9), other component unchanged
    za, ita = _z(p, [r0, r1], True)
    zb, itb = _z(p, [r0, r1], False)
    for x, y in zip(za, zb):
        assert np.linalg.norm(x - y) <= 1e-11 * np.linalg.norm(y)
    assert np.all(za[1][comps[0].skel.gidx] == 0.0)
    assert abs(ita - itb) <= 1


@pytest.mark.gpu
def test_block_bidiagonal_face_solves_equal_band_sweeps():
    """3D face solves through the block-bidiagonal form of the face factors (env DE_FB=1, opt-in: measured no faster)
    against the default row-by-row band sweeps, same inputs."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_06211_b200 import binding as B
    p = make_config("c4", nel=(24, 12, 12), sub=(6, 6, 6))
    T = build_topology(p)
    r = np.random.default_rng(43).normal(size=T.n_G)
    zs = []
    for fb in (True, False):
        if fb:
            os.environ["DE_FB"] = "1"
        try:
            S = B.Solver.from_problem(p, device=0)
        finally:
            os.environ.pop("DE_FB", None)
        try:
            S.factor()
            dr = torch.tensor(r, dtype=torch.float64, device="cuda")
            dz = torch.empty_like(dr)
            B.de_precond_apply_device(S.ctx, dr.data_ptr(), dz.data_ptr())
            zs.append(dz.cpu().numpy())
        finally:
            S.close()
    assert np.linalg.norm(zs[0] - zs[1]) <= 1e-10 * np.linalg.norm(zs[1])
