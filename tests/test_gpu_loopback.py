"""The multi-rank path of libde (nranks > 1: owned subdomain slabs, partial interface sums, the exchanges of g,
q and u, the cross-rank pivot agreement) executed on one GPU through a loopback group (include/de.h
de_loopback_create): G contexts, one host thread each, all-reduce = fixed-order sum of the ranks' device slots
behind host barriers (no kernel waits on another rank's kernel). DESIGN.md §8."""
import threading

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


def _run_ranks(p, G, fn, **opts):
    """Create G contexts in one loopback group and run fn(rank, solver) in G threads; returns the results."""
    from paper_1501_06211_b200 import binding as B
    g = B.de_loopback_create(G)
    out, err, solvers = [None] * G, [None] * G, [None] * G

    def work(r):
        try:
            solvers[r] = B.Solver.from_problem(p, device=0, rank=r, nranks=G, loopback=g, **opts)
            out[r] = fn(r, solvers[r])
        except Exception as ex:   # noqa: BLE001 - reported below
            err[r] = ex

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    if any(t.is_alive() for t in th):   # a rank is stuck: show where, and do not touch the contexts it is using
        import faulthandler
        import sys
        faulthandler.dump_traceback(file=sys.stderr, all_threads=True)
        pytest.fail(f"loopback ranks still running after 120 s: {[r for r, t in enumerate(th) if t.is_alive()]}; "
                    f"errors so far {err}")
    for s in solvers:
        if s is not None:
            s.close()
    B.de_loopback_destroy(g)
    for e in err:
        if e is not None:
            raise e
    return out


def _solve(r, S, p):
    S.factor()
    u, its, rel, _ = S.solve(p.rhs, p.rtol)
    cls, sub, red, nI, nG = S.dofmap()
    from paper_1501_06211_b200 import binding as B
    return u, its, rel, (cls, sub, red, nI, nG), B.de_get_owned(S.ctx)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_loopback_ranks_match_single_rank(G):
    from paper_1501_06211_b200 import binding as B
    p = make_config("c2")                                    # 8 x 4 subdomains: up to 8 slabs of one column
    S1 = B.Solver.from_problem(p, device=0)
    try:
        ref = _solve(0, S1, p)
    finally:
        S1.close()
    res = _run_ranks(p, G, lambda r, S: _solve(r, S, p))
    u1, its1, rel1, dm1, _ = ref
    owned = []
    for r, (u, its, rel, dm, own) in enumerate(res):
        assert np.array_equal(u, res[0][0])                  # every rank returns the same u, bitwise
        assert np.linalg.norm(u - u1) <= 1e-12 * np.linalg.norm(u1), (G, r)
        assert abs(its - its1) <= 2 and rel <= 1e-10
        for a, b in zip(dm, dm1):                             # the DOF map is bit-exact on every rank
            assert np.array_equal(np.asarray(a), np.asarray(b))
        owned.append(np.asarray(own))
    allown = np.sort(np.concatenate(owned))                  # the slabs partition the subdomains
    assert np.array_equal(allown, np.arange(32))
    px = 8
    for r, own in enumerate(owned):                          # rank r owns columns [r px / G, (r+1) px / G)
        cols = set(int(s) % px for s in own)
        assert cols == set(range(r * px // G, (r + 1) * px // G))


def test_loopback_pivot_failure_agreed_by_all_ranks():
    """A non-positive pivot on one rank's subdomain: every rank returns DE_ENOTSPD (none blocks in an exchange)."""
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    nx, ny = p.nel
    ex, ey = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    q = p.with_density(np.where(((ex >= 16) & (ey >= 8)).ravel(), 1e-120, 0.5))   # subdomain 3 (rank 1's slab)
    q.Emin = 0.0

    def fn(r, S):
        try:
            S.factor()
            return B.DE_OK, ""
        except B.DEError as ex:
            return ex.status, str(ex)

    res = _run_ranks(q, 2, fn)
    assert all(st == B.DE_ENOTSPD for st, _ in res)
    assert "subdomain 3" in res[1][1] and "another rank" in res[0][1]
