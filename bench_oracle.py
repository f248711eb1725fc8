"""bench_oracle.py — the oracle timed on the host's cores for bench.py (`cpu_baseline` leg and `--impl reference`).

Only bench.py imports this module (test/bench infrastructure: it executes oracle/, never the CUDA path).
The oracle runs as it stands (oracle/dd.py, oracle/precond.py, untuned); this file only distributes it the way
BASELINE.md §3 plans: os.cpu_count() forked worker processes over contiguous slices of the subdomains, one BLAS
thread each, shared-memory interface vectors, and one worker per displacement component for the preconditioner
(its components are independent).

One measured sample = factorisation of ALL subdomains (assembly + banded Cholesky, parallel) + `iters` full PCG
iterations (parallel Schur apply q = S p over all subdomains, parallel preconditioner z = H^-1 r, the PCG
vector updates on the main process). The BASELINE step (factor + the GPU's iteration count) is then
t_factor + n_iter * t_iter, extrapolated from those measured parts and labelled as such.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import statistics
import time

import numpy as np


def _limit_blas():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


class OraclePool:
    def __init__(self, prob, nworkers=None):
        from oracle.topology import build_topology
        from oracle.precond import build_components
        self.prob = prob
        self.topo = build_topology(prob)
        self.comps = build_components(prob, self.topo)
        nG = self.topo.n_G
        self.nw = max(1, nworkers or os.cpu_count() or 1)
        ctx = mp.get_context("fork")
        self.x = np.frombuffer(ctx.RawArray("d", nG), dtype=np.float64)
        self.q = np.frombuffer(ctx.RawArray("d", nG * self.nw), dtype=np.float64).reshape(self.nw, nG)
        self.r = np.frombuffer(ctx.RawArray("d", nG), dtype=np.float64)
        self.z = np.frombuffer(ctx.RawArray("d", nG), dtype=np.float64)
        nsub = self.topo.nsub
        cuts = np.linspace(0, nsub, self.nw + 1).astype(int)
        self.conns, self.procs = [], []
        for w in range(self.nw):
            a, b = ctx.Pipe()
            p = ctx.Process(target=self._schur_worker, args=(w, list(range(cuts[w], cuts[w + 1])), b), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.pconns = []
        for c in range(len(self.comps)):
            a, b = ctx.Pipe()
            p = ctx.Process(target=self._prec_worker, args=(c, b), daemon=True)
            p.start()
            self.pconns.append(a)
            self.procs.append(p)
        for cn in self.conns + self.pconns:
            cn.recv()   # ready

    # ---------------------------------------------------------------- workers (forked)
    def _schur_worker(self, w, subs, conn):
        from oracle.dd import subdomain_blocks, factor_subdomains, local_schur_apply
        _limit_blas()
        blocks = []
        conn.send("ready")
        while True:
            cmd = conn.recv()
            if cmd == "stop":
                return
            if cmd == "factor":
                blocks = factor_subdomains(subdomain_blocks(self.prob, self.topo, only=subs)) if subs else []
            elif cmd == "apply":
                q = self.q[w]
                q[:] = 0.0
                x = self.x
                for b in blocks:
                    np.add.at(q, b.R, local_schur_apply(b, x[b.R]))
            conn.send("done")

    def _prec_worker(self, c, conn):
        from oracle.precond import inverse_lanczos
        _limit_blas()
        cd = self.comps[c]
        g = cd.skel.gidx
        conn.send("ready")
        while True:
            cmd = conn.recv()
            if cmd == "stop":
                return
            rc = self.r[g]
            self.z[g] = inverse_lanczos(cd, rc, 10, 0.5, "X") if np.any(rc) else 0.0
            conn.send("done")

    # ---------------------------------------------------------------- main side
    def _all(self, conns, cmd):
        for cn in conns:
            cn.send(cmd)
        for cn in conns:
            cn.recv()

    def factor(self):
        t0 = time.perf_counter()
        self._all(self.conns, "factor")
        return time.perf_counter() - t0

    def schur(self, p):
        self.x[:] = p
        self._all(self.conns, "apply")
        return self.q.sum(axis=0)

    def precond(self, r):
        self.r[:] = r
        self._all(self.pconns, "prec")
        return self.z.copy()

    def pcg_iterations(self, n, seed=0):
        """n PCG iterations on S x = g with the oracle's operators (the iteration body of oracle/krylov.py pcg:
        q = S p, alpha, x/r updates, z = P r, beta, p update); returns seconds per iteration."""
        rng = np.random.default_rng(seed)
        g = rng.normal(size=self.topo.n_G)
        x = np.zeros_like(g)
        r = g.copy()
        z = self.precond(r)
        p = z.copy()
        rz = r @ z
        t0 = time.perf_counter()
        for _ in range(n):
            q = self.schur(p)
            alpha = rz / (p @ q)
            x += alpha * p
            r -= alpha * q
            z = self.precond(r)
            rz_new = r @ z
            p = z + (rz_new / rz) * p
            rz = rz_new
        return (time.perf_counter() - t0) / max(1, n)

    def close(self):
        for cn in self.conns + self.pconns:
            try:
                cn.send("stop")
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=5)


def measure(prob, gpu_iters, iters=3, repeats=3, pool=None):
    """Median over `repeats` samples of (t_factor, t_iter) on all host cores; returns a dict for bench.py."""
    own = pool is None
    pool = pool or OraclePool(prob)
    try:
        pool.factor()                     # warm-up (imports, page faults, lazy skeleton factorisations)
        pool.pcg_iterations(1)
        tf, ti = [], []
        for rep in range(repeats):
            tf.append(pool.factor())
            ti.append(pool.pcg_iterations(iters, seed=rep))
        t_factor, t_iter = statistics.median(tf), statistics.median(ti)
        n_free = int(np.sum(prob.fixed == 0))
        step = t_factor + gpu_iters * t_iter
        return {"t_factor": t_factor, "t_iter": t_iter, "step_s": step, "sample_s": t_factor + iters * t_iter,
                "value": n_free * gpu_iters / step / 1e6, "cores": pool.nw + len(pool.comps),
                "workers": pool.nw, "prec_workers": len(pool.comps),
                "sample": (f"measured on {pool.nw} worker processes (+{len(pool.comps)} preconditioner workers, one per "
                           f"component; 1 BLAS thread each; host os.cpu_count()={os.cpu_count()}): factorisation of all "
                           f"{pool.topo.nsub} subdomains t_factor={t_factor:.3f}s and {iters} full PCG iterations "
                           f"t_iter={t_iter:.4f}s (median of {repeats}); step = factor + {gpu_iters} iterations (the "
                           f"GPU's count) EXTRAPOLATED as t_factor + n*t_iter = {step:.1f}s")}
    finally:
        if own:
            pool.close()
