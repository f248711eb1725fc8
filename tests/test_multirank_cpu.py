"""World-size-2 gloo test (CPU) of the multi-GPU decomposition logic: every rank's libde
host setup owns a disjoint slab of subdomain columns covering all subdomains, and the replicated-interface
exchange — partial Schur sums over owned subdomains + one allreduce — equals the full interface operator.
The partial sums are computed with the oracle (no GPU here); the ownership comes from libde itself."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp
import torch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, kw, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from synthetic import make_config
    from paper_1501_06211_b200 import binding as B
    from oracle.topology import build_topology
    from oracle.dd import subdomain_blocks, factor_subdomains, local_schur_apply, schur_apply, condensed_rhs
    p = make_config(name, **kw)
    opt = B.de_default_options(host_only=1, rank=rank, nranks=world)
    ctx = B.de_setup(p.dim, p.nel, p.h, p.fixed, p.density, p.E0, p.Emin, p.p, p.nu, p.sub, opt)
    owned = B.de_get_owned(ctx)
    B.de_destroy(ctx)
    T = build_topology(p)
    blocks = factor_subdomains(subdomain_blocks(p, T, only=list(owned)))
    x = np.random.default_rng(7).normal(size=T.n_G)        # identical on every rank (replicated vector)
    q = np.zeros(T.n_G)
    for b in blocks:
        np.add.at(q, b.R, local_schur_apply(b, x[b.R]))
    qt = torch.from_numpy(q)
    dist.all_reduce(qt)                                    # the one exchange per PCG iteration
    own = torch.zeros(T.nsub, dtype=torch.int64)
    own[torch.from_numpy(owned.astype(np.int64))] = 1
    dist.all_reduce(own)
    if rank == 0:
        full = schur_apply(factor_subdomains(subdomain_blocks(p, T)), T.n_G, x)
        out.put((own.numpy().tolist(), float(np.linalg.norm(qt.numpy() - full) / np.linalg.norm(full)),
                 sorted(owned.tolist())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,kw,world", [("c2", dict(nel=(64, 32), sub=(16, 16)), 2),
                                           ("c4", dict(nel=(12, 6, 6), sub=(3, 3, 3)), 2),
                                           ("c2", dict(nel=(80, 16), sub=(16, 8)), 3)])
def test_sharded_interface_exchange(name, kw, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, kw, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    own, err, owned0 = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    assert all(v == 1 for v in own)            # disjoint cover: every subdomain owned exactly once
    assert err <= 1e-13
    assert owned0 == sorted(owned0) and len(owned0) > 0
