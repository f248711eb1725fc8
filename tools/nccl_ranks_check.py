"""Multi-rank path over NCCL, one process per GPU (launched by torchrun; tests/test_gpu_nccl.py runs it when the box
shows two or more GPUs): every rank solves config 2 with nranks = WORLD_SIZE (owned subdomain slabs, one ncclAllReduce
of the partial interface vector per iteration inside the captured PCG graph) and compares its u with a single-rank
solve on its own device: equal to 1e-12, iteration counts within 2, the same DOF map, DE_OK."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synthetic import make_config  # noqa: E402
from paper_1501_06211_b200 import binding as B  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [B.de_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    p = make_config("c2")
    S1 = B.Solver.from_problem(p, device=local)
    S1.factor()
    u1, its1, rel1, _ = S1.solve(p.rhs, p.rtol)
    dm1 = S1.dofmap()
    S1.close()
    S = B.Solver.from_problem(p, device=local, rank=rank, nranks=world, nccl_id=obj[0])
    S.factor()
    u, its, rel, st = S.solve(p.rhs, p.rtol)
    dm = S.dofmap()
    S.close()
    err = float(np.linalg.norm(u - u1) / np.linalg.norm(u1))
    ok = st == 0 and err <= 1e-12 and abs(its - its1) <= 2 and rel <= 1e-10 and \
        all(np.array_equal(np.asarray(a), np.asarray(b)) for a, b in zip(dm, dm1))
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    print(f"rank {rank}/{world}: its {its} (single {its1}), relres {rel:.2e}, |u-u1|/|u1| {err:.2e}, ok {ok}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) == 1 else 1)


if __name__ == "__main__":
    main()
