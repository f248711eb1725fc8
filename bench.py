#!/usr/bin/env python3
"""bench.py — interface-PCG MDOF·iter/s on B200 (BASELINE.json metric), driver contract.

A "step" is one pass of the whole hot path over one batch of synthetic input: the BASELINE
config-5 topology-optimisation sequence step (2048x1024 Q1 elements, 64x32 subdomains): new
densities (seeded +-5 % perturbation, clipped) -> de_factor (SIMP assembly + 2048 band Cholesky
factorisations) -> warm-started de_solve (condense, interface PCG with the inverse-Lanczos
H^_theta preconditioner to rtol 1e-10, back-substitution, true residual).
value = n_free * (PCG iterations) / step time / 1e6 over the K timed steps (whole job, all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl native|reference]
Multi-GPU: launched by torch.distributed.run; ranks shard subdomain columns, NCCL allreduce.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "interface-PCG MDOF*iter/s (rtol 1e-10)"
UNIT = "MDOF*iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def density_schedule(prob, n):
    from synthetic import density_sequence_step
    out = [prob.density.copy()]
    for t in range(1, n):
        out.append(density_sequence_step(out[-1], t))
    return out


# --------------------------------------------------------------------------- oracle (CPU) leg

def cpu_baseline(prob, gpu_iters, budget_s=20.0):
    """The oracle as it stands, on a bounded sample of the same workload: per-iteration cost
    (Schur apply over a subset of subdomains, scaled to all; one full preconditioner
    application; PCG vector work) and per-step factorisation cost (same subset, scaled)."""
    from oracle.topology import build_topology
    from oracle.dd import subdomain_blocks, factor_subdomains, local_schur_apply
    from oracle.precond import build_components, apply_precond
    topo = build_topology(prob)
    ns = min(topo.nsub, 64)
    sample = list(np.linspace(0, topo.nsub - 1, ns).astype(int))
    t0 = time.perf_counter()
    blocks = factor_subdomains(subdomain_blocks(prob, topo, only=sample))
    t_fac = (time.perf_counter() - t0) * topo.nsub / ns
    rng = np.random.default_rng(0)
    x = rng.normal(size=topo.n_G)
    reps, t_s = 0, 0.0
    while t_s < budget_s * 0.3 or reps < 1:
        t0 = time.perf_counter()
        for b in blocks:
            local_schur_apply(b, x[b.R])
        t_s += time.perf_counter() - t0
        reps += 1
    t_schur = t_s / reps * topo.nsub / ns
    comps = build_components(prob, topo)
    apply_precond(comps, x, "lanczos", 0.5, 10, "X")       # factorises the skeleton operators once
    reps, t_p = 0, 0.0
    while t_p < budget_s * 0.2 or reps < 1:
        t0 = time.perf_counter()
        apply_precond(comps, x, "lanczos", 0.5, 10, "X")
        t_p += time.perf_counter() - t0
        reps += 1
    t_prec = t_p / reps
    t_iter = t_schur + t_prec
    iters = max(1, gpu_iters)
    step = t_fac + iters * t_iter
    value = prob.ndof and (topo.n_I + topo.n_G) * iters / step / 1e6
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{ns}/{topo.nsub} subdomains (Schur apply + banded factorisation, scaled x{topo.nsub / ns:.0f}) "
                      f"+ full preconditioner application; step = factor + {iters} iterations (GPU count); "
                      f"t_iter={t_iter:.3f}s t_factor={t_fac:.2f}s; numpy/scipy single thread, host cpus={os.cpu_count()}",
            "s_per_iter": t_iter, "s_factor": t_fac}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synthetic import make_config
    prob = make_config(args.config)
    n_free = int(np.sum(prob.fixed == 0))
    gpu_iters = 900 if args.config == "c5" else 200
    cb = cpu_baseline(prob, gpu_iters, budget_s=8.0)
    steps = []
    for _ in range(args.warmup + args.steps):
        steps.append(cb["s_factor"] + gpu_iters * cb["s_per_iter"])
    ms = 1e3 * float(np.mean(steps[args.warmup:]))
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} (BASELINE config 5: 2048x1024 Q1, 64x32 subdomains, "
                                   "density-sequence step)"},
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0},
            "note": "oracle (oracle/) on host cores; bounded sample per step, scaled as stated in cpu_baseline.sample"}
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- native leg

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from synthetic import make_config
    from paper_1501_06211_b200.build import build
    from paper_1501_06211_b200 import binding as B

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if rank == 0:
        build()
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        obj = [B.de_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.current_stream()

    prob = make_config(args.config)
    nsteps = args.warmup + args.steps
    sched = density_schedule(prob, nsteps + 1)
    d_rho = [torch.tensor(r, dtype=torch.float64, device="cuda") for r in sched]
    d_rhs = torch.tensor(prob.rhs, dtype=torch.float64, device="cuda")
    d_u = torch.empty_like(d_rhs)

    solver = B.Solver.from_problem(prob.with_density(sched[0]), device=local, warm_start=1,
                                   rank=rank, nranks=world, nccl_id=nccl_id, stream=stream.cuda_stream)
    ctx = solver.ctx
    st0 = solver.stats()
    n_free = st0.n_free

    status_fail = []

    def step(t):
        B.de_update_densities_device(ctx, d_rho[t].data_ptr())
        B.de_factor(ctx)
        try:   # every step must return DE_OK (the refined iterate meets rtol, R17)
            its, rel, _ = B.de_solve_device(ctx, d_rhs.data_ptr(), prob.rtol, d_u.data_ptr())
        except B.DEError as ex:
            status_fail.append((t, ex.status))
            st_ = solver.stats()
            its, rel = st_.iterations, st_.relres_true
        return its, rel

    for t in range(args.warmup):                    # untimed warm-up (graph build, caches)
        step(t)
    torch.cuda.synchronize()
    B.de_set_profiling(ctx, True)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its_tot, rel_max, reldd_max, launches = 0, 0.0, 0.0, 0
    e0.record(stream)
    for t in range(args.warmup, nsteps):
        its, rel = step(t)
        its_tot += its
        rel_max = max(rel_max, rel)
        st_ = solver.stats()
        reldd_max = max(reldd_max, st_.relres_dd)
        launches += st_.kernels_launched + 5        # + factor kernels
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    k_ms, k_n = B.de_get_kernel_time(ctx)
    p_ms, p_n = B.de_get_prec_time(ctx)
    B.de_set_profiling(ctx, False)
    st = solver.stats()
    value = n_free * its_tot / (ms / 1e3) / 1e6
    ms_step = ms / args.steps

    # ------------------------------------------------ e2e: host buffers through the C-ABI
    e2e = None
    if not args.no_e2e:
        rhs_h = np.ascontiguousarray(prob.rhs)
        u_h = np.empty_like(rhs_h)
        rho_h = [np.ascontiguousarray(r) for r in sched]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_e = []
        its_e = 0
        for t in range(args.warmup, nsteps):
            ta = time.perf_counter()
            B.de_update_densities(ctx, rho_h[t])
            B.de_factor(ctx)
            try:
                _, its, rel, _ = B.de_solve(ctx, rhs_h, prob.rtol, u_h)
            except B.DEError as ex:
                status_fail.append(("e2e", t, ex.status))
                its = solver.stats().iterations
            t_e.append(time.perf_counter() - ta)
            its_e += its
        te = sum(t_e)
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": n_free * its_e / te / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(rho_h[0].nbytes + rhs_h.nbytes), "d2h_bytes_per_step": int(u_h.nbytes),
               "ms_per_step": 1e3 * te / args.steps}

    if rank != 0:
        solver.close()
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    pk = peaks()
    traffic = {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        if prof.get("config") == args.config and prof.get("n_gpus", 1) == world:
            traffic = prof.get("dram_bytes_per_launch", {})
    except Exception:
        pass
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if not pk.get("_fallback") else "fallback 6650 GB/s"

    def roofline(kernel, what, algo_bytes, launch_ms, launches):
        achieved = algo_bytes / (launch_ms / 1e3) / 1e9 if launch_ms > 0 else None
        return {"bound": "hbm", "kernel": f"{kernel} ({what})", "achieved": achieved, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": (achieved / pk["hbm_gbs"]) if achieved else None,
                "traffic": traffic.get(kernel), "algorithmic_bytes_per_launch": algo_bytes,
                "launch_ms": launch_ms, "launches_timed": launches,
                "share_of_step": (launch_ms * launches / ms) if launches else None, "peak_source": peak_src}

    schur_kernel = "k_schur_explicit" if st.schur_explicit else "k_schur_local"
    schur_bytes = st.bytes_schur_explicit if st.schur_explicit else st.bytes_schur
    roof_s = roofline(schur_kernel, "C2 Schur apply", schur_bytes, k_ms, k_n)
    roof_p = roofline("k_prec_coop", "C5 preconditioner application: k_prec_coop + k_prec_ritz + k_prec_combine, "
                      "event-timed as one", st.bytes_prec, p_ms, p_n) if p_n else None
    if roof_p and (roof_p["share_of_step"] or 0) > (roof_s["share_of_step"] or 0):
        roof, roof2 = roof_p, roof_s
    else:
        roof, roof2 = roof_s, roof_p
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(prob, its_tot // max(1, args.steps))
        cb = {k: v for k, v in cb.items() if k not in ("s_per_iter", "s_factor")}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: BASELINE config 5 step (2048x1024 Q1 plane stress, 64x32 "
                                   "subdomains of 32x32, SIMP p=3, density update -> refactor -> warm PCG rtol 1e-10)"
                       if args.config == "c5" else args.config,
                       "n_free": int(n_free), "n_gamma": int(st.n_Gamma), "subdomains": int(st.n_sub),
                       "preconditioner": "inverse Lanczos k=10, theta=0.5, exact inner solves (R10)",
                       "l2": "inputs larger than L2 (factor bands %.2f GB/rank)" % (st.bytes_factor / 1e9),
                       "parallelism": f"subdomain slabs x{world}"},
            "iterations_per_step": its_tot / args.steps, "true_relres_max": rel_max,
            "relres_dd_max": reldd_max, "solve_status_failures": status_fail,
            "solves_per_sec": 1e3 / ms_step, "factor_ms": st.ms_factor,
            "gpu_launches": int(launches), "clocks": clk, "roofline": roof, "roofline_secondary": roof2,
            "e2e": e2e, "cpu_baseline": cb}
    print(json.dumps(line))
    solver.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
