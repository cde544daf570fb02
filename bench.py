#!/usr/bin/env python3
"""Benchmark of the Epstein-zeta hot path on B200 ("Measurement").

Headline workload (BASELINE.json metric "Epstein-zeta evals/s ...; ATM fcc sum
wall time at 1-8 GPUs", config 3): one step = one complete ATM cohesive-energy
lattice sum for fcc on the fixed 12 x 128 x 128^2 graded Duffy grid
(25,165,824 nodes; per node one Z_3 and one Hessian of Z_5, i.e. 2 zeta
evaluations), sharded over the ranks with one NCCL all-reduce.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Rank 0 prints ONE JSON line.  value = zeta evaluations/s of the whole job
(device-timed, CUDA events, max over ranks); ms_per_step = ATM fcc sum wall
time; e2e = the same metric through the public API call
(distributed.atm_energy_distributed) from a cold cache, including host table
build, H2D uploads and the D2H of the result.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FCC_ATM_REF = 19.182931071876666   # reference integrate_product + Prop. 2.4 (tests/golden)
GRID = (128, 128, 3)               # n_u (graded u = t^3/2), n_v, grading
TERMS_PER_NODE = 900 + 1502        # reference enumeration: Z_3 (171+728+1) + Hessian Z_5 (171+1330+1)
# FP64 FLOPs per node of the fused ATM kernel (2*DFMA + DADD + DMUL), measured with ncu on the
# bench grid (profiles/r01_summary.md, v30: line kernel, split 0.13); used to turn the live kernel
# time into FLOP/s.  Re-measure whenever the kernel or the ATM split changes.
FLOPS_PER_NODE = 1578.0
FLOPS_SOURCE = "ncu r01 v30: 3.9712e+10 FP64 FLOPs per launch / 25,165,824 nodes"
# ncu r01 v30 dram__bytes_read.sum + dram__bytes_write.sum (plan staging; the tile partials stay in
# L2); the algorithmic HBM footprint of the integrand is zero (nodes generated on device)
TRAFFIC_PER_LAUNCH = 220416 + 0
NCU_UTIL = {"fp64_pipe_active": 0.570, "issue_active": 0.576, "lsu_wavefronts": 0.623,
            "warps_active": 0.309, "source": "ncu r01 v30 (--set full, one launch)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, local_rank: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = local_rank
        if vis:
            try:
                idx = int(vis.split(",")[local_rank])
            except (ValueError, IndexError):
                idx = local_rank
        self.idx = idx
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baselines
def cpu_atm_sample(n_nodes: int):
    """Oracle port (long-double C restatement of the reference algorithm) on a contiguous block of
    the C3 grid with every host thread; returns (evals/s, seconds, threads)."""
    from oracle import oracle as O
    from paper_2504_11989_b200 import named_lattice
    fcc = named_lattice("fcc")
    total = O.grid_nodes(3, GRID[0], GRID[1])
    lo = total // 2
    t0 = time.perf_counter()
    O.atm_grid(fcc.a, GRID[0], GRID[1], GRID[2], lo, lo + n_nodes)
    dt = time.perf_counter() - t0
    return 2.0 * n_nodes / dt, dt, O.nthreads()


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sample = 65536
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt, threads = cpu_atm_sample(sample)
        if i >= args.warmup:
            vals.append((v, dt))
    v = sum(x[0] for x in vals) / len(vals)
    ms = sum(x[1] for x in vals) / len(vals) * 1e3
    line = {
        "impl": "reference",
        "metric": "Epstein-zeta evals/s (FP64) on the ATM fcc sum",
        "value": v, "unit": "zeta evals/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 (long double oracle)", "data": "synthetic (fixed Duffy grid)",
        "config": config_block(world),
        "cpu_baseline": {"value": v, "unit": "zeta evals/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} contiguous nodes of the 25,165,824-node C3 grid per step "
                                   "(oracle/latsum_oracle.c, long double, all host threads)"},
        "e2e": {"value": v, "unit": "zeta evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference arm = oracle port of the reference algorithm (the reference is pure Python "
                "and is not installed on the GPU box); SURVEY.md section 6 lists the Python reference "
                "itself at 377 s (1 thread) / 102 s (8 threads) for the fcc ATM energy",
    }
    print(json.dumps(line), flush=True)


def config_block(world):
    return {"workload": "C3: ATM cohesive energy, fcc (unit NN distance), fixed Duffy grid 12 cells x "
                        "128 radial (graded u=t^3/2) x 128^2 angular = 25,165,824 nodes; per node Z_3 and "
                        "the Hessian of Z_5 (polynomial-weighted zeta)",
            "lattice": "fcc", "grid": {"n_u": GRID[0], "n_v": GRID[1], "grading": GRID[2]},
            "nodes_per_step": 25165824, "zeta_evals_per_node": 2, "terms_per_node": TERMS_PER_NODE,
            "parallelism": f"node-shard x{world} + 1 NCCL all-reduce" if world > 1 else "1 GPU",
            "l2": "node data generated on device; tables (<110 KB) live in shared memory; L2 flushed "
                  "(256 MB write) between timed steps"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_11989_b200 import _native as N
    from paper_2504_11989_b200 import named_lattice
    from paper_2504_11989_b200.distributed import ShardedIntegral, allreduce_partials, atm_energy_distributed
    from paper_2504_11989_b200.epstein import epstein_context
    from paper_2504_11989_b200.manybody import ATMGrid
    from paper_2504_11989_b200.quadrature import Plan, atm_plan, product_plan

    fcc = named_lattice("fcc")
    S = ShardedIntegral(atm_plan(fcc), *GRID)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step(evs=None):
        S.partials.zero_()
        if evs:
            evs[0].record(stream)
        S.plan.integrate_device(S.partials, S.n_u, S.n_v, S.grading, S.tile_lo, S.tile_hi)
        if evs:
            evs[1].record(stream)
        if world > 1:
            allreduce_partials(S.partials)  # C ABI: one ncclAllReduce on this stream
        Plan.reduce_device(S.partials, S.n_tiles, S.ncomp, S.out)
        if evs:
            evs[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    events = []
    for i in range(args.steps):
        flush.fill_(float(i))  # L2 flush between timed steps (outside the events)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        step(evs)
        events.append(evs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = sum(e[0].elapsed_time(e[2]) for e in events) / args.steps
    kern_ms = sum(e[0].elapsed_time(e[1]) for e in events) / args.steps
    t = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, kern_ms = float(t[0]), float(t[1])
    out = S.out.cpu().numpy()
    energy = (8.0 * out[0] - 3.0 * 8.0 * out[1]) / 6.0
    evals = 2.0 * S.n_nodes

    # ---- e2e through the public API (cold caches: host tables + H2D + kernel + D2H each call)
    e2e_ms = []
    # one untimed cold call first (first-call host paths, allocator), then the timed cold calls
    for it in range(max(1, args.e2e_steps) + 1):
        epstein_context.cache_clear()
        atm_plan.cache_clear()
        product_plan.cache_clear()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res = atm_energy_distributed(fcc, ATMGrid(*GRID))
        if it > 0:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_step_ms = float(te[0])
    # H2D per e2e call: the plan's tables (uploaded once per cold call) + the grid node arrays
    pinfo = atm_plan(fcc).info()
    h2d = int(pinfo.smem_bytes) + 8 * 2 * (GRID[0] + GRID[1])

    # ---- roofline of the dominant kernel (the fused ATM tile kernel)
    import ctypes as C
    pk, pms = C.c_double(0.0), C.c_double(0.0)
    N.check(N.lib().lz_fp64_peak(local, C.byref(pk), C.byref(pms)), "fp64 peak probe")
    local_nodes = min(S.local_nodes, S.n_nodes)
    achieved = FLOPS_PER_NODE * local_nodes / (kern_ms * 1e-3) / 1e12

    line = {
        "metric": "Epstein-zeta evals/s (FP64) on the ATM fcc sum; ms_per_step = ATM fcc sum wall time",
        "value": evals / (step_ms * 1e-3), "unit": "zeta evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (fixed Duffy grid generated on device)",
        "config": config_block(world),
        "terms_per_s": evals / 2.0 * TERMS_PER_NODE / (step_ms * 1e-3),
        "parity": {"atm_energy": energy, "reference": FCC_ATM_REF,
                   "rel_err": abs(energy - FCC_ATM_REF) / FCC_ATM_REF, "tolerance": 1e-10},
        "e2e": {"value": evals / (e2e_step_ms * 1e-3), "unit": "zeta evals/s",
                "ms_per_call": e2e_step_ms, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 16,
                "call": "paper_2504_11989_b200.distributed.atm_energy_distributed(fcc, ATMGrid(128,128,3)) "
                        "from cold caches", "energy": res.energy},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": pk.value, "unit": "TFLOP/s",
                     "frac": achieved / pk.value, "traffic": TRAFFIC_PER_LAUNCH,
                     "kernel": "lz::tile_kernel_l<20,1> (fused ATM integrand, line-factorised direct space)",
                     "kernel_ms": kern_ms, "flops_per_node": FLOPS_PER_NODE, "flops_source": FLOPS_SOURCE,
                     "peak_source": "measured live: DFMA-chain probe lz_fp64_peak (MEASURED_PEAKS.json has "
                                    "no FP64 entry)",
                     # utilisation counters of the same kernel from the ncu --set full capture
                     # (profiles/r01_atm_v30_metrics.json): the FLOP fraction counts DADD/DMUL as one
                     # FLOP although they occupy the FP64 pipe like a DFMA
                     "ncu": NCU_UTIL},
        "gpu_launches": 2 * args.steps,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, threads = cpu_atm_sample(131072)
        line["cpu_baseline"] = {"value": v, "unit": "zeta evals/s", "cores": threads, "kind": "port",
                                "sample": f"131072 contiguous nodes of the C3 grid ({dt:.1f} s), "
                                          "oracle/latsum_oracle.c (long double) on all host threads"}
    if rank == 0 and world == 1 and not args.no_secondary:
        line["secondary"] = secondary(np, torch)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def _time_cuda(fn, reps, torch):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _time_graph(fn, reps, torch):
    """Device time per call without host launch gaps: `reps` calls captured in one CUDA graph."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def secondary(np, torch):
    """Configs 1, 2, 4 on one GPU (device-timed), plus C1 through the numpy drop-in API."""
    from paper_2504_11989_b200 import named_lattice
    from paper_2504_11989_b200.epstein import EpsteinContext
    from paper_2504_11989_b200.quadrature import QuadratureConfig, integrate_product, product_plan
    out = {}
    sq = named_lattice("square")
    ctx = EpsteinContext(sq, 3.5, device=torch.cuda.current_device())
    for n, seed in ((4096, 0), (1 << 20, 1)):
        k = np.random.default_rng(seed).uniform(-0.5, 0.5, size=(n, 2))
        kt = torch.tensor(k, device="cuda")
        zt = torch.empty(n, dtype=torch.float64, device="cuda")
        ms_launch = _time_cuda(lambda: ctx.zeta_device(kt, out=zt), 20, torch)
        ms = _time_graph(lambda: ctx.zeta_device(kt, out=zt), 20, torch)
        kp = torch.from_numpy(k).pin_memory().numpy()   # pinned host input (contract: pinned H2D)
        zp = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
        ctx._eval_into(kp, zp)
        t0 = time.perf_counter()
        reps = 5
        for _ in range(reps):
            ctx._eval_into(kp, zp)
        e2e = (time.perf_counter() - t0) / reps
        out[f"c1_{n}"] = {"evals_per_s": n / (ms * 1e-3), "ms": ms, "ms_with_host_launch": ms_launch,
                          "e2e_evals_per_s": n / e2e, "terms_per_s": n * 105 / (ms * 1e-3),
                          "timing": "device, 20 calls replayed from one CUDA graph"}
    for name, nus, grid in (("c2_zeta333_sq_64x64", (3, 3, 3), (64, 64)),
                            ("c4_zeta51_sq_256x256", [4.0] * 51, (256, 256))):
        cfg = QuadratureConfig(grid_u=grid[0], grid_v=grid[1], estimate_error=False)
        integrate_product(sq, nus, cfg)
        plan = product_plan(sq, ((float(nus[0]), len(nus)),))
        nn, nt = plan.tiles(grid[0], grid[1], 1)
        part = torch.zeros(nt, dtype=torch.float64, device="cuda")
        ms = _time_cuda(lambda: plan.integrate_device(part, grid[0], grid[1], 1), 10, torch)
        t0 = time.perf_counter()
        v, _ = integrate_product(sq, nus, cfg)
        e2e = time.perf_counter() - t0
        out[name] = {"value": v, "nodes": nn, "kernel_ms": ms, "api_ms": e2e * 1e3,
                     "evals_per_s": nn / (ms * 1e-3)}
    # config 5: fcc/bcc LJ(12,6) + lambda ATM phase scan (two ATM sums + four zeta_at_zero on the
    # GPU, then the host enthalpy scan on the 64 x 64 (lambda, R) grids and lambda_c for 4 pressures)
    import numpy as np
    from paper_2504_11989_b200.manybody import ATMGrid
    from paper_2504_11989_b200.phase import LJParams, critical_coupling, lattice_constants, phase_scan
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lj = LJParams()
    fc = lattice_constants("fcc", lj, ATMGrid(128, 128, 3))
    bc = lattice_constants("bcc", lj, ATMGrid(128, 128, 3))
    t1 = time.perf_counter()
    lam = np.linspace(0.0, 2.0, 64)
    pts = phase_scan(fc, bc, lj, [0.0, 0.5, 1.0, 2.0], lam, np.linspace(0.9, 1.7, 64))
    pres = (0.0, 0.5, 1.0, 2.0)
    crit = dict(zip(pres, (float(v) for v in critical_coupling(fc, bc, lj, np.array(pres)))))
    t2 = time.perf_counter()
    out["c5_phase_scan"] = {"constants_ms": (t1 - t0) * 1e3, "scan_ms": (t2 - t1) * 1e3,
                            "lambda_c": crit, "k_atm_fcc": fc.k_atm, "k_atm_bcc": bc.k_atm,
                            "points": len(pts)}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
