#!/usr/bin/env python3
"""Benchmark of the Epstein-zeta hot path on B200.

Headline workload (BASELINE.json metric, config 3): one step = one complete ATM
cohesive-energy lattice sum for fcc on the fixed 12 x 128 x 128^2 graded Duffy
grid (25,165,824 nodes).  Per node the fused kernel evaluates one Hessian of
Z_5 (the polynomial-weighted zeta M_5) and takes Z_3 = tr M_5 from it, so a node
counts as ONE zeta evaluation.  The node grid is sharded over the ranks in 96
fixed chunks; ranks exchange chunk sums with one NCCL all-reduce.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

`--gpus N` without torchrun re-launches itself under torch.distributed.run with
N ranks.  Rank 0 prints ONE JSON line.  value = zeta evaluations/s of the whole
job (device-timed with CUDA events, max over ranks); ms_per_step = ATM fcc sum
wall time; e2e = the same metric through the public API
(distributed.atm_energy_distributed) including host table build, the H2D
uploads and the D2H of the result (cold: every library cache released; warm:
plan cached).  `--impl reference` times the reference's own CPU implementation
(the unmodified `latsum` package installed under baseline/_ref) on the same
node sample with every host core.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json "metric", verbatim in both arms (the driver pairs the arms by this string)
METRIC = "Epstein-zeta evals/s (FP64, % of FP64 peak); ATM fcc sum wall time at 1–8 GPUs"
UNIT = "zeta evals/s"
FCC_ATM_REF = 19.182931071876666   # reference integrate_product + Prop. 2.4 (tests/golden)
GRID = (128, 128, 3)               # n_u (graded u = t^3/2), n_v, grading
N_NODES = 12 * 128 * 128 * 128
TERMS_PER_NODE = 171 + 1330 + 1    # reference enumeration of the Hessian of Z_5
COUNTERS = os.path.join(ROOT, "profiles", "atm_kernel_current.json")
REF_SITE = os.path.join(ROOT, "baseline", "_ref")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-nodes", type=int, default=16384,
                    help="reference arm: nodes of the C3 grid per step (2 zeta evaluations each)")
    ap.add_argument("--ref-full-atm", action="store_true",
                    help="reference arm: also time the reference's own fcc ATM energy "
                         "(3 x integrate_product, ~100 s on 8 cores)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: become N ranks on this node."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


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


# ----------------------------------------------------------------------------- node sample
def c3_node_sample(n: int, seed: int = 7):
    """``n`` seeded random nodes of the C3 grid (uniform over cell, u and v indices), Cartesian k
    in the reference's Duffy coordinates (L/quadrature.py:136-177; u = t^3/2 graded GL)."""
    import numpy as np
    from paper_2504_11989_b200 import named_lattice
    from paper_2504_11989_b200.quadrature import angular_nodes, duffy_cells
    fcc = named_lattice("fcc")
    x, _ = np.polynomial.legendre.leggauss(GRID[0])
    u = 0.5 * ((x + 1.0) / 2.0) ** GRID[2]
    v, _ = angular_nodes(3, GRID[1])
    cells = duffy_cells(3)
    idx = np.random.default_rng(seed).integers(0, N_NODES, size=n)
    iu = idx % GRID[0]
    rest = idx // GRID[0]
    iv = rest % (GRID[1] ** 2)
    ic = rest // (GRID[1] ** 2)
    k = np.empty((n, 3))
    for c in range(len(cells)):
        sel = ic == c
        if sel.any():
            k[sel] = u[iu[sel], None] * cells[c].directions(fcc, v[iv[sel]])
    return k


# ----------------------------------------------------------------------------- reference CPU path
_REF_CTX = {}


def _ref_worker_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    sys.path.insert(0, REF_SITE)
    import latsum
    from latsum.epstein import epstein_context
    fcc = latsum.named_lattice("fcc")
    _REF_CTX["c3"] = epstein_context(fcc, 3.0)
    _REF_CTX["c5"] = epstein_context(fcc, 5.0)


def _ref_worker_eval(k):
    import numpy as np
    z3 = _REF_CTX["c3"].zeta(k)
    z5 = _REF_CTX["c5"].zeta(k)
    return float(np.sum(z3) + np.sum(z5))


def reference_available():
    return os.path.isdir(os.path.join(REF_SITE, "latsum"))


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ReferencePool:
    """The unmodified reference (baseline/_ref/latsum) evaluating Z_3 and Z_5 at C3 nodes, one
    process per host core (OPENBLAS_NUM_THREADS=1; processes, not threads --
    the reference's numpy/scipy path holds the GIL between calls)."""

    def __init__(self, procs: int):
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        self.procs = procs
        self.pool = ProcessPoolExecutor(procs, mp_context=mp.get_context("spawn"),
                                        initializer=_ref_worker_init)
        list(self.pool.map(_ref_worker_eval, [c3_node_sample(4, seed=99)] * procs))  # warm every worker

    def time(self, k):
        import numpy as np
        chunks = np.array_split(k, self.procs * 4)
        t0 = time.perf_counter()
        list(self.pool.map(_ref_worker_eval, chunks))
        dt = time.perf_counter() - t0
        return 2.0 * len(k) / dt, dt

    def close(self):
        self.pool.shutdown()


def port_sample(n_nodes: int):
    """Oracle port (long-double C restatement of the reference algorithm) on a contiguous block of
    the C3 grid with every host thread: (zeta evals/s counting one per node, seconds, threads)."""
    from oracle import oracle as O
    from paper_2504_11989_b200 import named_lattice
    fcc = named_lattice("fcc")
    lo = N_NODES // 2
    t0 = time.perf_counter()
    O.atm_grid(fcc.a, GRID[0], GRID[1], GRID[2], lo, lo + n_nodes)
    dt = time.perf_counter() - t0
    return n_nodes / dt, dt, O.nthreads()


def reference_full_atm(threads: int):
    """The reference's own fcc ATM energy: 3 x integrate_product + Prop. 2.4."""
    sys.path.insert(0, REF_SITE)
    import latsum
    from latsum.quadrature import integrate_product
    fcc = latsum.named_lattice("fcc")
    t0 = time.perf_counter()
    z333, _ = integrate_product(fcc, (3, 3, 3), threads=threads)
    zm155, _ = integrate_product(fcc, (-1, 5, 5), threads=threads)
    z135, _ = integrate_product(fcc, (1, 3, 5), threads=threads)
    e = z333 / 24 - 3 * zm155 / 16 + 3 * z135 / 8
    return time.perf_counter() - t0, e


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = cpu_cores()
    line = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded sample of the fixed C3 Duffy grid)",
            "config": config_block(world)}
    if reference_available():
        k = c3_node_sample(args.ref_nodes)
        pool = ReferencePool(cores)
        vals = []
        for i in range(args.warmup + args.steps):
            v, dt = pool.time(k)
            if i >= args.warmup:
                vals.append((v, dt))
        pool.close()
        v = sum(x[0] for x in vals) / len(vals)
        ms = sum(x[1] for x in vals) / len(vals) * 1e3
        sample = (f"{args.ref_nodes} seeded random nodes of the 25,165,824-node C3 grid per step, reference "
                  f"EpsteinContext.zeta for Z_3 and Z_5 at each (2 evaluations per node; the reference has no "
                  f"Hessian and its ATM route needs Z_-1, Z_1, Z_3, Z_5 per node), {cores} processes")
        kind = "reference"
        impl_note = ("unmodified reference latsum 0.1.0 (numpy/scipy), pip-installed from /root/reference/pkg "
                     "into baseline/_ref (baseline/install_reference.sh)")
    else:
        vals = []
        n = args.ref_nodes * 2
        for i in range(args.warmup + args.steps):
            v, dt, cores = port_sample(n)
            if i >= args.warmup:
                vals.append((v, dt))
        v = sum(x[0] for x in vals) / len(vals)
        ms = sum(x[1] for x in vals) / len(vals) * 1e3
        sample = f"{n} contiguous nodes of the C3 grid per step, oracle port, {cores} threads"
        kind = "port"
        impl_note = "baseline/_ref missing: oracle port (oracle/latsum_oracle.c) of the reference algorithm"
    line.update({"value": v, "ms_per_step": ms,
                 "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
                 "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                 "implementation": impl_note,
                 "note": "ms_per_step = wall time of one sample step (not an ATM sum); the reference's "
                         "own fcc ATM energy took 102 s on 8 threads in the survey container (SURVEY.md 6)"})
    if args.ref_full_atm and reference_available():
        secs, e = reference_full_atm(cores)
        line["reference_atm_sum"] = {"seconds": secs, "energy": e, "threads": cores}
    print(json.dumps(line), flush=True)


def config_block(world):
    return {"workload": "C3: ATM cohesive energy, fcc (unit NN distance), fixed Duffy grid 12 cells x "
                        "128 radial (graded u=t^3/2) x 128^2 angular = 25,165,824 nodes; per node one Hessian "
                        "of Z_5 (polynomial-weighted zeta M_5) and Z_3 = tr M_5",
            "lattice": "fcc", "grid": {"n_u": GRID[0], "n_v": GRID[1], "grading": GRID[2]},
            "nodes_per_step": N_NODES, "zeta_evals_per_node": 1, "terms_per_node": TERMS_PER_NODE,
            "parallelism": f"node-shard x{world} (96 fixed chunks) + 1 NCCL all-reduce of chunk sums"
                           if world > 1 else "1 GPU",
            "l2": "node data generated on device; tables (~50 KB) live in shared memory, the direct-space "
                  "row table (~18 MB, rebuilt every step by row_table_kernel) in L2; L2 flushed (256 MB write) "
                  "between timed steps"}


# ----------------------------------------------------------------------------- ours
def kernel_counters():
    """FP64 FLOPs per node of the ATM kernel from the committed ncu capture of the shipping build
    (profiles/atm_kernel_current.json, written by tools/ncu_metrics.py); stale if kernels.cu has
    changed since the capture."""
    with open(COUNTERS) as f:
        c = json.load(f)
    c["stale"] = c.get("csrc_sha1") != csrc_sha1()
    return c


def csrc_sha1():
    """sha1 over the sources that shape the ATM kernel's instruction stream (kernel, shared
    device headers, host plan builder); tools/ncu_metrics.py records the same digest."""
    h = hashlib.sha1()
    for name in ("kernels.cu", "lz_internal.h", "special.cuh", "capi.cpp", "context.cpp"):
        h.update(open(os.path.join(ROOT, "paper_2504_11989_b200", "csrc", name), "rb").read())
    return h.hexdigest()


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks need {world} visible GPUs, found {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_11989_b200 import _native as N
    from paper_2504_11989_b200 import named_lattice
    from paper_2504_11989_b200.distributed import ShardedIntegral, atm_energy_distributed
    from paper_2504_11989_b200.epstein import epstein_context
    from paper_2504_11989_b200.manybody import ATMGrid
    from paper_2504_11989_b200.quadrature import atm_plan, product_plan

    fcc = named_lattice("fcc")
    S = ShardedIntegral(atm_plan(fcc), *GRID)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        S.integrate()
        if evs:
            evs[1].record(stream)
        S.reduce()   # chunk sums, one ncclAllReduce of 96 x 2 doubles (W > 1), fixed-order total
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

    # ---- e2e through the public API, host buffers only (the lattice in, the energy out)
    def api_call():
        return atm_energy_distributed(fcc, ATMGrid(*GRID))

    def e2e(cold: bool, reps: int):
        ms, h2d, d2h = [], [], []
        for it in range(reps + 1):   # one untimed call first (first-call host paths, allocator)
            if cold:
                epstein_context.cache_clear()
                atm_plan.cache_clear()
                product_plan.cache_clear()
                import gc
                gc.collect()                       # contexts/plans freed -> device tables freed
                N.check(N.lib().lz_release_caches(local), "release caches")
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            import ctypes as C
            N.lib().lz_transfer_stats(None, None, 1)
            t0 = time.perf_counter()
            res = api_call()
            dt = (time.perf_counter() - t0) * 1e3
            hb, db = C.c_int64(0), C.c_int64(0)
            N.lib().lz_transfer_stats(C.byref(hb), C.byref(db), 1)
            if it > 0:
                ms.append(dt)
                h2d.append(hb.value)
                d2h.append(db.value)
        te = torch.tensor([sum(ms) / len(ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        # torch's own D2H of the two result doubles (ShardedIntegral.run().cpu()) is not a library copy
        return float(te[0]), int(max(h2d)), int(max(d2h)) + 16, res

    warm_ms, warm_h2d, warm_d2h, _ = e2e(False, max(1, args.e2e_steps))
    cold_ms, cold_h2d, cold_d2h, res = e2e(True, max(1, args.e2e_steps))

    # ---- roofline of the dominant kernel (the fused ATM tile kernel)
    import ctypes as C
    pk, pms = C.c_double(0.0), C.c_double(0.0)
    N.check(N.lib().lz_fp64_peak(local, C.byref(pk), C.byref(pms)), "fp64 peak probe")
    cnt = kernel_counters()
    local_nodes = min(S.local_nodes, N_NODES)
    achieved = cnt["flops_per_unit"] * local_nodes / (kern_ms * 1e-3) / 1e12
    evals = float(N_NODES)

    line = {
        "metric": METRIC,
        "value": evals / (step_ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (fixed Duffy grid generated on device)",
        "config": config_block(world),
        "atm_sum_ms": step_ms,
        "nodes_per_s": N_NODES / (step_ms * 1e-3),
        "hessian_evals_per_s": N_NODES / (step_ms * 1e-3),
        "zeta_values_per_s": 2.0 * N_NODES / (step_ms * 1e-3),
        "reference_terms_per_s": N_NODES * TERMS_PER_NODE / (step_ms * 1e-3),
        "parity": {"atm_energy": energy, "reference": FCC_ATM_REF,
                   "rel_err": abs(energy - FCC_ATM_REF) / FCC_ATM_REF, "tolerance": 1e-10},
        "e2e": {"value": evals / (cold_ms * 1e-3), "unit": UNIT, "ms_per_call": cold_ms,
                "h2d_bytes_per_step": cold_h2d, "d2h_bytes_per_step": cold_d2h,
                "bytes": "measured: lz_transfer_stats counts every host<->device copy the library issues",
                "call": "paper_2504_11989_b200.distributed.atm_energy_distributed(fcc, ATMGrid(128,128,3)) "
                        "with every cache released (Python context/plan caches and lz_release_caches): host "
                        "enumeration + table fits + H2D uploads + kernels + D2H of the energy",
                "energy": res.energy,
                "warm": {"value": evals / (warm_ms * 1e-3), "ms_per_call": warm_ms, "h2d_bytes_per_step": warm_h2d,
                         "d2h_bytes_per_step": warm_d2h, "call": "same call, plan cached"}},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": pk.value, "unit": "TFLOP/s",
                     "frac": achieved / pk.value, "traffic": cnt.get("dram_bytes_per_launch"),
                     "kernel": cnt.get("kernel"), "kernel_ms": kern_ms,
                     "flops_per_node": cnt["flops_per_unit"], "flops_source": cnt.get("source"),
                     "flops_per_reference_term": cnt["flops_per_unit"] / TERMS_PER_NODE,
                     "terms_evaluated_per_node": {
                         "reciprocal": 0.70, "q0": 1, "direct": "16 plane rotations per node (plane sums "
                         "shared by the 256 nodes of a line pair, from the per-(axis, radial node) row table)",
                         "source": "profiles/r02k_atm_segments.txt (execution counts of the term code)"},
                     "flops_stale": cnt["stale"],
                     "peak_source": "measured live: DFMA-chain probe lz_fp64_peak (MEASURED_PEAKS.json has "
                                    "no FP64 entry)",
                     "ncu": {k: cnt.get(k) for k in ("fp64_pipe_active", "issue_active", "lsu_wavefronts",
                                                     "warps_active", "registers")}},
        "exchange_bytes_per_step": S.exchange_bytes if world > 1 else 0,
        "gpu_launches": 4 * args.steps,   # row table + tile kernel + chunk reduce + total per step
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if reference_available():
            cores = cpu_cores()
            pool = ReferencePool(cores)
            k = c3_node_sample(8192)
            pool.time(k)
            v, dt = pool.time(k)
            pool.close()
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                                    "sample": f"8192 seeded random C3 nodes, unmodified reference zeta for Z_3 "
                                              f"and Z_5 (2 evaluations per node, {dt:.1f} s), {cores} processes"}
        pv, pdt, pthreads = port_sample(32768)
        line["cpu_port"] = {"value": pv, "unit": UNIT, "cores": pthreads, "kind": "port",
                            "sample": f"32768 contiguous C3 nodes ({pdt:.1f} s), oracle/latsum_oracle.c "
                                      "(long double), one evaluation per node as on the GPU"}
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


def shard_balance(torch):
    """Per-rank kernel time of the C3 grid split over W ranks, each shard timed alone on this GPU:
    max/mean is the load-balance ceiling of strong scaling."""
    from paper_2504_11989_b200 import named_lattice
    from paper_2504_11989_b200.distributed import ShardedIntegral
    from paper_2504_11989_b200.quadrature import atm_plan
    plan = atm_plan(named_lattice("fcc"))
    out = {}
    for world in (2, 4, 8):
        ms = []
        for r in range(world):
            s = ShardedIntegral(plan, *GRID, world=world, rank=r)
            s.world = 1
            ms.append(_time_cuda(s.integrate, 5, torch))
        mean = sum(ms) / len(ms)
        out[f"w{world}"] = {"shard_ms": ms, "max_over_mean": max(ms) / mean}
    return out


def secondary(np, torch):
    """Configs 1, 2, 4 on one GPU (device-timed), C1 through the numpy drop-in API, C5, shard
    balance."""
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
        t0 = time.perf_counter()
        v2, err2 = integrate_product(sq, nus)   # default contract: grid + error check (+ escalation)
        api = time.perf_counter() - t0
        out[name] = {"value": v, "nodes": nn, "kernel_ms": ms, "api_ms": e2e * 1e3,
                     "api_ms_default_cfg": api * 1e3, "default_cfg_err": err2,
                     "evals_per_s": nn / (ms * 1e-3)}
    # config 5: fcc/bcc LJ(12,6) + lambda ATM phase scan (two ATM sums + four zeta_at_zero on the
    # GPU, then the host enthalpy scan on the 64 x 64 (lambda, R) grids and lambda_c for 4 pressures)
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
    out["shard_balance"] = shard_balance(torch)
    # the bcc ATM sum of C5 on the same grid (17 planes per axis: four 32-item rounds of the plane
    # sums instead of fcc's three)
    from paper_2504_11989_b200.quadrature import atm_plan
    bplan = atm_plan(named_lattice("bcc"))
    _, bnt = bplan.tiles(*GRID)
    bpart = torch.zeros(bnt * 2, dtype=torch.float64, device="cuda")
    out["c3_bcc_atm_sum_ms"] = _time_cuda(lambda: bplan.integrate_device(bpart, *GRID), 10, torch)
    # the reference's own route to the fcc ATM energy (Prop. 2.4: three continued integrals with
    # its adaptive GK15/G7 refinement, method="adaptive", every round's zeta products on the GPU)
    fcc = named_lattice("fcc")
    acfg = QuadratureConfig(method="adaptive")
    integrate_product(fcc, (3, 3, 3), acfg)   # contexts and plans built outside the timing
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    zs = [integrate_product(fcc, nus, acfg)[0] for nus in ((3, 3, 3), (-1, 5, 5), (1, 3, 5))]
    t_ad = time.perf_counter() - t0
    e_ad = zs[0] / 24 - 3 * zs[1] / 16 + 3 * zs[2] / 8
    out["c3_prop24_adaptive"] = {"seconds": t_ad, "energy": e_ad,
                                 "rel_err_vs_reference": abs(e_ad - 19.182931071876666) / 19.182931071876666,
                                 "reference_seconds": {"threads_8": 102.0, "threads_1": 377.0,
                                                       "source": "SURVEY.md section 6 (reference run in the survey container)"}}
    # order-m derivatives at arbitrary k (moment kernel) and the device Taylor table at k = 0
    k3 = torch.tensor(np.random.default_rng(2).uniform(-0.45, 0.45, size=(1 << 14, 3)) @ fcc.a_inv_t.T,
                      device="cuda")
    c5 = EpsteinContext(fcc, 5.0, device=torch.cuda.current_device())
    der = {}
    for m in (4, 8, 12):
        c5.derivatives_device(k3, m)
        ms = _time_cuda(lambda: c5.derivatives_device(k3, m), 5, torch)
        der[f"order_{m}"] = {"points": int(k3.shape[0]), "ms": ms, "points_per_s": k3.shape[0] / (ms * 1e-3)}
    c3 = EpsteinContext(fcc, 3.0, device=torch.cuda.current_device())
    t0 = time.perf_counter()
    c3.reg_derivatives(8)
    der["taylor_table_order8_ms"] = (time.perf_counter() - t0) * 1e3
    out["fcc_nu5_derivatives"] = der
    return out


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
