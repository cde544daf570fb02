"""Small, fixed GPU workloads for ncu (one process, one GPU).

    python tools/profile_target.py atm      # one fused ATM integral, fcc, bench grid
    python tools/profile_target.py c1       # C1 throughput batch (2^20 points)
    python tools/profile_target.py e2e      # host-API overhead breakdown (no ncu)
    SWEEP=0.45,0.6 python tools/profile_target.py atm_sweep   # kernel ms vs theta split
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2504_11989_b200 import named_lattice
from paper_2504_11989_b200.epstein import EpsteinContext
from paper_2504_11989_b200.manybody import ATMGrid, atm_integrals
from paper_2504_11989_b200.quadrature import QuadratureConfig, atm_plan, integrate_product


def atm():
    fcc = named_lattice("fcc")
    plan = atm_plan(fcc)
    nn, nt = plan.tiles(128, 128, 3)
    part = torch.zeros(nt * 2, dtype=torch.float64, device="cuda")
    plan.integrate_device(part, 128, 128, 3)
    torch.cuda.synchronize()
    print("atm ok", nn, nt)


def atm_sweep():
    """Kernel time and energy of the fcc ATM sum vs the theta split (CUDA events, 5 reps)."""
    fcc = named_lattice(os.environ.get("LATTICE", "fcc"))
    scales = [float(v) for v in os.environ.get("SWEEP", "0.35,0.45,0.55,0.65,0.8").split(",")]
    for sc in scales:
        plan = atm_plan(fcc, sc * fcc.volume ** (-2.0 / 3.0))
        nn, nt = plan.tiles(128, 128, 3)
        part = torch.zeros(nt * 2, dtype=torch.float64, device="cuda")
        plan.integrate_device(part, 128, 128, 3)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            plan.integrate_device(part, 128, 128, 3)
        b.record()
        torch.cuda.synchronize()
        s2 = plan.integrate(128, 128, 3)
        e = 8.0 * (s2[0] - 3.0 * s2[1]) / 6.0
        info = plan.info()
        print(f"split {sc:.2f}: {a.elapsed_time(b) / 5:.3f} ms  n_dir {info.n_dir} runs {info.n_runs} "
              f"n_rec {info.n_rec} pieces {info.table_pieces} smem {info.smem_bytes}  E {e:.15f}")


def c1_small():
    sq = named_lattice("square")
    ctx = EpsteinContext(sq, 3.5, device=0)
    k = torch.tensor(np.random.default_rng(0).uniform(-0.5, 0.5, size=(4096, 2)), device="cuda")
    for _ in range(3):
        z, st = ctx.zeta_device(k)
    torch.cuda.synchronize()
    print("c1_small ok", float(z.sum()))


def c1():
    sq = named_lattice("square")
    ctx = EpsteinContext(sq, 3.5, device=0)
    k = torch.tensor(np.random.default_rng(1).uniform(-0.5, 0.5, size=(1 << 20, 2)), device="cuda")
    z, st = ctx.zeta_device(k)
    torch.cuda.synchronize()
    print("c1 ok", float(z.sum()))


def adaptive_fcc():
    """The reference's own route to the fcc ATM energy (Prop. 2.4: three meromorphically continued
    integrals through integrate_product, method="adaptive" = the reference's GK15/G7 refinement with
    every round's zeta products on the GPU), timed; the survey's reference timing is 102 s on 8
    threads (377 s on 1)."""
    from paper_2504_11989_b200.quadrature import integrate_product
    fcc = named_lattice("fcc")
    cfg = QuadratureConfig(method="adaptive")
    integrate_product(named_lattice("square"), (3, 3, 3), cfg)  # warm-up (contexts, kernels)
    out = {}
    t_all = time.perf_counter()
    for nus in ((3, 3, 3), (-1, 5, 5), (1, 3, 5)):
        t0 = time.perf_counter()
        v, err = integrate_product(fcc, nus, cfg)
        out[nus] = v
        print(f"fcc {nus}: {v!r} +- {err:.2e}  {time.perf_counter() - t0:.3f} s", flush=True)
    e = out[(3, 3, 3)] / 24 - 3 * out[(-1, 5, 5)] / 16 + 3 * out[(1, 3, 5)] / 8
    print(f"E_ATM (Prop. 2.4, adaptive) {e!r}  rel err vs reference {abs(e - 19.182931071876666) / 19.182931071876666:.2e}"
          f"  total {time.perf_counter() - t_all:.3f} s (reference: 102 s on 8 threads, 377 s on 1)")


def e2e_breakdown():
    """Where the cold-cache time of atm_energy_distributed goes (host plan vs device)."""
    from paper_2504_11989_b200.distributed import ShardedIntegral
    from paper_2504_11989_b200.epstein import epstein_context
    from paper_2504_11989_b200.quadrature import atm_plan, product_plan
    fcc = named_lattice("fcc")
    import gc
    from paper_2504_11989_b200 import _native as N
    for rep in range(4):
        epstein_context.cache_clear(); atm_plan.cache_clear(); product_plan.cache_clear()
        gc.collect()
        N.check(N.lib().lz_release_caches(0), "release caches")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if os.environ.get("SPLIT_PLAN"):
            from paper_2504_11989_b200.epstein import EpsteinContext as EC
            from paper_2504_11989_b200.quadrature import ATM_SPLIT_SCALE
            sp = ATM_SPLIT_SCALE * fcc.volume ** (-2.0 / 3)
            ta = time.perf_counter()
            z5 = EC(fcc, 5.0, sp, -2)
            tb = time.perf_counter()
            z3 = EC(fcc, 3.0, sp, deriv_order=-1)
            tc = time.perf_counter()
            print(f"  ctx z5 {1e3*(tb-ta):.2f} ms, ctx z3 {1e3*(tc-tb):.2f} ms (serial)")
        plan = atm_plan(fcc)  # plan-private contexts (in parallel) + plan build + upload
        t1 = time.perf_counter()
        s = ShardedIntegral(plan, 128, 128, 3)
        t2 = time.perf_counter()
        out = s.run().cpu().numpy()
        t3 = time.perf_counter()
        out = s.run().cpu().numpy()
        t4 = time.perf_counter()
        print(f"rep {rep}: cold atm_plan {1e3*(t1-t0):.2f} ms, ShardedIntegral {1e3*(t2-t1):.2f} ms, "
              f"run+d2h {1e3*(t3-t2):.2f} ms, warm run+d2h {1e3*(t4-t3):.2f} ms")


def c1_time():
    """Device time of the C1 zeta batches (4096 and 2^20 points), CUDA events."""
    sq = named_lattice("square")
    ctx = EpsteinContext(sq, 3.5, device=0)
    for n, seed in ((4096, 0), (1 << 20, 1)):
        k = torch.tensor(np.random.default_rng(seed).uniform(-0.5, 0.5, size=(n, 2)), device="cuda")
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            ctx.zeta_device(k, out=out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            ctx.zeta_device(k, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        print(f"n={n}: {ms:.4f} ms, {n / ms * 1e3:.3e} evals/s")
        # device time without host launch overhead: 20 launches replayed from a CUDA graph
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ctx.zeta_device(k, out=out)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    ctx.zeta_device(k, out=out)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        print(f"   graph replay: {a.elapsed_time(b) / 20:.4f} ms per batch")
        if n == 4096:
            for lanes in (1, 2, 4, 8, 16, 32):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    ctx.zeta_device(k, out=out, lanes_per_point=lanes)
                    torch.cuda.synchronize()
                    with torch.cuda.graph(g, stream=s):
                        for _ in range(20):
                            ctx.zeta_device(k, out=out, lanes_per_point=lanes)
                torch.cuda.synchronize()
                g.replay()
                torch.cuda.synchronize()
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                print(f"   lanes={lanes}: {a.elapsed_time(b) / 20:.4f} ms per batch (graph replay)")


def e2e():
    sq = named_lattice("square")
    ctx = EpsteinContext(sq, 3.5, device=0)
    for n in (1, 4096, 1 << 20):
        k = np.random.default_rng(0).uniform(-0.5, 0.5, size=(n, 2))
        kp = torch.from_numpy(k).pin_memory().numpy()
        ctx.zeta(k)
        for label, arr in (("pageable", k), ("pinned", kp)):
            t = time.perf_counter()
            for _ in range(10):
                ctx.zeta(arr)
            print(f"zeta n={n} {label}: {(time.perf_counter() - t) / 10 * 1e3:.3f} ms/call")
    cfg = QuadratureConfig(grid_u=256, grid_v=256, estimate_error=False)
    integrate_product(sq, [4.0] * 51, cfg)
    t = time.perf_counter()
    integrate_product(sq, [4.0] * 51, cfg)
    print(f"c4 integrate_product: {(time.perf_counter() - t) * 1e3:.3f} ms")
    t = time.perf_counter()
    atm_integrals(named_lattice("fcc"), ATMGrid(128, 128, 3))
    print(f"c3 atm_integrals warm: {(time.perf_counter() - t) * 1e3:.3f} ms")


if __name__ == "__main__":
    {"atm": atm, "c1": c1, "c1_time": c1_time, "e2e": e2e,
     "e2e_breakdown": e2e_breakdown, "atm_sweep": atm_sweep, "c1_small": c1_small, "adaptive_fcc": adaptive_fcc}[sys.argv[1]]()
