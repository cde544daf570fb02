"""A/B timing of the fcc ATM kernel (one process per variant; env vars / LATSUM_LIB select it).

    python tools/ab_time.py [reps]      -> one line: kernel ms (CUDA events, mean of reps after
                                           warm-up) and the ATM energy of the bench grid
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2504_11989_b200 import named_lattice
from paper_2504_11989_b200.quadrature import atm_plan


def main(reps=20):
    lat = named_lattice(os.environ.get("LATTICE", "fcc"))
    plan = atm_plan(lat)
    nn, nt = plan.tiles(128, 128, 3)
    part = torch.zeros(nt * 2, dtype=torch.float64, device="cuda")
    for _ in range(3):
        plan.integrate_device(part, 128, 128, 3)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.integrate_device(part, 128, 128, 3)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    s2 = plan.integrate(128, 128, 3)
    e = 8.0 * (s2[0] - 3.0 * s2[1]) / 6.0
    ts.sort()
    tag = os.environ.get("AB_TAG", "")
    print(f"{tag:24s} mean {sum(ts) / len(ts):.4f} ms  min {ts[0]:.4f}  median {ts[len(ts) // 2]:.4f}  "
          f"E {e:.15f}", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
