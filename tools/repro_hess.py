"""Stress repro: zeta_hessian of fcc nu = 5 at many theta splits (fresh contexts each time)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2504_11989_b200 import named_lattice
from paper_2504_11989_b200.epstein import EpsteinContext

fcc = named_lattice("fcc")
k = np.random.default_rng(7).uniform(-0.5, 0.5, size=(256, 3)) @ fcc.a_inv_t.T
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for rep in range(reps):
    for scale in (0.3, 0.35, 0.4, 0.5, 0.65, 1.0, 1.6):
        t = scale * fcc.volume ** (-2.0 / 3.0)
        H = EpsteinContext(fcc, 5.0, splitting=t, device=0).zeta_hessian(k)
        z = EpsteinContext(fcc, 3.0, splitting=t, device=0).zeta(k)
        tr = -np.trace(H, axis1=1, axis2=2) / (4 * np.pi ** 2)
        err = np.max(np.abs(tr - z) / np.maximum(np.abs(z), 1))
        if err > 1e-11:
            print("mismatch", rep, scale, err, flush=True)
    torch.cuda.synchronize()
    print("rep", rep, "ok", flush=True)
