"""Repro: product integrals on a skewed 2D lattice, permuted exponents (fresh contexts)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2504_11989_b200 import Lattice
from paper_2504_11989_b200.quadrature import QuadratureConfig, integrate_product

lat = Lattice(np.array([[0.67052951047905185, 6.9999999999999994e-15], [0.11973167945412462, 0.70000000000000007]]))
nus = [5.588392847354402, 4.149364479639103, 5.857816266896291]
cfg = QuadratureConfig(grid_u=64, grid_v=64, estimate_error=False)
bad = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    vals = [integrate_product(lat, p, cfg)[0] for p in (nus, [nus[1], nus[2], nus[0]], nus[::-1])]
    if max(vals) - min(vals) > 1e-12 * abs(vals[0]):
        bad += 1
        print("rep", rep, vals, flush=True)
print("bad", bad)
