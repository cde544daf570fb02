"""cProfile of the reference's Prop. 2.4 route (three adaptive continued integrals on fcc) through
integrate_product(method="adaptive"):  python tools/prof_adapt.py"""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
from paper_2504_11989_b200 import named_lattice
from paper_2504_11989_b200.quadrature import integrate_product, QuadratureConfig
fcc = named_lattice("fcc")
cfg = QuadratureConfig(method="adaptive")
integrate_product(named_lattice("square"), (3, 3, 3), cfg)
t0=time.perf_counter()
integrate_product(fcc, (1,3,5), cfg)
print("first (1,3,5)", time.perf_counter()-t0)
pr = cProfile.Profile(); pr.enable()
t0=time.perf_counter()
for nus in ((3, 3, 3), (-1, 5, 5), (1, 3, 5)):
    integrate_product(fcc, nus, cfg)
print("three integrals", time.perf_counter()-t0)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
