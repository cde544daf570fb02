"""latsum_b200: B200-native (sm_100a, FP64) Epstein-zeta lattice sums.

Drop-in for the reference package ``latsum`` (arXiv 2504.11989): the same
public names as L/__init__.py:1-18, with evaluation on the GPU through the C
ABI in include/latsum_b200.h.  Submodules: ``epstein`` (Z, Z_reg, shat,
polynomial-weighted zeta), ``quadrature`` (Duffy BZ quadrature of zeta
products), ``manybody`` (many-body zeta, ATM energy), ``phase`` (LJ+ATM
fcc/bcc scan), ``distributed`` (multi-GPU node sharding).
"""
from .errors import ConvergenceError, LatticeError, PoleError, TruncationWarning
from .lattice import BrillouinZone, Lattice, named_lattice, parse_lattice_spec

__version__ = "0.1.0"

__all__ = [
    "Lattice",
    "BrillouinZone",
    "named_lattice",
    "parse_lattice_spec",
    "LatticeError",
    "PoleError",
    "ConvergenceError",
    "TruncationWarning",
    "__version__",
]
