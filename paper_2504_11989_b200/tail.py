"""Meromorphic-continuation path of integrate_product for exponents nu <= d.

The reference (L/quadrature.py:400-452) splits the radial integral at epsilon,
integrates the inner part analytically from Taylor tables at k = 0 and the
outer part adaptively with the growing monomials subtracted.  In this build the
ATM energy does not need it (see manybody.py); the general path is the next
row of the scope table and is not available yet.
"""
from __future__ import annotations


def integrate_product_continued(lattice, contexts, cfg):
    raise NotImplementedError(
        "integrate_product with some nu <= d (meromorphic continuation) is not implemented on the "
        "B200 path yet; ATM energies are available through atm_cohesive_energy")
