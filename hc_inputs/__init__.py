"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds only *inputs*: polynomial systems F(x; p) written as sparse
term lists (problem formulations, §4 / Table 1), seeded parameter
instances, and fixture file I/O.  It contains none of the homotopy-continuation
arithmetic (no evaluation of H, no linear solves, no tracking): both `oracle/`
and `paper_2112_03444_b200/` consume what it produces, and neither shares code
with the other through it.
"""
from .poly import Poly, var_x, var_p, const
from .descriptor import SystemDesc, desc_from_equations
from . import systems, rng, fixtures

__all__ = ["Poly", "var_x", "var_p", "const", "SystemDesc", "desc_from_equations",
           "systems", "rng", "fixtures"]
