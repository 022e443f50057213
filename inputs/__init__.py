"""inputs — seeded synthetic input generators shared by the oracle side and the
CUDA side (tests, bench, smoke).  This package holds none of the method's
arithmetic: it only draws random numbers and assembles the SPD test matrices
the configs in BASELINE.json describe (DESIGN.md §"Input recipe").
"""
from .gen import *  # noqa: F401,F403
