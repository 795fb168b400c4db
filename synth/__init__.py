"""Seeded synthetic inputs for the iFCTN-TC PAM sweep (configs C1–C5).

This module is shared by both sides of the parity check (the oracle under oracle/ and the
CUDA path under paper_2511_16358_b200/). It holds none of the method's arithmetic: no
contraction, no Gram/RHS, no solve, no refill. It only draws random numbers and shapes
them into a truth tensor, a mask and an initial factor set.
"""
from .generate import (CONFIGS, MSI_GRID, TRAFFIC_GRID, Problem, grid_rank_matrix, init_factors, make_config,  # noqa: F401
                       make_problem, mask_count)
