"""ORACLE -- test infrastructure, not product code.

A plain, slow, fp64 CPU evaluation of PAPER.md Eq. probDef by Alg. 1 per problem.
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference) may import it.
It shares no code with paper_1207_2169_b200/ (the CUDA path) and never imports it.
See oracle/gls.py for the step-by-step citations and DESIGN.md §4 for the pins.
oracle/estimate.py: the variance-component estimation step (readings E1-E4), pinned by
tests/test_oracle_estimate.py.
"""
from . import estimate  # noqa: F401
from .gls import (STATUS_COLLINEAR, STATUS_NONFINITE, STATUS_OK, assemble_covariance, cholesky_lower,
                  forward_substitute, gls_sequence, gls_single, small_cholesky, small_spd_solve)

__all__ = ["STATUS_OK", "STATUS_COLLINEAR", "STATUS_NONFINITE", "assemble_covariance", "cholesky_lower",
           "forward_substitute", "gls_single", "gls_sequence", "small_cholesky", "small_spd_solve"]
