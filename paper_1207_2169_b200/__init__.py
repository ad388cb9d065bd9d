"""B200-native CLAK-Eig GLS-sequence hot path (arXiv 1207.2169, Alg. 4) behind the C-ABI libgwas.so.

The package holds only the CUDA sources (csrc/), the in-tree build (build.py) and a thin ctypes binding
(_lib.py, api.py).  There is no CPU fallback: importing fails if libgwas.so is missing.
"""
from ._lib import GwasError, lib  # noqa: F401  (loads libgwas.so or raises ImportError)
from .api import Gwas, gemm_tn  # noqa: F401

__all__ = ["Gwas", "GwasError", "gemm_tn", "lib"]
