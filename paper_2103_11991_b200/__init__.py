"""B200-native two-phase hash SpGEMM (C = A*B on CSR), after Kokkos Kernels
(arXiv 2103.11991, Sec. 2.2.1).  The compute path is libkk_spgemm.so (CUDA, sm_100a)
behind the C ABI in include/kk_spgemm.h; this package is its thin Python binding.
"""
from .spgemm import CsrMatrix, SpGEMM, spadd, spgemm, spgemm_jacobi  # noqa: F401
from . import _ffi  # noqa: F401

__all__ = ["CsrMatrix", "SpGEMM", "spadd", "spgemm", "spgemm_jacobi"]
