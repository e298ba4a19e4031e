"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package builds input matrices only. It holds none of the SpGEMM method's
arithmetic (no products, no accumulation, no counting of C): see DESIGN.md §3
for the recipe of every workload.
"""
from .generators import (  # noqa: F401
    CSR,
    stencil_laplacian,
    laplacian_2d_5pt,
    laplacian_3d_7pt,
    laplacian_3d_27pt,
    block_stencil_27pt,
    aggregation_prolongator,
    transpose_pattern_ones,
    transpose,
    random_value,
    uniform01,
    rmat,
    random_csr,
    config,
    CONFIGS,
)
