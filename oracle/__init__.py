"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 numpy implementation of arXiv 2011.07632's hot path
(tree -> H2 by proxy-point ID -> Alg. 4 SPD-HSS construction -> recursive HSS
solve -> PCG).  It exists to prove the CUDA path correct.

Rules:
  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
    --impl reference leg may import anything under oracle/.  The product
    package paper_2011_07632_b200 never imports it and never falls back to it.
  * Shares no code with the CUDA path (no kernels, headers, helpers or table
    generators).  Only the seeded input generators in synth/ serve both.
  * Each function cites the PAPER.md passage (P:line, section / equation /
    algorithm label) or the DESIGN.md reading (R1..R22) it follows.
  * Library primitives used as single steps: numpy matmul, numpy.linalg
    cholesky/eigh, scipy.linalg.solve_triangular.  QRCP is written out
    (Businger-Golub with recomputed norms, lowest-index tie-break, R4) because
    its pivot rule is part of the parity contract.

Parity status of each function is listed in DESIGN.md §Oracle pins; functions
with no independent pin carry "parity unpinned" in their docstring.
"""
from .kernels import kernel_matrix, kernel_value
from .tree import Tree, build_tree, interaction_lists, Lists
from .linalg import NotPD, cholesky, qrcp, sym_sqrt_pair
from .h2 import H2, h2_build, h2_matvec, h2_densify, proxy_points, halton
from .spdhss import (HSS, spdhss_build, hss_matvec, hss_densify, hss_solve,
                     pcg, block_jacobi_solve, spdhss_build_adaptive, alg1_generalized, special_products, hss_error)

__all__ = [n for n in dir() if not n.startswith("_")]
