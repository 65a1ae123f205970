"""CPU oracle for RSRS -- TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT PATH.

A plain, slow, obviously correct CPU implementation (numpy/scipy, LAPACK,
FP64 / complex128) of what the hot path computes, written from PAPER.md
(arXiv 2311.01451) step by step.  It shares no code with the CUDA path
(paper_2311_01451_b200/); neither imports the other.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import it.

Pins (tests/test_oracle_*.py, tests/test_workloads_t11.py, run with -m "not gpu"):
Fig. 1 tree example, brute-force neighbours, nullification identities
(PAPER.md:266-291), extraction exactness on block-sparse operators (Fig. 2b), ID
bounds and exact low-rank recovery, the sample-consistency invariant
Y = A_g Omega after every step, the decoupling invariant, the
zero-far-field special case, dense LU solve / relerr at c1 (g = c_id = 1 and the
frozen c1 configuration), the sphere at c5's frozen parameters vs dense LU, the
tolerance schedule, solve(apply(x)) = x, the
colour-parallel execution (bit-identical to the sequential order), the coupling
estimator and noise level against the explicitly tracked operator (f1), the
triangular form against dense LU (f4), the T11 workload against dense LU (f3).
Parity unpinned: exact skeleton index sets at near-tie pivots (covered only by
the +-2 rank and 10 eps solution tolerances); see DESIGN.md.
"""
from .tree import build_tree, Tree, Level, morton_encode, morton_decode  # noqa: F401
from .rsrs import (factor, solve, apply, Factorization, Step, RSRSError,  # noqa: F401
                   null_basis, pinv_right, row_id, atol_schedule, coupling_estimate,
                   noise_level, noise_aware_atol)
