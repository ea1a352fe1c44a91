"""CPU oracle for the SCM hot path of MC-PDIPM (arXiv 1310.6919).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import anything under oracle/.  The
product path (paper_1310_6919_b200/) never imports it and fails loudly when its
CUDA library is missing.

The oracle shares no code with the CUDA path (no kernels, headers, helpers or
table generators); its only common input is the seeded instance generator in
instances/, which holds none of the method's arithmetic.  Everything is plain,
slow and fp64, each function citing the PAPER.md passage it follows:

* symbolic.py  - extended sparsity pattern E by the elimination game,
                 etree, fundamental supernodes as cliques.
* algorithm1.py- Algorithm 1 literally: reversal P_r, Cholesky, L_r = P_r M_r^{-T} P_r,
                 first |S_r| columns into L-hat; L-hat -> (L, D).
* ldl.py       - plain left-looking sparse LDL^T of Y on E (type (v)).
* scm.py       - B_kl = trace(A_k X-hat A_l Y^{-1}) (P:380 Eq. SCM), dense
                 mode and sampled-column mode via per-RHS solves (P:686-688 Eq. newSCM2).
* cholesky.py  - LAPACK potrf of B (type (i)).
* direction.py - the HKM search direction as printed: g, dz (Eq. SCE), dY, dX-hat and dX on
                 E (P-MATRIX, Eq. newdX/newdX2), mu, step lengths
                 alpha_p per clique (Eq. primal_length2) and alpha_d.

Parity status of every function is listed in DESIGN.md §Oracle pins; every
function here is pinned by a `-m "not gpu"` test against values the paper or
mathematics fixes (tests/test_oracle_*.py).  None is "parity unpinned".
"""
from . import symbolic, algorithm1, ldl, scm, cholesky, direction  # noqa: F401
