"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct CPU implementation of the
Newton-step solve of arXiv 2403.15913 (§III-§V) that the CUDA library
is checked against.  It shares no code with the CUDA path
(paper_2403_15913_b200/) and never imports it; only the seeded input
generators in inputs/ serve both.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import, call, link or execute anything under
oracle/.  The product path must never route through it.

Tiers:
  * Tier T (oracle/dense.py): dense K_aug assembly, Bunch–Kaufman LDLᵀ with
    inertia, dense condensation / Lifted-KKT / HyKKT formulas, for tiny
    systems.
  * Tier S (oracle/sparse.py + oracle/csrc/sparse_oracle.c): the specified
    nested-dissection ordering, elimination tree, column counts and L pattern,
    a simple left-looking column Cholesky, triangular solves, unpreconditioned
    CG on S_γ, Richardson refinement on K_aug, slack/dual recovery.

Parity status per function is listed in DESIGN.md §4 ("pins").
"""
