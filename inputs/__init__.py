"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no condensation, factorization,
Schur complement, CG or refinement).  It only builds the *problem data* the
method consumes: the distillation-column NLP of PAPER.md §VI.A —
its sparsity patterns and derivative values at synthetic interior-point
iterates — and small random saddle-point instances for unit tests.

Everything here is deterministic given the seeds.
"""
