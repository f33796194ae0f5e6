"""fp64 CPU oracle for the GA-NGMRES transport-optimization hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the C-ABI library
``libtopt.so`` and its Python binding ``paper_2510_08782_b200``) may import,
call, link or execute anything in this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) use it.

What it is: a plain, slow, obviously-correct fp64 implementation of what the
paper (arXiv 2510.08782, ``PAPER.md``) defines, following the paper's steps in
the paper's order, with the readings R1..R30 of SURVEY.md §8(c) wherever the
paper is silent or garbled (all listed in DESIGN.md §3).  Library primitives
(numpy FFTs, SVD) serve as single steps; no blocking, fusion or reordering.

Modules
  spectral   Fourier grid, derivatives, regularisation symbol L, (alpha L)^-1,
             Leray projector, discrete inner product
  interp     periodic tricubic Lagrange interpolation at node + displacement
             (reading R5)
  transport  RK2 characteristic feet, forward/adjoint SL sweeps, static
             source factors (R6-R8)
  gradient   objective (1.1a), reduced gradient (2.2), preconditioned
             direction (2.5)/(2.6)
  solver     Armijo with memory, FP map q (2.7), NGMRES(w) Alg.1, AA(w)
             Alg.2, GA-NGMRES(w;sigma,tau) Alg.3
  flowmap    flow map y and det(grad y) (figure captions P:323, P:781, P:866;
             reading R32)

Parity pins: every function is pinned by tests in ``tests/test_oracle_*.py``
against closed forms, invariants and brute force.
"""
from . import spectral, interp, transport, gradient, solver, flowmap  # noqa: F401
