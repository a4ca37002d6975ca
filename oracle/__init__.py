"""CPU ORACLE for the ChASE hot path (arXiv 2309.15595) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import or call anything in this package.  The product path
(``paper_2309_15595_b200``) never imports it and has no CPU fallback.

Plain, slow, obviously-correct fp64 NumPy implementations, written from PAPER.md in the
paper's order and notation (``P:NNN`` = /root/reference/PAPER.md line, ``S:NNN`` = SPEC.md
line).  A library matmul (numpy ``@``) serves as the HEMM step; everything else (Chebyshev
scalars, Cholesky, triangular solves, Householder QR, Alg.4 dispatch, Alg.5 estimate) is
written out loop by loop.  Shares no code with the CUDA path.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): closed-form Chebyshev values (cos/cosh form),
brute-force eigendecomposition for N <= 64, the FFT closed form of the DFT-phase matrices,
SPEC's hand-computed examples under tests/golden/, QR invariants and LAPACK Householder QR.
Every function here is pinned; none is "parity unpinned".

``oracle/cpp/chase_oracle.cpp`` (binding ``oracle.cpp_oracle``) is the same filter and CholeskyQR
family as plain C++17 triple loops with OpenMP over output rows (the north star's "plain, slow
CPU filter and CholeskyQR with triple loops"), pinned by tests/test_oracle_cpp.py with the same
closed forms and golden cases; bench.py times it as ``cpu_baseline`` and the reference arm.
"""
from .filter import chebyshev_scalars, chebyshev_filter, filter_schedule, filter_record  # noqa: F401
from .qr import (gram, potrf_upper, trsm_right_upper, shift_value, cholesky_qr, caqr,  # noqa: F401
                 cond_est, select_variant, householder_qr, householder_factor, larfg,
                 frobenius_sq)
from .grid import distributed_filter, step_partial  # noqa: F401
from .residual import residuals  # noqa: F401
from .rayleigh_ritz import rayleigh_ritz  # noqa: F401
