"""CPU oracle for the bandix-b200 hot path.  TEST INFRASTRUCTURE ONLY.

This package restates, batched over a leading system axis, the arithmetic of
the reference package ``bandix`` 0.1.0 (``/root/reference/pkg/src/bandix``):
every function follows the reference's scalar operation order exactly (one
IEEE-754 binary64 rounding per operation, no FMA), so on identical inputs it
is bit-identical to the reference.  Each function cites the reference
``file:line`` it follows.

Parity status: PINNED.  ``tests/golden/*.npz`` hold outputs produced by the
reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src``); ``tests/test_oracle_golden.py`` asserts the
restatement equals those vectors bit-for-bit.  Where the reference has no code
(stride m > 2 and Stone's alpha for SIP; fp64 limits of the symbolic solvers at
N=2048) the restatement is pinned at the reference-representable twin
(m=2, alpha=0; small-N exact solves) and the rest is documented as an
extension in DESIGN.md.

Who may import this package: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- only as the
checker or the timed CPU baseline, never as the product path.  The product
(``paper_1804_09666_b200``) never imports it.
"""

STATUS_OK = 0
STATUS_ZERO_PIVOT = 1
STATUS_SINGULAR = 2
STATUS_MAX_ITER = 3
STATUS_DIVERGED = 4
STATUS_ZERO_DIAG = 5
STATUS_WINDOW_OVERFLOW = 6
STATUS_NOT_GRID = 7
STATUS_REDUCTION_PIVOT = 8
STATUS_STAGNATED = 9
