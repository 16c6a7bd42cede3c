"""CPU oracle for the NFSGLFT hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy (and plain C for the window loops), the
algorithm of the reference `sglnufft` package (arXiv 1809.10786) for the
forward NFSGLFT and its adjoint.  Every function cites the reference
file:line it follows (paths relative to the reference's
`pkg/src/sglnufft/`).

It exists only as the checker: `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s CPU-baseline leg / `--impl reference` arm may import it.  The
product package `paper_1809_10786_b200` never imports it and has no CPU
fallback.

Pinning: the restatement is checked against golden vectors produced by the
reference itself (`tests/golden/make_golden.py`, run in the build container
where the reference is importable) and against the reference's own
known-answer tests (see `tests/test_oracle.py`).
"""
from .sgl_oracle import (  # noqa: F401
    OraclePlan,
    coeff_count,
    oracle_plan,
    oracle_forward,
    oracle_adjoint,
    evaluate_direct,
    evaluate_direct_adjoint,
    rel_linf,
)
