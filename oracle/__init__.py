"""CPU oracle for the nodal-DG Maxwell hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference package's algorithm for the
path the B200 operator replaces (see ``dg_oracle`` for file:line citations
into /root/reference/pkg/src/simtdg).  It is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it.  The product package
(``paper_0901_1024_b200``) never imports it and has no CPU fallback.

Parity of the oracle itself is pinned against outputs of the real reference,
generated in the build container by ``oracle/make_golden.py`` and committed
as ``tests/golden/*.npz`` (tests/test_oracle_golden.py).
"""

from .dg_oracle import (  # noqa: F401
    RK_A,
    RK_B,
    RK_C,
    OracleOperator,
    build_oracle_operator,
    oracle_connectivity,
    oracle_geometry,
    oracle_sigma,
    pec_mirror,
    rk4_step,
    upwind_bracket,
)
