"""Algorithmic flop/byte model of one element-stage.

An *element-stage* is one RHS evaluation plus the LSRK register update for one
element; one RK4 step is 5 element-stages per element.  These counts are fixed
by the algorithm, not by the implementation, and are what every throughput and
roofline number in bench.py is computed from.
"""

from __future__ import annotations

from .refelem import simplex_node_count


def flops_per_element_stage(order: int) -> int:
    n_p, n_fp = simplex_node_count(order)
    return (18 * (2 * n_p - 1) * n_p       # D_r, D_s, D_t on 6 fields
            + 66 * n_p                      # geometric factors + curls
            + 66 * 4 * n_fp                 # upwind flux + face scaling
            + 6 * (8 * n_fp - 1) * n_p      # LIFT on 6 fields
            + 18 * n_p                      # 1/J, 1/eps, 1/mu, combine
            + 30 * n_p)                     # LSRK update


def bytes_per_element_stage(order: int, word: int) -> int:
    """Compulsory HBM bytes: u, res read+write (24 Np words) + 26 geometry + 8 connectivity words."""
    n_p, _ = simplex_node_count(order)
    return word * (24 * n_p + 34)


def dofs(order: int, num_elements: int) -> int:
    return 6 * simplex_node_count(order)[0] * num_elements
