"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no Sinkhorn, no cell solve, no
flow update).  It only produces the problem data the paper's experiments are
shaped like:

* quantised Gaussian-mixture images (App. A.2, "Gaussian
  mixtures with random variances, means and magnitudes");
* the four-bumps image of §5.2;
* the initial coupling pi^0 = (id, T)_# mu for a rotation(+contraction) map T
  (§5.4, Eq. T0), discretised by integer
  bilinear splatting so that every number is an exact dyadic rational;
* random feasible flows w and random integer min-cost-flow instances
  (test inputs for the flow-update steps).

Every value is an integer count times 2^-E, so mu, nu and the initial
basic-cell Y-marginals are exactly representable in fp32 and fp64 and the
min-cost-flow supplies q_i = m_i 2^E are exact int64.
"""
from .generators import (  # noqa: F401
    SplitMix64,
    Problem,
    gaussian_mixture_counts,
    four_bumps_counts,
    rotation_map,
    splat_coupling,
    make_problem,
    random_flow,
    random_mcf_instance,
    exponent_E,
)
