"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct fp64 CPU implementation of what the
B200 hot path computes (arXiv 2405.09400, PAPER.md): single-scale entropic
domain decomposition (Alg. 1/2) with the GPU-style bounding
box state of App. A (Alg. 4), the flow update (Def.
flow-update PAPER.md:416-436, product gluing candidate PAPER.md:552) and the
hybrid schedule (Alg. 3), plus the diagnostics of App. A.2.2
 and a dense global Sinkhorn reference.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product path
(paper_2405_09400_b200) never imports it and shares no code with it; the two
meet only through the seeded generators in synth/.

Each function cites the passage it follows.  Where the paper is silent the
DESIGN.md reading (R#) is named.  Parity status per function is listed in
DESIGN.md "Oracle pins"; functions with no independent pin say
"parity unpinned" in their docstring.
"""
from .partitions import basic_partition, composite_partition, partition_graph_connected  # noqa: F401
from .sinkhorn import cell_sinkhorn, dense_sinkhorn, lse, y_update_at  # noqa: F401
from .domdec import OracleState, init_state, domdec_sweep, basic_to_composite, balance, truncate_box  # noqa: F401
from .flow import (edge_costs, integer_instance, min_cost_flow, mcf_bruteforce,  # noqa: F401
                   apply_flow, flow_update, flow_objective)
from .diagnostics import (marginal_errors, transport_cost, primal_score, dual_score,  # noqa: F401
                          stitch_alpha, pd_gap, y_response, dense_state_plan)
from .schedule import run  # noqa: F401
