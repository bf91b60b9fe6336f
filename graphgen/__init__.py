"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the MWU method: it only draws graphs and
sparse matrices (the BASELINE.json configs c1-c5, their reduced same-recipe
instances, small closed-form graph families and random positive LPs).  Both
`oracle/` and the product path consume its outputs; neither is imported here.
"""
from .generators import (  # noqa: F401
    Graph, CsrLP, bipartite_uniform, erdos_renyi, rmat, bipartite_zipf,
    complete_graph, complete_bipartite, star_graph, path_graph, cycle_graph,
    circulant_regular, random_small_graph, hub_graph, random_small_bipartite,
    random_planted_lp, infeasible_lp, config_graph, CONFIGS, disjoint_union, plus_random_edges,
    rgg, biadjacency, gmatch_instance,
)
