"""B200-native frontier BFS / Bellman-Ford (arxiv 1805.05208, GBBS hot path).

The product is libgbbs.so (C ABI in include/gbbs.h, kernels in csrc/); this
package is its thin Python binding.  Importing it loads libgbbs.so and raises
if it is missing — there is no fallback path.
"""
from .gbbs import (GBBS_BORROW, GBBS_INF, GBBS_MODE_AUTO, GBBS_MODE_DENSE, GBBS_MODE_SPARSE,  # noqa: F401
                   GBBS_NO_VALIDATE, GBBS_SYMMETRIC, GbbsError, Graph, gbbs_bellman_ford, gbbs_betweenness, gbbs_bfs,
                   gbbs_graph_create, gbbs_graph_destroy, gbbs_widest_path, last_error, make_opts, make_stats,
                   round_records)
