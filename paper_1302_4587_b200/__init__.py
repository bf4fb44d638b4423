"""B200-native local max maximal matching (arXiv 1302.4587), drop-in for locmax.

Public surface mirrors the reference package's matching path
(``/root/reference/pkg/src/locmax/__init__.py``): ``Graph``, ``Matching``,
``RoundStats``, ``PhaseTrace``, ``matching_from_edge_ids``,
``validate_matching``, ``build_graph``, ``run_matcher`` and the engine entry
point ``local_max_b200`` (the ``local_max_seq`` contract,
``matchers.py:61-122``), computed by hand-written sm_100a kernels in
``csrc/`` behind the C ABI in ``include/lmx.h``.
"""

from .builders import build_graph, gen_rgg, gen_rmat
from .engine import (Engine, RbmDidNotConverge, default_engine, load_library, local_max_b200, pram_local_max_b200,
                     rbm_b200, run_matcher)
from .graph import (
    Graph,
    Matching,
    MatchingCheck,
    PhaseTrace,
    RoundStats,
    matching_from_edge_ids,
    validate_matching,
)

local_max = local_max_b200

__version__ = "0.1.0"

__all__ = [
    "Engine", "Graph", "Matching", "MatchingCheck", "PhaseTrace", "RoundStats",
    "build_graph", "default_engine", "gen_rgg", "gen_rmat", "load_library", "local_max", "local_max_b200",
    "matching_from_edge_ids", "run_matcher", "validate_matching", "rbm_b200", "RbmDidNotConverge",
    "pram_local_max_b200",
]
