"""B200-native TOAST hot path (arXiv 2508.15010): batched evaluation of MCTS
rollouts over the sharding-decision space.  C ABI: include/toast.h
(libtoast.so, sm_100a kernels); Python binding: paper_2508_15010_b200.toast."""
from . import toast  # noqa: F401  (fails loudly if libtoast.so is missing)
from .toast import (Analysis, SearchOptions, SearchState, ToastError, as_costs, build_analysis, eval_batch,  # noqa: F401
                    load_graph, materialize, nda, rollout_batch, search)
