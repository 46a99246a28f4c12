"""B200-native TOAST hot path (arXiv 2508.15010): batched evaluation of MCTS
rollouts over the sharding-decision space.  C ABI: include/toast.h
(libtoast.so, sm_100a kernels); Python binding: paper_2508_15010_b200.toast
(loaded on first use; it fails loudly if libtoast.so is missing)."""

_EXPORTS = ("Analysis", "SearchOptions", "SearchState", "ToastError", "as_costs", "as_scores", "build_analysis",
            "eval_batch", "eval_scores", "load_graph", "lower", "materialize", "nda", "rollout_batch", "rollout_scores",
            "search")


def __getattr__(name):
    if name in _EXPORTS:
        from . import toast
        return getattr(toast, name)
    raise AttributeError(name)
