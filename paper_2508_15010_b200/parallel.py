"""Multi-GPU plumbing around libtoast: one process per GPU,
torch.distributed (NCCL on GPUs, gloo on CPU) for the few-hundred-byte
per-round exchange of root-parallel search, and disjoint Philox id ranges for
weak-scaled batched evaluation.  No data-path collective exists: candidates
are independent."""
from __future__ import annotations

import numpy as np

from . import toast as T

EXPORT_DTYPE = np.dtype([
    ("best_score", "<f8"), ("best_key", "<u8"), ("best_seq", "<u2", (32,)), ("evals", "<i8"),
    ("elapsed_s", "<f8"), ("rank", "<i4"), ("pad", "<i4"), ("best", T.COST_DTYPE)])


def export_dtype(n_actions: int) -> np.dtype:
    """The full per-rank record: the header above, then (visits, value_sum) of
    every root child, indexed by action id (include/toast.h toast_root_stat)."""
    return np.dtype([("hdr", EXPORT_DTYPE), ("root", T.ROOT_STAT_DTYPE, (n_actions,))])


def all_gather_bytes(buf: np.ndarray, group=None) -> np.ndarray:
    """all_gather of one fixed-size byte record per rank -> [world * nbytes] uint8."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    x = torch.from_numpy(np.ascontiguousarray(buf, dtype=np.uint8)).to(dev)
    out = torch.empty(world * x.numel(), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, x, group=group)
    return out.cpu().numpy()


def search_root_parallel(a: "T.Analysis", opts: "T.SearchOptions", group=None, stream=None, trace=None,
                         root_stats=None):
    """Root-parallel MCTS (R16): every rank grows its own tree (seed + rank);
    after each round the ranks all-gather their export records (best sequence
    and root visit statistics) and every rank imports the same bytes, so the
    global best, the summed root statistics and the stop decision agree.
    root_stats: optional list that receives the final summed root statistics."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    st = T.SearchState(a, opts, rank, world, stream=stream)
    while True:
        rec = st.round()
        gathered = all_gather_bytes(rec, group)
        stop = st.import_(gathered)
        if trace is not None:
            g = gathered.reshape(world, -1)[:, :EXPORT_DTYPE.itemsize].copy().view(EXPORT_DTYPE)
            trace.append(float(g["best_score"].min()))
        if stop:
            break
    if root_stats is not None:
        root_stats.append(st.root_stats())
    return st.end()


def rank_id_base(rank: int, per_rank: int) -> int:
    """Disjoint Philox counter ranges per rank for weak-scaled rollouts."""
    return rank << 40
