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
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    st = T.SearchState(a, opts, rank, world, stream=stream)
    nccl = dist.get_backend(group) == "nccl"
    if nccl:   # the exchange stays in device memory (toast_search_round_dev / _import_dev)
        dev = torch.device("cuda", torch.cuda.current_device())
        rec_d = torch.empty(st.export_bytes, dtype=torch.uint8, device=dev)
        all_d = torch.empty(world * st.export_bytes, dtype=torch.uint8, device=dev)
        cur = torch.cuda.current_stream(dev)
    while True:
        if nccl:
            st.round_dev(rec_d, stream=cur)
            dist.all_gather_into_tensor(all_d, rec_d, group=group)
            stop = st.import_dev(all_d, stream=cur)
            gathered = all_d.cpu().numpy() if trace is not None else None
        else:
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


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def rank_id_base(rank: int, per_rank: int) -> int:
    """Disjoint Philox counter ranges per rank for weak-scaled rollouts."""
    return rank << 40


def shard_range(n: int, rank: int, world: int) -> tuple:
    """The contiguous rows [lo, hi) of an n-row batch that rank evaluates:
    the first n % world ranks take one row more."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def eval_sharded(a: "T.Analysis", seqs, group=None, stream=None, compact: bool = False, _evaluate=None):
    """Data-parallel toast_eval_batch over the ranks of `group`:
    every rank holds the same global batch seqs (uint16[n][32], device tensor on
    NCCL), evaluates its contiguous rows [lo, hi) with the library, and one
    all_gather_into_tensor of the fixed-size result records (the last ranks'
    slices padded to the largest) gives every rank all n results in batch
    order.  Returns a uint8 [n, record bytes] tensor (256-B toast_cost, or 16-B
    toast_score when compact).  There is no exchange inside the evaluation:
    candidates are independent.  _evaluate(seqs_slice, out_slice) replaces the
    library call in host-logic tests only."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = int(seqs.shape[0])
    rec = 16 if compact else 256
    lo, hi = shard_range(n, rank, world)
    width = shard_range(n, 0, world)[1]            # the largest slice
    cuda = seqs.device.type == "cuda"
    # everything (the zero fill, the evaluation) runs on `stream`; the current
    # stream, which the collective is ordered on, waits for it
    side = stream if (cuda and stream is not None) else None
    if side is not None and not isinstance(side, torch.cuda.Stream):
        side = torch.cuda.ExternalStream(int(getattr(side, "cuda_stream", side)))
    ctx = torch.cuda.stream(side) if side is not None else _nullctx()
    with ctx:
        local = torch.zeros((width, rec), dtype=torch.uint8, device=seqs.device)
        if hi > lo:
            if _evaluate is not None:
                _evaluate(seqs[lo:hi], local[: hi - lo])
            elif compact:
                T.eval_scores(a, seqs[lo:hi], local[: hi - lo], stream=side)
            else:
                T.eval_batch(a, seqs[lo:hi], local[: hi - lo], stream=side)
    if side is not None:
        torch.cuda.current_stream().wait_stream(side)
        local.record_stream(torch.cuda.current_stream())
    gathered = torch.empty((world * width, rec), dtype=torch.uint8, device=seqs.device)
    dist.all_gather_into_tensor(gathered, local, group=group)
    parts = [gathered[r * width: r * width + (shard_range(n, r, world)[1] - shard_range(n, r, world)[0])]
             for r in range(world)]
    return torch.cat(parts, dim=0)
