"""The N > 1 path on CPU: world_size-2 gloo process group, the per-round
all-gather of toast_search_export records and the library's import logic
(the same code the NCCL ranks run), with the round's records built from
oracle rollouts of each rank's seed."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2508_15010_b200 import parallel as P
        from paper_2508_15010_b200 import toast as T
        from workloads import configs
        c = configs.get("gpt2")
        a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=-1)
        o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth)
        opts = T.SearchOptions(seed=10, patience=2, max_evals=10 ** 9)
        st = T.SearchState(a, opts, rank, world)
        na = len(a.dump()["actions"]) + 1
        RD = P.export_dtype(na)
        assert st.export_bytes == RD.itemsize
        out = []
        for rnd in range(4):
            # this rank's "round": a batch of rollouts for its own seed; best = min (score, key)
            seqs, costs = o.rollout(np.zeros((64, 32), np.uint16), seed=opts.seed + rank, id_base=rnd * 64)
            i = int(np.lexsort((costs["state_key"], costs["score"]))[0])
            rec = np.zeros(1, dtype=RD)
            h = rec["hdr"]
            h["best_score"] = costs["score"][i]
            h["best_key"] = costs["state_key"][i]
            h["best_seq"] = seqs[i]
            h["evals"] = 65 * (rnd + 1)
            h["elapsed_s"] = 0.1 * rnd
            h["rank"] = rank
            h["best"] = costs[i]
            rec["hdr"] = h
            # root statistics: visits / reward sums of the root children this rank's rollouts started with
            root = np.zeros(na, dtype=T.ROOT_STAT_DTYPE)
            for s_, c_ in zip(seqs, costs):
                root["visits"][s_[0]] += 1
                root["value_sum"][s_[0]] -= c_["score"]
            rec["root"] = root
            gathered = P.all_gather_bytes(rec.view(np.uint8).reshape(-1))
            stop = st.import_(gathered)
            g = gathered.view(RD)
            rs = st.root_stats()
            assert np.array_equal(rs["visits"], g["root"]["visits"].sum(axis=0))
            assert np.array_equal(rs["value_sum"], g["root"]["value_sum"][0] + g["root"]["value_sum"][1])
            out.append((stop, float(g["hdr"]["best_score"].min()), int(g["hdr"]["evals"].sum()),
                        int(rs["visits"].sum())))
            if stop:
                break
        res = st.end()
        q.put((rank, out, float(res["best"]["score"]), res["best_seq"].tolist(), int(res["evals"])))
    finally:
        dist.destroy_process_group()


def test_root_parallel_exchange_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, out0, s0, q0, e0), (r1, out1, s1, q1, e1) = res
    # identical decisions, identical global best, on both ranks
    assert out0 == out1
    assert (s0, q0, e0) == (s1, q1, e1)
    # the global best is the best of both ranks' records; evals and root visits are summed
    assert s0 == min(o[1] for o in out0)
    assert all(o[3] == 128 for o in out0)
    assert e0 == out0[-1][2]
    # patience 2: it stops after two non-improving rounds or runs all 4
    stops = [o[0] for o in out0]
    assert stops.count(True) <= 1 and (not any(stops[:-1]))


def _eval_worker(rank, world, port, n, q):
    """eval_sharded's slicing and gather on gloo, with a stand-in evaluator that
    writes each row's global index into its record (the library needs a GPU)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_15010_b200 import parallel as P
        seqs = torch.arange(n * 32, dtype=torch.int16).reshape(n, 32) if n else torch.zeros((0, 32), dtype=torch.int16)
        seen = []

        def fake(sl, out):
            seen.append(int(sl.shape[0]))
            out.view(torch.int64)[:, 0] = sl[:, 0].to(torch.int64) // 32   # the global row index
            out.view(torch.int64)[:, 1] = rank

        res = P.eval_sharded(None, seqs, _evaluate=fake)
        q.put((rank, res.view(torch.int64)[:, 0].tolist(), res.view(torch.int64)[:, 1].tolist(), seen))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [0, 7, 101])
def test_eval_sharded_two_ranks(n):
    """contiguous per-rank slices (ragged last slice, empty batch),
    one all-gather, every rank ends with all n records in batch order."""
    from paper_2508_15010_b200.parallel import shard_range
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_eval_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rows, owner, seen in res:
        assert rows == list(range(n))
        expect = []
        for r in range(world):
            lo_r, hi_r = shard_range(n, r, world)
            expect += [r] * (hi_r - lo_r)
        assert owner == expect
        lo, hi = shard_range(n, rank, world)
        assert seen == ([hi - lo] if hi > lo else [])
