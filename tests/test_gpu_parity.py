"""GPU parity: libtoast's sm_100a kernels vs the CPU oracle, element by element.

Bar (BASELINE north star): shardings, collective choice, byte
counts, peak memory, FLOPs and state keys bit-exact; runtime/score within
1e-6 relative — asserted here as bit-exact, which is stricter (both sides
evaluate the same IEEE double expression in the same order without FMA).
Inputs: oracle rollouts (C15 policy), uniform random ids (status paths),
hand-built 30-action sequences, and the bench's full-size launch.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from workloads import candidates, configs

pytestmark = pytest.mark.gpu

FIELDS_INT = ("peak_bytes", "flops", "flops_hi", "state_key", "status", "n_collectives")


def _T():
    from paper_2508_15010_b200 import toast as T
    return T


_cache = {}


def setup(name, **over):
    key = (name, tuple(sorted(over.items())))
    if key not in _cache:
        T = _T()
        c = configs.get(name)
        dm = over.get("dm", c.dm)
        a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0)
        o = Oracle(c.ir, c.axes, c.flops_per_sec, dm, c.penalty_c, c.min_dims, c.max_depth)
        _cache[key] = (a, o)
    return _cache[key]


def gpu_eval(a, seqs: np.ndarray) -> np.ndarray:
    import torch
    T = _T()
    d_seqs = torch.from_numpy(np.ascontiguousarray(seqs).view(np.int16)).cuda()
    d_out = torch.empty((len(seqs), 256), dtype=torch.uint8, device="cuda")
    T.eval_batch(a, d_seqs, d_out)
    torch.cuda.synchronize()
    return T.as_costs(d_out)


def gpu_rollout(a, prefixes: np.ndarray, seed: int, id_base: int):
    import torch
    T = _T()
    d_pre = torch.from_numpy(np.ascontiguousarray(prefixes).view(np.int16)).cuda()
    d_seq = torch.empty_like(d_pre)
    d_out = torch.empty((len(prefixes), 256), dtype=torch.uint8, device="cuda")
    T.rollout_batch(a, d_pre, seed, id_base, d_seq, d_out)
    torch.cuda.synchronize()
    return d_seq.cpu().numpy().view(np.uint16), T.as_costs(d_out)


def assert_same(g: np.ndarray, o: np.ndarray, ctx=""):
    assert len(g) == len(o)
    for f in FIELDS_INT:
        bad = np.nonzero(g[f] != o[f])[0]
        assert len(bad) == 0, (ctx, f, bad[:5], g[f][bad[:5]], o[f][bad[:5]])
    for f in ("payload", "count"):
        bad = np.nonzero((g[f] != o[f]).reshape(len(g), -1).any(1))[0]
        assert len(bad) == 0, (ctx, f, bad[:5])
    for f in ("runtime_s", "score"):
        # the north-star tolerance (1e-6 relative) ...
        rel = np.abs(g[f] - o[f]) / np.maximum(np.abs(o[f]), 1e-300)
        assert (rel <= 1e-6).all(), (ctx, f, rel.max())
        # ... and, stricter, bit equality
        bad = np.nonzero(g[f].view(np.uint64) != o[f].view(np.uint64))[0]
        assert len(bad) == 0, (ctx, f, bad[:5], g[f][bad[:5]], o[f][bad[:5]])


ALL = ["mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_1ax_np2", "gpt2_3ax", "gpt2_3ax_np2", "gpt2_4ax", "gpt2_4ax_np2",
       "gpt24", "gns16", "unet", "llama80"]
# the small configs the oracle evaluates thousands of times in seconds
SMALL = ("mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_1ax_np2", "gpt2_3ax", "gpt2_3ax_np2", "gpt2_4ax", "gpt2_4ax_np2")
# one config per kernel instantiation (mesh axes, every axis a power of two)
VARIANT_CONFIG = {(1, 1): "attn_toy", (1, 0): "gpt2_1ax_np2", (2, 1): "gpt2", (2, 0): "gpt2_np2", (3, 1): "gpt2_3ax",
                  (3, 0): "gpt2_3ax_np2", (4, 1): "gpt2_4ax", (4, 0): "gpt2_4ax_np2"}


@pytest.mark.parametrize("name", ALL)
def test_eval_parity_on_oracle_rollouts(name):
    a, o = setup(name)
    n = 3000 if name in SMALL else 100 if name == "llama80" else 300
    seqs, oc = o.rollout(np.zeros((n, 32), np.uint16), seed=1234, threads=8)
    assert_same(gpu_eval(a, seqs), oc, name)


@pytest.mark.parametrize("name", ["mlp_c", "gpt2", "gpt2_3ax", "gpt2_3ax_np2", "gpt2_4ax_np2", "unet"])
def test_eval_parity_uniform_ids_and_status(name):
    """Raw random ids: exercises BAD_ACTION_ID, DUP, RES_MISMATCH, NONZERO_AFTER_STOP
    next to valid sequences (ragged lengths 0..30)."""
    a, o = setup(name)
    seqs = candidates.uniform(2000 if name != "unet" else 400, o.n_actions + 2, seed=7, bad_frac=0.05)
    oc = o.eval(seqs, threads=8)
    assert set(np.unique(oc["status"])) >= {0}
    assert len(np.unique(oc["status"])) >= 3
    assert_same(gpu_eval(a, seqs), oc, name)


def _legal_long(o: Oracle, n: int, seed: int, length: int = 30) -> np.ndarray:
    """Sequences that keep choosing legal actions (C15 kill rule restated) with
    STOP disabled, up to `length` actions — the worst-case batch."""
    d = o.dump()
    acts = d["actions"]
    groups = [sc[2] for sc in d["scolors"]]
    rng = np.random.default_rng(seed)

    def kills(x, y):
        cx, rx, ax = acts[x - 1]
        cy, ry, ay = acts[y - 1]
        if cx == cy and ax == ay:
            return True
        for i, gx in enumerate(groups[cx]):
            for j, gy in enumerate(groups[cy]):
                if gx == gy and ((rx >> i) ^ (ry >> j)) & 1:
                    return True
        return False

    out = np.zeros((n, 32), np.uint16)
    for r in range(n):
        legal = list(range(1, len(acts) + 1))
        k = 0
        while legal and k < length:
            a = legal[rng.integers(len(legal))]
            out[r, k] = a
            k += 1
            legal = [b for b in legal if not kills(a, b)]
    return out


@pytest.mark.parametrize("name", ["unet", "gpt24", "gns16", "mlp_c", "gpt2_3ax", "gpt2_3ax_np2", "gpt2_1ax_np2",
                                  "llama80"])
def test_eval_parity_worst_case_long_sequences(name):
    a, o = setup(name)
    seqs = _legal_long(o, 60 if name == "llama80" else 200, seed=3)
    oc = o.eval(seqs, threads=8)
    assert (oc["status"] == 0).all()
    assert_same(gpu_eval(a, seqs), oc, name)


def test_eval_host_pointer_path_and_edges():
    """Host (numpy) buffers go through device scratch; n = 0 and n = 1 work."""
    T = _T()
    a, o = setup("gpt2")
    seqs, oc = o.rollout(np.zeros((257, 32), np.uint16), seed=9)
    out = np.zeros(257, dtype=T.COST_DTYPE)
    T.eval_batch(a, seqs, out)
    assert_same(out, oc, "host")
    one = np.zeros(1, dtype=T.COST_DTYPE)
    T.eval_batch(a, seqs[:1], one)
    assert_same(one, oc[:1], "n=1")
    T.eval_batch(a, seqs[:0], one[:0], n=0)


@pytest.mark.parametrize("name", ["mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_1ax_np2", "gpt2_3ax", "gpt2_3ax_np2",
                                  "gpt2_4ax", "gpt2_4ax_np2", "gpt24", "unet", "gns16", "llama80"])
def test_rollout_parity(name):
    """K2 vs C15: same (seed, id) -> same sequence and same cost record."""
    a, o = setup(name)
    n = 2000 if name in SMALL else 100 if name == "llama80" else 200
    pre = np.zeros((n, 32), np.uint16)
    # half the rows start from a (legal) prefix drawn by the oracle
    s0, _ = o.rollout(np.zeros((n // 2, 32), np.uint16), seed=77)
    for i in range(n // 2):
        L = int((s0[i] != 0).sum())
        k = i % (L + 1)
        pre[i, :k] = s0[i, :k]
    seed, id_base = 0xDEADBEEF12345, (1 << 33) + 17
    os_, oc = o.rollout(pre, seed=seed, id_base=id_base, threads=8)
    gs, gc = gpu_rollout(a, pre, seed, id_base)
    assert np.array_equal(gs, os_)
    assert_same(gc, oc, name)


def test_rollout_bad_prefix_is_not_extended():
    a, o = setup("mlp_c")
    pre = np.zeros((3, 32), np.uint16)
    pre[0, 0] = 999      # bad id
    pre[1, [0, 2]] = 1   # nonzero after STOP
    pre[2, 0] = 1
    os_, oc = o.rollout(pre, seed=1)
    gs, gc = gpu_rollout(a, pre, 1, 0)
    assert np.array_equal(gs, os_) and np.array_equal(gs[:2], pre[:2])
    assert_same(gc, oc)


@pytest.mark.parametrize("name,samples", [("gpt24", 48), ("unet", 24), ("gns16", 24), ("llama80", 200)])
def test_full_size_bench_launch_sampled(name, samples):
    """Every BASELINE config at full size in bench.py's launch configuration
    (2^18 rollouts rounded down to whole waves, from the empty prefix, bench's
    seed): a sample of outputs is recomputed one by one by the oracle
    (sequence and record); size-independent properties hold for all rows."""
    a, o = setup(name)
    wave = a.preferred_batch()
    n = max(wave, ((1 << 18) // wave) * wave)
    seed, id_base = 2024, 3 * n
    gs, gc = gpu_rollout(a, np.zeros((n, 32), np.uint16), seed, id_base)
    assert (gc["status"] == 0).all()
    idx = np.random.default_rng(0).choice(n, size=samples, replace=False)
    for i in idx:
        s1, c1 = o.rollout(np.zeros((1, 32), np.uint16), seed=seed, id_base=id_base + int(i))
        assert np.array_equal(gs[i], s1[0])
        assert_same(gc[i:i + 1], c1, f"row {i}")
    # properties that hold at any size
    t0, p0, _ = o.baseline()
    assert (gc["peak_bytes"] <= p0).all()
    assert (gc["score"] > 0).all()


@pytest.mark.slow
def test_llama80_sampled():
    a, o = setup("llama80")
    n = 4096
    gs, gc = gpu_rollout(a, np.zeros((n, 32), np.uint16), 5, 0)
    for i in np.random.default_rng(1).choice(n, size=8, replace=False):
        s1, c1 = o.rollout(np.zeros((1, 32), np.uint16), seed=5, id_base=int(i))
        assert np.array_equal(gs[i], s1[0])
        assert_same(gc[i:i + 1], c1)


@pytest.mark.parametrize("name,dm", [("mlp_c", None), ("attn_toy", 700), ("gpt2", None)])
def test_search_trace_parity(name, dm):
    """C16 implemented twice (oracle on CPU, library on host+GPU): same seed ->
    same rounds, evaluation count and best state."""
    T = _T()
    a, o = setup(name, dm=dm) if dm else setup(name)
    for tp in (0, 1):   # a tree of sequences, and with transpositions (reading R24)
        opts = T.SearchOptions(seed=3, max_evals=3000, leaves_per_round=4, rollouts_per_leaf=8, patience=3,
                               transpositions=tp)
        r = T.search(a, opts)
        ro, _ = o.search(seed=3, max_evals=3000, L=4, R=8, patience=3, transpositions=tp)
        assert int(r["rounds"]) == int(ro["rounds"]), tp
        assert int(r["evals"]) == int(ro["evals"]), tp
        assert np.array_equal(r["best_seq"], ro["best_seq"]), tp
        assert r["best"]["score"] == ro["best"]["score"], tp
    opts = T.SearchOptions(seed=3, max_evals=3000, leaves_per_round=4, rollouts_per_leaf=8, patience=3)
    r = T.search(a, opts)
    ro, _ = o.search(seed=3, max_evals=3000, L=4, R=8, patience=3)
    assert int(r["rounds"]) == int(ro["rounds"])
    assert int(r["evals"]) == int(ro["evals"])
    assert np.array_equal(r["best_seq"], ro["best_seq"])
    assert r["best"]["score"] == ro["best"]["score"]


def test_search_mlp_c_finds_bruteforce_optimum():
    T = _T()
    a, o = setup("mlp_c")
    _, best, bc = o.bruteforce()
    r = T.search(a, T.SearchOptions(seed=0, max_evals=20000, leaves_per_round=8, rollouts_per_leaf=32, patience=4))
    assert r["best"]["score"] == bc["score"]


def test_root_parallel_search_nccl_single_rank():
    """The multi-GPU search driver at world size 1 over NCCL — the exchange in
    device memory (toast_search_round_dev / toast_search_import_dev, SURVEY
    §8(b)) — reproduces toast_search exactly (same seed, same trajectory)."""
    import os
    import socket

    import torch.distributed as dist
    T = _T()
    from paper_2508_15010_b200 import parallel as P
    a, o = setup("gpt2")
    opts = T.SearchOptions(seed=4, max_evals=20000, leaves_per_round=8, rollouts_per_leaf=32, patience=3)
    ref = T.search(a, opts)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        trace = []
        r = P.search_root_parallel(a, opts, trace=trace)
    finally:
        dist.destroy_process_group()
    assert int(r["rounds"]) == int(ref["rounds"]) and int(r["evals"]) == int(ref["evals"])
    assert np.array_equal(r["best_seq"], ref["best_seq"]) and r["best"]["score"] == ref["best"]["score"]
    assert len(trace) == int(r["rounds"]) and trace[-1] == r["best"]["score"]


def test_eval_sharded_nccl_single_rank():
    """parallel.eval_sharded over NCCL at world size 1: the
    gathered records equal toast_eval_batch's, full and compact."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    T = _T()
    from paper_2508_15010_b200 import parallel as P
    a, o = setup("gpt2")
    seqs, oc = o.rollout(np.zeros((1000, 32), np.uint16), seed=8)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        d = torch.from_numpy(np.ascontiguousarray(seqs).view(np.int16)).cuda()
        full = P.eval_sharded(a, d)
        comp = P.eval_sharded(a, d, compact=True)
        side = torch.cuda.Stream()              # a caller's stream other than the current one
        full_side = P.eval_sharded(a, d, stream=side)
    finally:
        dist.destroy_process_group()
    assert T.as_costs(full).tobytes() == oc.tobytes()
    assert T.as_costs(full_side).tobytes() == oc.tobytes()
    sc = T.as_scores(comp)
    assert (sc["score"].view(np.uint64) == oc["score"].view(np.uint64)).all() and (sc["state_key"] == oc["state_key"]).all()


def test_random_programs_parity_including_repeated_operands():
    """Random programs (repeated operands such as mul(x, x) / matmul(x, x) take
    the per-edge path; the rest go through edge templates), two meshes, oracle
    rollouts and raw ids, compared record by record."""
    from workloads import models
    T = _T()
    n_rep = 0
    for seed in range(24):
        ir = models.random_program(seed, n_ops=18)
        n_rep += sum(1 for l in ir.splitlines() if "(" in l and len(set(x.strip() for x in l[l.index("(") + 1:l.rindex(")")].split(","))) == 1 and "," in l)
        for axes in ([("a", 2, 1e10), ("b", 4, 1e11)], [("a", 3, 1e10), ("b", 2, 2e10)]):
            try:
                o = Oracle(ir, axes, 1e12, 1 << 12, 100.0, 1, 30)
            except Exception:
                continue
            a = T.build_analysis(ir, axes, 1e12, 1 << 12, 100.0, 1, 30, cuda_device=0)
            seqs, oc = o.rollout(np.zeros((256, 32), np.uint16), seed=seed)
            assert_same(gpu_eval(a, seqs), oc, f"random {seed} {axes}")
            raw = candidates.uniform(128, o.n_actions + 1, seed=seed)
            assert_same(gpu_eval(a, raw), o.eval(raw), f"random raw {seed}")
    assert n_rep > 0   # the per-edge (repeated operand) path was exercised


@pytest.mark.parametrize("n", [1, 31, 33, 64, 200, 1000])
def test_small_batches_split_across_warps(n):
    """Batches below one wave are swept by K > 1 warps per block (segmented
    liveness scan); results must not depend on K."""
    a, o = setup("gpt24")
    seqs, oc = o.rollout(np.zeros((n, 32), np.uint16), seed=n)
    assert_same(gpu_eval(a, seqs), oc, f"n={n}")


def test_pinned_host_pipeline_matches_device_path():
    """Pinned host buffers take the chunked two-stream pipeline; results equal
    the device-resident call (and hence the oracle) record for record."""
    import torch
    T = _T()
    a, o = setup("gpt24")
    n = 2 * a.preferred_batch() + 77
    h_pre = torch.zeros((n, 32), dtype=torch.int16).pin_memory()
    h_seq = torch.empty_like(h_pre).pin_memory()
    h_out = torch.empty((n, 256), dtype=torch.uint8).pin_memory()
    T.rollout_batch(a, h_pre, 99, 5, h_seq, h_out)
    gs, gc = gpu_rollout(a, np.zeros((n, 32), np.uint16), 99, 5)
    assert np.array_equal(h_seq.numpy().view(np.uint16), gs)
    assert h_out.numpy().tobytes() == gc.tobytes()
    idx = np.random.default_rng(2).choice(n, 16, replace=False)
    for i in idx:
        s1, c1 = o.rollout(np.zeros((1, 32), np.uint16), seed=99, id_base=5 + int(i))
        assert np.array_equal(gs[i], s1[0])
        assert_same(gc[i:i + 1], c1)


# --------------------------------------------------------------------------- NEXT-2: critical path (R22)
_cp_cache = {}


def setup_cp(name):
    if name not in _cp_cache:
        T = _T()
        c = configs.get(name)
        a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0,
                             cost_model=T.COST_CRITICAL_PATH, dedup=T.DEDUP_OFF)   # the one-kernel path
        o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cost_model=1)
        _cp_cache[name] = (a, o)
    return _cp_cache[name]


@pytest.mark.parametrize("name", ["mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_1ax_np2", "gpt2_3ax", "gpt2_3ax_np2",
                                  "gpt2_4ax", "gpt2_4ax_np2", "gns16", "unet", "llama80"])
def test_critical_path_rollout_parity(name):
    """Reading R22: rollouts + evaluation under the critical-path cost model,
    bit-exact to the oracle's critical path (runtime, score and every field)."""
    a, o = setup_cp(name)
    n = 2048 if name in SMALL else 48 if name == "llama80" else 256
    pre = np.zeros((n, 32), np.uint16)
    os_, oc = o.rollout(pre, seed=9, id_base=5)
    gs, gc = gpu_rollout(a, pre, 9, 5)
    assert np.array_equal(gs, os_)
    assert_same(gc, oc, name)
    assert_same(gpu_eval(a, os_), oc, name)


def test_critical_path_full_size_sampled():
    """GPT-24 at full bench size under R22: sampled rows recomputed by the oracle."""
    a, o = setup_cp("gpt24")
    wave = a.preferred_batch()
    n = max(wave, ((1 << 18) // wave) * wave)
    gs, gc = gpu_rollout(a, np.zeros((n, 32), np.uint16), 2024, 0)
    assert (gc["status"] == 0).all()
    for i in np.random.default_rng(2).choice(n, size=12, replace=False):
        s1, c1 = o.rollout(np.zeros((1, 32), np.uint16), seed=2024, id_base=int(i))
        assert np.array_equal(gs[i], s1[0])
        assert_same(gc[i:i + 1], c1, f"row {i}")


@pytest.mark.parametrize("grouping", [0, 1])
def test_critical_path_random_programs(grouping):
    """R22 on random programs (unary chains, diamonds and repeated operands —
    the walk's aliases, never-communicating and dominated edges, in-bundle
    forwarding — and a size-3 axis), under both conflict groupings."""
    T = _T()
    from workloads import models
    ran = 0
    for seed in range(60):
        ir = models.random_program(seed, n_ops=20 + seed % 3 * 10, max_ext=8)
        axes = [("a", 2, 1e10), ("b", 3, 1e11)] if seed % 2 else [("a", 2, 1e10), ("b", 4, 1e11)]
        try:
            a = T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=0, cost_model=T.COST_CRITICAL_PATH,
                                 dedup=T.DEDUP_OFF if seed % 2 else T.DEDUP_ON,
                                 grouping=grouping)
        except T.ToastError:
            continue
        o = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cost_model=1, grouping=grouping)
        pre = np.zeros((256, 32), np.uint16)
        os_, oc = o.rollout(pre, seed=seed)
        gs, gc = gpu_rollout(a, pre, seed, 0)
        assert np.array_equal(gs, os_)
        assert_same(gc, oc, ir)
        ran += 1
    assert ran >= 30


@pytest.mark.parametrize("name", ["mlp_c", "gpt2", "gpt2_4ax_np2", "unet"])
def test_compact_scores_equal_full_records(name):
    """toast_eval_scores / toast_rollout_scores: the 16-B results are the full
    records' score and state key bit for bit (NaN | status for a bad candidate),
    on device pointers and through the pinned host-buffer pipeline."""
    import torch
    T = _T()
    a, o = setup(name)
    n = 4096 if name != "unet" else 1024
    seqs = candidates.uniform(n, o.n_actions + 2, seed=3, bad_frac=0.05)
    full = gpu_eval(a, seqs)
    d_seqs = torch.from_numpy(np.ascontiguousarray(seqs).view(np.int16)).cuda()
    d_sc = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    T.eval_scores(a, d_seqs, d_sc)
    torch.cuda.synchronize()
    sc = T.as_scores(d_sc)
    ok = full["status"] == 0
    assert ok.any() and (~ok).any()
    assert (sc["score"][ok].view(np.uint64) == full["score"][ok].view(np.uint64)).all()
    assert (sc["state_key"][ok] == full["state_key"][ok]).all()
    assert np.isnan(sc["score"][~ok]).all() and (sc["state_key"][~ok] == full["status"][~ok]).all()
    # rollouts, device and pinned host buffers (large enough for the chunked pipeline)
    m = max(2 * a.preferred_batch() + 77, 4096)
    pre = np.zeros((m, 32), np.uint16)
    gs, gc = gpu_rollout(a, pre, 21, 9)
    h_pre = torch.zeros((m, 32), dtype=torch.int16).pin_memory()
    h_seq = torch.empty_like(h_pre).pin_memory()
    h_sc = torch.empty((m, 16), dtype=torch.uint8).pin_memory()
    T.rollout_scores(a, h_pre, 21, 9, h_seq, h_sc)
    hs = T.as_scores(h_sc)
    assert np.array_equal(h_seq.numpy().view(np.uint16), gs)
    assert (hs["score"].view(np.uint64) == gc["score"].view(np.uint64)).all()
    assert (hs["state_key"] == gc["state_key"]).all()


def test_critical_path_concurrent_streams_and_host_pipeline():
    """R22's per-launch finish-slot scratch: the pinned host-buffer pipeline
    (chunks on several streams) and two calls racing on two streams give the
    device path's records bit for bit."""
    import torch
    T = _T()
    a, o = setup_cp("gpt2")
    m = 3 * a.preferred_batch() + 123
    pre = np.zeros((m, 32), np.uint16)
    gs, gc = gpu_rollout(a, pre, 31, 0)
    h_pre = torch.zeros((m, 32), dtype=torch.int16).pin_memory()
    h_seq = torch.empty_like(h_pre).pin_memory()
    h_out = torch.empty((m, 256), dtype=torch.uint8).pin_memory()
    T.rollout_batch(a, h_pre, 31, 0, h_seq, h_out)
    assert np.array_equal(h_seq.numpy().view(np.uint16), gs)
    assert T.as_costs(h_out).tobytes() == gc.tobytes()
    d_seqs = torch.from_numpy(np.ascontiguousarray(gs).view(np.int16)).cuda()
    outs = [torch.empty((m, 256), dtype=torch.uint8, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for rep in range(3):
        for s, out in zip(streams, outs):
            T.eval_batch(a, d_seqs, out, stream=s)
    torch.cuda.synchronize()
    for out in outs:
        assert T.as_costs(out).tobytes() == gc.tobytes()
    # sampled rows against the oracle
    for i in np.random.default_rng(5).choice(m, size=16, replace=False):
        s1, c1 = o.rollout(np.zeros((1, 32), np.uint16), seed=31, id_base=int(i))
        assert np.array_equal(gs[i], s1[0])
        assert_same(gc[i:i + 1], c1, f"row {i}")


@pytest.mark.parametrize("name", ["gpt2", "unet", "gpt2_4ax_np2"])
def test_results_independent_of_k_and_residency(name):
    """The measured K and residency (TOAST_FORCE_K / TOAST_FORCE_BLOCKS pin them)
    change only the schedule: rollouts and records are bit-identical."""
    import os
    T = _T()
    c = configs.get(name)
    a0, _o = setup(name)
    n = 3 * a0.preferred_batch() + 17
    pre = np.zeros((n, 32), np.uint16)
    s0, c0 = gpu_rollout(a0, pre, 13, 4)
    for K, B in ((1, 3), (2, 5), (4, 2), (8, 1)):
        os.environ["TOAST_FORCE_K"], os.environ["TOAST_FORCE_BLOCKS"] = str(K), str(B)
        try:
            a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth,
                                 cuda_device=0)
        finally:
            del os.environ["TOAST_FORCE_K"], os.environ["TOAST_FORCE_BLOCKS"]
        assert a.kernel_tables()["warps_per_batch"] == K
        s1, c1 = gpu_rollout(a, pre, 13, 4)
        assert np.array_equal(s1, s0) and c1.tobytes() == c0.tobytes(), (K, B)


def test_cli_partitions_a_program(tmp_path, capsys):
    """python -m paper_2508_15010_b200: search on cuda:0, then the best state's
    record and lowered program; on MLP-c the best equals the oracle's
    exhaustive optimum (C17)."""
    from paper_2508_15010_b200.__main__ import main
    a, o = setup("mlp_c")
    _, _best, bc = o.bruteforce()
    c = configs.get("mlp_c")
    f = tmp_path / "mlp_c.ir"
    f.write_text(c.ir)
    mesh = ",".join(f"{n}={s}:{bw!r}" for n, s, bw in c.axes)
    assert main(["--ir", str(f), "--mesh", mesh, "--flops", repr(c.flops_per_sec), "--dm", str(c.dm),
                 "--min-dims", str(c.min_dims), "--budget", "20000"]) == 0
    out = capsys.readouterr().out
    assert f"best score {float(bc['score']):.6g}" in out
    assert "return" in out and "mesh" in out
    assert main(["--config", "gpt2", "--cost-model", "cp", "--grouping", "contraction", "--budget", "20000",
                 "--no-program"]) == 0
    assert main(["--ir", str(f), "--mesh", mesh, "--flops", repr(c.flops_per_sec), "--dm", str(c.dm),
                 "--min-dims", str(c.min_dims), "--budget", "20000", "--dedup", "--transpositions"]) == 0
    assert f"best score {float(bc['score']):.6g}" in capsys.readouterr().out


def test_search_device_exchange_refuses_host_buffers():
    """toast_search_round_dev / toast_search_import_dev take device memory only
    (TOAST_E_INVALID_ARG for a host buffer), and a device round's record equals
    the host round's of the same search state."""
    import torch
    T = _T()
    a, _ = setup("gpt2")
    opts = T.SearchOptions(seed=2, max_evals=5000, leaves_per_round=4, rollouts_per_leaf=8)
    st_h, st_d = T.SearchState(a, opts, 0, 1), T.SearchState(a, opts, 0, 1)
    with pytest.raises(T.ToastError) as e:
        st_d.round_dev(np.zeros(st_d.export_bytes, np.uint8))
    assert e.value.code == "TOAST_E_INVALID_ARG"
    rec_h = st_h.round()
    dev = torch.empty(st_d.export_bytes, dtype=torch.uint8, device="cuda")
    st_d.round_dev(dev)
    rec_d = dev.cpu().numpy()
    hdr = 8 + 8 + 64 + 8   # best score, key, sequence, evals (elapsed_s and after differ by the clock)
    assert rec_h[:hdr].tobytes() == rec_d[:hdr].tobytes()
    assert rec_h[hdr + 8 + 8:].tobytes() == rec_d[hdr + 8 + 8:].tobytes()
    assert st_h.import_(rec_h) == st_d.import_dev(dev)
    st_h.end()
    st_d.end()


@pytest.mark.parametrize("cost_model", [0, 1])
@pytest.mark.parametrize("variant", sorted(VARIANT_CONFIG))
def test_every_kernel_instantiation_matches_the_oracle(variant, cost_model):
    """Each of the 32 kernels (toast_eval_kernel / toast_rollout_kernel x mesh
    axes 1-4 x power-of-two or not x sum / critical-path model) is the one the
    analysis dispatches (its kernel_variant) and is bit-exact to the oracle on
    rollouts from the root and from prefixes and on their re-evaluation."""
    name = VARIANT_CONFIG[variant]
    a, o = setup_cp(name) if cost_model else setup(name)
    assert a.kernel_tables()["kernel_variant"] == [variant[0], variant[1], cost_model]
    n = 1000
    pre = np.zeros((n, 32), np.uint16)
    s0, _ = o.rollout(np.zeros((n // 2, 32), np.uint16), seed=31)
    for i in range(n // 2):
        pre[i, :i % 3] = s0[i, :i % 3]
    os_, oc = o.rollout(pre, seed=8, id_base=1 << 40, threads=8)
    gs, gc = gpu_rollout(a, pre, 8, 1 << 40)
    assert np.array_equal(gs, os_)
    assert_same(gc, oc, (name, cost_model))
    assert_same(gpu_eval(a, os_), oc, (name, cost_model))


def test_llama80_worst_case_and_sampled_critical_path():
    """Llama-80 (the 3-axis BASELINE config) under the critical-path model:
    maximal-length sequences evaluated, and a bench-sized launch sampled."""
    a, o = setup_cp("llama80")
    seqs = _legal_long(o, 24, seed=5)
    assert_same(gpu_eval(a, seqs), o.eval(seqs, threads=8), "llama80 cp worst case")
    n = 32 * 148 * 4
    gs, gc = gpu_rollout(a, np.zeros((n, 32), np.uint16), 77, 0)
    for i in np.random.default_rng(4).choice(n, size=24, replace=False):
        s1, c1 = o.rollout(np.zeros((1, 32), np.uint16), seed=77, id_base=int(i))
        assert np.array_equal(gs[i], s1[0])
        assert_same(gc[i:i + 1], c1, f"row {i}")


def test_checked_library_race_and_bounds():
    """Race / bounds evidence without compute-sanitizer (closed on this pool):
    the checked library (kernels.cu TOAST_CHECKED, built by build()) traps on
    any out-of-bounds shared-memory access or table index, poisons every
    shared-memory region as soon as it dies (the sequence staging after
    decode, the event bitmaps after H2a, the class maps under the
    accumulators, the record staging, everything between batches) and sleeps
    pseudo-random times per warp at every barrier and per lane at every
    cross-lane exchange.  scripts/sanitize.py runs every kernel instantiation
    (1-4 mesh axes, power of two or not, sum and critical-path models) at
    K = 1, 2, 4 and 8 warps per batch on a ragged batch through it: all
    bit-identical to the oracle."""
    import os
    import subprocess
    import sys
    from paper_2508_15010_b200 import build as B
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    assert os.path.exists(B.LIB_CHECKED), "build() builds the checked library"
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "sanitize.py")], capture_output=True, text=True,
                       env=dict(os.environ, TOAST_LIB=B.LIB_CHECKED), timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "all bit-identical to the oracle" in r.stdout
    assert r.stdout.count(": ok") == 8 * 2 * 4 + 8 * 2


def test_checked_library_catches_a_planted_race():
    """The checker is not vacuous: the same library with the barrier between
    warp 0's decode and the other warps' reads of its results removed
    (TOAST_CHK_MUTANT) fails the K > 1 runs of scripts/sanitize.py."""
    import os
    import subprocess
    import sys
    from paper_2508_15010_b200 import build as B
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    assert os.path.exists(B.LIB_MUTANT), "build() builds the mutant library"
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "sanitize.py"), "gpt2", "gpt2_3ax"],
                       capture_output=True, text=True, env=dict(os.environ, TOAST_LIB=B.LIB_MUTANT), timeout=900)
    assert r.returncode != 0, r.stdout[-2000:]
    assert "gpt2 cost_model=0 K=1: ok" in r.stdout          # one-warp blocks never needed that barrier
    assert "gpt2 cost_model=0 K=2: ok" not in r.stdout      # the first multi-warp run is caught


_dd_cache = {}


def setup_dedup(name, cost_model=0):
    key = (name, cost_model)
    if key not in _dd_cache:
        T = _T()
        c = configs.get(name)
        a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0,
                             cost_model=cost_model, dedup=1)
        o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cost_model=cost_model)
        _dd_cache[key] = (a, o)
    return _dd_cache[key]


@pytest.mark.parametrize("cost_model", [0, 1])
@pytest.mark.parametrize("name", ["mlp_c", "gpt2", "gpt2_np2", "gpt2_3ax", "gpt2_3ax_np2", "gpt2_4ax_np2", "gpt2_1ax_np2",
                                  "unet", "gns16"])
def test_dedup_rollouts_bit_identical(name, cost_model):
    """NEXT-3: with dedup on, a rollout launch costs each distinct
    materialised state once and copies its record to every candidate that
    reached it — sequences and records bit-identical to the oracle's, with
    prefixes, a bad prefix (its error record) and a ragged tail, full and
    compact records, device and pinned-host buffers."""
    import torch
    T = _T()
    a, o = setup_dedup(name, cost_model)
    n = 3001 if name not in ("unet", "gns16") else 601
    pre = np.zeros((n, 32), np.uint16)
    s0, _ = o.rollout(np.zeros((n // 2, 32), np.uint16), seed=41)
    for i in range(n // 2):
        pre[i, :i % 3] = s0[i, :i % 3]
    pre[7, 0] = 60000                     # a bad id: the error record
    os_, oc = o.rollout(pre, seed=12, id_base=99, threads=8)
    gs, gc = gpu_rollout(a, pre, 12, 99)
    assert np.array_equal(gs, os_)
    assert_same(gc, oc, (name, cost_model, "dedup"))
    assert len(np.unique(oc["state_key"][oc["status"] == 0])) < n   # there were duplicates to share
    # compact records through the pinned host pipeline
    h_pre = torch.from_numpy(pre.view(np.int16)).pin_memory()
    h_seq = torch.empty_like(h_pre).pin_memory()
    h_sc = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
    T.rollout_scores(a, h_pre, 12, 99, h_seq, h_sc)
    sc = T.as_scores(h_sc)
    ok = oc["status"] == 0
    assert np.array_equal(h_seq.numpy().view(np.uint16), os_)
    assert (sc["score"][ok].view(np.uint64) == oc["score"][ok].view(np.uint64)).all()
    assert (sc["state_key"][ok] == oc["state_key"][ok]).all()
    assert np.isnan(sc["score"][~ok]).all() and (sc["state_key"][~ok] == oc["status"][~ok]).all()


def test_dedup_full_size_and_search():
    """GPT-24 at the bench's launch size with dedup: sampled rows equal the
    oracle's, every row equals the one-kernel path's; a search with dedup on
    follows the same trajectory as without (same evals, rounds, best)."""
    T = _T()
    a, o = setup_dedup("gpt24")
    a1, _ = setup("gpt24")
    wave = a1.preferred_batch()
    n = max(wave, ((1 << 18) // wave) * wave)
    gs, gc = gpu_rollout(a, np.zeros((n, 32), np.uint16), 2024, 0)
    gs1, gc1 = gpu_rollout(a1, np.zeros((n, 32), np.uint16), 2024, 0)
    assert np.array_equal(gs, gs1) and gc.tobytes() == gc1.tobytes()
    for i in np.random.default_rng(3).choice(n, size=16, replace=False):
        s1, c1 = o.rollout(np.zeros((1, 32), np.uint16), seed=2024, id_base=int(i))
        assert np.array_equal(gs[i], s1[0])
        assert_same(gc[i:i + 1], c1, f"row {i}")
    opts = T.SearchOptions(seed=1, max_evals=200000, leaves_per_round=16, rollouts_per_leaf=64, patience=3)
    r, r1 = T.search(a, opts), T.search(a1, opts)
    assert int(r["evals"]) == int(r1["evals"]) and int(r["rounds"]) == int(r1["rounds"])
    assert r["best"].tobytes() == r1["best"].tobytes() and np.array_equal(r["best_seq"], r1["best_seq"])


def _root_parallel_worker(rank, world, port, out_dir):
    import json
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_15010_b200 import parallel as P
        from paper_2508_15010_b200 import toast as T
        import torch
        torch.cuda.set_device(0)
        c = configs.get("gpt2")
        a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0)
        opts = T.SearchOptions(seed=11, max_evals=60000, leaves_per_round=8, rollouts_per_leaf=32, patience=4)
        st = T.SearchState(a, opts, rank, world)
        own = None
        rounds = 0
        while True:                        # the library's own rounds, exchanged over gloo
            rec = st.round()
            own = rec.copy()
            stop = st.import_(P.all_gather_bytes(rec))
            rounds += 1
            if stop:
                break
        summed = st.root_stats()
        res = st.end()
        hdr = P.EXPORT_DTYPE.itemsize
        own_root = own[hdr:].view(T.ROOT_STAT_DTYPE)
        json.dump({"best_seq": [int(x) for x in res["best_seq"]], "score": float(res["best"]["score"]),
                   "best_bytes": res["best"].tobytes().hex(), "evals": int(res["evals"]), "rounds": rounds,
                   "summed_visits": summed["visits"].tolist(), "summed_values": summed["value_sum"].tolist(),
                   "own_visits": own_root["visits"].tolist(), "own_values": own_root["value_sum"].tolist()},
                  open(os.path.join(out_dir, f"rank{rank}.json"), "w"))
    finally:
        dist.destroy_process_group()


def test_root_parallel_search_two_ranks_library_rounds(tmp_path):
    """Root-parallel search ("many trajectories in
    parallel") with the library's own rounds on two ranks (two processes on
    cuda:0, gloo between them; the ranks' kernels never wait on each other):
    every rank ends with the same global best, the root statistics every rank
    reports are the sum of the ranks' own, and the best is the oracle's score
    for its sequence."""
    import json
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_root_parallel_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r = [json.load(open(tmp_path / f"rank{k}.json")) for k in range(2)]
    assert r[0]["best_seq"] == r[1]["best_seq"] and r[0]["best_bytes"] == r[1]["best_bytes"]
    assert r[0]["evals"] == r[1]["evals"] and r[0]["rounds"] == r[1]["rounds"]
    assert r[0]["summed_visits"] == r[1]["summed_visits"]
    assert r[0]["summed_visits"] == [x + y for x, y in zip(r[0]["own_visits"], r[1]["own_visits"])]
    assert r[0]["summed_values"] == [x + y for x, y in zip(r[0]["own_values"], r[1]["own_values"])]
    assert r[0]["own_values"] != r[1]["own_values"]          # the ranks' rollouts differ (seed + rank)
    _, o = setup("gpt2")
    c = o.eval(np.array([r[0]["best_seq"]], np.uint16))[0]
    assert c["status"] == 0 and float(c["score"]) == r[0]["score"]
