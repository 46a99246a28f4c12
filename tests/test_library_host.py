"""CPU-side checks of libtoast: the C ABI loads and exports every symbol
include/toast.h declares, the H0 analysis equals the oracle's exactly, the
host-side materialisation agrees, and errors come back as status codes."""
import os
import re

import numpy as np
import pytest

from oracle.oracle import Oracle
from workloads import configs, models

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2508_15010_b200 import toast as T
    return T


def test_exports_every_header_symbol():
    T = _lib()
    hdr = open(os.path.join(ROOT, "include", "toast.h")).read()
    declared = set(re.findall(r"^(?:toast_status|size_t|const char\*|void)\s+(toast_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 18
    import ctypes
    lib = ctypes.CDLL(T.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(T.EXPORTED)


def _both(name):
    T = _lib()
    c = configs.get(name)
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=-1)
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth)
    return a, o, c


@pytest.mark.parametrize("name", ["mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_4ax", "gpt2_4ax_np2", "gpt24", "gns16",
                                  "unet"])
def test_h0_analysis_equals_oracle(name):
    """H0 parity: loop table, components, super-colors, conflicts, sets, sides,
    WL signatures, groups, action table and baseline are identical."""
    a, o, _ = _both(name)
    da, do = a.dump(), o.dump()
    assert da.keys() == do.keys()
    for k in do:
        assert da[k] == do[k], k


@pytest.mark.slow
def test_h0_analysis_equals_oracle_llama80():
    a, o, _ = _both("llama80")
    assert a.dump() == o.dump()


def test_h0_random_programs():
    T = _lib()
    for seed in range(30):
        ir = models.random_program(seed, n_ops=16)
        axes = [("a", 2, 1e10), ("b", 4, 1e11)]
        a = T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=-1)
        o = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1, 30)
        assert a.dump() == o.dump(), ir


@pytest.mark.parametrize("name", ["mlp_c", "gpt2", "unet"])
def test_host_materialize_equals_oracle(name):
    T = _lib()
    a, o, _ = _both(name)
    seqs, _c = o.rollout(np.zeros((200, 32), np.uint16), seed=5)
    for s in seqs:
        lst = [int(x) for x in s if x]
        assert np.array_equal(T.materialize(a, lst), o.materialize(lst))


def test_baseline_record_equals_oracle_empty_eval():
    T = _lib()
    for name in ("mlp_c", "gpt2", "gns16"):
        a, o, _ = _both(name)
        b = a.baseline()
        e = o.eval(np.zeros((1, 32), np.uint16))[0]
        for f in ("runtime_s", "score", "peak_bytes", "flops", "flops_hi", "state_key", "status", "n_collectives"):
            assert b[f] == e[f], f


@pytest.mark.parametrize("src,code", [
    ("def f(x: f32[2,3], y: f32[4,5]) {\n  z = matmul(x, y)\n  return z\n}\n", "TOAST_E_SHAPE"),
    ("def f(x: f32[2,2]) {\n  z = matmul(x, q)\n  return z\n}\n", "TOAST_E_UNDEFINED"),
    ("def f(x: f32[2,2]) {\n  z = matmul(x, x)\n  z = matmul(x, x)\n  return z\n}\n", "TOAST_E_DUPLICATE"),
    ("def f(x: f32[2,2]) {\n  z = matmul(x x)\n  return z\n}\n", "TOAST_E_PARSE"),
    ("def f(x: f32[2,2]) {\n  z = frobnicate(x)\n  return z\n}\n", "TOAST_E_PARSE"),
])
def test_parse_errors(src, code):
    T = _lib()
    with pytest.raises(T.ToastError) as e:
        T.load_graph(src, [("a", 2, 1e10)], 1e12, 1 << 40, cuda_device=-1)
    assert e.value.code == code


def test_parse_error_location_and_binding_name():
    T = _lib()
    with pytest.raises(T.ToastError) as e:
        T.load_graph("def f(x: f32[2,2]) {\n  z = matmul(x x)\n  return z\n}\n", [("a", 2, 1e10)], 1e12, 1, cuda_device=-1)
    assert "2:" in str(e.value)
    with pytest.raises(T.ToastError) as e:
        T.load_graph("def f(x: f32[2,3], y: f32[4,5]) {\n  zz = matmul(x, y)\n  return zz\n}\n", [("a", 2, 1e10)], 1e12, 1,
                     cuda_device=-1)
    assert "'zz'" in str(e.value)


def test_mesh_machine_degenerate_limit_errors():
    T = _lib()
    ir = open(os.path.join(ROOT, "tests", "golden", "mlp_c.ir")).read()
    for axes in ([("a", 1, 1e10)], [("a", 2, 1e10), ("a", 2, 1e10)], [("a", 2, 0.0)], [("a", 2, 1.0)] * 0,
                 [(f"a{i}", 2, 1.0) for i in range(5)]):
        with pytest.raises(T.ToastError) as e:
            T.load_graph(ir, axes, 1e12, 1, cuda_device=-1)
        assert e.value.code == "TOAST_E_MESH"
    with pytest.raises(T.ToastError) as e:
        T.load_graph(ir, [("a", 2, 1e10)], 0.0, 1, cuda_device=-1)
    assert e.value.code == "TOAST_E_MACHINE"
    g = T.load_graph("def id(x: f32[4,8]) {\n  y = relu(x)\n  return y\n}\n", [("a", 2, 1e10)], 1e12, 1, cuda_device=-1)
    with pytest.raises(T.ToastError) as e:
        T.nda(g, 1, 30)
    assert e.value.code == "TOAST_E_DEGENERATE"
    g = T.load_graph(ir, [("a", 2, 1e10)], 1e12, 1, cuda_device=-1)
    with pytest.raises(T.ToastError) as e:
        T.nda(g, 1, 33)
    assert e.value.code == "TOAST_E_INVALID_ARG"


def test_no_cpu_fallback_without_device():
    """A host-only analysis refuses to evaluate: there is no CPU path."""
    T = _lib()
    a, _, _ = _both("mlp_c")
    seqs = np.zeros((4, 32), np.uint16)
    out = np.zeros(4, dtype=T.COST_DTYPE)
    with pytest.raises(T.ToastError) as e:
        T.eval_batch(a, seqs, out)
    assert e.value.code == "TOAST_E_CUDA"
    sc = np.zeros(4, dtype=T.SCORE_DTYPE)
    outs = np.zeros((4, 32), np.uint16)
    for call in (lambda: T.eval_scores(a, seqs, sc), lambda: T.rollout_scores(a, seqs, 1, 0, outs, sc),
                 lambda: T.rollout_batch(a, seqs, 1, 0, outs, out)):
        with pytest.raises(T.ToastError) as e:
            call()
        assert e.value.code == "TOAST_E_CUDA"


@pytest.mark.parametrize("name", ["mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_4ax_np2", "gns16"])
def test_peak_frontier_holds_the_peak(name):
    """Reading R19: the library's peak-memory frontier (the ops H0 keeps after
    dropping every op another op dominates over the whole weight box) contains
    an op attaining the oracle's peak, for every candidate.  The oracle's
    per-op liveness profile M_t (C12) is the plain definition; the
    frontier comes from the library's own H0 tables."""
    a, o, c = _both(name)
    kt = a.kernel_tables()
    front = np.array(kt["frontier_ops"], dtype=np.int64)
    assert len(front) >= 1 and kt["n_points"] == len(front)
    assert len(front) < a.dump()["n_ops"] or a.dump()["n_ops"] <= 8
    small = a.dump()["n_ops"] < 100
    seqs, costs = o.rollout(np.zeros((300 if small else 100, 32), np.uint16), seed=11, id_base=0)
    # plus sequences of the maximum depth (stop disabled): the most-sharded states
    deep = _deep_sequences(o, 100 if small else 12, seed=5)
    for seq in list(seqs) + deep:
        prof = o.profile(seq)
        assert prof.max() == prof[front].max(), (name, list(seq))


def _deep_sequences(o, n, seed):
    """n random legal sequences that keep adding actions until none is legal."""
    rng = np.random.default_rng(seed)
    out = []
    na = o.n_actions
    for _ in range(n):
        seq = []
        for _d in range(30):
            cand = [x for x in rng.permutation(np.arange(1, na)) if _legal(o, seq, int(x))]
            if not cand:
                break
            seq.append(int(cand[0]))
        out.append(np.array(seq + [0] * (32 - len(seq)), np.uint16))
    return out


def _legal(o, seq, x):
    s = np.zeros((1, 32), np.uint16)
    s[0, :len(seq) + 1] = seq + [x]
    return int(o.eval(s)[0]["status"]) == 0


def test_peak_frontier_random_programs():
    """R19 on random programs (repeated operands included, so some frontier
    points carry special edges), with a non-power-of-two mesh axis."""
    T = _lib()
    ran = 0
    for seed in range(40):
        ir = models.random_program(seed, n_ops=24, max_ext=12)
        axes = [("a", 2, 1e10), ("b", 3, 1e11)] if seed % 2 else [("a", 2, 1e10), ("b", 4, 1e11)]
        try:
            a = T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=-1)
        except T.ToastError as e:   # a documented TOAST_E_LIMIT (e.g. > 8 SetGroups in one super-color)
            assert "LIMIT" in str(e)
            continue
        ran += 1
        o = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1, 30)
        front = np.array(a.kernel_tables()["frontier_ops"], dtype=np.int64)
        seqs, _c = o.rollout(np.zeros((60, 32), np.uint16), seed=seed)
        for seq in list(seqs) + _deep_sequences(o, 10, seed=seed):
            prof = o.profile(seq)
            assert prof.max() == prof[front].max(), (ir, list(seq))
    assert ran >= 30


def test_lower_and_materialize_refuse_invalid_sequences():
    """toast_lower / toast_materialize run the decode checks of C9 (the kernels'
    H1): a repeated (super-color, axis), a resolution that disagrees with a
    fixed SetGroup bit, a nonzero id after STOP or a bad id is refused with
    TOAST_E_INVALID_ARG — exactly when the oracle flags the sequence — and a
    color repeated five times returns at once (it used to hang)."""
    import ctypes
    from workloads import candidates
    T = _lib()
    a, o, _ = _both("mlp_c")
    for bad in ([1, 1], [3, 6], [1, 0, 2], [1, 1, 1, 1, 1], [999]):
        s = np.zeros((1, 32), np.uint16)
        s[0, :len(bad)] = bad
        assert int(o.eval(s)[0]["status"]) != 0, bad
        for f in (T.lower, T.materialize):
            with pytest.raises(T.ToastError) as e:
                f(a, bad)
            assert e.value.code == "TOAST_E_INVALID_ARG"
    seqs = candidates.uniform(400, o.n_actions + 1, seed=11, bad_frac=0.1)
    st = o.eval(seqs)["status"]
    assert (st != 0).sum() > 50 and (st == 0).sum() > 20
    for s, bits in zip(seqs, st):
        n = ctypes.c_size_t()
        rc = T._lib.toast_lower(a.handle, np.ascontiguousarray(s).ctypes.data, None, 0, ctypes.byref(n))
        assert (rc != 0) == (bits != 0), (s, bits)


def test_nda_dedup_option_values():
    """toast_nda_opts.dedup: 0 off, 1 on, 2 auto (on under the critical-path
    model); anything else is TOAST_E_INVALID_ARG."""
    T = _lib()
    c = configs.get("mlp_c")
    for d in (0, 1, 2):
        T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=-1,
                         dedup=d)
    for d in (-1, 3):
        with pytest.raises(T.ToastError) as e:
            T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth,
                             cuda_device=-1, dedup=d)
        assert e.value.code == "TOAST_E_INVALID_ARG"
