"""NEXT-1: toast_lower emits the device-local program of a
sequence; the sharded interpreter (tests/sharded_interp.py) runs it on every
device of the mesh and checks that it computes the unsharded program, that
every layout change is the one its collective performs, and that the payload
each collective declares is the ring model's.  The lowered collectives, per
(axis, kind), must also total the cost record the oracle computes (C11) — so
the cost model's collective choice is pinned to a program that provably
computes the right values, not only to the paper's examples.  CPU only."""
import os
import re

import numpy as np
import pytest

from oracle.oracle import Oracle
from workloads import models
import sharded_interp as SI

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KINDS = ["all_gather", "reduce_scatter", "all_reduce", "all_to_all"]   # toast_cost.payload order


def _T():
    from paper_2508_15010_b200 import toast as T
    return T


def golden(name):
    return open(os.path.join(GOLD, name)).read()


def action_id(d, loop, r, axis):
    sc = d["loops"][loop][5]
    for i, a in enumerate(d["actions"]):
        if a == [sc, r, axis]:
            return i + 1
    raise KeyError((loop, r, axis))


def _check_program(ir, axes, seqs, costs, inputs, F=1e12):
    T = _T()
    a = T.build_analysis(ir, axes, F, 1 << 40, 100.0, 1, 30, cuda_device=-1)
    for s, c in zip(seqs, costs):
        lst = [int(x) for x in s if x]
        low = T.lower(a, lst)
        pay = SI.run_lowered(low, ir, inputs)
        counts = {}
        for kind in KINDS:
            for m in re.finditer(r"= " + kind + r"\{axis=(\d+)", low):
                counts[(int(m.group(1)), kind)] = counts.get((int(m.group(1)), kind), 0) + 1
        for A in range(len(axes)):
            for k, kind in enumerate(KINDS):
                assert pay.get((A, kind), 0) == int(c["payload"][A][k]), (lst, A, kind, low)
                assert counts.get((A, kind), 0) == int(c["count"][A][k]), (lst, A, kind, low)
        assert sum(counts.values()) == int(c["n_collectives"])


def _deep(o, n, seed):
    """n random legal sequences extended until no action is legal (the most-sharded states)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        seq = []
        for _d in range(30):
            nxt = None
            for x in rng.permutation(np.arange(1, o.n_actions)):
                s = np.zeros((1, 32), np.uint16)
                s[0, :len(seq) + 1] = seq + [int(x)]
                if int(o.eval(s)[0]["status"]) == 0:
                    nxt = int(x)
                    break
            if nxt is None:
                break
            seq.append(nxt)
        out.append(np.array(seq + [0] * (32 - len(seq)), np.uint16))
    return out


def test_fig2c_lowered_program():
    """Fig. 2c: B->b, U->m lowers to x[256{b},32], w1[32,64{m}],
    w2[64{m},16] and exactly one all_reduce{m} of the partial w, 8,192 B
    (S:386), and the program computes the unsharded mlp."""
    T = _T()
    ir = golden("mlp_fig2.ir")
    axes = [("b", 2, 1e10), ("m", 2, 1e11)]
    a = T.build_analysis(ir, axes, 1e9, 1 << 40, 100.0, 1, 30, cuda_device=-1)
    d = a.dump()
    low = T.lower(a, [action_id(d, 0, 0, 0), action_id(d, 3, 0, 1)])
    lines = [l for l in low.splitlines() if l.startswith("%")]
    assert "local[128,32] layout[1,0]" in lines[0]            # x: [256{b}, 32]
    assert "local[32,32] layout[0,2]" in lines[1]             # w1: [32, 64{m}]
    assert "local[32,16] layout[2,0]" in lines[2]             # w2: [64{m}, 16]
    colls = [l for l in lines if re.search(r"= (all_gather|all_to_all|reduce_scatter|all_reduce|slice)\{", l)]
    assert len(colls) == 1 and colls[0].startswith("%w.1 = all_reduce{axis=1}(%w)") and colls[0].endswith("bytes=8192")
    assert "partial[2]" in [l for l in lines if l.startswith("%w = matmul")][0]
    assert low.strip().endswith("return %w.1")
    SI.run_lowered(low, ir, SI.random_inputs(ir, 0))


def test_fig5b_lowered_sequence_resolution():
    """Fig. 5b: sharding S on the sequence resolution lowers to an
    all_gather{s} of k and a reduce_scatter{s} of the partial z, 64 B each."""
    T = _T()
    ir = golden("attn_fig5.ir")
    axes = [("s", 2, 1e10)]
    a = T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=-1)
    o = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1)
    d = a.dump()
    found = False
    for r in (0, 1):
        seq = [action_id(d, 0, r, 0)]
        low = T.lower(a, seq)
        SI.run_lowered(low, ir, SI.random_inputs(ir, r))
        colls = re.findall(r"= (all_gather|all_to_all|reduce_scatter|all_reduce)\{[^}]*\}\((%[\w.]+)\).* bytes=(\d+)", low)
        if any(c[0] == "reduce_scatter" for c in colls):
            assert sorted(colls) == [("all_gather", "%k", "64"), ("reduce_scatter", "%z", "64")]
            found = True
        c = o.eval(Oracle.seqs([seq]))[0]
        assert sum(int(b) for _, _, b in colls) == int(c["payload"].sum())
    assert found


GOLDENS = [("mlp_fig2.ir", 1e9), ("mlp_c.ir", 1e12), ("attn_fig5.ir", 1e12), ("g_matmul_add.ir", 1e12),
           ("f_transpose.ir", 1e12)]
MESHES = [[("a", 2, 1e10), ("b", 2, 1e11)], [("a", 2, 1e10), ("b", 4, 1e11)], [("a", 4, 1e10)]]


@pytest.mark.parametrize("name,F", GOLDENS)
@pytest.mark.parametrize("mesh", range(len(MESHES)))
def test_lowered_goldens_compute_the_unsharded_program(name, F, mesh):
    ir = golden(name)
    axes = MESHES[mesh]
    o = Oracle(ir, axes, F, 1 << 40, 100.0, 1)
    seqs, costs = o.rollout(np.zeros((60, 32), np.uint16), seed=mesh)
    deep = _deep(o, 10, seed=mesh)
    seqs = list(seqs) + deep
    costs = list(costs) + list(o.eval(np.stack(deep)))
    _check_program(ir, axes, seqs, costs, SI.random_inputs(ir, mesh), F)


def test_lowered_random_programs_compute_the_unsharded_program():
    """40 random programs (repeated operands included) on a 2x4 mesh."""
    T = _T()
    ran = 0
    for seed in range(40):
        ir = models.random_program(seed, n_ops=16)
        axes = [("a", 2, 1e10), ("b", 4, 1e11)]
        try:
            T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=-1)
        except T.ToastError as e:   # documented limits, or a program without a contraction (TOAST_E_DEGENERATE)
            assert "LIMIT" in str(e) or "DEGENERATE" in str(e)
            continue
        o = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1)
        seqs, costs = o.rollout(np.zeros((20, 32), np.uint16), seed=seed)
        deep = _deep(o, 3, seed=seed)
        with np.errstate(over="ignore", invalid="ignore"):
            _check_program(ir, axes, list(seqs) + deep, list(costs) + list(o.eval(np.stack(deep))),
                           SI.random_inputs(ir, seed))
        ran += 1
    assert ran >= 30


def test_interpreter_rejects_a_wrong_program():
    """The interpreter is not vacuous: dropping the all_reduce of Fig. 2c, or
    mislabelling its payload, is caught."""
    T = _T()
    ir = golden("mlp_fig2.ir")
    axes = [("b", 2, 1e10), ("m", 2, 1e11)]
    a = T.build_analysis(ir, axes, 1e9, 1 << 40, 100.0, 1, 30, cuda_device=-1)
    d = a.dump()
    low = T.lower(a, [action_id(d, 0, 0, 0), action_id(d, 3, 0, 1)])
    inp = SI.random_inputs(ir, 0)
    no_ar = "\n".join(l for l in low.splitlines() if "all_reduce" not in l).replace("return %w.1", "return %w")
    with pytest.raises(SI.ShardError):
        SI.run_lowered(no_ar, ir, inp)
    with pytest.raises(SI.ShardError):
        SI.run_lowered(low.replace("bytes=8192", "bytes=4096"), ir, inp)
    # a layout the op does not produce
    with pytest.raises(SI.ShardError):
        SI.run_lowered(low.replace("%z = relu(%y) f32 [256,64] local[128,32] layout[1,2]",
                                   "%z = relu(%y) f32 [256,64] local[128,64] layout[1,0]"), ir, inp)
