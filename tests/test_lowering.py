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


def count_collectives(low):
    """{(axis, kind): number of collectives} over the lowered program (an
    all_to_all listing several moves counts once per moved axis)"""
    counts = {}
    for m in re.finditer(r"= (" + "|".join(KINDS) + r")((?:\+?\{[^}]*\})+)\(", low):
        for ax in re.findall(r"\{axis=(\d+)", m.group(2)):
            counts[(int(ax), m.group(1))] = counts.get((int(ax), m.group(1)), 0) + 1
    return counts


def _check_program(ir, axes, seqs, costs, inputs, F=1e12):
    T = _T()
    a = T.build_analysis(ir, axes, F, 1 << 40, 100.0, 1, 30, cuda_device=-1)
    for s, c in zip(seqs, costs):
        lst = [int(x) for x in s if x]
        low = T.lower(a, lst)
        pay = SI.run_lowered(low, ir, inputs)
        counts = count_collectives(low)
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


# ---------------------------------------------------------------------------
# The extension ops (SURVEY §8(c) C1 rows beyond Fig. 3: dot_general, conv2d
# and its backward ops, resample, concat, slice, pad, gather, segment_sum) —
# "populated ahead of time for every op in our array IR, analogously to
# PartIR/Shardy"; dot_general / convolution are the matmul-class
# ops.  Their loop rules are pinned here by what the lowered program
# computes, not by a restated table.
# ---------------------------------------------------------------------------
EXT_KINDS = ("dot_general", "conv2d", "conv2d_bwd_input", "conv2d_bwd_filter", "resample", "concat", "slice", "pad",
             "gather", "segment_sum")
EXT_MESHES = [[("a", 2, 1e10), ("b", 4, 1e11)], [("a", 2, 1e10), ("b", 2, 1e10), ("c", 2, 1e11)],
              [("a", 2, 1e10), ("b", 3, 1e10), ("c", 2, 1e11)]]


def _check_ext(ir, axes, n_roll, n_deep, seed, stats):
    T = _T()
    try:
        a = T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=-1)
    except T.ToastError as e:    # documented limits (e.g. > 8 SetGroups in one super-color)
        assert "LIMIT" in str(e), e
        return False
    o = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1)
    seqs, costs = o.rollout(np.zeros((n_roll, 32), np.uint16), seed=seed)
    seqs, costs = list(seqs), list(costs)
    if n_deep:
        deep = _deep(o, n_deep, seed=seed)
        seqs += deep
        costs += list(o.eval(np.stack(deep)))
    inputs = SI.random_inputs(ir, seed)
    for s, c in zip(seqs, costs):
        lst = [int(x) for x in s if x]
        low = T.lower(a, lst)
        pay = SI.run_lowered(low, ir, inputs, stats=stats)
        counts = count_collectives(low)
        for A in range(len(axes)):
            for k, kind in enumerate(KINDS):
                assert pay.get((A, kind), 0) == int(c["payload"][A][k]), (lst, A, kind)
                assert counts.get((A, kind), 0) == int(c["count"][A][k]), (lst, A, kind)
        assert sum(counts.values()) == int(c["n_collectives"])
    return True


def _assert_ext_coverage(stats, kinds):
    """every extension op kind ran, with a sharded result dim, and every kind
    with a reduction loop also left a partial result somewhere"""
    partial_kinds = {"dot_general", "conv2d", "conv2d_bwd_input", "conv2d_bwd_filter", "segment_sum"}
    for k in kinds:
        assert k in stats and stats[k][0] > 0, (k, "never lowered")
        assert stats[k][1] > 0, (k, "never sharded")
        if k in partial_kinds:
            assert stats[k][2] > 0, (k, "never partial")


def test_lowered_random_extension_programs_compute_the_unsharded_program():
    """40 random programs over every extension op kind (repeated operands such
    as dot_general(x, x) and concat([x, x]) included) on a 2x4, a 2x2x2 and a
    non-power-of-two 2x3x2 mesh: the lowered program computes the unsharded
    one on every device and its collectives total the oracle's C11 record."""
    stats, ran = {}, 0
    for seed in range(40):
        ir = models.random_program(seed, n_ops=16, ext=True)
        for mi, axes in enumerate(EXT_MESHES):
            ran += _check_ext(ir, axes, 16, 1 if mi == 0 else 0, seed, stats)
    assert ran >= 100
    _assert_ext_coverage(stats, EXT_KINDS)


TOY = {
    "gpt": lambda: models.gpt(layers=2, B=4, S=8, D=8, H=2, Dh=4, F=16, V=16, name="gpt_toy"),
    "llama": lambda: models.llama(layers=2, B=4, S=8, D=8, Hkv=2, G=2, Dh=4, F=16, V=16, name="llama_toy"),
    "gns": lambda: models.gns(steps=2, Nn=8, Ne=16, hidden=8, latent=8, node_in=4, edge_in=4, out_dim=2,
                              name="gns_toy"),
    "unet": lambda: models.unet(B=2, HW=8, C=(4, 8), heads=2, in_ch=2, temb=4, blocks_down=1, blocks_up=2,
                                name="unet_toy"),
}
TOY_KINDS = {"gpt": ("dot_general", "gather"), "llama": ("dot_general", "gather", "concat", "slice", "pad"),
             "gns": ("dot_general", "gather", "segment_sum", "concat", "slice"),
             "unet": ("dot_general", "conv2d", "conv2d_bwd_input", "conv2d_bwd_filter", "resample", "concat", "slice")}


@pytest.mark.parametrize("model", sorted(TOY))
@pytest.mark.parametrize("mesh", range(len(EXT_MESHES)))
def test_lowered_toy_models_compute_the_unsharded_program(model, mesh):
    """The BASELINE generators at toy widths (2 layers / steps; forward,
    backward and Adam), on 2- and 3-axis meshes: oracle rollouts and a
    maximal-depth sequence lower to programs that compute the unsharded
    training step, with the oracle's collective totals."""
    stats = {}
    assert _check_ext(TOY[model](), EXT_MESHES[mesh], 12, 1 if mesh < 2 else 0, 100 + mesh, stats)
    if mesh < 2:    # the 2x3x2 mesh leaves most toy extents indivisible by 3
        _assert_ext_coverage(stats, TOY_KINDS[model])


# Programs a wrong loop rule would produce, written out by hand (mesh a=2).
# Each must be rejected both with the interpreter's derived layouts (strict)
# and by the values alone (strict=False trusts the declared layouts).
_WRONG = {
    # X loops (reading G23 / C1): sharding them has no local semantics
    "conv2d spatial dim sharded": ("def f(x: f32[2,4,4,2], w: f32[3,3,2,2]) {\n  y = conv2d(x, w)\n  return y\n}\n", """mesh a=2
%x = param f32 [2,4,4,2] local[2,2,4,2] layout[0,1,0,0] partial[0]
%w = param f32 [3,3,2,2] local[3,3,2,2] layout[0,0,0,0] partial[0]
%y = conv2d(%x, %w) f32 [2,4,4,2] local[2,2,4,2] layout[0,1,0,0] partial[0]
return %y"""),
    "gather table rows sharded": ("def f(t: f32[8,2], i: i32[4]) {\n  y = gather(t, i)\n  return y\n}\n", """mesh a=2
%t = param f32 [8,2] local[4,2] layout[1,0] partial[0]
%i = param i32 [4] local[4] layout[0] partial[0]
%y = gather(%t, %i) f32 [4,2] local[4,2] layout[0,0] partial[0]
return %y"""),
    "segment_sum segments sharded": ("def f(x: f32[4,2], i: i32[4]) {\n  y = segment_sum[8](x, i)\n  return y\n}\n", """mesh a=2
%x = param f32 [4,2] local[4,2] layout[0,0] partial[0]
%i = param i32 [4] local[4] layout[0] partial[0]
%y = segment_sum[8](%x, %i) f32 [8,2] local[4,2] layout[1,0] partial[0]
return %y"""),
    "concat dim sharded": ("def f(x: f32[4,2], z: f32[4,2]) {\n  y = concat[0](x, z)\n  return y\n}\n", """mesh a=2
%x = param f32 [4,2] local[2,2] layout[1,0] partial[0]
%z = param f32 [4,2] local[2,2] layout[1,0] partial[0]
%y = concat[0](%x, %z) f32 [8,2] local[4,2] layout[1,0] partial[0]
return %y"""),
    "slice dim sharded": ("def f(x: f32[8,2]) {\n  y = slice[0,2,4](x)\n  return y\n}\n", """mesh a=2
%x = param f32 [8,2] local[4,2] layout[1,0] partial[0]
%y = slice[0,2,4](%x) f32 [4,2] local[2,2] layout[1,0] partial[0]
return %y"""),
    "pad dim sharded": ("def f(x: f32[4,2]) {\n  y = pad[0,1,1](x)\n  return y\n}\n", """mesh a=2
%x = param f32 [4,2] local[2,2] layout[1,0] partial[0]
%y = pad[0,1,1](%x) f32 [6,2] local[3,2] layout[1,0] partial[0]
return %y"""),
    # R loops: a sharded reduction loop leaves partial sums that a use must reduce (G27)
    "segment_sum members marked P": ("def f(x: f32[4,2], i: i32[4]) {\n  y = segment_sum[8](x, i)\n  return y\n}\n", """mesh a=2
%x = param f32 [4,2] local[2,2] layout[1,0] partial[0]
%i = param i32 [4] local[2] layout[1] partial[0]
%y = segment_sum[8](%x, %i) f32 [8,2] local[8,2] layout[0,0] partial[0]
return %y"""),
    "dot_general contracting dim marked P": ("def f(x: f32[2,4], z: f32[4,2]) {\n  y = dot_general[;;1;0](x, z)\n  return y\n}\n", """mesh a=2
%x = param f32 [2,4] local[2,2] layout[0,1] partial[0]
%z = param f32 [4,2] local[2,2] layout[1,0] partial[0]
%y = dot_general[;;1;0](%x, %z) f32 [2,2] local[2,2] layout[0,0] partial[0]
return %y"""),
    "conv2d input channels marked P": ("def f(x: f32[2,4,4,2], w: f32[3,3,2,2]) {\n  y = conv2d(x, w)\n  return y\n}\n", """mesh a=2
%x = param f32 [2,4,4,2] local[2,4,4,1] layout[0,0,0,1] partial[0]
%w = param f32 [3,3,2,2] local[3,3,1,2] layout[0,0,1,0] partial[0]
%y = conv2d(%x, %w) f32 [2,4,4,2] local[2,4,4,2] layout[0,0,0,0] partial[0]
return %y"""),
    "conv2d_bwd_input output channels marked P": ("def f(d: f32[2,4,4,2], w: f32[3,3,2,2]) {\n  y = conv2d_bwd_input(d, w)\n  return y\n}\n", """mesh a=2
%d = param f32 [2,4,4,2] local[2,4,4,1] layout[0,0,0,1] partial[0]
%w = param f32 [3,3,2,2] local[3,3,2,1] layout[0,0,0,1] partial[0]
%y = conv2d_bwd_input(%d, %w) f32 [2,4,4,2] local[2,4,4,2] layout[0,0,0,0] partial[0]
return %y"""),
    "conv2d_bwd_filter batch marked P": ("def f(x: f32[2,4,4,2], d: f32[2,4,4,2]) {\n  y = conv2d_bwd_filter[3,3](x, d)\n  return y\n}\n", """mesh a=2
%x = param f32 [2,4,4,2] local[1,4,4,2] layout[1,0,0,0] partial[0]
%d = param f32 [2,4,4,2] local[1,4,4,2] layout[1,0,0,0] partial[0]
%y = conv2d_bwd_filter[3,3](%x, %d) f32 [3,3,2,2] local[3,3,2,2] layout[0,0,0,0] partial[0]
return %y"""),
    # P loops identified with the wrong result dim
    "dot_general batch dim taken as a free dim": ("def f(x: f32[4,2,3], z: f32[4,3,2]) {\n  y = dot_general[0;0;2;1](x, z)\n  return y\n}\n", """mesh a=2
%x = param f32 [4,2,3] local[2,2,3] layout[1,0,0] partial[0]
%z = param f32 [4,3,2] local[2,3,2] layout[1,0,0] partial[0]
%y = dot_general[0;0;2;1](%x, %z) f32 [4,2,2] local[4,1,2] layout[0,1,0] partial[0]
return %y"""),
    "gather feature dim taken from the index": ("def f(t: f32[8,2], i: i32[4]) {\n  y = gather(t, i)\n  return y\n}\n", """mesh a=2
%t = param f32 [8,2] local[8,1] layout[0,1] partial[0]
%i = param i32 [4] local[4] layout[0] partial[0]
%y = gather(%t, %i) f32 [4,2] local[2,2] layout[1,0] partial[0]
return %y"""),
}


@pytest.mark.parametrize("case", sorted(_WRONG))
@pytest.mark.parametrize("strict", [True, False])
def test_interpreter_rejects_wrong_extension_rules(case, strict):
    """Not vacuous: the programs a plausible slip in an extension op's loop rule
    would lower to (an unshardable dim sharded, a reduction loop treated as
    parallel, a dim identified with the wrong result dim) are rejected — by
    the derived layouts and, with strict=False, by the values alone."""
    ir, low = _WRONG[case]
    with pytest.raises(SI.ShardError):
        SI.run_lowered(low, ir, SI.random_inputs(ir, 1), strict=strict)


def test_interpreter_accepts_the_right_extension_rules():
    """The corrected forms of the partial-sum cases above (the reduction loop's
    partial result all-reduced) compute the unsharded program."""
    fixed = 0
    for case, (ir, low) in _WRONG.items():
        if "marked P" not in case:
            continue
        lines = low.splitlines()
        y = lines[-2]
        lines[-2] = y.replace("partial[0]", "partial[1]")
        gl = re.search(r"f32 (\[[^\]]*\]) local(\[[^\]]*\]) layout(\[[^\]]*\])", y)
        lines.insert(-1, f"%y.1 = all_reduce{{axis=0}}(%y) f32 {gl.group(1)} local{gl.group(2)} layout{gl.group(3)} "
                         f"partial[0] bytes={4 * int(np.prod(eval(gl.group(2))))}")
        lines[-1] = "return %y.1"
        SI.run_lowered("\n".join(lines), ir, SI.random_inputs(ir, 1))
        fixed += 1
    assert fixed == 5


def test_blocked_all_to_all_moves_run_as_one_collective():
    """Reading R20: a weight whose two axes swap dims with extents too small to
    hold both at once (the toy U-Net's square 3x3 filters on {a:2, b:4}) has no
    divisible single-axis all_to_all order; the lowering lists both moves in
    one all_to_all (each axis charged as its own, as C11 counts them) and the
    program still computes the unsharded training step."""
    T = _T()
    ir, axes = TOY["unet"](), EXT_MESHES[0]
    a = T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=-1)
    o = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1)
    for seed in range(100, 110):
        seq = _deep(o, 1, seed=seed)[0]
        low = T.lower(a, [int(x) for x in seq if x])
        if "}+{" not in low:
            continue
        pay = SI.run_lowered(low, ir, SI.random_inputs(ir, seed))
        c = o.eval(np.stack([seq]))[0]
        for A in range(len(axes)):
            assert pay.get((A, "all_to_all"), 0) == int(c["payload"][A][3])
        counts = count_collectives(low)
        assert all(counts.get((A, "all_to_all"), 0) == int(c["count"][A][3]) for A in range(len(axes)))
        return
    raise AssertionError("no maximal-depth toy U-Net sequence needed a combined all_to_all")
