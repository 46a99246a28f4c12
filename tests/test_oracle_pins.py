"""Pins for the oracle (SURVEY §8(c) "What pins each part").

Every expected value here comes from the paper (worked examples, cited), a
closed form, an invariant, a library known-answer vector, or brute force —
never from the oracle itself and never from the CUDA path.
"""
import itertools
import re
import json
import os

import numpy as np
import pytest

from oracle.oracle import AG, AR, A2A, RS, Oracle, OracleError, philox4x32_10
from workloads import configs, models

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DER = json.load(open(os.path.join(GOLD, "derived.json")))


def golden(name):
    return open(os.path.join(GOLD, name)).read()


def action_id(d, loop, r, axis):
    """id of action (super-color containing `loop`, r, axis) in the dump."""
    sc = d["loops"][loop][5]
    for i, a in enumerate(d["actions"]):
        if a == [sc, r, axis]:
            return i + 1
    raise KeyError((loop, r, axis))


def value_dim_components(d, o: Oracle, rank_by_op):
    """Partition of value dims (op, dim) by component, as sets of (op, dim)."""
    groups = {}
    for op, rank in rank_by_op.items():
        for i in range(rank):
            groups.setdefault(d["loops"][o.def_loop(op, i)][4], set()).add((op, i))
    return sorted(sorted(g) for g in groups.values())


# --------------------------------------------------------------------------- C1–C2
def test_fig4c_mlp_colors():
    """Fig. 4c: I∪M gives x:[B,X], w1:[X,U], w2:[U,W], y,z:[B,U], w:[B,W]."""
    o = Oracle(golden("mlp_fig2.ir"), [("b", 2, 1e10)], 1e9, 1 << 40, 100.0, 1)
    d = o.dump()
    # ops: x0 w1 1 w2 2 y 3 z 4 w 5 ret 6
    parts = value_dim_components(d, o, {0: 2, 1: 2, 2: 2, 3: 2, 4: 2, 5: 2})
    B = [(0, 0), (3, 0), (4, 0), (5, 0)]
    X = [(0, 1), (1, 0)]
    U = [(1, 1), (2, 0), (3, 1), (4, 1)]
    W = [(2, 1), (5, 1)]
    assert parts == sorted([B, X, U, W])


def test_fig4b_ionly_one_class_per_op_loop():
    """Fig. 4b: matmul(x:[A1,X1], w1:[X1,A2]):[A1,A2] — identified with I only."""
    o = Oracle(golden("mlp_fig2.ir"), [("b", 2, 1e10)], 1e9, 1 << 40, 100.0, 1)
    t = 3  # y = matmul(x, w1)
    assert o.use_loop(t, 0, 0) == o.def_loop(t, 0)       # A1
    assert o.use_loop(t, 0, 1) == o.use_loop(t, 1, 0)    # X1
    assert o.use_loop(t, 1, 1) == o.def_loop(t, 1)       # A2
    assert len({o.use_loop(t, 0, 0), o.use_loop(t, 0, 1), o.use_loop(t, 1, 1)}) == 3
    # Fig. 4a: 6 param names + 6 use sites x 2 dims + 3 results x 2 dims;
    # M has one edge per use dim (12); I = 3 (matmul) + 2 (ReLU) + 3 (matmul) = 8
    names, m, ident = o.nda_sizes()
    assert (names, m, ident) == (6 + 12 + 6, 12, 8)


def test_identity_program_edges():
    """`id(x){return x}` has exactly rank(x) M edges and no identities;
    S:391: a program with no contraction has baseline runtime 0 -> degenerate."""
    with pytest.raises(OracleError) as e:
        Oracle("def id(x: f32[4,8]) {\n  return x\n}\n", [("b", 2, 1e10)], 1e9, 1 << 40)
    assert e.value.code == "E_DEGENERATE"
    o = Oracle("def id(x: f32[4,8], a: f32[2,2], b: f32[2,2]) {\n  y = matmul(a, b)\n  return x, y\n}\n",
               [("b", 2, 1e10)], 1e9, 1 << 40, 100.0, 1)
    d = o.dump()
    assert d["n_edges"] == 2 + 2 + 2 + 2
    assert d["conflicts"] == []


# --------------------------------------------------------------------------- C3–C5
def test_attention_five_conflicts_one_set():
    """P:891 five conflicts; P:940-946 one compatibility set, two resolutions."""
    o = Oracle(golden("attn_fig5.ir"), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
    d = o.dump()
    assert len(d["conflicts"]) == DER["attn_fig5"]["n_conflicts"]
    assert len(set(c[3] for c in d["conflicts"])) == DER["attn_fig5"]["n_sets"]
    # each conflict's ops: a, b(reduce), c(broadcast), d(div), z
    ops = [c[0] for c in d["conflicts"]]
    assert ops == [8, 9, 10, 11, 12]
    # the S super-color offers exactly two resolutions on the one axis
    sc = d["loops"][d["conflicts"][0][1]][5]
    assert sorted(a[1] for a in d["actions"] if a[0] == sc) == [0, 1]


def test_f_transpose_conflict():
    """z = matmul(x, transpose(x)) is conflicted; with the return as a
    use site that is two pairs in one set (SURVEY §8(c) C3-C5 pins)."""
    o = Oracle(golden("f_transpose.ir"), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
    d = o.dump()
    assert len(d["conflicts"]) == 2
    assert [c[0] for c in d["conflicts"]] == [2, 3]     # matmul, ret
    assert len(set(c[3] for c in d["conflicts"])) == 1


def test_h_no_conflict_and_mlp_no_conflict():
    """h(x) uses x twice yet has no conflict; Fig. 2 mlp has none."""
    # h has no contraction -> degenerate baseline; check conflicts via a carrier matmul
    ir = golden("h_reduce_bcast.ir").replace("def h(x: f32[8,4])", "def h(x: f32[8,4], pa: f32[2,2], pb: f32[2,2])")
    ir = ir.replace("  return w", "  mm = matmul(pa, pb)\n  return w, mm")
    o = Oracle(ir, [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
    assert o.dump()["conflicts"] == []
    o = Oracle(golden("mlp_fig2.ir"), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
    assert o.dump()["conflicts"] == []


def test_g_conflict_resolutions_rs_vs_ag():
    """[comment] P:1005-1034: g(t,u) has one conflict (u-def, matmul) in one set;
    one resolution reduce-scatters, the other all-gathers t."""
    o = Oracle(golden("g_matmul_add.ir"), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
    d = o.dump()
    assert [c[0] for c in d["conflicts"]] == [1, 2]
    assert len(set(c[3] for c in d["conflicts"])) == 1
    seen = {}
    for r in (0, 1):
        a = action_id(d, 3, r, 0)   # loop 3 = u dim 1 (the B component)
        c = o.eval(Oracle.seqs([[a]]))[0]
        kinds = tuple(int(x) for x in c["count"][0])
        seen[r] = kinds
        m = o.materialize([a])
        u0, u1 = o.def_loop(1, 0), o.def_loop(1, 1)
        if kinds == (0, 1, 0, 0):
            assert m[u0] == 1 and m[u1] == 0          # "shard u dim 0" -> reduce_scatter
        else:
            assert kinds == (1, 0, 0, 0)              # all_gather of t
            assert m[u0] == 0 and m[u1] == 1
    assert sorted(seen.values()) == [(0, 1, 0, 0), (1, 0, 0, 0)]


def test_linearity_theorem_random_programs():
    """[comment] Thm P:1106-1110 / SPEC S:278: single-use variables never conflict."""
    for seed in range(100):
        ir = models.random_program(seed, n_ops=10, linear=True)
        o = Oracle(ir, [("a", 2, 1e10), ("b", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
        assert o.dump()["conflicts"] == [], ir


def test_setgroups_independent_of_layers():
    """§3.6: isomorphic sets of repeated layers share one resolution."""
    n_actions = set()
    for L in (1, 2, 3, 4, 6):
        o = Oracle(models.stacked_attn(L), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
        d = o.dump()
        assert len(d["set_group"]) == L           # one compatibility set per layer
        assert d["n_groups"] == 1                 # all isomorphic -> one SetGroup
        if L >= 2:
            n_actions.add(len(d["actions"]))
    assert len(n_actions) == 1


# --------------------------------------------------------------------------- C9–C13
def test_fig2b_batch_no_communication_and_batch_law():
    """P:365 batch partitioning needs no communication; P:1462 runtime / b."""
    for b in (2, 4, 8):
        o = Oracle(golden("mlp_fig2.ir"), [("b", b, 1e10)], 1e9, 1 << 40, 100.0, 1)
        d = o.dump()
        t0, p0, f0 = o.baseline()
        assert f0 == 1048576 + 524288
        c = o.eval(Oracle.seqs([[action_id(d, 0, 0, 0)]]))[0]
        assert c["n_collectives"] == 0 and int(c["payload"].sum()) == 0
        assert int(c["flops"]) * b == f0
        assert c["score"] == 1.0 / b                        # RT = 1/b exactly, MP = 0


def test_fig2c_megatron_one_allreduce():
    """Fig. 2c: B->b, U->m gives exactly one all_reduce{m}."""
    o = Oracle(golden("mlp_fig2.ir"), [("b", 2, 1e10), ("m", 2, 1e11)], 1e9, 1 << 40, 100.0, 1)
    d = o.dump()
    g = DER["mlp_fig2"]
    t0, p0, f0 = o.baseline()
    assert (p0, f0) == (g["peak0"], g["flops0"])
    seq = [action_id(d, 0, 0, 0), action_id(d, 3, 0, 1)]   # (B,b), (U,m)
    c = o.eval(Oracle.seqs([seq]))[0]
    gc = DER["mlp_fig2c"]
    assert c["n_collectives"] == 1
    assert int(c["count"][1][AR]) == 1 and int(c["payload"][1][AR]) == gc["ar_m_payload"]
    assert (int(c["peak_bytes"]), int(c["flops"])) == (gc["peak"], gc["flops"])
    # device-local annotations of Fig. 2c: x [256{b},32], w1 [32,64{m}], w2 [64{m},16]
    m = o.materialize(seq)
    assert [m[o.def_loop(0, i)] for i in (0, 1)] == [1, 0]
    assert [m[o.def_loop(1, i)] for i in (0, 1)] == [0, 2]
    assert [m[o.def_loop(2, i)] for i in (0, 1)] == [2, 0]


def test_fig5b_sequence_resolution_collectives():
    """Fig. 5b: sequence sharding = all_gather{s}(k) + reduce_scatter{s}(z);
    the other resolution = two all_gathers and one AR of b (reading G22)."""
    o = Oracle(golden("attn_fig5.ir"), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
    d = o.dump()
    got = {}
    for r in (0, 1):
        c = o.eval(Oracle.seqs([[action_id(d, 0, r, 0)]]))[0]   # loop 0 = x dim 0 (S)
        got[r] = c
    seq_r = [r for r in (0, 1) if got[r]["count"][0][RS] == 1]
    assert len(seq_r) == 1
    seq_r = seq_r[0]
    other = 1 - seq_r
    cs, co = got[seq_r], got[other]
    assert (int(cs["count"][0][AG]), int(cs["count"][0][RS]), int(cs["count"][0][AR])) == (1, 1, 0)
    assert int(cs["payload"][0][AG]) == 64 and int(cs["payload"][0][RS]) == 64
    assert (int(co["count"][0][AG]), int(co["count"][0][RS]), int(co["count"][0][AR])) == (2, 0, 1)
    assert int(co["payload"][0][AG]) == 128 and int(co["payload"][0][AR]) == 32
    # Fig. 5b annotations: a:[S, S{s}], b:[S{s}], c:[S, S{s}], d:[S, S{s}], z_ partial -> z:[S{s},H2] after RS
    m = o.materialize([action_id(d, 0, seq_r, 0)])
    ops = {"x": 0, "k": 4, "v": 5, "q": 6, "qt": 7, "a": 8, "b": 9, "c": 10, "d": 11, "z": 12}
    ann = {k: [int(m[o.def_loop(t, i)]) for i in range(2 if k != "b" else 1)] for k, t in ops.items()}
    assert ann == {"x": [1, 0], "k": [1, 0], "v": [1, 0], "q": [1, 0], "qt": [0, 1], "a": [0, 1],
                   "b": [1], "c": [0, 1], "d": [0, 1], "z": [0, 0]}


def test_mlp_c_derived_table():
    """SURVEY §8(c) DERIVED MLP-c goldens (M1)."""
    c = configs.get("mlp_c")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims)
    d = o.dump()
    g = DER["mlp_c"]
    t0, p0, f0 = o.baseline()
    assert (p0, f0) == (g["peak0"], g["flops0"])
    sc_members = {}
    for l, row in enumerate(d["loops"]):
        sc_members.setdefault(row[5], []).append(l)
    assert sorted(sc_members.values()) == sorted(g["loop_supercolors"].values())
    assert [c[:3] for c in d["conflicts"]] == g["conflicts"]
    assert sorted(c[4] for c in d["conflicts"]) == g["side0"]
    assert d["actions"] == g["actions"]
    for r, key in ((0, "H_r0_m"), (1, "H_r1_m")):
        cst = o.eval(Oracle.seqs([[action_id(d, 2, r, 1)]]))[0]
        e = g[key]
        assert int(cst["peak_bytes"]) == e["peak"] and int(cst["flops"]) == e["flops"]
        assert int(cst["payload"][1][AR]) == e["ar_m"] and int(cst["count"][1][AR]) == 1
        if r == 0:
            assert int(cst["payload"][1][RS]) == e["rs_m"] and int(cst["count"][1][AG]) == 0
        else:
            assert int(cst["payload"][1][AG]) == e["ag_m"] and int(cst["count"][1][RS]) == 0
    # DM = 131072: r=0 pays a memory penalty, r=1 does not
    s0 = o.eval(Oracle.seqs([[action_id(d, 2, 0, 1)]]))[0]
    s1 = o.eval(Oracle.seqs([[action_id(d, 2, 1, 1)]]))[0]
    assert s0["score"] > s0["runtime_s"] / t0 and s1["score"] == s1["runtime_s"] / t0


def test_memory_penalty_closed_form():
    """RT(∅) = 1; MP = C·(peak−DM)/peak0 if peak > DM else 0."""
    ir = golden("mlp_fig2.ir")
    o = Oracle(ir, [("b", 2, 1e10)], 1e9, 135168 // 2, 100.0, 1)
    c = o.eval(Oracle.seqs([[]]))[0]
    assert c["score"] == 1.0 + 50.0                    # half of peak0 over DM, C = 100
    o = Oracle(ir, [("b", 2, 1e10)], 1e9, 135168, 100.0, 1)
    assert o.eval(Oracle.seqs([[]]))[0]["score"] == 1.0  # peak == DM -> no penalty


# --------------------------------------------------------------------------- C12 brute force
def _bruteforce_unsharded_peak(ir: str) -> int:
    """Independent liveness: max over program points of the bytes of values v with
    def(v) <= t <= last_use(v), parsed straight from the text."""
    lines = [l.strip() for l in ir.splitlines() if l.strip() and not l.strip().startswith("#")]
    hdr = lines[0]
    params = hdr[hdr.index("(") + 1: hdr.rindex(")")]
    vals = []   # (name, bytes)
    import re
    for m in re.finditer(r"(\w+):\s*(\w+)\[([0-9,]*)\]", params):
        n, dt, sh = m.groups()
        b = {"f32": 4, "bf16": 2, "i32": 4}[dt]
        for e in (sh.split(",") if sh else []):
            b *= int(e)
        vals.append([n, b])
    return vals, lines


def test_liveness_bruteforce_random_programs():
    """Unsharded peak equals the brute-force live-set maximum, using
    shapes re-derived from an independent dense interpretation of each program."""
    for seed in range(40):
        ir = models.random_program(seed, n_ops=14)
        o = Oracle(ir, [("a", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
        # shapes via the builder that generated the program (independent of the oracle)
        import re
        shapes = {}
        lines = [l.strip() for l in ir.splitlines()]
        hdr = lines[0]
        for m in re.finditer(r"(\w+):\s*(\w+)\[([0-9,]*)\]", hdr):
            shapes[m.group(1)] = [int(e) for e in m.group(3).split(",")] if m.group(3) else []
        defs = list(shapes)               # program points: params first
        uses = {}
        body = [l for l in lines[1:] if "=" in l]
        for l in body:
            out, rhs = [s.strip() for s in l.split("=", 1)]
            kind = rhs.split("(")[0].split("[")[0]
            attrs = rhs[rhs.index("[") + 1: rhs.index("]")] if "[" in rhs.split("(")[0] else ""
            args = [a.strip() for a in rhs[rhs.index("(") + 1: rhs.rindex(")")].split(",")]
            s0 = shapes[args[0]]
            if kind == "matmul":
                sh = [s0[0], shapes[args[1]][1]]
            elif kind == "transpose":
                perm = [int(x) for x in attrs.split(",")]
                sh = [s0[p] for p in perm]
            elif kind == "reduce":
                ds = [int(x) for x in attrs.split(",")[:-1]]
                sh = [e for i, e in enumerate(s0) if i not in ds]
            elif kind == "broadcast":
                l_, e_ = [int(x) for x in attrs.split(",")]
                sh = s0[:l_] + [e_] + s0[l_:]
            else:
                sh = list(s0)
            shapes[out] = sh
            t = len(defs)
            defs.append(out)
            for a in args:
                uses.setdefault(a, []).append(t)
        rets = [a.strip() for a in lines[-2].replace("return", "").split(",")]
        for i, a in enumerate(rets):
            uses.setdefault(a, []).append(len(defs) + i)
        npoints = len(defs) + len(rets)
        size = {v: 4 * int(np.prod(shapes[v])) if shapes[v] else 4 for v in defs}
        last = {v: max(uses.get(v, [defs.index(v)])) for v in defs}
        peak = 0
        for t in range(npoints):
            live = sum(size[v] for i, v in enumerate(defs) if i <= t <= last[v])
            peak = max(peak, live)
        assert o.baseline()[1] == peak, (seed, ir)


# --------------------------------------------------------------------------- invariants
def _check_state_invariants(o: Oracle, d: dict, seqs, costs):
    loops = d["loops"]
    nA = len(o.axes)
    sizes = [a[1] for a in o.axes]
    side0 = {}
    for c in d["conflicts"]:
        other = c[2] if c[4] == c[1] else c[1]
        side0[(c[1], c[2])] = (c[4], other, d["set_group"][c[3]])
    t0, p0, _ = o.baseline()
    for s, cst in zip(seqs, costs):
        assert cst["status"] == 0
        m = o.materialize([int(x) for x in s if x])
        # (1) one axis shards at most one loop of an op
        by_op = {}
        for l, row in enumerate(loops):
            if m[l]:
                assert not (by_op.get(row[0], 0) & m[l])
                by_op[row[0]] = by_op.get(row[0], 0) | m[l]
            # (2) local extent = global / prod(axis sizes), exactly
            prod = 1
            for A in range(nA):
                if m[l] >> A & 1:
                    prod *= sizes[A]
            assert row[2] % prod == 0
            if row[3] == 2:
                assert m[l] == 0                               # X loops never sharded
        # (3) consistency within a conflict group: the deselected endpoint is never sharded
        fixed = {}
        for a in s:
            if not a:
                break
            sc, r, _ = d["actions"][a - 1]
            for t, gid in enumerate(d["scolors"][sc][2]):
                fixed[gid] = (r >> t) & 1
        for (u, v), (s0, s1, gid) in side0.items():
            if gid in fixed:
                assert m[s1 if fixed[gid] == 0 else s0] == 0
        # (4) sharded peak never exceeds unsharded peak (north star invariant)
        assert int(cst["peak_bytes"]) <= p0


@pytest.mark.parametrize("name", ["mlp_c", "gpt2"])
def test_state_invariants_on_rollouts(name):
    c = configs.get(name)
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims)
    d = o.dump()
    seqs, costs = o.rollout(np.zeros((60, 32), np.uint16), seed=7)
    _check_state_invariants(o, d, seqs, costs)


def test_zero_collectives_without_conflicts_or_reductions():
    """North star: "collective bytes are zero when there is no conflict" — for a
    color with no conflict, no R loop and no X loop, a single action that shards
    every loop of the color (no skip) inserts no collective."""
    checked = 0
    for seed in range(60):
        ir = models.random_program(seed, n_ops=12)
        o = Oracle(ir, [("a", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
        d = o.dump()
        conf_sc = {d["loops"][c[1]][5] for c in d["conflicts"]}
        for ai, (sc, r, ax) in enumerate(d["actions"]):
            members = [l for l, row in enumerate(d["loops"]) if row[5] == sc]
            if sc in conf_sc or any(d["loops"][l][3] != 0 for l in members):
                continue
            m = o.materialize([ai + 1])
            if not all(m[l] for l in members):
                continue          # a divisibility skip happened
            c = o.eval(Oracle.seqs([[ai + 1]]))[0]
            assert c["n_collectives"] == 0 and int(c["payload"].sum()) == 0
            checked += 1
    assert checked > 20


def test_state_key_identifies_sharding():
    """P:1435-1440 / C14: key(s1) == key(s2) iff the materialized masks are equal;
    commuting actions on disjoint axes give the same key."""
    c = configs.get("mlp_c")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims)
    d = o.dump()
    seqs, costs = o.rollout(np.zeros((3000, 32), np.uint16), seed=3)
    by_key = {}
    for s, cst in zip(seqs, costs):
        m = o.materialize([int(x) for x in s if x]).tobytes()
        k = int(cst["state_key"])
        if k in by_key:
            assert by_key[k] == m
        by_key[k] = m
    inv = {}
    for k, m in by_key.items():
        assert m not in inv
        inv[m] = k
    a, b = action_id(d, 0, 0, 0), action_id(d, 5, 0, 1)   # (B,b), (O,m)
    c1, c2 = o.eval(Oracle.seqs([[a, b], [b, a]]))
    assert c1["state_key"] == c2["state_key"]
    assert o.eval(Oracle.seqs([[]]))[0]["state_key"] == 0


# --------------------------------------------------------------------------- C9 decode status
def test_decode_status_flags():
    c = configs.get("mlp_c")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims)
    n = o.n_actions
    cs = o.eval(Oracle.seqs([[n], [1, 1], [3, 6], [1, 0, 2], [9999]]))
    assert [int(x["status"]) for x in cs] == [1, 2, 4, 8, 1]
    assert all(int(x["peak_bytes"]) == 0 and x["score"] == 0.0 for x in cs)


# --------------------------------------------------------------------------- C15
def test_philox_known_answers():
    """Random123 kat_vectors for philox4x32-10."""
    kat = [([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
           ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
           ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
            [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1])]
    for ctr, key, exp in kat:
        assert philox4x32_10(ctr, key) == exp


def test_rollout_depth_and_legality():
    """Trajectories end at STOP or depth 30; chosen actions stay legal."""
    c = configs.get("gpt2")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims)
    seqs, costs = o.rollout(np.zeros((300, 32), np.uint16), seed=11)
    lens = (seqs != 0).sum(1)
    assert lens.max() <= 30 and lens.min() >= 1          # p_stop(0) = 0
    assert (costs["status"] == 0).all()
    # depth distribution: p_stop = d/30 -> mean length well below 30
    assert 2 < lens.mean() < 12


# --------------------------------------------------------------------------- C16/C17
@pytest.mark.parametrize("tp", [0, 1])
def test_search_reaches_bruteforce_optimum_mlp_c(tp):
    """MCTS best equals the exhaustive optimum at desk scale
    (as a tree of sequences, and with transpositions, reading R24)."""
    c = configs.get("mlp_c")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims)
    n, best, bc = o.bruteforce()
    assert n > 1000
    r, trace = o.search(seed=0, max_evals=4000, L=4, R=8, patience=4, transpositions=tp)
    assert r["best"]["score"] == bc["score"]
    assert np.all(np.diff(trace) <= 0)


@pytest.mark.parametrize("tp", [0, 1])
@pytest.mark.parametrize("dm", [1 << 40, 700, 400])
def test_search_reaches_bruteforce_optimum_attn(dm, tp):
    """toy attention with DM below the unsharded peak forces sharding."""
    c = configs.get("attn_toy")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, dm, c.penalty_c, c.min_dims)
    n, best, bc = o.bruteforce()
    r, _ = o.search(seed=1, max_evals=4000, L=4, R=8, patience=4, transpositions=tp)
    assert r["best"]["score"] == bc["score"]


def test_transpositions_keep_each_state_once():
    """Reading R24 ("any action sequence yielding the same sharded
    model resolves to the same unique state"): on MLP-c, whose 3,849 legal
    sequences reach far fewer distinct states, a search with transpositions
    spends its rounds on distinct states — it reaches the exhaustive optimum
    with no more evaluations than the tree of sequences, and the exhaustive
    count of distinct states (by state key) is well below the sequence count."""
    c = configs.get("mlp_c")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims)
    n, best, bc = o.bruteforce()
    # every legal sequence's state key (the exhaustive enumeration of C17 restated as a DFS here)
    acts = o.dump()["actions"]
    groups = [sc[2] for sc in o.dump()["scolors"]]

    def kills(x, y):
        cx, rx, ax = acts[x - 1]
        cy, ry, ay = acts[y - 1]
        if cx == cy and ax == ay:
            return True
        return any(gx == gy and ((rx >> i) ^ (ry >> j)) & 1 for i, gx in enumerate(groups[cx])
                   for j, gy in enumerate(groups[cy]))
    seqs = []

    def dfs(seq, legal):
        seqs.append(seq)
        for x in legal:
            dfs(seq + [x], [y for y in legal if not kills(x, y)])
    dfs([], list(range(1, len(acts) + 1)))
    keys = o.eval(Oracle.seqs(seqs))["state_key"]
    assert len(seqs) == n and len(np.unique(keys)) < len(seqs) // 4
    r0, _ = o.search(seed=0, max_evals=100000, L=4, R=8, patience=1000, target_score=float(bc["score"]))
    r1, _ = o.search(seed=0, max_evals=100000, L=4, R=8, patience=1000, target_score=float(bc["score"]),
                     transpositions=1)
    assert r1["hit_target"] and r0["hit_target"]
    assert int(r1["evals"]) <= int(r0["evals"])


# --------------------------------------------------------------------------- parser errors
@pytest.mark.parametrize("src,code", [
    ("def f(x: f32[2,3], y: f32[4,5]) {\n  z = matmul(x, y)\n  return z\n}\n", "E_SHAPE"),
    ("def f(x: f32[2,2]) {\n  z = matmul(x, q)\n  return z\n}\n", "E_UNDEFINED"),
    ("def f(x: f32[2,2]) {\n  z = matmul(x, x)\n  z = matmul(x, x)\n  return z\n}\n", "E_DUPLICATE"),
    ("def f(x: f32[2,2]) {\n  z = matmul(x x)\n  return z\n}\n", "E_PARSE"),
])
def test_parser_errors(src, code):
    with pytest.raises(OracleError) as e:
        Oracle(src, [("a", 2, 1e10)], 1e12, 1 << 40)
    assert e.value.code == code


# --------------------------------------------------------------------------- C6 by brute force
def _iso(g1, g2):
    """Labelled-graph isomorphism by backtracking: node labels (op kind, role,
    loop type, side mask), directed M edges, undirected conflict edges."""
    n1 = {v[0]: tuple(v[1:]) for v in g1["nodes"]}
    n2 = {v[0]: tuple(v[1:]) for v in g2["nodes"]}
    if sorted(n1.values()) != sorted(n2.values()) or len(g1["medges"]) != len(g2["medges"]) \
            or len(g1["cedges"]) != len(g2["cedges"]):
        return False
    m1, m2 = {tuple(e) for e in g1["medges"]}, {tuple(e) for e in g2["medges"]}
    c1 = {frozenset(e) for e in g1["cedges"]}
    c2 = {frozenset(e) for e in g2["cedges"]}
    order = sorted(n1, key=lambda v: sum(1 for w in n1 if n1[w] == n1[v]))   # rarest labels first
    used, mp = set(), {}

    def ok(v, w):
        for (a, b) in m1:
            if a == v and b in mp and (w, mp[b]) not in m2:
                return False
            if b == v and a in mp and (mp[a], w) not in m2:
                return False
        for e in c1:
            if v in e:
                (u,) = e - {v} if len(e) == 2 else (v,)
                if u in mp and frozenset((w, mp[u])) not in c2:
                    return False
        return True

    def go(i):
        if i == len(order):
            return True
        v = order[i]
        for w in n2:
            if w in used or n2[w] != n1[v] or not ok(v, w):
                continue
            mp[v] = w
            used.add(w)
            if go(i + 1):
                return True
            del mp[v]
            used.discard(w)
        return False

    return go(0)


F_BLOCKS = """
  yt1 = transpose[1,0](y1)
  f1 = matmul(y1, yt1)
  yt2 = transpose[1,0](y2)
  f2 = matmul(y2, yt2)
"""


def _attn_and_f(layers=2):
    ir = models.stacked_attn(layers)
    head, rest = ir.split(") {", 1)
    body, ret = rest.rsplit("  return ", 1)
    return head + ", y1: f32[8,4], y2: f32[16,4]) {" + body + F_BLOCKS + "  return " + ret.replace("\n}", ", f1, f2\n}")


def test_setgroups_are_the_isomorphism_classes():
    """§3.6: sets share a SetGroup iff they are isomorphic.  Checked by
    brute-force labelled-graph isomorphism of the graphs the C6 hash reads, on
    two attention layers plus two x·xᵀ blocks (two classes of two sets each)
    and on random programs with several sets."""
    cases = [_attn_and_f(2)] + [models.random_program(s, n_ops=24) for s in range(60)]
    multi = 0
    pairs = {True: 0, False: 0}
    for ir in cases:
        try:
            o = Oracle(ir, [("a", 2, 1e10), ("b", 4, 1e11)], 1e12, 1 << 40, 100.0, 1)
        except OracleError:
            continue
        d, gs = o.dump(), o.set_graphs()
        if len(gs) < 2:
            continue
        multi += 1
        grp = d["set_group"]
        for i in range(len(gs)):
            for j in range(i + 1, len(gs)):
                if max(len(gs[i]["nodes"]), len(gs[j]["nodes"])) > 14:
                    continue
                iso = _iso(gs[i], gs[j])
                assert iso == (grp[i] == grp[j]), (ir, i, j)
                pairs[iso] += 1
    assert multi >= 3
    assert pairs[True] >= 100 and pairs[False] >= 500, pairs   # comparisons made, not just programs seen
    d = Oracle(_attn_and_f(2), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1).dump()
    assert len(d["set_group"]) == 4 and d["n_groups"] == 2


# --------------------------------------------------------------------------- C7 argument groups
def _param_partition(ir, names, axes=(("s", 2, 1e10),)):
    """Partition of the parameters' (name, dim) pairs by super-color."""
    o = Oracle(ir, list(axes), 1e12, 1 << 40, 100.0, 1)
    d = o.dump()
    groups = {}
    for op, (name, rank) in enumerate(names):
        for i in range(rank):
            groups.setdefault(d["loops"][o.def_loop(op, i)][5], set()).add((name, i))
    return sorted(sorted(g) for g in groups.values()), d


def _attn_params(L):
    return [("x", 2)] + [(f"{w}{l}", 2) for l in range(L) for w in ("wq", "wk", "wv")]


def test_argument_groups_mirror_layers():
    """§4.4: weights of repeated layers are grouped, so every
    layer's weights share super-colors with layer 0's and the number of
    super-colors does not grow with the number of layers (from two layers on:
    chaining layer 0's output into layer 1 already joins the feature dims)."""
    n_sc = set()
    for L in (2, 3, 4, 6):
        part, d = _param_partition(models.stacked_attn(L), _attn_params(L))
        n_sc.add(len(d["scolors"]))
        for l in range(1, L):
            for w in ("wq", "wk", "wv"):
                for i in range(2):
                    assert any((f"{w}0", i) in g and (f"{w}{l}", i) in g for g in part), (L, w, l, i)
    assert len(n_sc) == 1


def test_argument_groups_depend_on_uses_only():
    """Keys are "constructed from all uses": renaming the parameters and
    permuting their declaration order leaves the grouping unchanged."""
    import random
    L = 2
    ir = models.stacked_attn(L)
    names = _attn_params(L)
    base, _ = _param_partition(ir, names)
    head, rest = ir.split("(", 1)
    params, body = rest.split(") {", 1)
    decl = [f"{n}: {t}" for n, t in re.findall(r"(\w+)\s*:\s*(\w+\[[^\]]*\])", params)]
    assert len(decl) == len(names)
    rng = random.Random(3)
    for trial in range(4):
        perm = list(range(len(decl)))
        rng.shuffle(perm)
        ren = {n: f"r{trial}_{k}" for k, (n, _) in enumerate(names)}
        new_decl = []
        for k in perm:
            n, ty = decl[k].split(":", 1)
            new_decl.append(f"{ren[n.strip()]}:{ty}")
        new_body = body
        for n in sorted(ren, key=len, reverse=True):
            new_body = re.sub(rf"\b{n}\b", ren[n], new_body)
        ir2 = f"{head}({', '.join(new_decl)}) {{{new_body}"
        part2, _ = _param_partition(ir2, [(ren[names[k][0]], names[k][1]) for k in perm])
        inv = {v: k for k, v in ren.items()}
        assert sorted(sorted((inv[n], i) for n, i in g) for g in part2) == base


def test_set_graphs_rebuilt_by_hand():
    """The labelled graphs C6 hashes, rebuilt by hand from the paper's
    attention layer (Fig. 5; the five conflicts of P:891 at the
    score matmul, the reduce, the broadcast, the div and the output matmul,
    joined by the M edges of the score's uses) and from the x·xᵀ block
    (the matmul's (i, j) and the returned value's two dims): the
    oracle's graphs are isomorphic to these, label for label (op kind, role,
    loop type P=0 / R=1, side 1 / 2)."""
    def graph(nodes, medges, cedges):
        return {"nodes": [[k] + list(v) for k, v in nodes.items()], "medges": medges, "cedges": cedges}
    attn = graph({"a0": ("matmul", 0, 0, 1), "a1": ("matmul", 1, 0, 2),          # a = matmul(k, qt): i, j
                  "r0": ("reduce", 0, 1, 1), "r1": ("reduce", 1, 0, 2),          # b = reduce[0](a): dim 0 reduced
                  "b0": ("broadcast", 0, 0, 1), "b1": ("broadcast", 1, 0, 2),    # c = broadcast[0](b)
                  "d0": ("div", 0, 0, 1), "d1": ("div", 1, 0, 2),                # d = div(a, c)
                  "z0": ("matmul", 0, 0, 1), "zk": ("matmul", 2, 1, 2)},         # z = matmul(d, v): i, k
                 [["a0", "r0"], ["a0", "d0"], ["a1", "r1"], ["a1", "d1"], ["b0", "d0"], ["b1", "d1"],
                  ["d0", "z0"], ["d1", "zk"]],
                 [["a0", "a1"], ["r0", "r1"], ["b0", "b1"], ["d0", "d1"], ["z0", "zk"]])
    xxt = graph({"i": ("matmul", 0, 0, 1), "j": ("matmul", 1, 0, 2), "s0": ("ret", 0, 0, 1), "s1": ("ret", 1, 0, 2)},
                [["i", "s0"], ["j", "s1"]], [["i", "j"], ["s0", "s1"]])
    o = Oracle(_attn_and_f(2), [("s", 2, 1e10)], 1e12, 1 << 40, 100.0, 1)
    gs = o.set_graphs()
    assert len(gs) == 4
    assert [_iso(g, attn) for g in gs] == [True, True, False, False]
    assert [_iso(g, xxt) for g in gs] == [False, False, True, True]
