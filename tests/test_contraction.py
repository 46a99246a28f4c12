"""NEXT-4: the dimension-graph contraction heuristic (reading R23;
[comment] §3.5) as an alternative to compatibility sets.

Pins of the oracle (no GPU): the paper's listings — the attention layer's
conflicts all identified as compatible and the "paths going across"
listing whose vertical edges are not all contracted
 — and the definition itself, checked by brute force on small
programs from the contracted graph the oracle reports: no conflict's endpoints
share a node or are joined by a directed path, every edge left uncontracted
would join one (the greedy pass is maximal), conflict-free components contract
to one node, and sets are exactly the conflicts on one unordered node pair.
Then library == oracle on the H0 dump (host), and GPU rollouts/evals under a
contraction analysis bit-identical to the oracle's (-m gpu).
"""
import os
from collections import defaultdict, deque

import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError
from workloads import configs, models

CONTRACTION = 1
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# x carries a conflict between N and O (x = t t^T: both dims come
# from t's dim 0), y = transpose(x), then add(x, y).
INCOMPATIBLE = """def g(t: f32[8,4]) {
  tt = transpose[1,0](t)
  x = matmul(t, tt)
  y = transpose[1,0](x)
  z = add(x, y)
  return z
}
"""


def _oracle(ir, axes=(("s", 2, 1e10),), grouping=CONTRACTION, min_dims=1):
    return Oracle(ir, list(axes), 1e12, 1 << 40, 100.0, min_dims, 30, grouping=grouping)


def _adj(edges, cnode):
    adj = defaultdict(set)
    for a, b in edges:
        if cnode[a] != cnode[b]:
            adj[cnode[a]].add(cnode[b])
    return adj


def _reach(adj, src):
    seen, q = {src}, deque([src])
    while q:
        x = q.popleft()
        for y in adj[x]:
            if y not in seen:
                seen.add(y)
                q.append(y)
    return seen


def _conflict_joined(edges, cnode, conflicts):
    adj = _adj(edges, cnode)
    for _op, u, v, _s, _s0 in conflicts:
        U, V = cnode[u], cnode[v]
        if U == V or V in _reach(adj, U) or U in _reach(adj, V):
            return True
    return False


def check_definition(o: Oracle):
    """Brute-force check of the contraction result against its definition."""
    d = o.dump()
    edges = [tuple(e) for e in o.edges()]
    cnode = d["cnode"]
    conf = d["conflicts"]
    # nodes are named by their smallest member loop, and only M edges are contracted
    comp = [l[4] for l in d["loops"]]
    for l, c in enumerate(cnode):
        assert cnode[c] == c and c <= l and comp[c] == comp[l]
    # no conflict is joined by the contraction
    assert not _conflict_joined(edges, cnode, conf)
    # maximal: contracting any remaining edge would join a conflict
    rejected = 0
    for a, b in edges:
        A, B = cnode[a], cnode[b]
        if A == B:
            continue
        rejected += 1
        m = min(A, B)
        trial = [m if c in (A, B) else c for c in cnode]
        assert _conflict_joined(edges, trial, conf), (a, b)
    # a component without conflicts contracts to a single node
    conf_comps = {comp[u] for _op, u, _v, _s, _s0 in conf}
    for l, c in enumerate(cnode):
        if comp[l] not in conf_comps:
            assert c == comp[l]
    # counts: every accepted contraction merges two nodes
    assert d["contracted"] == len(cnode) - len(set(cnode))
    # a skipped edge stays skipped (contraction only adds paths), so the skips are the split edges
    assert d["contract_rejected"] == rejected and d["n_boxes"] == 0
    # sets = conflicts on one unordered pair of contracted nodes, numbered by smallest conflict
    key_set, first = {}, []
    for i, (_op, u, v, s, s0) in enumerate(conf):
        k = tuple(sorted((cnode[u], cnode[v])))
        if k not in key_set:
            key_set[k] = len(first)
            first.append(i)
        assert s == key_set[k]
        root_u = cnode[conf[first[s]][1]]
        assert s0 == (u if cnode[u] == root_u else v)
    return d


def test_attention_conflicts_all_identified_compatible():
    """P:1336 "(correctly) identify all conflicts in the forward attention layer as
    compatible": the five conflicts of Fig. 5 form one set whose two
    resolutions are the compatibility-set ones."""
    o1 = _oracle(open(os.path.join(GOLD, "attn_fig5.ir")).read())
    d1 = check_definition(o1)
    assert len(d1["conflicts"]) == 5
    assert {c[3] for c in d1["conflicts"]} == {0}
    d0 = _oracle(open(os.path.join(GOLD, "attn_fig5.ir")).read(), grouping=0).dump()
    assert [c[4] for c in d1["conflicts"]] == [c[4] for c in d0["conflicts"]]   # same sides
    assert d1["actions"] == d0["actions"] and d1["n_groups"] == d0["n_groups"] == 1


def test_paths_going_across_are_not_contracted():
    """with paths going across between the conflict in x
    (N, O) and the one in the add (L, R), not all vertical edges N->L, O->R are
    contracted, and the two conflicts are not identified."""
    o = _oracle(INCOMPATIBLE)
    d = check_definition(o)
    # ops: t 0, tt 1, x 2, y 3, z 4, ret 5
    N, O = o.def_loop(2, 0), o.def_loop(2, 1)
    L, R = o.use_loop(4, 0, 0), o.use_loop(4, 0, 1)
    cn = d["cnode"]
    assert not (cn[N] == cn[L] and cn[O] == cn[R])
    set_of = {(c[1], c[2]): c[3] for c in d["conflicts"]}
    sx = set_of[tuple(sorted((N, O)))]
    sz = set_of[tuple(sorted((L, R)))]
    assert sx != sz


def test_mlp_box_contracted():
    """P:1350 on the M1 pattern (SURVEY §8(c) MLP-c): the w1-def conflict and the
    matmul's (j, k) conflict form a box with no path across; both vertical edges
    are contracted and the two conflicts share one set, as with compatibility sets."""
    c = configs.get("mlp_c")
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, grouping=CONTRACTION)
    d = check_definition(o)
    assert [x[3] for x in d["conflicts"]] == [0, 0]
    d0 = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth).dump()
    assert d["conflicts"] == d0["conflicts"] and d["actions"] == d0["actions"]


@pytest.mark.parametrize("seed", range(40))
def test_definition_on_random_programs(seed):
    ir = models.random_program(seed, n_ops=12)
    try:
        o = _oracle(ir, (("a", 2, 1e10), ("b", 4, 1e11)))
    except OracleError as e:
        assert e.code == "E_LIMIT"
        return
    check_definition(o)


def test_linear_programs_contract_each_component():
    """Single-use programs have no conflicts, so every component
    contracts to one node."""
    for seed in range(20):
        o = _oracle(models.random_program(seed, n_ops=10, linear=True), (("a", 2, 1e10),))
        d = check_definition(o)
        assert d["conflicts"] == [] and d["contract_rejected"] == 0
        assert d["cnode"] == [l[4] for l in d["loops"]]


def test_stacked_layers_share_setgroups():
    """§3.6 on top of the heuristic: the number of SetGroups, hence the
    action count, does not grow with the number of stacked attention layers."""
    n_actions, n_groups = set(), set()
    for L in (2, 3, 4):
        d = check_definition(_oracle(models.stacked_attn(L)))
        n_actions.add(len(d["actions"]))
        n_groups.add(d["n_groups"])
    assert len(n_actions) == 1 and len(n_groups) == 1


# ------------------------------------------------------------------ library == oracle (host)
def _T():
    from paper_2508_15010_b200 import toast as T
    return T


@pytest.mark.parametrize("name", ["mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_4ax"])
def test_library_h0_equals_oracle(name):
    T = _T()
    c = configs.get(name)
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=-1,
                         grouping=T.GROUP_CONTRACTION)
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, grouping=CONTRACTION)
    da, do = a.dump(), o.dump()
    assert da.keys() == do.keys()
    for k in do:
        assert da[k] == do[k], k


def test_library_h0_equals_oracle_random():
    T = _T()
    for seed in range(40):
        ir = models.random_program(seed, n_ops=16)
        axes = [("a", 2, 1e10), ("b", 4, 1e11)]
        ea = eo = None
        try:
            da = T.build_analysis(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, cuda_device=-1,
                                  grouping=T.GROUP_CONTRACTION).dump()
        except T.ToastError as e:
            ea = e
        try:
            do = Oracle(ir, axes, 1e12, 1 << 40, 100.0, 1, 30, grouping=CONTRACTION).dump()
        except OracleError as e:
            eo = e
        assert (ea is None) == (eo is None), ir
        if ea is None:
            assert da == do, ir


def test_invalid_grouping_is_an_error():
    T = _T()
    c = configs.get("mlp_c")
    g = T.load_graph(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, -1)
    with pytest.raises(T.ToastError) as e:
        T.nda(g, 1, 30, 0, grouping=7)
    assert "conflict_grouping" in str(e.value)
    with pytest.raises(OracleError):
        Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, 1, 30, grouping=7)


# ------------------------------------------------------------------ GPU parity under the heuristic
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mlp_c", "gpt2", "gpt2_4ax"])
def test_gpu_rollout_and_eval_parity(name):
    import torch
    T = _T()
    c = configs.get(name)
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0,
                         grouping=T.GROUP_CONTRACTION)
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, grouping=CONTRACTION)
    n = 3000
    pre = torch.zeros((n, 32), dtype=torch.int16, device="cuda")
    seqs = torch.empty_like(pre)
    out = torch.empty((n, 256), dtype=torch.uint8, device="cuda")
    T.rollout_batch(a, pre, 77, 0, seqs, out)
    out2 = torch.empty_like(out)
    T.eval_batch(a, seqs, out2)
    torch.cuda.synchronize()
    g_seqs = seqs.cpu().numpy().view(np.uint16)
    o_seqs, oc = o.rollout(np.zeros((n, 32), np.uint16), seed=77, id_base=0)
    assert np.array_equal(g_seqs, o_seqs)
    assert T.as_costs(out).tobytes() == oc.tobytes()
    assert T.as_costs(out2).tobytes() == oc.tobytes()


@pytest.mark.gpu
def test_gpu_critical_path_under_contraction():
    """Both analysis options together (R22 cost model, R23 grouping): rollouts and
    evals bit-identical to the oracle's."""
    import torch
    T = _T()
    c = configs.get("gpt2")
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0,
                         cost_model=T.COST_CRITICAL_PATH, grouping=T.GROUP_CONTRACTION, dedup=T.DEDUP_OFF)
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cost_model=1,
               grouping=CONTRACTION)
    n = 2048
    pre = torch.zeros((n, 32), dtype=torch.int16, device="cuda")
    seqs = torch.empty_like(pre)
    out = torch.empty((n, 256), dtype=torch.uint8, device="cuda")
    T.rollout_batch(a, pre, 11, 3, seqs, out)
    torch.cuda.synchronize()
    o_seqs, oc = o.rollout(np.zeros((n, 32), np.uint16), seed=11, id_base=3)
    assert np.array_equal(seqs.cpu().numpy().view(np.uint16), o_seqs)
    assert T.as_costs(out).tobytes() == oc.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mlp_c", "attn_toy"])
def test_gpu_search_under_contraction_finds_bruteforce_optimum(name):
    """C16/C17 under R23: the GPU search reaches the oracle's exhaustive optimum
    over the heuristic's action space, and the search trace equals the oracle's."""
    T = _T()
    c = configs.get(name)
    dm = 700 if name == "attn_toy" else c.dm
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0,
                         grouping=T.GROUP_CONTRACTION)
    o = Oracle(c.ir, c.axes, c.flops_per_sec, dm, c.penalty_c, c.min_dims, c.max_depth, grouping=CONTRACTION)
    _, _best, bc = o.bruteforce()
    r = T.search(a, T.SearchOptions(seed=0, max_evals=20000, leaves_per_round=8, rollouts_per_leaf=32, patience=4))
    assert r["best"]["score"] == bc["score"]
    opts = T.SearchOptions(seed=3, max_evals=3000, leaves_per_round=4, rollouts_per_leaf=8, patience=3)
    r = T.search(a, opts)
    ro, _ = o.search(seed=3, max_evals=3000, L=4, R=8, patience=3)
    assert int(r["rounds"]) == int(ro["rounds"]) and int(r["evals"]) == int(ro["evals"])
    assert np.array_equal(r["best_seq"], ro["best_seq"]) and r["best"]["score"] == ro["best"]["score"]


@pytest.mark.parametrize("name", ["gpt24", "unet"])
def test_library_contraction_definition_at_full_size(name):
    """The library's contraction of the full-size configs checked against the
    definition directly: no conflict joined by the contracted graph, and
    every uncontracted edge would join one (maximal) — the latter through the
    merged node only, since a merge creates exactly the paths through it.  The M
    edges come from the oracle's loop table (equal to the library's, pinned by
    test_library_host.py::test_h0_analysis_equals_oracle)."""
    T = _T()
    c = configs.get(name)
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=-1,
                         grouping=T.GROUP_CONTRACTION)
    d = a.dump()
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth)
    assert d["loops"] == o.dump()["loops"]
    edges = [tuple(e) for e in o.edges()]
    cn = d["cnode"]
    conf = d["conflicts"]
    adj, radj = _adj(edges, cn), defaultdict(set)
    for x, ys in list(adj.items()):
        for y in ys:
            radj[y].add(x)
    partners = defaultdict(set)
    for _op, u, v, _s, _s0 in conf:
        partners[cn[u]].add(cn[v])
        partners[cn[v]].add(cn[u])
    # no conflict joined: for every node with conflict endpoints, no partner node is reachable from it
    for U, ps in partners.items():
        assert U not in ps
        assert not (ps & _reach(adj, U)), U
    # maximal: merging the two nodes of any split edge joins a conflict through the merged node
    split = {(cn[a_], cn[b]) for a_, b in edges if cn[a_] != cn[b]}
    assert len(split) > 0 and d["contract_rejected"] >= len(split)
    for X, Y in split:
        fwd = _reach(adj, X) | _reach(adj, Y)
        bwd = _reach(radj, X) | _reach(radj, Y)
        joined = any(partners[p] & fwd for p in bwd if p in partners)
        assert joined, (X, Y)
    # sets = unordered node pairs
    key_set = {}
    for _op, u, v, s, _s0 in conf:
        k = tuple(sorted((cn[u], cn[v])))
        assert key_set.setdefault(k, s) == s
    assert len(set(key_set.values())) == len(key_set)
