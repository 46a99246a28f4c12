"""Reading R22 ("runtime cost is accumulated along
the critical path"): the oracle's critical-path runtime pinned by closed forms
— a chain's critical path is the sum of its durations, parallel branches take
the max, a reduced partial adds its all_reduce after the producing op (Fig. 2c)
— and by properties (never above the straight-line sum, never below the
longest single op, the batch law).  CPU only."""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle
from workloads import configs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return open(os.path.join(GOLD, name)).read()


def action_id(d, loop, r, axis):
    sc = d["loops"][loop][5]
    for i, a in enumerate(d["actions"]):
        if a == [sc, r, axis]:
            return i + 1
    raise KeyError((loop, r, axis))


def test_chain_critical_path_is_the_sum():
    """Fig. 2a mlp is a chain x -> y -> z -> w: its critical path is the sum of
    the two matmuls' times, 1,048,576 / F + 524,288 / F."""
    F = 1e9
    o = Oracle(golden("mlp_fig2.ir"), [("b", 2, 1e10)], F, 1 << 40, 100.0, 1, cost_model=1)
    t0, _, _ = o.baseline()
    assert t0 == (0.0 + 1048576 / F) + 524288 / F
    s = Oracle(golden("mlp_fig2.ir"), [("b", 2, 1e10)], F, 1 << 40, 100.0, 1, cost_model=0)
    assert abs(t0 - s.baseline()[0]) <= 1e-15 * t0


BRANCHES = """def br(x: f32[64,32], w1: f32[32,128], w2: f32[32,16], w3: f32[16,128]) {
  y1 = matmul(x, w1)
  y2 = matmul(x, w2)
  y3 = matmul(y2, w3)
  z = add(y1, y3)
  return z
}"""


def test_parallel_branches_take_the_max():
    """y1 and y2 -> y3 run in parallel; the critical path is max(c(y1), c(y2) + c(y3))
    while the straight-line sum adds all three."""
    F = 1e12
    c1, c2, c3 = 2 * 64 * 32 * 128 / F, 2 * 64 * 32 * 16 / F, 2 * 64 * 16 * 128 / F
    o = Oracle(BRANCHES, [("a", 2, 1e10)], F, 1 << 40, 100.0, 1, cost_model=1)
    t0, _, _ = o.baseline()
    assert t0 == max(c1, c2 + c3)
    s = Oracle(BRANCHES, [("a", 2, 1e10)], F, 1 << 40, 100.0, 1, cost_model=0)
    assert abs(s.baseline()[0] - (c1 + c2 + c3)) <= 1e-15 * (c1 + c2 + c3)


def test_fig2c_all_reduce_on_the_critical_path():
    """Fig. 2c: B->b, U->m.  Both matmuls run on local shards
    (y: 2*128*32*32, w: 2*128*32*16 flops) and the all_reduce{m} of w (8,192 B,
    ring time (n-1)*2*8192/n / bw_m) follows on the path to the return."""
    F, bw = 1e9, 1e11
    o = Oracle(golden("mlp_fig2.ir"), [("b", 2, 1e10), ("m", 2, bw)], F, 1 << 40, 100.0, 1, cost_model=1)
    d = o.dump()
    c = o.eval(Oracle.seqs([[action_id(d, 0, 0, 0), action_id(d, 3, 0, 1)]]))[0]
    cy, cw = (2 * 128 * 32 * 32) / F, (2 * 128 * 32 * 16) / F
    # the edge's collective time, axis by axis in mesh order (b carries nothing)
    term_b = ((2 - 1.0) * (0.0 + 0.0) + ((2 - 1.0) * (2.0 * 0.0 + 0.0)) / 2) / 1e10
    term_m = ((2 - 1.0) * (0.0 + 0.0) + ((2 - 1.0) * (2.0 * 8192.0 + 0.0)) / 2) / bw
    m_ar = (0.0 + term_b) + term_m
    assert c["runtime_s"] == ((0.0 + cy) + cw) + m_ar
    assert int(c["payload"][1][2]) == 8192 and int(c["n_collectives"]) == 1


@pytest.mark.parametrize("name", ["mlp_c", "gpt2", "attn_toy"])
def test_critical_path_properties(name):
    """For every rollout: critical path <= straight-line sum (every path is a
    subset of the sum's terms), >= the longest single op's compute time, and
    every other field (payloads, peak, FLOPs, key) is the sum model's."""
    c = configs.get(name)
    o1 = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cost_model=1)
    o0 = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cost_model=0)
    seqs, c1 = o1.rollout(np.zeros((300, 32), np.uint16), seed=4)
    c0 = o0.eval(seqs)
    ok = c1["status"] == 0
    assert ok.any()
    assert (c1["runtime_s"][ok] <= c0["runtime_s"][ok] * (1 + 1e-12)).all()
    assert (c1["runtime_s"][ok] > 0).all()
    for f in ("peak_bytes", "flops", "state_key", "payload", "count", "n_collectives", "status"):
        assert np.array_equal(c1[f], c0[f]), f
    t01, _, _ = o1.baseline()
    t00, _, _ = o0.baseline()
    assert t01 <= t00 * (1 + 1e-12)


def test_batch_law_critical_path():
    """Pure batch sharding over b devices divides every op's work by b and
    moves no data: RT = 1/b on the critical path too."""
    for b in (2, 4, 8):
        o = Oracle(golden("mlp_fig2.ir"), [("b", b, 1e10)], 1e9, 1 << 40, 100.0, 1, cost_model=1)
        d = o.dump()
        c = o.eval(Oracle.seqs([[action_id(d, 0, 0, 0)]]))[0]
        assert abs(c["score"] - 1.0 / b) <= 1e-15
