"""A sharded interpreter for the device-local programs of toast_lower (SURVEY
§8(f) NEXT-1) — TEST INFRASTRUCTURE.

It runs the original program on global float64 arrays (its own IR parser and
op semantics, written from the IR grammar), then runs the
lowered program on every device of the mesh: every value is a
local array per device plus its layout (per dim, the mesh axes sharding it)
and its partial axes.  A shard is the canonical block of the layout (block
index mixed-radix in the device's coordinates, highest mesh axis major —
reading R21).

* A compute op sees only its device's local operands.  Operands whose dims
  the op ties (elementwise operands, a matmul's contraction dim) must have
  the same layout there, no operand may be partial (every use reduces a
  partial value, reading G27), and the result's layout and partial axes are
  DERIVED from the operands and compared with the ones the lowering declares
  (a sharded contracted / reduced dim leaves the result partial over its axes).
* A collective redistributes the value as its name says over the groups of
  devices that differ in one mesh coordinate: the interpreter reassembles
  the value (one global array per combination of partial-axis coordinates,
  checking that replicas agree), combines the partials an all_reduce /
  reduce_scatter removes (sum, or the reduction's own combiner), and hands
  every device the canonical block of the new layout.  Each step's declared
  layout change must be the collective's (all_gather: axis A leaves dim i;
  all_to_all: A moves from dim i to dim j; reduce_scatter: A leaves the
  partial set and joins dim j; all_reduce: A leaves the partial set; slice:
  A joins dim j), and its declared payload must be the ring model's
  (G13: all_gather / all_to_all the input shard, reduce_scatter the output
  shard, all_reduce the buffer).
* Every returned value, reassembled, must equal the unsharded result.

What this does not check is the device ORDER a multi-axis dim needs (an
all_gather of the major axis of a two-axis dim leaves a strided block that a
real runtime fixes with a permute the cost model does not charge) — see
DESIGN.md reading R21.
"""
from __future__ import annotations

import itertools
import re

import numpy as np


# ------------------------------------------------------------------ op semantics (global and local alike)
UNARY = {
    "relu": lambda x, c: np.maximum(x, 0.0), "neg": lambda x, c: -x, "exp": lambda x, c: np.exp(x),
    "log": lambda x, c: np.log(np.abs(x) + 1.0), "tanh": lambda x, c: np.tanh(x), "abs": lambda x, c: np.abs(x),
    "square": lambda x, c: x * x, "sigmoid": lambda x, c: 1.0 / (1.0 + np.exp(-x)),
    "scale": lambda x, c: x * float(c[0]), "add_s": lambda x, c: x + float(c[0]),
}
BINARY = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": lambda a, b: a / b,
          "max": np.maximum, "min": np.minimum}
COMBINE = {"add": np.add, "max": np.maximum, "min": np.minimum, "mul": np.multiply}
REDUCE = {"add": np.sum, "max": np.max, "min": np.min, "mul": np.prod}


def _attrs(a: str):
    return [g.split(",") if g else [] for g in a.split(";")] if a else []


def apply_op(kind: str, attrs, args, out_shape=None):
    """numpy semantics of one IR op; out_shape (local) fixes a broadcast's new extent."""
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        return _apply(kind, attrs, args, out_shape)


def _apply(kind, attrs, args, out_shape):
    if kind in UNARY:
        return UNARY[kind](args[0], attrs[0] if attrs else None)
    if kind in BINARY:
        return BINARY[kind](args[0], args[1])
    if kind == "transpose":
        return np.transpose(args[0], [int(p) for p in attrs[0]])
    if kind == "reduce":
        dims = tuple(int(d) for d in attrs[0][:-1])
        return REDUCE[attrs[0][-1]](args[0], axis=dims)
    if kind == "broadcast":
        l, e = int(attrs[0][0]), int(attrs[0][1])
        if out_shape is not None:
            e = out_shape[l]
        return np.repeat(np.expand_dims(args[0], l), e, axis=l)
    if kind == "matmul":
        return args[0] @ args[1]
    raise NotImplementedError(kind)


# ------------------------------------------------------------------ the original program
_DEF = re.compile(r"def\s+\w+\s*\((.*?)\)\s*\{(.*)\}", re.S)


def parse_ir(text: str):
    text = "\n".join(l.split("#", 1)[0] for l in text.splitlines())
    m = _DEF.search(text)
    params = []
    for p in re.finditer(r"(\w+)\s*:\s*(\w+)\s*\[([^\]]*)\]", m.group(1)):
        params.append((p.group(1), p.group(2), tuple(int(x) for x in p.group(3).split(",") if x.strip())))
    body, rets = [], []
    for line in m.group(2).splitlines():
        line = line.strip()
        if not line:
            continue
        if line.startswith("return"):
            rets = [r.strip() for r in line[len("return"):].split(",")]
            continue
        b = re.match(r"(\w+)\s*=\s*(\w+)(?:\[([^\]]*)\])?\s*\(([^)]*)\)", line)
        body.append((b.group(1), b.group(2), _attrs(b.group(3) or ""), [x.strip() for x in b.group(4).split(",") if x.strip()]))
    return params, body, rets


def run_global(ir: str, inputs: dict):
    params, body, rets = parse_ir(ir)
    env = dict(inputs)
    for name, kind, attrs, ops in body:
        env[name] = apply_op(kind, attrs, [env[o] for o in ops])
    return {r: env[r] for r in rets}, rets


def random_inputs(ir: str, seed: int):
    rng = np.random.default_rng(seed)
    params, _, _ = parse_ir(ir)
    return {n: rng.integers(-3, 4, size=shape).astype(np.float64) / 2.0 for n, _, shape in params}


# ------------------------------------------------------------------ the lowered program
_STMT = re.compile(r"(%[\w.]+)\s*=\s*([\w]+)(?:\[([^\]]*)\])?(?:\{([^}]*)\})?(?:\(([^)]*)\))?\s+(\w+)\s+\[([^\]]*)\]"
                   r"\s+local\[([^\]]*)\]\s+layout\[([^\]]*)\]\s+partial\[(\d+)\](?:\s+bytes=(\d+))?")


def _ints(s):
    return [int(x) for x in s.split(",") if x.strip()]


class ShardError(AssertionError):
    pass


ELEM = {"f32": 4, "bf16": 2, "f16": 2, "i32": 4, "f64": 8, "i64": 8}


def run_lowered(low: str, ir: str, inputs: dict):
    """Execute the lowered program on every device.  Returns the payload totals
    {(axis, collective name): bytes}; raises ShardError on any inconsistency."""
    lines = [l for l in low.splitlines() if l.strip() and not l.startswith("#")]
    sizes = [int(kv.split("=")[1]) for kv in lines[0].split()[1:]]
    NA = len(sizes)
    devices = list(itertools.product(*[range(n) for n in sizes]))
    G, _ = run_global(ir, inputs)
    env = {}          # name -> (local data per device, layout, partial, combiner)
    payload = {}

    def block(d, n, mask):
        k, b = 1, 0
        for A in reversed(range(NA)):
            if (mask >> A) & 1:
                b = b * sizes[A] + d[A]
                k *= sizes[A]
        if n % k:
            raise ShardError(f"extent {n} not divisible by {k}")
        w = n // k
        return slice(b * w, (b + 1) * w)

    def shard(glob, d, layout):
        return glob[tuple(block(d, glob.shape[i], layout[i]) for i in range(glob.ndim))]

    def pcoord(d, partial):
        return tuple(d[A] for A in range(NA) if (partial >> A) & 1)

    def reassemble(name, data, layout, partial, gshape):
        """one global array per partial-coordinate tuple; replicas must agree"""
        out = {}
        for d in devices:
            key = pcoord(d, partial)
            g = out.setdefault(key, np.full(gshape, np.nan))
            sl = tuple(block(d, gshape[i], layout[i]) for i in range(len(gshape)))
            cur = g[sl]
            if not np.all(np.isnan(cur)) and not np.allclose(cur, data[d], rtol=1e-9, atol=1e-9, equal_nan=True):
                raise ShardError(f"{name}: replicas disagree")
            g[sl] = data[d]
        return out

    for line in lines[1:]:
        if line.startswith("return"):
            outs = [x.strip() for x in line[len("return"):].split(",")]
            break
        m = _STMT.match(line)
        if not m:
            raise ShardError(f"cannot parse: {line}")
        name, op, attr, coll, args, dtype, gsh, lsh, lay, part, nbytes = m.groups()
        gshape, lshape, layout, part = _ints(gsh), _ints(lsh), _ints(lay), int(part)
        args = [x.strip() for x in (args or "").split(",") if x.strip()]
        for i in range(len(gshape)):
            k = 1
            for A in range(NA):
                if (layout[i] >> A) & 1:
                    k *= sizes[A]
            if gshape[i] % k or gshape[i] // k != lshape[i]:
                raise ShardError(f"{name}: local extent {lshape[i]} does not match layout {layout[i]}")
        if op == "param":
            if part:
                raise ShardError(f"{name}: a parameter cannot be partial")
            env[name] = ({d: shard(inputs[name[1:]], d, layout) for d in devices}, layout, 0, "add")
            continue
        if coll:
            kv = {x.split("=")[0]: int(x.split("=")[1]) for x in coll.split(",")}
            A, bit = kv["axis"], 1 << kv["axis"]
            data, L0, P0, comb = env[args[0]]
            want = list(L0)
            P1 = P0
            if op == "all_gather":
                i = kv["dim"]
                if not want[i] & bit:
                    raise ShardError(f"{name}: all_gather of an axis the dim does not hold")
                want[i] &= ~bit
            elif op == "all_to_all":
                i, j = kv["from"], kv["to"]
                if not want[i] & bit or want[j] & bit:
                    raise ShardError(f"{name}: bad all_to_all")
                want[i] &= ~bit
                want[j] |= bit
            elif op in ("reduce_scatter", "all_reduce"):
                if not P0 & bit:
                    raise ShardError(f"{name}: {op} of a value not partial over axis {A}")
                P1 = P0 & ~bit
                if op == "reduce_scatter":
                    if want[kv["dim"]] & bit:
                        raise ShardError(f"{name}: bad reduce_scatter")
                    want[kv["dim"]] |= bit
            elif op == "slice":
                if want[kv["dim"]] & bit or P0 & bit:
                    raise ShardError(f"{name}: bad slice")
                want[kv["dim"]] |= bit
            else:
                raise ShardError(op)
            if want != layout or P1 != part:
                raise ShardError(f"{name}: {op} gives layout {want} partial {P1}, declared {layout} partial {part}")
            glob = reassemble(args[0], data, L0, P0, gshape)
            if P1 != P0:   # combine the partials over axis A
                merged = {}
                for key, g in glob.items():
                    # key lists the coordinates of P0's axes in mesh order; drop axis A's
                    axes0 = [x for x in range(NA) if (P0 >> x) & 1]
                    k1 = tuple(c for x, c in zip(axes0, key) if x != A)
                    merged[k1] = g if k1 not in merged else COMBINE[comb](merged[k1], g)
                glob = merged
            new = {d: shard(glob[pcoord(d, P1)], d, layout) for d in devices}
            if nbytes is not None:
                elem = ELEM[dtype]
                d0 = devices[0]
                moved = (data[d0].size if op in ("all_gather", "all_to_all", "all_reduce") else new[d0].size) * elem
                if int(nbytes) != moved:
                    raise ShardError(f"{name}: declared {nbytes} bytes, the ring model charges {moved}")
                payload[(A, op)] = payload.get((A, op), 0) + int(nbytes)
            elif op != "slice":
                raise ShardError(f"{name}: collective without a payload")
            env[name] = (new, layout, P1, comb)
            continue
        # compute op on local operands
        kind, attrs = op, _attrs(attr or "")
        vals = [env[x] for x in args]
        for v in vals:
            if v[2]:
                raise ShardError(f"{name}: operand is partial (every use must reduce it)")
        Ls = [v[1] for v in vals]
        derived_p, comb = 0, "add"
        if kind in UNARY:
            derived = list(Ls[0])
        elif kind in BINARY:
            if Ls[0] != Ls[1]:
                raise ShardError(f"{name}: elementwise operands have layouts {Ls[0]} and {Ls[1]}")
            derived = list(Ls[0])
        elif kind == "transpose":
            derived = [Ls[0][int(p)] for p in attrs[0]]
        elif kind == "reduce":
            dims = [int(x) for x in attrs[0][:-1]]
            derived = [Ls[0][q] for q in range(len(Ls[0])) if q not in dims]
            for q in dims:
                derived_p |= Ls[0][q]
            comb = attrs[0][-1]
        elif kind == "broadcast":
            l = int(attrs[0][0])
            derived = list(Ls[0][:l]) + [layout[l]] + list(Ls[0][l:])   # the new dim: as declared
        elif kind == "matmul":
            if Ls[0][1] != Ls[1][0]:
                raise ShardError(f"{name}: contraction layouts {Ls[0][1]} and {Ls[1][0]} differ")
            derived = [Ls[0][0], Ls[1][1]]
            derived_p = Ls[0][1]
        else:
            raise NotImplementedError(kind)
        if derived != layout or derived_p != part:
            raise ShardError(f"{name}: the op gives layout {derived} partial {derived_p}, declared {layout} partial {part}")
        data = {d: apply_op(kind, attrs, [v[0][d] for v in vals], out_shape=lshape) for d in devices}
        for d in devices:
            if list(data[d].shape) != lshape:
                raise ShardError(f"{name}: local shape {list(data[d].shape)} != declared {lshape}")
        env[name] = (data, layout, part, comb)
    for o in outs:
        data, L, P, _ = env[o]
        if P:
            raise ShardError(f"returned {o} is still partial")
        ref = G[o[1:].split(".")[0]]
        glob = reassemble(o, data, L, 0, list(ref.shape))[()]
        if not np.allclose(glob, ref, rtol=1e-9, atol=1e-9, equal_nan=True):
            raise ShardError(f"returned {o} differs from the unsharded program")
    return payload
