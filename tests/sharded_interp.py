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
# Elementwise ops are total, bounded stand-ins for their names (log(|x|+1),
# 1/(|x|+1), ...): an elementwise function commutes with any sharding, so the
# check does not depend on which function it is, and bounded functions keep
# deep programs (backward + Adam) finite so the comparison stays sharp.
def _sig(x):
    return 1.0 / (1.0 + np.exp(-np.clip(x, -30.0, 30.0)))


UNARY = {
    "relu": lambda x, c: np.maximum(x, 0.0), "neg": lambda x, c: -x, "exp": lambda x, c: np.exp(np.clip(x, -30.0, 30.0)),
    "log": lambda x, c: np.log(np.abs(x) + 1.0), "tanh": lambda x, c: np.tanh(x), "abs": lambda x, c: np.abs(x),
    "square": lambda x, c: x * x, "sigmoid": lambda x, c: _sig(x),
    "scale": lambda x, c: x * float(c[0]), "add_s": lambda x, c: x + float(c[0]),
    "recip": lambda x, c: 1.0 / (np.abs(x) + 1.0), "rsqrt": lambda x, c: 1.0 / np.sqrt(np.abs(x) + 1.0),
    "sqrt": lambda x, c: np.sqrt(np.abs(x)), "gelu": lambda x, c: x * _sig(1.702 * x), "silu": lambda x, c: x * _sig(x),
    "sign": lambda x, c: np.sign(x), "ones_like": lambda x, c: np.ones_like(x),
    "pow_s": lambda x, c: np.abs(x) ** float(c[0]), "convert": lambda x, c: x, "stop_gradient": lambda x, c: x,
    "cos": lambda x, c: np.cos(x), "sin": lambda x, c: np.sin(x),
}
BINARY = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": lambda a, b: a * b / (b * b + 1e-6),
          "max": np.maximum, "min": np.minimum, "pow": lambda a, b: (np.abs(a) + 1.0) ** np.clip(b, -2.0, 2.0)}
COMBINE = {"add": np.add, "max": np.maximum, "min": np.minimum, "mul": np.multiply}
REDUCE = {"add": np.sum, "max": np.max, "min": np.min, "mul": np.prod}


def _unary(kind):
    if kind in UNARY:
        return UNARY[kind]
    if kind.startswith("d_"):      # the derivative of an elementwise function: elementwise too
        return lambda x, c: np.tanh(x) + 0.5
    return None


def _attrs(a: str):
    return [g.split(",") if g else [] for g in a.split(";")] if a else []


def _ints1(attrs, g=0):
    return [int(v) for v in attrs[g]] if g < len(attrs) else []


def apply_op(kind: str, attrs, args, out_shape=None):
    """numpy semantics of one IR op; out_shape (local) fixes a broadcast's new
    extent and a segment_sum's segment count."""
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        return _apply(kind, attrs, args, out_shape)


def _index(idx, n):
    """gather / segment_sum indices: the i32 values, taken mod the table's rows
    (a total function, so any input is a valid index)"""
    return np.mod(np.floor(idx).astype(np.int64), n)


def _conv_same(x, w):
    """conv2d, NHWC x HWIO -> NHWC, stride 1, 'same' zero padding"""
    KH, KW = w.shape[0], w.shape[1]
    ph, pw = (KH - 1) // 2, (KW - 1) // 2
    N, H, W, _ = x.shape
    xp = np.pad(x, ((0, 0), (ph, KH - 1 - ph), (pw, KW - 1 - pw), (0, 0)))
    out = np.zeros((N, H, W, w.shape[3]))
    for i in range(KH):
        for j in range(KW):
            out += np.einsum("nhwc,cd->nhwd", xp[:, i:i + H, j:j + W, :], w[i, j])
    return out


def _conv_bwd_input(dy, w):
    """the adjoint of _conv_same in x: dx[n,h,w,c] = sum dy[n,h-i+ph,w-j+pw,d] w[i,j,c,d]"""
    KH, KW = w.shape[0], w.shape[1]
    ph, pw = (KH - 1) // 2, (KW - 1) // 2
    N, H, W, _ = dy.shape
    dp = np.pad(dy, ((0, 0), (KH - 1 - ph, ph), (KW - 1 - pw, pw), (0, 0)))
    out = np.zeros((N, H, W, w.shape[2]))
    for i in range(KH):
        for j in range(KW):
            a, b = KH - 1 - i, KW - 1 - j
            out += np.einsum("nhwd,cd->nhwc", dp[:, a:a + H, b:b + W, :], w[i, j])
    return out


def _conv_bwd_filter(x, dy, KH, KW):
    """the adjoint of _conv_same in w: dw[i,j,c,d] = sum x[n,h+i-ph,w+j-pw,c] dy[n,h,w,d]"""
    ph, pw = (KH - 1) // 2, (KW - 1) // 2
    N, H, W, _ = x.shape
    xp = np.pad(x, ((0, 0), (ph, KH - 1 - ph), (pw, KW - 1 - pw), (0, 0)))
    out = np.zeros((KH, KW, x.shape[3], dy.shape[3]))
    for i in range(KH):
        for j in range(KW):
            out[i, j] = np.einsum("nhwc,nhwd->cd", xp[:, i:i + H, j:j + W, :], dy)
    return out


def _dot_general(a, b, lb, rb, lc, rc):
    """result dims: batch (lhs order), lhs free, rhs free; contracting dims summed"""
    letters = iter("abcdefghijklmnopqrstuvwxyz")
    sa = [None] * a.ndim
    sb = [None] * b.ndim
    for x, y in list(zip(lb, rb)) + list(zip(lc, rc)):
        sa[x] = sb[y] = next(letters)
    for i in range(a.ndim):
        if sa[i] is None:
            sa[i] = next(letters)
    for i in range(b.ndim):
        if sb[i] is None:
            sb[i] = next(letters)
    res = [sa[x] for x in lb] + [sa[i] for i in range(a.ndim) if i not in lb and i not in lc] + \
          [sb[i] for i in range(b.ndim) if i not in rb and i not in rc]
    return np.einsum("".join(sa) + "," + "".join(sb) + "->" + "".join(res), a, b)


def _apply(kind, attrs, args, out_shape):
    f = _unary(kind)
    if f is not None:
        return f(args[0], attrs[0] if attrs else None)
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
    if kind == "dot_general":
        return _dot_general(args[0], args[1], *[_ints1(attrs, g) for g in range(4)])
    if kind == "conv2d":
        return _conv_same(args[0], args[1])
    if kind == "conv2d_bwd_input":
        return _conv_bwd_input(args[0], args[1])
    if kind == "conv2d_bwd_filter":
        kh, kw = _ints1(attrs)
        return _conv_bwd_filter(args[0], args[1], kh, kw)
    if kind == "resample":
        mode, fct = attrs[0][0], int(attrs[0][1])
        x = args[0]
        if mode == "up":       # nearest neighbour
            return np.repeat(np.repeat(x, fct, axis=1), fct, axis=2)
        N, H, W, C = x.shape   # average pooling over f x f windows
        return x.reshape(N, H // fct, fct, W // fct, fct, C).mean(axis=(2, 4))
    if kind == "concat":
        return np.concatenate(args, axis=int(attrs[0][0]))
    if kind == "slice":
        d, s, n = _ints1(attrs)
        return np.take(args[0], np.arange(s, s + n), axis=d)
    if kind == "pad":
        d, lo, hi = _ints1(attrs)
        w = [(0, 0)] * args[0].ndim
        w[d] = (lo, hi)
        return np.pad(args[0], w)
    if kind == "gather":          # tbl[n,f], idx[e..] -> [e.., f]
        tbl, idx = args
        return tbl[_index(idx, tbl.shape[0])]
    if kind == "segment_sum":     # dat[e.., f], idx[e..] -> [n, f]
        dat, idx = args
        n = out_shape[0] if out_shape is not None else int(attrs[0][0])
        out = np.zeros((n, dat.shape[-1]))
        np.add.at(out, _index(idx, n).reshape(-1), dat.reshape(-1, dat.shape[-1]))
        return out
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
    out = {}
    for n, dt, shape in params:
        if dt == "i32":    # indices / labels: small non-negative integers
            out[n] = rng.integers(0, 8, size=shape).astype(np.float64)
        else:
            out[n] = rng.integers(-3, 4, size=shape).astype(np.float64) / 2.0
    return out


def close(a, b) -> bool:
    """equal up to summation order: |a - b| <= 1e-9 (max |b| + 1) elementwise"""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return False
    fin = np.isfinite(b)
    if not np.array_equal(np.isfinite(a), fin):
        return False
    if not fin.any():
        return True
    tol = 1e-9 * (np.max(np.abs(b[fin])) + 1.0)
    return bool(np.all(np.abs(a[fin] - b[fin]) <= tol))


# ------------------------------------------------------------------ the lowered program
# a collective carries one {key=value,...} group per move; an all_to_all whose
# single-axis moves block one another lists them all, joined by '+', with one
# payload per move (reading R20)
_STMT = re.compile(r"(%[\w.]+)\s*=\s*([\w]+)(?:\[([^\]]*)\])?((?:\+?\{[^}]*\})*)(?:\(([^)]*)\))?\s+(\w+)\s+\[([^\]]*)\]"
                   r"\s+local\[([^\]]*)\]\s+layout\[([^\]]*)\]\s+partial\[(\d+)\](?:\s+bytes=(\d+(?:\+\d+)*))?")


def _ints(s):
    return [int(x) for x in s.split(",") if x.strip()]


class ShardError(AssertionError):
    pass


ELEM = {"f32": 4, "bf16": 2, "f16": 2, "i32": 4, "f64": 8, "i64": 8}


def run_lowered(low: str, ir: str, inputs: dict, strict: bool = True, stats: dict | None = None):
    """Execute the lowered program on every device.  Returns the payload totals
    {(axis, collective name): bytes}; raises ShardError on any inconsistency.

    strict=False trusts every compute op's declared layout and partial axes
    (no comparison with the derived ones), so only the values decide — the
    tests use it to show that the values alone catch a wrong rule.  stats, if
    given, collects per op kind how often a result dim was sharded and how
    often the result was partial (coverage of the rules exercised)."""
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
            if not np.all(np.isnan(cur)) and not close(cur, data[d]):
                raise ShardError(f"{name}: replicas disagree")
            g[sl] = data[d]
        return out

    def _multi_all_to_all(name, op, groups, args, dtype, gshape, layout, part, nbytes):
        """one all_to_all over the product of several axes: every move at once"""
        if op != "all_to_all":
            raise ShardError(f"{name}: only an all_to_all may list several moves")
        data, L0, P0, comb = env[args[0]]
        want = list(L0)
        for kv in groups:
            bit, i, j = 1 << kv["axis"], kv["from"], kv["to"]
            if not L0[i] & bit or want[j] & bit:
                raise ShardError(f"{name}: bad all_to_all move {kv}")
            want[i] &= ~bit
            want[j] |= bit
        if want != layout or P0 != part:
            raise ShardError(f"{name}: all_to_all gives layout {want}, declared {layout}")
        glob = reassemble(args[0], data, L0, P0, gshape)
        new = {d: shard(glob[pcoord(d, P0)], d, layout) for d in devices}
        each = [int(b) for b in (nbytes or "").split("+") if b]
        if len(each) != len(groups):
            raise ShardError(f"{name}: one payload per move")
        moved = data[devices[0]].size * ELEM[dtype]
        for kv, b in zip(groups, each):
            if b != moved:
                raise ShardError(f"{name}: declared {b} bytes, the ring model charges {moved}")
            payload[(kv["axis"], op)] = payload.get((kv["axis"], op), 0) + b
        env[name] = (new, layout, P0, comb)

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
        seen = part
        for m_ in layout:
            if m_ & seen:
                raise ShardError(f"{name}: a mesh axis shards two dims (or a dim and the partial sum)")
            seen |= m_
        if op == "param":
            if part:
                raise ShardError(f"{name}: a parameter cannot be partial")
            env[name] = ({d: shard(inputs[name[1:]], d, layout) for d in devices}, layout, 0, "add")
            continue
        if coll:
            groups = [{x.split("=")[0]: int(x.split("=")[1]) for x in grp.split(",")}
                      for grp in re.findall(r"\{([^}]*)\}", coll)]
            if len(groups) > 1:
                _multi_all_to_all(name, op, groups, args, dtype, gshape, layout, part, nbytes)
                continue
            kv = groups[0]
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
        if _unary(kind) is not None:
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
        elif kind == "dot_general":
            lb, rb, lc, rc = [_ints1(attrs, g) for g in range(4)]
            La, Lb = Ls
            for x, y in list(zip(lb, rb)) + list(zip(lc, rc)):
                if La[x] != Lb[y]:
                    raise ShardError(f"{name}: tied dims {x}/{y} have layouts {La[x]} and {Lb[y]}")
            for x in lc:               # a sharded contracting dim leaves partial sums
                derived_p |= La[x]
            derived = [La[x] for x in lb] + [La[i] for i in range(len(La)) if i not in lb and i not in lc] + \
                      [Lb[i] for i in range(len(Lb)) if i not in rb and i not in rc]
        elif kind in ("conv2d", "conv2d_bwd_input"):
            Lx, Lw = Ls
            cx, cw = (3, 2) if kind == "conv2d" else (3, 3)   # contracted channel of the input / of the filter
            if Lx[cx] != Lw[cw]:
                raise ShardError(f"{name}: contracted channels have layouts {Lx[cx]} and {Lw[cw]}")
            if Lw[0] or Lw[1]:
                raise ShardError(f"{name}: a sharded filter window has no local convolution")
            derived_p = Lx[cx]
            derived = [Lx[0], Lx[1], Lx[2], Lw[3] if kind == "conv2d" else Lw[2]]
        elif kind == "conv2d_bwd_filter":
            Lx, Ld = Ls
            for i in range(3):         # N, H, W are summed over
                if Lx[i] != Ld[i]:
                    raise ShardError(f"{name}: summed dim {i} has layouts {Lx[i]} and {Ld[i]}")
                derived_p |= Lx[i]
            derived = [0, 0, Lx[3], Ld[3]]
        elif kind in ("resample", "slice", "pad"):
            derived = list(Ls[0])
        elif kind == "concat":
            if any(L != Ls[0] for L in Ls):
                raise ShardError(f"{name}: concatenated operands have layouts {Ls}")
            derived = list(Ls[0])
        elif kind == "gather":
            Lt, Li = Ls
            derived = list(Li) + [Lt[1]]
        elif kind == "segment_sum":
            Ld, Li = Ls
            ke = len(Li)
            if list(Ld[:ke]) != list(Li):
                raise ShardError(f"{name}: data and index layouts {Ld[:ke]} and {Li} differ")
            for x in Ld[:ke]:          # a sharded segment-member dim leaves partial sums
                derived_p |= x
            derived = [layout[0], Ld[ke]]   # the segment dim: as declared (the values decide)
        else:
            raise NotImplementedError(kind)
        if stats is not None:
            st = stats.setdefault(kind, [0, 0, 0])
            st[0] += 1
            st[1] += any(layout)
            st[2] += part != 0
        if strict and (derived != layout or derived_p != part):
            raise ShardError(f"{name}: the op gives layout {derived} partial {derived_p}, declared {layout} partial {part}")
        try:
            data = {d: apply_op(kind, attrs, [v[0][d] for v in vals], out_shape=lshape) for d in devices}
        except (IndexError, ValueError) as e:   # the op has no meaning on these local blocks
            raise ShardError(f"{name}: the local operands do not fit the op ({e})")
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
        if not close(glob, ref):
            raise ShardError(f"returned {o} differs from the unsharded program")
    return payload
