"""Text-IR builder for the synthetic workloads (input generation only).

This module emits straight-line tensor programs in the text IR (DESIGN.md
§"IR") — a forward pass, a reverse-mode backward pass and Adam — shaped like
the paper's models (§5.1).  It holds none of the
method's arithmetic: no names, loops, conflicts, shardings or costs; it only
writes programs.  Both the oracle and the CUDA path consume its output.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class _Param:
    name: str
    dtype: str
    shape: tuple
    trainable: bool
    kind: str  # "weight" | "opt" | "data"


@dataclass
class _Rec:
    out: str
    kind: str
    attrs: object
    operands: tuple
    diff: bool


def _fmt_attr(a) -> str:
    if a is None:
        return ""
    if isinstance(a, str):
        return f"[{a}]"
    return "[" + ",".join(str(x) for x in a) + "]"


class Builder:
    def __init__(self, name: str):
        self.name = name
        self.params: list[_Param] = []
        self.lines: list[str] = []
        self.shape: dict[str, tuple] = {}
        self.dtype: dict[str, str] = {}
        self.tape: list[_Rec] = []
        self._n = 0
        self.returns: list[str] = []

    # ------------------------------------------------------------------
    def _fresh(self, hint: str) -> str:
        self._n += 1
        return f"{hint}{self._n}"

    def param(self, name: str, dtype: str, shape, trainable: bool = True, kind: str = "weight") -> str:
        assert name not in self.shape, name
        self.params.append(_Param(name, dtype, tuple(shape), trainable, kind))
        self.shape[name] = tuple(shape)
        self.dtype[name] = dtype
        return name

    def data(self, name: str, dtype: str, shape) -> str:
        return self.param(name, dtype, shape, trainable=False, kind="data")

    def _emit(self, kind, operands, shape, dtype, attrs=None, diff=True, hint="v") -> str:
        out = self._fresh(hint)
        self.lines.append(f"  {out} = {kind}{_fmt_attr(attrs)}({', '.join(operands)})")
        self.shape[out] = tuple(shape)
        self.dtype[out] = dtype
        self.tape.append(_Rec(out, kind, attrs, tuple(operands), diff))
        return out

    # ---------------------------------------------------------------- ops
    def unary(self, kind: str, x: str, attr=None, diff=True) -> str:
        return self._emit(kind, [x], self.shape[x], self.dtype[x], attrs=attr, diff=diff)

    def convert(self, x: str, dt: str) -> str:
        if self.dtype[x] == dt:
            return x
        return self._emit("convert", [x], self.shape[x], dt, attrs=dt)

    def scale(self, x: str, c: float) -> str:
        return self.unary("scale", x, [repr(float(c))])

    def add_s(self, x: str, c: float) -> str:
        return self.unary("add_s", x, [repr(float(c))])

    def binary(self, kind: str, a: str, b: str) -> str:
        assert self.shape[a] == self.shape[b], (kind, a, b, self.shape[a], self.shape[b])
        return self._emit(kind, [a, b], self.shape[a], self.dtype[a])

    def add(self, a, b):
        return self.binary("add", a, b)

    def sub(self, a, b):
        return self.binary("sub", a, b)

    def mul(self, a, b):
        return self.binary("mul", a, b)

    def div(self, a, b):
        return self.binary("div", a, b)

    def transpose(self, x: str, perm) -> str:
        perm = list(perm)
        if perm == list(range(len(perm))):
            return x
        s = self.shape[x]
        return self._emit("transpose", [x], [s[p] for p in perm], self.dtype[x], attrs=perm)

    def reduce(self, x: str, dims, comb: str = "add", diff=True) -> str:
        dims = sorted(dims)
        s = self.shape[x]
        return self._emit("reduce", [x], [e for i, e in enumerate(s) if i not in dims], self.dtype[x],
                          attrs=list(dims) + [comb], diff=diff)

    def broadcast(self, x: str, l: int, e: int) -> str:
        s = list(self.shape[x])
        s.insert(l, e)
        return self._emit("broadcast", [x], s, self.dtype[x], attrs=[l, e])

    def broadcast_to(self, x: str, target_shape, positions) -> str:
        """Insert the dims at `positions` (ascending, in the target) of target_shape."""
        for p in sorted(positions):
            x = self.broadcast(x, p, target_shape[p])
        assert self.shape[x] == tuple(target_shape), (self.shape[x], target_shape)
        return x

    def dot_general(self, a: str, b: str, lb, rb, lc, rc) -> str:
        sa, sb = self.shape[a], self.shape[b]
        lf = [i for i in range(len(sa)) if i not in lb and i not in lc]
        rf = [i for i in range(len(sb)) if i not in rb and i not in rc]
        for x, y in zip(lb, rb):
            assert sa[x] == sb[y]
        for x, y in zip(lc, rc):
            assert sa[x] == sb[y], (a, b, sa, sb, lc, rc)
        shape = [sa[i] for i in lb] + [sa[i] for i in lf] + [sb[i] for i in rf]
        attrs = ";".join(",".join(str(v) for v in g) for g in (lb, rb, lc, rc))
        return self._emit("dot_general", [a, b], shape, self.dtype[a], attrs=attrs)

    def matmul(self, a: str, b: str) -> str:
        sa, sb = self.shape[a], self.shape[b]
        assert len(sa) == 2 and len(sb) == 2 and sa[1] == sb[0]
        return self._emit("matmul", [a, b], [sa[0], sb[1]], self.dtype[a])

    def conv2d(self, x: str, w: str) -> str:
        sx, sw = self.shape[x], self.shape[w]
        assert sx[3] == sw[2]
        return self._emit("conv2d", [x, w], [sx[0], sx[1], sx[2], sw[3]], self.dtype[x])

    def conv2d_bwd_input(self, dy: str, w: str) -> str:
        sd, sw = self.shape[dy], self.shape[w]
        return self._emit("conv2d_bwd_input", [dy, w], [sd[0], sd[1], sd[2], sw[2]], self.dtype[dy])

    def conv2d_bwd_filter(self, x: str, dy: str, kh: int, kw: int) -> str:
        sx, sd = self.shape[x], self.shape[dy]
        return self._emit("conv2d_bwd_filter", [x, dy], [kh, kw, sx[3], sd[3]], self.dtype[x], attrs=[kh, kw])

    def resample(self, x: str, mode: str, f: int) -> str:
        s = list(self.shape[x])
        if mode == "up":
            s[1] *= f
            s[2] *= f
        else:
            s[1] //= f
            s[2] //= f
        return self._emit("resample", [x], s, self.dtype[x], attrs=[mode, f])

    def concat(self, xs, d: int) -> str:
        s = list(self.shape[xs[0]])
        s[d] = sum(self.shape[x][d] for x in xs)
        return self._emit("concat", list(xs), s, self.dtype[xs[0]], attrs=[d])

    def slice(self, x: str, d: int, start: int, length: int) -> str:
        s = list(self.shape[x])
        s[d] = length
        return self._emit("slice", [x], s, self.dtype[x], attrs=[d, start, length])

    def pad(self, x: str, d: int, lo: int, hi: int) -> str:
        s = list(self.shape[x])
        s[d] += lo + hi
        return self._emit("pad", [x], s, self.dtype[x], attrs=[d, lo, hi])

    def gather(self, tbl: str, idx: str) -> str:
        st, si = self.shape[tbl], self.shape[idx]
        return self._emit("gather", [tbl, idx], list(si) + [st[1]], self.dtype[tbl])

    def segment_sum(self, dat: str, idx: str, n: int) -> str:
        sd = self.shape[dat]
        return self._emit("segment_sum", [dat, idx], [n, sd[-1]], self.dtype[dat], attrs=[n])

    # ------------------------------------------------------- autodiff
    def _acc(self, grads, x, g):
        if x in grads:
            grads[x] = self.add(grads[x], g)
        else:
            grads[x] = g

    def backward(self, loss: str) -> dict:
        """Reverse-mode VJPs over the recorded forward ops; weight gradients
        appear at their natural backward position."""
        fwd = list(self.tape)
        grads = {loss: self.unary("ones_like", loss)}
        for rec in reversed(fwd):
            if rec.out not in grads or not rec.diff:
                continue
            gy = grads.pop(rec.out)
            for x, gx in self._vjp(rec, gy):
                if gx is not None and self._needs_grad(x):
                    self._acc(grads, x, gx)
        return grads

    def _needs_grad(self, x) -> bool:
        for p in self.params:
            if p.name == x:
                return p.trainable
        return self.dtype.get(x) != "i32"

    def _vjp(self, r: _Rec, gy: str):
        k, ops = r.kind, r.operands
        if k == "ones_like":
            return []
        if k == "convert":
            return [(ops[0], self.convert(gy, self.dtype[ops[0]]))]
        if k in ("scale",):
            return [(ops[0], self.unary("scale", gy, r.attrs))]
        if k in ("add_s", "stop_gradient"):
            return [(ops[0], gy)] if k == "add_s" else []
        if k == "neg":
            return [(ops[0], self.unary("neg", gy))]
        if k == "exp":
            return [(ops[0], self.mul(gy, r.out))]
        if k == "log":
            return [(ops[0], self.div(gy, ops[0]))]
        if k in ("relu", "gelu", "silu", "tanh", "sigmoid", "rsqrt", "sqrt", "recip", "square", "cos", "sin", "abs"):
            return [(ops[0], self.mul(gy, self.unary("d_" + k, ops[0])))]
        if k == "add":
            return [(ops[0], gy), (ops[1], gy)]
        if k == "sub":
            return [(ops[0], gy), (ops[1], self.unary("neg", gy))]
        if k == "mul":
            return [(ops[0], self.mul(gy, ops[1])), (ops[1], self.mul(gy, ops[0]))]
        if k == "div":
            ga = self.div(gy, ops[1])
            gb = self.unary("neg", self.div(self.mul(gy, r.out), ops[1]))
            return [(ops[0], ga), (ops[1], gb)]
        if k in ("max", "min"):
            return [(ops[0], self.mul(gy, self.unary("d_" + k, ops[0]))),
                    (ops[1], self.mul(gy, self.unary("d_" + k, ops[1])))]
        if k == "transpose":
            perm = list(r.attrs)
            inv = [0] * len(perm)
            for j, p in enumerate(perm):
                inv[p] = j
            return [(ops[0], self.transpose(gy, inv))]
        if k == "reduce":
            dims = list(r.attrs[:-1])
            return [(ops[0], self.broadcast_to(gy, self.shape[ops[0]], dims))]
        if k == "broadcast":
            return [(ops[0], self.reduce(gy, [r.attrs[0]], "add"))]
        if k == "matmul":
            a, b = ops
            return [(a, self.dot_general(gy, b, [], [], [1], [1])),
                    (b, self.dot_general(a, gy, [], [], [0], [0]))]
        if k == "dot_general":
            return self._vjp_dot(r, gy)
        if k == "conv2d":
            x, w = ops
            sw = self.shape[w]
            return [(x, self.conv2d_bwd_input(gy, w)), (w, self.conv2d_bwd_filter(x, gy, sw[0], sw[1]))]
        if k == "resample":
            mode, f = r.attrs
            return [(ops[0], self.resample(gy, "down" if mode == "up" else "up", f))]
        if k == "concat":
            d = r.attrs[0]
            out, off = [], 0
            for x in ops:
                n = self.shape[x][d]
                out.append((x, self.slice(gy, d, off, n)))
                off += n
            return out
        if k == "slice":
            d, s, n = r.attrs
            ext = self.shape[ops[0]][d]
            return [(ops[0], self.pad(gy, d, s, ext - s - n))]
        if k == "pad":
            d, lo, hi = r.attrs
            return [(ops[0], self.slice(gy, d, lo, self.shape[ops[0]][d]))]
        if k == "gather":
            tbl, idx = ops
            return [(tbl, self.segment_sum(gy, idx, self.shape[tbl][0]))]
        if k == "segment_sum":
            dat, idx = ops
            return [(dat, self.gather(gy, idx))]
        raise NotImplementedError(k)

    def _vjp_dot(self, r: _Rec, gy: str):
        a, b = r.operands
        lb, rb, lc, rc = [[int(v) for v in g.split(",")] if g else [] for g in r.attrs.split(";")]
        sa, sb = self.shape[a], self.shape[b]
        lf = [i for i in range(len(sa)) if i not in lb and i not in lc]
        rf = [i for i in range(len(sb)) if i not in rb and i not in rc]
        nb, nlf, nrf = len(lb), len(lf), len(rf)
        # dA = gy (x) B over rfree, batched over batch
        ga = self.dot_general(gy, b, list(range(nb)), rb, list(range(nb + nlf, nb + nlf + nrf)), rf)
        rem_b = sorted(range(len(sb)), key=lambda i: i)
        rem_b = [i for i in rem_b if i in rc]  # B's remaining dims, ascending
        a_dims = list(lb) + list(lf) + [lc[rc.index(i)] for i in rem_b]
        perm_a = [a_dims.index(j) for j in range(len(sa))]
        ga = self.transpose(ga, perm_a)
        # dB = A (x) gy over lfree, batched
        gb = self.dot_general(a, gy, lb, list(range(nb)), lf, list(range(nb, nb + nlf)))
        rem_a = [i for i in range(len(sa)) if i in lc]
        b_dims = list(rb) + [rc[lc.index(i)] for i in rem_a] + list(rf)
        perm_b = [b_dims.index(j) for j in range(len(sb))]
        gb = self.transpose(gb, perm_b)
        return [(a, ga), (b, gb)]

    # ------------------------------------------------------------ Adam
    def adam(self, grads: dict, b1=0.9, b2=0.95, lr=3e-4, eps=1e-8):
        """Adam with fp32 moments; one update per trainable weight,
        in parameter declaration order."""
        weights = [p for p in self.params if p.kind == "weight" and p.trainable]
        ms, vs = {}, {}
        for p in weights:
            ms[p.name] = self.param("m_" + p.name, "f32", p.shape, trainable=False, kind="opt")
            vs[p.name] = self.param("v_" + p.name, "f32", p.shape, trainable=False, kind="opt")
        outs = []
        for p in weights:
            if p.name not in grads:
                continue
            g = self.convert(grads[p.name], "f32")
            m2 = self.add(self.scale(ms[p.name], b1), self.scale(g, 1 - b1))
            v2 = self.add(self.scale(vs[p.name], b2), self.scale(self.unary("square", g), 1 - b2))
            u = self.div(m2, self.add_s(self.unary("sqrt", v2), eps))
            u = self.convert(self.scale(u, -lr), p.dtype)
            p2 = self.add(p.name, u)
            outs += [p2, m2, v2]
        self.returns = outs
        return outs

    # ------------------------------------------------------------ text
    def text(self, returns=None) -> str:
        rets = returns if returns is not None else self.returns
        order = ([p for p in self.params if p.kind == "weight"] + [p for p in self.params if p.kind == "opt" and p.name.startswith("m_")]
                 + [p for p in self.params if p.kind == "opt" and p.name.startswith("v_")]
                 + [p for p in self.params if p.kind == "data"])
        hdr = ", ".join(f"{p.name}: {p.dtype}[{','.join(str(e) for e in p.shape)}]" for p in order)
        body = "\n".join(self.lines)
        return f"def {self.name}({hdr}) {{\n{body}\n  return {', '.join(rets)}\n}}\n"
