"""Synthetic training-step programs shaped like the paper's models.

Sources for the structure (§5.1):
  * GPT / Llama decoders: T2B/T7B-like widths, Adam,
    no rematerialisation.
  * GNS: encoder / message passing / decoder, 3-layer MLPs, hidden 1024,
    latent 2048.
  * U-Net: 9 residual down blocks, 12 up blocks, 32-head attention between
    them.
Emission order (SURVEY §8(d) "Generator conventions"): params (weights, Adam
m, v, data) -> forward -> loss -> backward -> Adam -> return.

Input generation only: nothing here computes any part of the method.
"""
from __future__ import annotations

from .ir import Builder


# ---------------------------------------------------------------------------
# paper worked examples (tests/golden holds the literal listings)
# ---------------------------------------------------------------------------
def stacked_attn(layers: int, S: int = 8, D: int = 4) -> str:
    """L copies of Fig. 5a attention chained through a residual-free
    stack: layer l's output feeds layer l+1's x.  Used for the §3.6 invariant
    "resolutions independent of the number of layers"."""
    hdr, body = [], []
    hdr.append(f"x: f32[{S},{D}]")
    x = "x"
    for l in range(layers):
        for w in ("wq", "wk", "wv"):
            hdr.append(f"{w}{l}: f32[{D},{D}]")
        body += [
            f"  k{l} = matmul({x}, wk{l})",
            f"  v{l} = matmul({x}, wv{l})",
            f"  q{l} = matmul({x}, wq{l})",
            f"  qt{l} = transpose[1,0](q{l})",
            f"  a{l} = matmul(k{l}, qt{l})",
            f"  b{l} = reduce[0,add](a{l})",
            f"  c{l} = broadcast[0,{S}](b{l})",
            f"  d{l} = div(a{l}, c{l})",
            f"  z{l} = matmul(d{l}, v{l})",
        ]
        x = f"z{l}"
    return f"def attn{layers}({', '.join(hdr)}) {{\n" + "\n".join(body) + f"\n  return {x}\n}}\n"


# ---------------------------------------------------------------------------
# shared blocks
# ---------------------------------------------------------------------------
def rmsnorm(g: Builder, x: str, gain: str) -> str:
    s = g.shape[x]
    last = len(s) - 1
    ms = g.reduce(g.unary("square", x), [last])
    ms = g.add_s(g.scale(ms, 1.0 / s[last]), 1e-6)
    r = g.broadcast(g.unary("rsqrt", ms), last, s[last])
    y = g.mul(x, r)
    gb = g.broadcast_to(gain, s, list(range(last)))
    return g.mul(y, gb)


def softmax(g: Builder, x: str, axis: int) -> str:
    s = g.shape[x]
    mx = g.reduce(x, [axis], "max", diff=False)
    e = g.unary("exp", g.sub(x, g.broadcast(mx, axis, s[axis])))
    se = g.reduce(e, [axis])
    return g.div(e, g.broadcast(se, axis, s[axis]))


def cross_entropy(g: Builder, logits: str, labels: str) -> str:
    s = g.shape[logits]
    last = len(s) - 1
    mx = g.reduce(logits, [last], "max", diff=False)
    sh = g.sub(logits, g.broadcast(mx, last, s[last]))
    lse = g.unary("log", g.reduce(g.unary("exp", sh), [last]))
    logp = g.sub(sh, g.broadcast(lse, last, s[last]))
    oh = g.broadcast(g.convert(labels, g.dtype[logits]), last, s[last])
    picked = g.reduce(g.mul(logp, oh), [last])
    tot = g.reduce(picked, list(range(len(g.shape[picked]))))
    n = 1
    for e in g.shape[picked]:
        n *= e
    return g.scale(tot, -1.0 / n)


# ---------------------------------------------------------------------------
# M2: GPT-style decoder
# ---------------------------------------------------------------------------
def gpt(layers=24, B=64, S=2048, D=2048, H=16, Dh=128, F=8192, V=50304, dt="bf16", name="gpt") -> str:
    g = Builder(name)
    emb = g.param("emb", dt, [V, D])
    Ls = []
    for l in range(layers):
        Ls.append(dict(
            g1=g.param(f"g1_{l}", dt, [D]), wq=g.param(f"wq_{l}", dt, [D, H, Dh]),
            wk=g.param(f"wk_{l}", dt, [D, H, Dh]), wv=g.param(f"wv_{l}", dt, [D, H, Dh]),
            wo=g.param(f"wo_{l}", dt, [H, Dh, D]), g2=g.param(f"g2_{l}", dt, [D]),
            w1=g.param(f"w1_{l}", dt, [D, F]), w2=g.param(f"w2_{l}", dt, [F, D])))
    gf = g.param("gf", dt, [D])
    wu = g.param("wu", dt, [D, V])
    tok = g.data("tok", "i32", [B, S])
    lab = g.data("labels", "i32", [B, S])
    mask = g.param("mask", dt, [S, S], trainable=False, kind="data")

    h = g.gather(emb, tok)                                         # [B,S,D]
    for P in Ls:
        n = rmsnorm(g, h, P["g1"])
        q = g.dot_general(n, P["wq"], [], [], [2], [0])            # [B,S,H,Dh]
        k = g.dot_general(n, P["wk"], [], [], [2], [0])
        v = g.dot_general(n, P["wv"], [], [], [2], [0])
        s = g.dot_general(q, k, [0, 2], [0, 2], [3], [3])          # [B,H,Sq,Sk]  seq-seq conflict
        s = g.scale(s, Dh ** -0.5)
        s = g.add(s, g.broadcast_to(mask, [B, H, S, S], [0, 1]))
        p = softmax(g, s, 3)
        o = g.dot_general(p, v, [0, 1], [0, 2], [3], [1])          # [B,H,Sq,Dh]
        a = g.dot_general(o, P["wo"], [], [], [1, 3], [0, 1])      # [B,S,D]
        h = g.add(h, a)
        n2 = rmsnorm(g, h, P["g2"])
        u = g.unary("gelu", g.dot_general(n2, P["w1"], [], [], [2], [0]))
        d = g.dot_general(u, P["w2"], [], [], [2], [0])
        h = g.add(h, d)
    hf = rmsnorm(g, h, gf)
    logits = g.dot_general(hf, wu, [], [], [2], [0])               # [B,S,V]
    loss = cross_entropy(g, logits, lab)
    grads = g.backward(loss)
    g.adam(grads)
    return g.text()


# ---------------------------------------------------------------------------
# M5: Llama-style decoder (GQA, RoPE, SwiGLU)
# ---------------------------------------------------------------------------
def rope(g: Builder, x: str, cos: str, sin: str, s_dim: int) -> str:
    s = g.shape[x]
    last = len(s) - 1
    half = s[last] // 2
    x1 = g.slice(x, last, 0, half)
    x2 = g.slice(x, last, half, half)
    rot = g.concat([g.unary("neg", x2), x1], last)
    pos = [i for i in range(len(s)) if i not in (s_dim, last)]
    cb = g.broadcast_to(cos, s, pos)
    sb = g.broadcast_to(sin, s, pos)
    return g.add(g.mul(x, cb), g.mul(rot, sb))


def llama(layers=80, B=256, S=4096, D=8192, Hkv=8, G=8, Dh=128, F=28672, V=32000, dt="bf16", name="llama") -> str:
    g = Builder(name)
    emb = g.param("emb", dt, [V, D])
    Ls = []
    for l in range(layers):
        Ls.append(dict(
            g1=g.param(f"g1_{l}", dt, [D]), wq=g.param(f"wq_{l}", dt, [D, Hkv, G, Dh]),
            wk=g.param(f"wk_{l}", dt, [D, Hkv, Dh]), wv=g.param(f"wv_{l}", dt, [D, Hkv, Dh]),
            wo=g.param(f"wo_{l}", dt, [Hkv, G, Dh, D]), g2=g.param(f"g2_{l}", dt, [D]),
            wg=g.param(f"wg_{l}", dt, [D, F]), wu=g.param(f"wu_{l}", dt, [D, F]),
            wd=g.param(f"wd_{l}", dt, [F, D])))
    gf = g.param("gf", dt, [D])
    wout = g.param("wout", dt, [D, V])
    tok = g.data("tok", "i32", [B, S])
    lab = g.data("labels", "i32", [B, S])
    mask = g.param("mask", dt, [S, S], trainable=False, kind="data")
    cos = g.param("rope_cos", dt, [S, Dh], trainable=False, kind="data")
    sin = g.param("rope_sin", dt, [S, Dh], trainable=False, kind="data")

    h = g.gather(emb, tok)                                          # [B,S,D]
    for P in Ls:
        n = rmsnorm(g, h, P["g1"])
        q = g.dot_general(n, P["wq"], [], [], [2], [0])             # [B,S,Hkv,G,Dh]
        k = g.dot_general(n, P["wk"], [], [], [2], [0])             # [B,S,Hkv,Dh]
        v = g.dot_general(n, P["wv"], [], [], [2], [0])
        q = rope(g, q, cos, sin, 1)
        k = rope(g, k, cos, sin, 1)
        s = g.dot_general(q, k, [0, 2], [0, 2], [4], [3])           # [B,Hkv,Sq,G,Sk]
        s = g.scale(s, Dh ** -0.5)
        s = g.add(s, g.broadcast_to(mask, [B, Hkv, S, G, S], [0, 1, 3]))
        p = softmax(g, s, 4)
        o = g.dot_general(p, v, [0, 1], [0, 2], [4], [1])           # [B,Hkv,Sq,G,Dh]
        a = g.dot_general(o, P["wo"], [], [], [1, 3, 4], [0, 1, 2]) # [B,S,D]
        h = g.add(h, a)
        n2 = rmsnorm(g, h, P["g2"])
        gt = g.unary("silu", g.dot_general(n2, P["wg"], [], [], [2], [0]))
        up = g.dot_general(n2, P["wu"], [], [], [2], [0])
        d = g.dot_general(g.mul(gt, up), P["wd"], [], [], [2], [0])
        h = g.add(h, d)
    hf = rmsnorm(g, h, gf)
    logits = g.dot_general(hf, wout, [], [], [2], [0])
    loss = cross_entropy(g, logits, lab)
    grads = g.backward(loss)
    g.adam(grads)
    return g.text()


# ---------------------------------------------------------------------------
# M4: Graph Network Simulator
# ---------------------------------------------------------------------------
def _linear(g: Builder, x: str, w: str, b: str) -> str:
    s = g.shape[x]
    y = g.dot_general(x, w, [], [], [len(s) - 1], [0])
    return g.add(y, g.broadcast_to(b, g.shape[y], list(range(len(g.shape[y]) - 1))))


def _mlp3(g: Builder, x: str, P: dict, norm: bool) -> str:
    h = g.unary("relu", _linear(g, x, P["w0"], P["b0"]))
    h = g.unary("relu", _linear(g, h, P["w1"], P["b1"]))
    h = _linear(g, h, P["w2"], P["b2"])
    if norm:
        h = rmsnorm(g, h, P["ln"])
    return h


def _mlp3_params(g: Builder, pre: str, din: int, hid: int, dout: int, dt: str, norm: bool) -> dict:
    P = dict(w0=g.param(pre + "w0", dt, [din, hid]), b0=g.param(pre + "b0", dt, [hid]),
             w1=g.param(pre + "w1", dt, [hid, hid]), b1=g.param(pre + "b1", dt, [hid]),
             w2=g.param(pre + "w2", dt, [hid, dout]), b2=g.param(pre + "b2", dt, [dout]))
    if norm:
        P["ln"] = g.param(pre + "ln", dt, [dout])
    return P


def gns(steps=16, Nn=2048, Ne=65536, hidden=1024, latent=2048, node_in=16, edge_in=8, out_dim=4,
        dt="bf16", name="gns") -> str:
    g = Builder(name)
    enc_n = _mlp3_params(g, "encn_", node_in, hidden, latent, dt, True)
    enc_e = _mlp3_params(g, "ence_", edge_in, hidden, latent, dt, True)
    stepP = []
    for s in range(steps):
        stepP.append((_mlp3_params(g, f"e{s}_", 3 * latent, hidden, latent, dt, True),
                      _mlp3_params(g, f"n{s}_", 2 * latent, hidden, latent, dt, True)))
    dec = _mlp3_params(g, "dec_", latent, hidden, out_dim, dt, False)
    xn = g.data("node_feat", dt, [Nn, node_in])
    xe = g.data("edge_feat", dt, [Ne, edge_in])
    snd = g.data("senders", "i32", [Ne])
    rcv = g.data("receivers", "i32", [Ne])
    tgt = g.data("target", dt, [Nn, out_dim])

    x = _mlp3(g, xn, enc_n, True)                 # [Nn, latent]
    e = _mlp3(g, xe, enc_e, True)                 # [Ne, latent]
    for Pe, Pn in stepP:
        xs = g.gather(x, snd)
        xr = g.gather(x, rcv)
        e_new = _mlp3(g, g.concat([xs, xr, e], 1), Pe, True)
        e = g.add(e, e_new)
        agg = g.segment_sum(e, rcv, Nn)
        x_new = _mlp3(g, g.concat([x, agg], 1), Pn, True)
        x = g.add(x, x_new)
    y = _mlp3(g, x, dec, False)
    diff = g.sub(y, tgt)
    loss = g.scale(g.reduce(g.unary("square", diff), [0, 1]), 1.0 / (Nn * out_dim))
    grads = g.backward(loss)
    g.adam(grads)
    return g.text()


# ---------------------------------------------------------------------------
# M3: U-Net (diffusion)
# ---------------------------------------------------------------------------
def _chan_norm(g: Builder, x: str, gain: str) -> str:
    return rmsnorm(g, x, gain)


def unet(B=32, HW=64, C=(320, 640, 1280), heads=32, in_ch=4, temb=320, blocks_down=3, blocks_up=4,
         dt="bf16", name="unet") -> str:
    g = Builder(name)
    specs = []  # (name, cin, cout)
    # plan the channel flow first so params are declared before the body
    c0 = C[0]
    down = []
    skips = [c0]
    cur = c0
    for lvl, c in enumerate(C):
        for b in range(blocks_down):
            down.append((f"d{lvl}b{b}", cur, c))
            cur = c
            skips.append(c)
        if lvl + 1 < len(C):
            skips.append(c)  # after downsample
    up = []
    for lvl in reversed(range(len(C))):
        c = C[lvl]
        for b in range(blocks_up):
            sc = skips.pop()
            up.append((f"u{lvl}b{b}", cur + sc, c))
            cur = c
    w_in = g.param("conv_in", dt, [3, 3, in_ch, c0])
    P = {}
    for nm, ci, co in down + up:
        P[nm] = dict(g1=g.param(nm + "_g1", dt, [ci]), w1=g.param(nm + "_w1", dt, [3, 3, ci, co]),
                     wt=g.param(nm + "_wt", dt, [temb, co]), g2=g.param(nm + "_g2", dt, [co]),
                     w2=g.param(nm + "_w2", dt, [3, 3, co, co]))
        if ci != co:
            P[nm]["ws"] = g.param(nm + "_ws", dt, [1, 1, ci, co])
    Cb = C[-1]
    Dh = Cb // heads
    att = dict(g=g.param("att_g", dt, [Cb]), wq=g.param("att_wq", dt, [Cb, heads, Dh]),
               wk=g.param("att_wk", dt, [Cb, heads, Dh]), wv=g.param("att_wv", dt, [Cb, heads, Dh]),
               wo=g.param("att_wo", dt, [heads, Dh, Cb]))
    g_out = g.param("out_g", dt, [c0])
    w_out = g.param("conv_out", dt, [3, 3, c0, in_ch])
    x = g.data("latent", dt, [B, HW, HW, in_ch])
    t = g.data("t_emb", dt, [B, temb])
    noise = g.data("noise", dt, [B, HW, HW, in_ch])

    ts = g.unary("silu", t)

    def resblock(h, p):
        s = g.shape[h]
        y = g.conv2d(g.unary("silu", _chan_norm(g, h, p["g1"])), p["w1"])
        te = g.dot_general(ts, p["wt"], [], [], [1], [0])           # [B, cout]
        y = g.add(y, g.broadcast_to(te, g.shape[y], [1, 2]))
        y = g.conv2d(g.unary("silu", _chan_norm(g, y, p["g2"])), p["w2"])
        sk = g.conv2d(h, p["ws"]) if "ws" in p else h
        return g.add(sk, y)

    h = g.conv2d(x, w_in)
    stack = [h]
    di = 0
    for lvl, c in enumerate(C):
        for b in range(blocks_down):
            h = resblock(h, P[down[di][0]])
            di += 1
            stack.append(h)
        if lvl + 1 < len(C):
            h = g.resample(h, "down", 2)
            stack.append(h)
    # bottleneck attention over (H, W) with `heads` heads
    n = _chan_norm(g, h, att["g"])
    q = g.dot_general(n, att["wq"], [], [], [3], [0])                # [B,H,W,N,Dh]
    k = g.dot_general(n, att["wk"], [], [], [3], [0])
    v = g.dot_general(n, att["wv"], [], [], [3], [0])
    s = g.dot_general(q, k, [0, 3], [0, 3], [4], [4])                # [B,N,H,W,H',W']
    s = g.scale(s, Dh ** -0.5)
    sh = g.shape[s]
    mx = g.reduce(s, [4, 5], "max", diff=False)
    e = g.unary("exp", g.sub(s, g.broadcast_to(mx, sh, [4, 5])))
    se = g.reduce(e, [4, 5])
    p = g.div(e, g.broadcast_to(se, sh, [4, 5]))
    o = g.dot_general(p, v, [0, 1], [0, 3], [4, 5], [1, 2])          # [B,N,H,W,Dh]
    a = g.dot_general(o, att["wo"], [], [], [1, 4], [0, 1])          # [B,H,W,C]
    h = g.add(h, a)
    ui = 0
    for lvl in reversed(range(len(C))):
        for b in range(blocks_up):
            h = g.concat([h, stack.pop()], 3)
            h = resblock(h, P[up[ui][0]])
            ui += 1
        if lvl > 0:
            h = g.resample(h, "up", 2)
    y = g.conv2d(g.unary("silu", _chan_norm(g, h, g_out)), w_out)
    diff = g.sub(y, noise)
    loss = g.scale(g.reduce(g.unary("square", diff), [0, 1, 2, 3]), 1.0 / (B * HW * HW * in_ch))
    grads = g.backward(loss)
    g.adam(grads)
    return g.text()


# ---------------------------------------------------------------------------
# small random programs for property tests (seeded)
# ---------------------------------------------------------------------------
def random_program(seed: int, n_ops: int = 12, linear: bool = False, max_ext: int = 8, ext: bool = False) -> str:
    """A random straight-line program over unary/binary/transpose/reduce/
    broadcast/matmul.  With linear=True every variable is used exactly once
    (the [comment] linearity theorem).  With ext=True the
    program also uses every extension op kind of the BASELINE generators
    (random_program_ext)."""
    if ext:
        return random_program_ext(seed, n_ops)
    import random
    rng = random.Random(seed)
    exts = [2, 4, 8][: max(1, [2, 4, 8].index(max_ext) + 1)] if max_ext in (2, 4, 8) else [2, 4]
    g = Builder(f"r{seed}")
    avail = []  # (name, uses_left)
    n_params = rng.randint(2, 4)
    for i in range(n_params):
        r = rng.randint(1, 3)
        shape = [rng.choice(exts) for _ in range(r)]
        avail.append(g.param(f"p{i}", "f32", shape))
    uses = {a: 0 for a in avail}

    def pick(pred=lambda n: True):
        cands = [a for a in avail if pred(a) and (not linear or uses[a] == 0)]
        if not cands:
            return None
        return rng.choice(cands)

    for _ in range(n_ops):
        kind = rng.choice(["unary", "binary", "transpose", "reduce", "broadcast", "matmul", "matmul"])
        out = None
        if kind == "unary":
            x = pick()
            if x is None:
                break
            out = g.unary(rng.choice(["relu", "exp", "neg"]), x)
            uses[x] += 1
        elif kind == "binary":
            x = pick()
            if x is None:
                break
            y = pick(lambda n: n != x and g.shape[n] == g.shape[x]) if linear else pick(lambda n: g.shape[n] == g.shape[x])
            if y is None:
                continue
            out = g.binary(rng.choice(["add", "mul", "sub"]), x, y)
            uses[x] += 1
            uses[y] += 1
        elif kind == "transpose":
            x = pick(lambda n: len(g.shape[n]) >= 2)
            if x is None:
                continue
            perm = list(range(len(g.shape[x])))
            rng.shuffle(perm)
            if perm == sorted(perm):
                perm = perm[::-1]
            out = g.transpose(x, perm)
            uses[x] += 1
        elif kind == "reduce":
            x = pick(lambda n: len(g.shape[n]) >= 2)
            if x is None:
                continue
            out = g.reduce(x, [rng.randrange(len(g.shape[x]))], "add")
            uses[x] += 1
        elif kind == "broadcast":
            x = pick(lambda n: len(g.shape[n]) <= 2)
            if x is None:
                continue
            out = g.broadcast(x, rng.randint(0, len(g.shape[x])), rng.choice(exts))
            uses[x] += 1
        elif kind == "matmul":
            x = pick(lambda n: len(g.shape[n]) == 2)
            if x is None:
                continue
            y = pick(lambda n: len(g.shape[n]) == 2 and g.shape[n][0] == g.shape[x][1] and (not linear or n != x))
            if y is None:
                continue
            out = g.matmul(x, y)
            uses[x] += 1
            uses[y] += 1
        if out is not None:
            avail.append(out)
            uses[out] = 0
    if linear:
        rets = [a for a in avail if uses[a] == 0]
    else:
        rets = [avail[-1]]
    if not any(k in "\n".join(g.lines) for k in ("matmul",)):
        # guarantee a contraction so the baseline runtime is non-zero
        a = g.param("pa", "f32", [2, 2])
        b = g.param("pb", "f32", [2, 2])
        rets = rets + [g.matmul(a, b)]
    return g.text(returns=rets)


def random_program_ext(seed: int, n_ops: int = 16) -> str:
    """A random straight-line program over the op kinds the BASELINE
    generators emit beyond Fig. 3's: dot_general (random batch / contracting
    dims, including a value contracted with itself), conv2d and its two
    backward ops (1x1 and 3x3 filters), resample up/down, concat (including a
    value concatenated with itself), slice, pad, gather and segment_sum (i32
    index params, shared between ops as in GNS), plus the elementwise /
    reduce / broadcast / transpose ops that glue them.  Extents are 2, 4, 8 and
    the odd extents pad creates; the first ops are a conv pair and a
    dot_general so every program has a contraction."""
    import random
    rng = random.Random(seed)
    g = Builder(f"x{seed}")
    E = [2, 4, 8]
    vals = []           # values usable as operands
    idx_params = {}     # index shape -> i32 param
    n_p = [0]

    def newp(shape, dt="f32"):
        n_p[0] += 1
        return g.param(f"p{n_p[0]}", dt, list(shape))

    def idx(shape):
        shape = tuple(shape)
        if shape not in idx_params or rng.random() < 0.3:
            n_p[0] += 1
            idx_params[shape] = g.data(f"i{n_p[0]}", "i32", list(shape))
        return idx_params[shape]

    def rank(r):
        c = [v for v in vals if len(g.shape[v]) == r]
        return rng.choice(c) if c else None

    # seed values: an image-like tensor and a couple of matrices / 3-tensors
    img = newp([rng.choice([2, 4]), 4, 4, rng.choice(E)])
    vals += [img, newp([rng.choice(E), rng.choice(E)]), newp([rng.choice(E), rng.choice(E), rng.choice(E)])]
    w0 = newp([3, 3, g.shape[img][3], rng.choice(E)])
    vals.append(g.conv2d(img, w0))
    m = vals[1]
    vals.append(g.dot_general(m, newp([g.shape[m][1], rng.choice(E)]), [], [], [1], [0]))

    kinds = ["dot", "dot", "self_dot", "conv", "conv_bwd", "resample", "concat", "slice", "pad", "gather",
             "segment_sum", "unary", "binary", "reduce", "broadcast", "transpose"]
    for _ in range(n_ops):
        k = rng.choice(kinds)
        out = None
        if k == "dot":
            x = rng.choice(vals)
            s = g.shape[x]
            dims = list(range(len(s)))
            rng.shuffle(dims)
            nb = rng.randint(0, max(0, len(s) - 1)) if len(s) >= 2 else 0
            nb = min(nb, 1)
            lb, lc = dims[:nb], dims[nb:nb + rng.randint(1, max(1, len(s) - nb))]
            if not lc:
                continue
            free = [rng.choice(E) for _ in range(rng.randint(0, 1))]
            # rhs dims in a random order: batch, contracting, free
            items = [("b", i) for i in range(len(lb))] + [("c", i) for i in range(len(lc))] + [("f", i) for i in range(len(free))]
            rng.shuffle(items)
            shape, rb, rc = [], [0] * len(lb), [0] * len(lc)
            for pos, (t, i) in enumerate(items):
                if t == "b":
                    rb[i] = pos
                    shape.append(s[lb[i]])
                elif t == "c":
                    rc[i] = pos
                    shape.append(s[lc[i]])
                else:
                    shape.append(free[i])
            y = rank(len(shape)) if rng.random() < 0.3 else None
            if y is None or list(g.shape[y]) != shape:
                y = newp(shape)
            out = g.dot_general(x, y, lb, rb, lc, rc)
        elif k == "self_dot":      # x . x^T-like: contract one dim of a value with itself (a conflict)
            x = rng.choice([v for v in vals if len(g.shape[v]) in (2, 3)] or vals)
            s = g.shape[x]
            if len(s) < 2:
                continue
            c = len(s) - 1
            b = [0] if len(s) == 3 else []
            out = g.dot_general(x, x, b, b, [c], [c])
        elif k == "conv":
            x = rank(4)
            if x is None:
                continue
            kk = rng.choice([1, 3])
            out = g.conv2d(x, newp([kk, kk, g.shape[x][3], rng.choice(E)]))
        elif k == "conv_bwd":
            x = rank(4)
            if x is None:
                continue
            kk = rng.choice([1, 3])
            co = rng.choice(E)
            w = newp([kk, kk, g.shape[x][3], co])
            y = g.conv2d(x, w)
            vals.append(y)
            if rng.random() < 0.5:
                out = g.conv2d_bwd_input(y, w)
            else:
                out = g.conv2d_bwd_filter(x, y, kk, kk)
        elif k == "resample":
            x = rank(4)
            if x is None:
                continue
            s = g.shape[x]
            if s[1] >= 4 and s[1] % 2 == 0 and s[2] % 2 == 0 and rng.random() < 0.5:
                out = g.resample(x, "down", 2)
            elif s[1] <= 4:
                out = g.resample(x, "up", 2)
            else:
                continue
        elif k == "concat":
            x = rng.choice(vals)
            d = rng.randrange(len(g.shape[x]))
            others = [v for v in vals if v != x and len(g.shape[v]) == len(g.shape[x])
                      and all(g.shape[v][i] == g.shape[x][i] for i in range(len(g.shape[x])) if i != d)]
            y = rng.choice(others) if others and rng.random() < 0.6 else x   # concat([x, x]): a repeated operand
            out = g.concat([x, y], d)
        elif k == "slice":
            x = rng.choice(vals)
            d = rng.randrange(len(g.shape[x]))
            e = g.shape[x][d]
            if e < 2:
                continue
            out = g.slice(x, d, rng.randrange(0, e // 2 + 1), e // 2)
        elif k == "pad":
            x = rng.choice(vals)
            d = rng.randrange(len(g.shape[x]))
            lo = rng.choice([0, 1, 2])
            out = g.pad(x, d, lo, 2 - lo if rng.random() < 0.7 else 1 - min(lo, 1))
        elif k == "gather":
            t = rank(2)
            if t is None:
                continue
            ishape = [rng.choice(E)] if rng.random() < 0.7 else [rng.choice(E), rng.choice(E)]
            out = g.gather(t, idx(ishape))
        elif k == "segment_sum":
            x = rng.choice([v for v in vals if len(g.shape[v]) in (2, 3)] or vals)
            s = g.shape[x]
            if len(s) < 2:
                continue
            out = g.segment_sum(x, idx(s[:-1]), rng.choice(E))
        elif k == "unary":
            x = rng.choice(vals)
            out = g.unary(rng.choice(["relu", "exp", "neg", "silu"]), x)
        elif k == "binary":
            x = rng.choice(vals)
            same = [v for v in vals if g.shape[v] == g.shape[x]]
            out = g.binary(rng.choice(["add", "mul", "sub"]), x, rng.choice(same))
        elif k == "reduce":
            x = rng.choice([v for v in vals if len(g.shape[v]) >= 2] or vals)
            if len(g.shape[x]) < 2:
                continue
            out = g.reduce(x, [rng.randrange(len(g.shape[x]))], rng.choice(["add", "add", "max"]))
        elif k == "broadcast":
            x = rng.choice([v for v in vals if len(g.shape[v]) <= 3] or vals)
            if len(g.shape[x]) > 3:
                continue
            out = g.broadcast(x, rng.randint(0, len(g.shape[x])), rng.choice(E))
        elif k == "transpose":
            x = rng.choice([v for v in vals if len(g.shape[v]) >= 2] or vals)
            perm = list(range(len(g.shape[x])))
            if len(perm) < 2:
                continue
            rng.shuffle(perm)
            out = g.transpose(x, perm)
        if out is not None and out not in vals and len(g.shape[out]) >= 1:
            vals.append(out)
    return g.text(returns=[vals[-1], vals[4]] if vals[-1] != vals[4] else [vals[-1]])
