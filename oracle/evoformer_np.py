"""CPU oracle: a numpy restatement of the reference's Parallel Evoformer
block forward AND backward, plus the BP=1 train step built on it.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it,
and there only as the checker / the timed CPU baseline.

Where the reference records ops on a reverse-mode tape
(/root/reference/pkg/src/branchpar/tensor.py), this restatement writes
each sub-op as an explicit forward that returns a cache and an explicit
vector-Jacobian product.  The formulas follow the reference line by line
(citations below use ``src/X.py:N`` for
``/root/reference/pkg/src/branchpar/X.py`` line N).

Parity status: PINNED.  ``tests/test_oracle.py`` checks every sub-op
forward/backward and the whole train step against golden vectors produced
by running the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import numpy as np

MSA_SUBOPS = ("row_attn", "col_attn", "msa_transition", "opm")
PAIR_SUBOPS = ("tri_mult_out", "tri_mult_in", "tri_attn_start", "tri_attn_end",
               "pair_transition")
SUBOPS = MSA_SUBOPS + PAIR_SUBOPS


class Dims:
    """Model dimensions (src/evoformer.py:43-79).  c_head = c_m // h."""

    def __init__(self, s, r, c_m, c_z, h, c_opm=32, t_factor=4, n_blocks=1,
                 eps=1e-5, variant="parallel"):
        self.s, self.r, self.c_m, self.c_z, self.h = s, r, c_m, c_z, h
        self.c_opm, self.t_factor, self.n_blocks = c_opm, t_factor, n_blocks
        self.eps, self.variant = eps, variant
        assert c_m % h == 0

    @property
    def c_head(self):
        return self.c_m // self.h

    @property
    def hc(self):
        return self.h * self.c_head

    @classmethod
    def of(cls, cfg):
        return cls(cfg.s, cfg.r, cfg.c_m, cfg.c_z, cfg.h, cfg.c_opm,
                   cfg.t_factor, cfg.n_blocks, cfg.eps,
                   getattr(cfg, "variant", "parallel"))


# ---------------------------------------------------------------------------
# parameters (src/evoformer.py:139-218): same names, shapes, RNG order
# ---------------------------------------------------------------------------

def param_specs(d: Dims, subop: str):
    """(suffix, shape, kind) per tensor; kind W | b0 | g1 | ln_g | ln_b."""
    cm, cz, hc, h, c, t = d.c_m, d.c_z, d.hc, d.h, d.c_opm, d.t_factor
    attn_core = [("q_w", None, "W"), ("k_w", None, "W"), ("v_w", None, "W")]
    if subop in ("row_attn", "col_attn"):
        out = [("ln_g", (cm,), "ln_g"), ("ln_b", (cm,), "ln_b")]
        if subop == "row_attn":
            out += [("lnz_g", (cz,), "ln_g"), ("lnz_b", (cz,), "ln_b")]
        out += [(n, (cm, hc), k) for n, _, k in attn_core]
        out += [("gate_w", (cm, hc), "W"), ("gate_b", (hc,), "g1")]
        if subop == "row_attn":
            out += [("bias_w", (cz, h), "W")]
        out += [("out_w", (hc, cm), "W"), ("out_b", (cm,), "b0")]
        return out
    if subop in ("msa_transition", "pair_transition"):
        cx = cm if subop == "msa_transition" else cz
        return [("ln_g", (cx,), "ln_g"), ("ln_b", (cx,), "ln_b"),
                ("w1", (cx, t * cx), "W"), ("b1", (t * cx,), "b0"),
                ("w2", (t * cx, cx), "W"), ("b2", (cx,), "b0")]
    if subop == "opm":
        return [("ln_g", (cm,), "ln_g"), ("ln_b", (cm,), "ln_b"),
                ("a_w", (cm, c), "W"), ("a_b", (c,), "b0"),
                ("b_w", (cm, c), "W"), ("b_b", (c,), "b0"),
                ("out_w", (c * c, cz), "W"), ("out_b", (cz,), "b0")]
    if subop in ("tri_mult_out", "tri_mult_in"):
        return [("ln_g", (cz,), "ln_g"), ("ln_b", (cz,), "ln_b"),
                ("a_gate_w", (cz, c), "W"), ("a_gate_b", (c,), "g1"),
                ("a_w", (cz, c), "W"), ("a_b", (c,), "b0"),
                ("b_gate_w", (cz, c), "W"), ("b_gate_b", (c,), "g1"),
                ("b_w", (cz, c), "W"), ("b_b", (c,), "b0"),
                ("out_gate_w", (cz, cz), "W"), ("out_gate_b", (cz,), "g1"),
                ("p_ln_g", (c,), "ln_g"), ("p_ln_b", (c,), "ln_b"),
                ("out_w", (c, cz), "W"), ("out_b", (cz,), "b0")]
    if subop in ("tri_attn_start", "tri_attn_end"):
        return [("ln_g", (cz,), "ln_g"), ("ln_b", (cz,), "ln_b"),
                ("q_w", (cz, hc), "W"), ("k_w", (cz, hc), "W"),
                ("v_w", (cz, hc), "W"), ("bias_w", (cz, h), "W"),
                ("gate_w", (cz, hc), "W"), ("gate_b", (hc,), "g1"),
                ("out_w", (hc, cz), "W"), ("out_b", (cz,), "b0")]
    raise KeyError(subop)


def init_params(d: Dims, seed: int, dtype=np.float64) -> dict:
    """src/evoformer.py:193-218: only weights consume the PCG64 stream,
    drawn f64 in block -> SUBOPS -> spec order, then cast."""
    rng = np.random.default_rng(seed)
    out = {}
    for blk in range(d.n_blocks):
        for subop in SUBOPS:
            for suffix, shape, kind in param_specs(d, subop):
                if kind == "W":
                    arr = rng.uniform(-0.02, 0.02, size=shape)
                elif kind in ("g1", "ln_g"):
                    arr = np.ones(shape)
                else:
                    arr = np.zeros(shape)
                out[f"blk{blk}.{subop}.{suffix}"] = arr.astype(dtype)
    return out


def make_batch(d: Dims, seed: int, n: int, dtype=np.float64):
    """src/schedules.py:177-185 (m then z per sample, one rng)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        m = rng.standard_normal((d.s, d.r, d.c_m)).astype(dtype)
        z = rng.standard_normal((d.r, d.r, d.c_z)).astype(dtype)
        out.append((m, z))
    return out


# ---------------------------------------------------------------------------
# primitive ops and their VJPs (src/tensor.py)
# ---------------------------------------------------------------------------

def sigmoid(x):
    """Two-branch stable sigmoid, src/tensor.py:259-269."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def softmax(x):
    """Max-shifted softmax over the last axis, src/tensor.py:352-357."""
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def softmax_vjp(dy, y):
    """src/tensor.py:359-361: y * (dy - sum(dy*y))."""
    return y * (dy - (dy * y).sum(axis=-1, keepdims=True))


def ln_fwd(x, g, b, eps):
    """src/tensor.py:375-381: population variance, inv = 1/sqrt(var+eps)."""
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + eps)
    xhat = xc * inv
    return xhat * g + b, (xhat, inv)


def ln_vjp(dy, cache, g):
    """src/tensor.py:384-390."""
    xhat, inv = cache
    d = xhat.shape[-1]
    dxh = dy * g
    m1 = dxh.mean(axis=-1, keepdims=True)
    m2 = (dxh * xhat).mean(axis=-1, keepdims=True)
    dx = inv * (dxh - m1 - xhat * m2)
    dg = (dy * xhat).reshape(-1, d).sum(axis=0)
    db = dy.reshape(-1, d).sum(axis=0)
    return dx, dg, db


def lin(x, w, b=None):
    """x @ w (+ b) on the last axis, W stored [d_in, d_out]
    (src/tensor.py:314-331)."""
    y = np.matmul(x, w)
    return y if b is None else y + b


def lin_vjp(dy, x, w, with_bias=True):
    """src/tensor.py:337-343: dx = dy W^T, dW = x^T dy (rows flattened),
    db = row sum of dy."""
    d_in, d_out = w.shape
    dx = np.matmul(dy, w.T)
    x2 = x.reshape(-1, d_in)
    g2 = dy.reshape(-1, d_out)
    dw = np.matmul(x2.T, g2)
    db = g2.sum(axis=0) if with_bias else None
    return dx, dw, db


class Grads(dict):
    """name -> accumulated gradient array."""

    def add(self, name, g):
        if name in self:
            self[name] = self[name] + g
        else:
            self[name] = np.array(g, copy=True)


# ---------------------------------------------------------------------------
# gated attention (src/evoformer.py:268-286)
# ---------------------------------------------------------------------------

def _split_heads(x, h, c):
    B, L = x.shape[0], x.shape[1]
    return x.reshape(B, L, h, c).transpose(0, 2, 1, 3)


def _merge_heads(x):
    B, h, L, c = x.shape
    return x.transpose(0, 2, 1, 3).reshape(B, L, h * c)


def gated_attn_fwd(P, px, xh, bias, d: Dims):
    """xh [B,L,c_in]; bias [h,L,L] or None broadcast over B."""
    h, c = d.h, d.c_head
    scale = c ** -0.5
    q = _split_heads(lin(xh, P[f"{px}.q_w"]), h, c)
    k = _split_heads(lin(xh, P[f"{px}.k_w"]), h, c)
    v = _split_heads(lin(xh, P[f"{px}.v_w"]), h, c)
    qs = q * scale                                   # scale before q k^T (:278)
    logits = np.matmul(qs, k.transpose(0, 1, 3, 2))
    if bias is not None:
        logits = logits + bias
    att = softmax(logits)
    ctx = np.matmul(att, v)
    merged = _merge_heads(ctx)
    gate = sigmoid(lin(xh, P[f"{px}.gate_w"], P[f"{px}.gate_b"]))
    gm = gate * merged                              # gate before out-proj (:285)
    out = lin(gm, P[f"{px}.out_w"], P[f"{px}.out_b"])
    cache = dict(xh=xh, qs=qs, k=k, v=v, att=att, merged=merged, gate=gate,
                 gm=gm, has_bias=bias is not None)
    return out, cache


def gated_attn_vjp(dout, cache, P, px, d: Dims, G: Grads):
    """Returns (dxh, dbias or None); parameter grads go into G."""
    h, c = d.h, d.c_head
    scale = c ** -0.5
    xh = cache["xh"]
    dgm, dwo, dbo = lin_vjp(dout, cache["gm"], P[f"{px}.out_w"])
    G.add(f"{px}.out_w", dwo)
    G.add(f"{px}.out_b", dbo)
    gate, merged = cache["gate"], cache["merged"]
    dgate_pre = dgm * merged * gate * (1.0 - gate)
    dmerged = dgm * gate
    dxh, dwg, dbg = lin_vjp(dgate_pre, xh, P[f"{px}.gate_w"])
    G.add(f"{px}.gate_w", dwg)
    G.add(f"{px}.gate_b", dbg)
    dctx = _split_heads(dmerged, h, c)
    att, v, qs, k = cache["att"], cache["v"], cache["qs"], cache["k"]
    datt = np.matmul(dctx, v.transpose(0, 1, 3, 2))
    dv = np.matmul(att.transpose(0, 1, 3, 2), dctx)
    dlog = softmax_vjp(datt, att)
    dbias = dlog.sum(axis=0) if cache["has_bias"] else None
    dqs = np.matmul(dlog, k)
    dk = np.matmul(dlog.transpose(0, 1, 3, 2), qs)
    dq = dqs * scale
    for name, dt in (("q_w", dq), ("k_w", dk), ("v_w", dv)):
        dx_, dw_, _ = lin_vjp(_merge_heads(dt), xh, P[f"{px}.{name}"], False)
        G.add(f"{px}.{name}", dw_)
        dxh = dxh + dx_
    return dxh, dbias


# ---------------------------------------------------------------------------
# the nine sub-ops (src/evoformer.py:289-420), forward + VJP
# ---------------------------------------------------------------------------

def row_attn_fwd(P, px, m, z, d):
    """src/evoformer.py:289-297."""
    mh, lc_m = ln_fwd(m, P[f"{px}.ln_g"], P[f"{px}.ln_b"], d.eps)
    zh, lc_z = ln_fwd(z, P[f"{px}.lnz_g"], P[f"{px}.lnz_b"], d.eps)
    bias = lin(zh, P[f"{px}.bias_w"]).transpose(2, 0, 1)   # [h, r, r]
    out, ac = gated_attn_fwd(P, px, mh, bias, d)
    return out, dict(lc_m=lc_m, lc_z=lc_z, zh=zh, ac=ac)


def row_attn_vjp(dout, cache, P, px, d, G):
    dmh, dbias = gated_attn_vjp(dout, cache["ac"], P, px, d, G)
    dbp = dbias.transpose(1, 2, 0)                          # [r, r, h]
    dzh, dwb, _ = lin_vjp(dbp, cache["zh"], P[f"{px}.bias_w"], False)
    G.add(f"{px}.bias_w", dwb)
    dz, dg, db = ln_vjp(dzh, cache["lc_z"], P[f"{px}.lnz_g"])
    G.add(f"{px}.lnz_g", dg)
    G.add(f"{px}.lnz_b", db)
    dm, dg, db = ln_vjp(dmh, cache["lc_m"], P[f"{px}.ln_g"])
    G.add(f"{px}.ln_g", dg)
    G.add(f"{px}.ln_b", db)
    return dm, dz


def col_attn_fwd(P, px, m, d):
    """src/evoformer.py:300-311: row attention on m^T, no bias."""
    mp = m.transpose(1, 0, 2)
    mh, lc = ln_fwd(mp, P[f"{px}.ln_g"], P[f"{px}.ln_b"], d.eps)
    out, ac = gated_attn_fwd(P, px, mh, None, d)
    return out.transpose(1, 0, 2), dict(lc=lc, ac=ac)


def col_attn_vjp(dout, cache, P, px, d, G):
    dmh, _ = gated_attn_vjp(dout.transpose(1, 0, 2), cache["ac"], P, px, d, G)
    dmp, dg, db = ln_vjp(dmh, cache["lc"], P[f"{px}.ln_g"])
    G.add(f"{px}.ln_g", dg)
    G.add(f"{px}.ln_b", db)
    return dmp.transpose(1, 0, 2)


def transition_fwd(P, px, x, d):
    """src/evoformer.py:314-329: relu(LN(x) W1 + b1) W2 + b2."""
    xh, lc = ln_fwd(x, P[f"{px}.ln_g"], P[f"{px}.ln_b"], d.eps)
    pre = lin(xh, P[f"{px}.w1"], P[f"{px}.b1"])
    hid = np.maximum(pre, 0.0)
    out = lin(hid, P[f"{px}.w2"], P[f"{px}.b2"])
    return out, dict(lc=lc, xh=xh, pre=pre, hid=hid)


def transition_vjp(dout, cache, P, px, d, G):
    dhid, dw2, db2 = lin_vjp(dout, cache["hid"], P[f"{px}.w2"])
    G.add(f"{px}.w2", dw2)
    G.add(f"{px}.b2", db2)
    dpre = dhid * (cache["pre"] > 0)                       # src/tensor.py:274-280
    dxh, dw1, db1 = lin_vjp(dpre, cache["xh"], P[f"{px}.w1"])
    G.add(f"{px}.w1", dw1)
    G.add(f"{px}.b1", db1)
    dx, dg, db = ln_vjp(dxh, cache["lc"], P[f"{px}.ln_g"])
    G.add(f"{px}.ln_g", dg)
    G.add(f"{px}.ln_b", db)
    return dx


def opm_fwd(P, px, m, d):
    """src/evoformer.py:332-352 (unsharded): scale 1/s before out-proj,
    channel pair (p, q) flattened as p*c + q."""
    s, r, c = d.s, d.r, d.c_opm
    mh, lc = ln_fwd(m, P[f"{px}.ln_g"], P[f"{px}.ln_b"], d.eps)
    a = lin(mh, P[f"{px}.a_w"], P[f"{px}.a_b"])
    b = lin(mh, P[f"{px}.b_w"], P[f"{px}.b_b"])
    # raw[(i,p),(j,q)] = sum_s a[s,(i,p)] b[s,(j,q)]  (a BLAS matmul, :343-347)
    raw = np.matmul(a.reshape(s, r * c).T, b.reshape(s, r * c))
    o = raw.reshape(r, c, r, c).transpose(0, 2, 1, 3).reshape(r, r, c * c)
    os_ = o * (1.0 / s)
    out = lin(os_, P[f"{px}.out_w"], P[f"{px}.out_b"])
    return out, dict(lc=lc, mh=mh, a=a, b=b, os=os_)


def opm_vjp(dout, cache, P, px, d, G):
    s, r, c = d.s, d.r, d.c_opm
    dos, dwo, dbo = lin_vjp(dout, cache["os"], P[f"{px}.out_w"])
    G.add(f"{px}.out_w", dwo)
    G.add(f"{px}.out_b", dbo)
    do = (dos * (1.0 / s)).reshape(r, r, c, c)
    a, b, mh = cache["a"], cache["b"], cache["mh"]
    draw = do.transpose(0, 2, 1, 3).reshape(r * c, r * c)      # [(i,p),(j,q)]
    da = np.matmul(b.reshape(s, r * c), draw.T).reshape(s, r, c)
    db = np.matmul(a.reshape(s, r * c), draw).reshape(s, r, c)
    dmh_a, dwa, dba = lin_vjp(da, mh, P[f"{px}.a_w"])
    dmh_b, dwb, dbb = lin_vjp(db, mh, P[f"{px}.b_w"])
    G.add(f"{px}.a_w", dwa)
    G.add(f"{px}.a_b", dba)
    G.add(f"{px}.b_w", dwb)
    G.add(f"{px}.b_b", dbb)
    dm, dg, dbeta = ln_vjp(dmh_a + dmh_b, cache["lc"], P[f"{px}.ln_g"])
    G.add(f"{px}.ln_g", dg)
    G.add(f"{px}.ln_b", dbeta)
    return dm


def tri_mult_fwd(P, px, z, d, incoming):
    """src/evoformer.py:359-397 (unsharded)."""
    zh, lc = ln_fwd(z, P[f"{px}.ln_g"], P[f"{px}.ln_b"], d.eps)
    proj = {}
    for tag in ("a", "b"):
        gp = sigmoid(lin(zh, P[f"{px}.{tag}_gate_w"], P[f"{px}.{tag}_gate_b"]))
        val = lin(zh, P[f"{px}.{tag}_w"], P[f"{px}.{tag}_b"])
        proj[tag] = (gp, val, gp * val)
    a, b = proj["a"][2], proj["b"][2]
    ac, bc = a.transpose(2, 0, 1), b.transpose(2, 0, 1)     # [c, ., .]
    if incoming:
        p = np.matmul(ac.transpose(0, 2, 1), bc)               # sum_k a[k,i] b[k,j]
    else:
        p = np.matmul(ac, bc.transpose(0, 2, 1))               # sum_k a[i,k] b[j,k]
    p = np.ascontiguousarray(p.transpose(1, 2, 0))
    pn, lcp = ln_fwd(p, P[f"{px}.p_ln_g"], P[f"{px}.p_ln_b"], d.eps)
    o = lin(pn, P[f"{px}.out_w"], P[f"{px}.out_b"])
    g = sigmoid(lin(zh, P[f"{px}.out_gate_w"], P[f"{px}.out_gate_b"]))
    return g * o, dict(lc=lc, zh=zh, proj=proj, lcp=lcp, pn=pn, o=o, g=g,
                       incoming=incoming)


def tri_mult_vjp(dout, cache, P, px, d, G):
    g, o, zh = cache["g"], cache["o"], cache["zh"]
    dgp = dout * o * g * (1.0 - g)
    do = dout * g
    dzh, dw, db = lin_vjp(dgp, zh, P[f"{px}.out_gate_w"])
    G.add(f"{px}.out_gate_w", dw)
    G.add(f"{px}.out_gate_b", db)
    dpn, dw, db = lin_vjp(do, cache["pn"], P[f"{px}.out_w"])
    G.add(f"{px}.out_w", dw)
    G.add(f"{px}.out_b", db)
    dp, dg_, db_ = ln_vjp(dpn, cache["lcp"], P[f"{px}.p_ln_g"])
    G.add(f"{px}.p_ln_g", dg_)
    G.add(f"{px}.p_ln_b", db_)
    a, b = cache["proj"]["a"][2], cache["proj"]["b"][2]
    dpc = dp.transpose(2, 0, 1)                                 # [c, i, j]
    ac, bc = a.transpose(2, 0, 1), b.transpose(2, 0, 1)
    if cache["incoming"]:
        da = np.matmul(bc, dpc.transpose(0, 2, 1)).transpose(1, 2, 0)   # [k,i,c]
        dbb = np.matmul(ac, dpc).transpose(1, 2, 0)                     # [k,j,c]
    else:
        da = np.matmul(dpc, bc).transpose(1, 2, 0)                      # [i,k,c]
        dbb = np.matmul(dpc.transpose(0, 2, 1), ac).transpose(1, 2, 0)  # [j,k,c]
    for tag, dt in (("a", da), ("b", dbb)):
        gp, val, _ = cache["proj"][tag]
        dgpre = dt * val * gp * (1.0 - gp)
        dval = dt * gp
        dx1, dw1, db1 = lin_vjp(dgpre, zh, P[f"{px}.{tag}_gate_w"])
        dx2, dw2, db2 = lin_vjp(dval, zh, P[f"{px}.{tag}_w"])
        G.add(f"{px}.{tag}_gate_w", dw1)
        G.add(f"{px}.{tag}_gate_b", db1)
        G.add(f"{px}.{tag}_w", dw2)
        G.add(f"{px}.{tag}_b", db2)
        dzh = dzh + dx1 + dx2
    dz, dg_, db_ = ln_vjp(dzh, cache["lc"], P[f"{px}.ln_g"])
    G.add(f"{px}.ln_g", dg_)
    G.add(f"{px}.ln_b", db_)
    return dz


def tri_attn_fwd(P, px, z, d, ending):
    """src/evoformer.py:400-420: start attends within rows with bias
    b[h,j,k] = LN(z)[j,k] W_b; end is start on z^T, transposed back."""
    zz = z.transpose(1, 0, 2) if ending else z
    zh, lc = ln_fwd(zz, P[f"{px}.ln_g"], P[f"{px}.ln_b"], d.eps)
    bias = lin(zh, P[f"{px}.bias_w"]).transpose(2, 0, 1)
    out, ac = gated_attn_fwd(P, px, zh, bias, d)
    if ending:
        out = out.transpose(1, 0, 2)
    return out, dict(lc=lc, zh=zh, ac=ac, ending=ending)


def tri_attn_vjp(dout, cache, P, px, d, G):
    ending = cache["ending"]
    dd = dout.transpose(1, 0, 2) if ending else dout
    dzh, dbias = gated_attn_vjp(dd, cache["ac"], P, px, d, G)
    dzh_b, dwb, _ = lin_vjp(dbias.transpose(1, 2, 0), cache["zh"],
                            P[f"{px}.bias_w"], False)
    G.add(f"{px}.bias_w", dwb)
    dzz, dg, db = ln_vjp(dzh + dzh_b, cache["lc"], P[f"{px}.ln_g"])
    G.add(f"{px}.ln_g", dg)
    G.add(f"{px}.ln_b", db)
    return dzz.transpose(1, 0, 2) if ending else dzz


def subop_fwd(name, P, px, m, z, d):
    """Dispatch one sub-op forward; returns (delta, cache)."""
    if name == "row_attn":
        return row_attn_fwd(P, px, m, z, d)
    if name == "col_attn":
        return col_attn_fwd(P, px, m, d)
    if name == "msa_transition":
        return transition_fwd(P, px, m, d)
    if name == "opm":
        return opm_fwd(P, px, m, d)
    if name == "pair_transition":
        return transition_fwd(P, px, z, d)
    if name.startswith("tri_mult"):
        return tri_mult_fwd(P, px, z, d, name.endswith("_in"))
    if name.startswith("tri_attn"):
        return tri_attn_fwd(P, px, z, d, name.endswith("_end"))
    raise KeyError(name)


def subop_vjp(name, ddelta, cache, P, px, d, G):
    """Returns (dm or None, dz or None)."""
    if name == "row_attn":
        return row_attn_vjp(ddelta, cache, P, px, d, G)
    if name == "col_attn":
        return col_attn_vjp(ddelta, cache, P, px, d, G), None
    if name in ("msa_transition",):
        return transition_vjp(ddelta, cache, P, px, d, G), None
    if name == "opm":
        return opm_vjp(ddelta, cache, P, px, d, G), None
    if name == "pair_transition":
        return None, transition_vjp(ddelta, cache, P, px, d, G)
    if name.startswith("tri_mult"):
        return None, tri_mult_vjp(ddelta, cache, P, px, d, G)
    if name.startswith("tri_attn"):
        return None, tri_attn_vjp(ddelta, cache, P, px, d, G)
    raise KeyError(name)


# ---------------------------------------------------------------------------
# tracks, parallel block, stack, train step (src/evoformer.py:427-467,
# src/schedules.py:194-211)
# ---------------------------------------------------------------------------

MSA_TRACK = ("row_attn", "col_attn", "msa_transition")
PAIR_TRACK = PAIR_SUBOPS


def _msa_track_fwd(P, blk, m, z, d, caches):
    for name in MSA_TRACK:
        delta, caches[name] = subop_fwd(name, P, f"blk{blk}.{name}", m, z, d)
        m = m + delta
    return m


def _pair_track_fwd(P, blk, z, d, caches):
    for name in PAIR_TRACK:
        delta, caches[name] = subop_fwd(name, P, f"blk{blk}.{name}", None, z, d)
        z = z + delta
    return z


def _pair_track_vjp(dz, caches, P, blk, d, G):
    """Gradient wrt the pair-track input (residuals included)."""
    for name in reversed(PAIR_TRACK):
        dz = dz + subop_vjp(name, dz, caches[name], P, f"blk{blk}.{name}", d, G)[1]
    return dz


def _msa_track_vjp(dm, caches, P, blk, d, G):
    """(gradient wrt the MSA-track input m, its gradient wrt z: dz_row)."""
    dz_row = None
    for name in reversed(MSA_TRACK):
        dm_part, dz_part = subop_vjp(name, dm, caches[name], P, f"blk{blk}.{name}", d, G)
        dm = dm + dm_part
        if dz_part is not None:
            dz_row = dz_part
    return dm, dz_row


def block_fwd_variant(P, blk, m, z, d):
    """af2 / multimer wirings (src/evoformer.py:448-455).
    af2:      m' = msa_track(m, z); z1 = z + opm(m'); z' = pair_track(z1)
    multimer: z1 = z + opm(m); m' = msa_track(m, z1); z' = pair_track(z1)"""
    caches = {}
    if d.variant == "af2":
        m_c = _msa_track_fwd(P, blk, m, z, d, caches)
        o, caches["opm"] = opm_fwd(P, f"blk{blk}.opm", m_c, d)
        z1 = z + o
    else:
        o, caches["opm"] = opm_fwd(P, f"blk{blk}.opm", m, d)
        z1 = z + o
        m_c = _msa_track_fwd(P, blk, m, z1, d, caches)
    return m_c, _pair_track_fwd(P, blk, z1, d, caches), caches


def block_vjp_variant(dm_out, dz_out, caches, P, blk, d, G):
    dz1 = _pair_track_vjp(dz_out, caches, P, blk, d, G)
    if d.variant == "af2":
        dm1 = dm_out + subop_vjp("opm", dz1, caches["opm"], P, f"blk{blk}.opm", d, G)[0]
        dm, dz_row = _msa_track_vjp(dm1, caches, P, blk, d, G)
        return dm, dz1 + dz_row
    dm1, dz_row = _msa_track_vjp(dm_out, caches, P, blk, d, G)
    dz1 = dz1 + dz_row
    dm = dm1 + subop_vjp("opm", dz1, caches["opm"], P, f"blk{blk}.opm", d, G)[0]
    return dm, dz1


def block_fwd(P, blk, m, z, d):
    """Parallel wiring (src/evoformer.py:456-461): both tracks read the
    block inputs; z' = pair_track(z) + opm(msa_track(m, z))."""
    if d.variant != "parallel":
        return block_fwd_variant(P, blk, m, z, d)
    caches = {}
    m_c = m
    for name in MSA_TRACK:
        delta, caches[name] = subop_fwd(name, P, f"blk{blk}.{name}", m_c, z, d)
        m_c = m_c + delta
    z_c = z
    for name in PAIR_TRACK:
        delta, caches[name] = subop_fwd(name, P, f"blk{blk}.{name}", m_c, z_c, d)
        z_c = z_c + delta
    o, caches["opm"] = opm_fwd(P, f"blk{blk}.opm", m_c, d)
    return m_c, z_c + o, caches


def block_vjp(dm_out, dz_out, caches, P, blk, d, G):
    """Returns (dm_in, dz_in).  dz_in = dz_pair + dz_row, the same two
    operands the BP schedule sums (src/schedules.py:253, 293)."""
    if d.variant != "parallel":
        return block_vjp_variant(dm_out, dz_out, caches, P, blk, d, G)
    dm = dm_out + subop_vjp("opm", dz_out, caches["opm"], P, f"blk{blk}.opm",
                            d, G)[0]
    dz = dz_out
    for name in reversed(PAIR_TRACK):
        dz = dz + subop_vjp(name, dz, caches[name], P, f"blk{blk}.{name}", d, G)[1]
    dz_pair = dz
    dz_row = None
    for name in reversed(MSA_TRACK):
        dm_part, dz_part = subop_vjp(name, dm, caches[name], P,
                                     f"blk{blk}.{name}", d, G)
        dm = dm + dm_part
        if dz_part is not None:
            dz_row = dz_part
    return dm, dz_pair + dz_row


def train_step(P, m, z, d):
    """BP=1 step (src/schedules.py:198-211, loss :194-195).

    Returns dict(m_out, z_out, loss, dm, dz, grads)."""
    caches = []
    m_c, z_c = m, z
    for blk in range(d.n_blocks):
        m_c, z_c, c = block_fwd(P, blk, m_c, z_c, d)
        caches.append(c)
    loss = np.mean(m_c * m_c) + np.mean(z_c * z_c)
    dm = m_c * (2.0 / m_c.size)
    dz = z_c * (2.0 / z_c.size)
    G = Grads()
    for blk in reversed(range(d.n_blocks)):
        dm, dz = block_vjp(dm, dz, caches[blk], P, blk, d, G)
    for name in P:
        if name not in G:
            G[name] = np.zeros_like(P[name])
    return dict(m_out=m_c, z_out=z_c, loss=float(loss), dm=dm, dz=dz,
                grads=dict(G))


def composed_step(Pe, de: Dims, Pm, dm_: Dims, m_e, m, z):
    """two ``evoformer_stack`` calls on one tape
    (src/evoformer.py:464-467): the extra-MSA stack (Pe, de) runs on
    (m_e, z), its m_e output is dropped, its z output feeds the main stack
    (Pm, dm_); loss on the main outputs (src/schedules.py:194-195).

    Returns dict(m_out, z_out, loss, dm_e, dm, dz, grads_e, grads_m)."""
    ce, cm = [], []
    me_c, z_c = m_e, z
    for blk in range(de.n_blocks):
        me_c, z_c, c = block_fwd(Pe, blk, me_c, z_c, de)
        ce.append(c)
    m_c = m
    for blk in range(dm_.n_blocks):
        m_c, z_c, c = block_fwd(Pm, blk, m_c, z_c, dm_)
        cm.append(c)
    loss = np.mean(m_c * m_c) + np.mean(z_c * z_c)
    dm = m_c * (2.0 / m_c.size)
    dz = z_c * (2.0 / z_c.size)
    Gm, Ge = Grads(), Grads()
    for blk in reversed(range(dm_.n_blocks)):
        dm, dz = block_vjp(dm, dz, cm[blk], Pm, blk, dm_, Gm)
    dme = np.zeros_like(me_c)
    for blk in reversed(range(de.n_blocks)):
        dme, dz = block_vjp(dme, dz, ce[blk], Pe, blk, de, Ge)
    for P, G in ((Pe, Ge), (Pm, Gm)):
        for name in P:
            if name not in G:
                G[name] = np.zeros_like(P[name])
    return dict(m_out=m_c, z_out=z_c, loss=float(loss), dm_e=dme, dm=dm, dz=dz,
                grads_e=dict(Ge), grads_m=dict(Gm))


def run_single(d: Dims, P: dict, seed: int = 32, dtype=np.float64):
    """Oracle counterpart of src/schedules.py:387-399."""
    m, z = make_batch(d, seed, 1, dtype)[0]
    return train_step(P, m, z, d)


def block_flops(d: Dims) -> int:
    """Forward multiply-add FLOPs of one parallel block: the reference
    tape's ``madds`` counter (src/tensor.py:302, 333), equal to
    src/costmodel.py:66-85 ``op_flops``.  fwd+bwd = 3x this."""
    s, r, cm, cz, h, c, t = d.s, d.r, d.c_m, d.c_z, d.h, d.c_opm, d.t_factor
    hc, ch = d.hc, d.c_head
    M, Z = s * r, r * r
    f = 0
    # row attn: q,k,v,gate,out projections + bias proj + QK^T + PV
    f += 2 * M * cm * hc * 4 + 2 * M * hc * cm + 2 * Z * cz * h
    f += 2 * 2 * s * h * r * r * ch
    # col attn
    f += 2 * M * cm * hc * 4 + 2 * M * hc * cm + 2 * 2 * r * h * s * s * ch
    # msa transition
    f += 2 * 2 * M * cm * t * cm
    # opm: a,b proj, outer product, out proj
    f += 2 * 2 * M * cm * c + 2 * Z * c * c * s + 2 * Z * c * c * cz
    # tri mult x2: 4 proj (c) + out gate (cz) + contraction + out proj
    f += 2 * (2 * Z * cz * (4 * c + cz) + 2 * Z * r * c + 2 * Z * c * cz)
    # tri attn x2: q,k,v,gate + out + bias + QK^T + PV
    f += 2 * (2 * Z * cz * hc * 4 + 2 * Z * hc * cz + 2 * Z * cz * h
              + 2 * 2 * r * h * r * r * ch)
    # pair transition
    f += 2 * 2 * Z * cz * t * cz
    return f
