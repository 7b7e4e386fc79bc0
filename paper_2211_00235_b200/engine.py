"""Forward/backward of the nine sub-ops and the parallel block as
sequences of native launches (paper_2211_00235_b200/csrc via kernels.py).

Numerics contract (SURVEY.md 8(a')): the residual streams m, z and every
gradient that crosses a sub-op boundary are fp32; GEMM operands and
saved activations use the activation dtype `act` (bf16 for the
performance path, fp32 for the parity path); every accumulation is fp32.

Each sub-op mirrors one reference function (src/evoformer.py:289-420);
the backward is the explicit VJP of the reference tape's ops
(src/tensor.py).  Layouts (rows = positions, row-major):
  m    [s*r, c_m]  row (si, i)        z    [r*r, c_z]  row (i, j)
  proj [rows, 4*hc] = q | k | v | sigmoid(gate)     (attention sub-ops)
  bias [h, r*r] head-major, row = z row               (pair bias)
  tri-mult: proj [r*r, 4c+c_z] = a | b | sig(ga) | sig(gb) | sig(g_out),
            a_cf, b_cf, p_cf channel-first [c, r, r]
  opm: ab [2, s*r, c]; o [r, r, c, c] (flatten (p,q) -> p*c+q, :348-350)
"""

from __future__ import annotations

import torch

from . import kernels as K
from ._native import EPI_NONE, EPI_RELU, EPI_SIGMOID_FROM
from .kernels import Mat

import os

MSA_SUBOPS = ("row_attn", "col_attn", "msa_transition", "opm")
MSA_TRACK = ("row_attn", "col_attn", "msa_transition")
# the pair track on a second CUDA stream, concurrent with the MSA track
# (block_fwd / block_bwd); EVO_BRANCH_STREAMS=0 runs them back to back
BRANCH_STREAMS = os.environ.get("EVO_BRANCH_STREAMS", "1") != "0"
_SIDE = {}


def side_stream(dev):
    """The per-device second stream of the two-track block."""
    key = torch.device(dev)
    s = _SIDE.get(key)
    if s is None:
        s = _SIDE[key] = torch.cuda.Stream(device=key)
    return s


# weight-gradient GEMMs (and their bias column sums) off the critical path:
# on a helper stream of the current stream, joined at the end of the sub-op
# backward that forked them; EVO_DW_STREAMS=0 keeps them in line
DW_STREAMS = os.environ.get("EVO_DW_STREAMS", "1") != "0"
_HELPER = {}


def helper_stream(cur):
    key = (cur.device, cur.cuda_stream)
    s = _HELPER.get(key)
    if s is None:
        s = _HELPER[key] = torch.cuda.Stream(device=cur.device)
    return s


class OffPath:
    """``with off.path(): ...`` runs the enclosed launches (which only write
    gradient banks) on the current stream's helper stream after everything
    issued so far; ``off.join()`` makes the current stream wait for them.
    The enclosed launches' inputs stay referenced by the caller until the
    join, so the allocator cannot recycle them early."""

    def __init__(self):
        self.pending = []

    def path(self):
        return _OffCtx(self)

    def join(self):
        for cur, hs in self.pending:
            cur.wait_stream(hs)
        self.pending = []


class _OffCtx:
    def __init__(self, off):
        self.off, self.ctx = off, None

    def __enter__(self):
        if not DW_STREAMS:
            return self
        cur = torch.cuda.current_stream()
        hs = helper_stream(cur)
        hs.wait_stream(cur)
        self.off.pending.append((cur, hs))
        self.ctx = torch.cuda.stream(hs)
        self.ctx.__enter__()
        return self

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)
        return False


# 3-product bf16 first projection in the transitions (see transition_fwd);
# EVO_SPLIT_TRANSITION=0 turns it off (plain bf16 operands)
SPLIT_TRANSITION = os.environ.get("EVO_SPLIT_TRANSITION", "1") != "0"
PAIR_SUBOPS = ("tri_mult_out", "tri_mult_in", "tri_attn_start", "tri_attn_end",
               "pair_transition")
F32 = torch.float32


def _empty(shape, dtype, dev):
    return torch.empty(shape, dtype=dtype, device=dev)


# ---------------------------------------------------------------------------
# parameter packing: fp32 masters -> act-dtype operand buffers (once/step)
# ---------------------------------------------------------------------------

class GradBank:
    """Flat fp32 gradient buffer of one branch of one block; packed grad
    tensors are views into it (one buffer per branch => one collective per
    branch for the BP owner broadcast and the DP allreduce)."""

    def __init__(self, numel: int, dev):
        self.flat = torch.zeros(numel, dtype=F32, device=dev)
        self.pos = 0

    def take(self, *shape):
        n = 1
        for s in shape:
            n *= s
        v = self.flat[self.pos:self.pos + n].view(*shape)
        self.pos += n
        return v


def _cat_cols(dev, act, rows, parts):
    """Pack [rows, sum(cols)] act-dtype from fp32 [rows, cols_i] params."""
    total = sum(p.shape[1] for p in parts)
    out = _empty((rows, total), act, dev)
    col = 0
    for p in parts:
        K.copy2d(p, rows, p.shape[1], out, s_rs=p.shape[1], d_rs=total, d_off=col)
        col += p.shape[1]
    return out


def _cat_vec(dev, parts):
    total = sum(p.shape[0] for p in parts)
    out = _empty((total,), F32, dev)
    col = 0
    for p in parts:
        K.copy2d(p, 1, p.shape[0], out, s_rs=p.shape[0], d_rs=total, d_off=col)
        col += p.shape[0]
    return out


def _to_act(dev, act, p):
    if p.dtype == act:
        return p
    out = _empty(p.shape, act, dev)
    K.copy2d(p, p.shape[0], p.shape[1], out, s_rs=p.shape[1], d_rs=p.shape[1])
    return out


class Packed(dict):
    pass


def pack_subop(P, px, name, cfg, act, dev):
    """Operand buffers for one sub-op (see module docstring for layouts)."""
    g = lambda s: P[f"{px}.{s}"]
    pk = Packed()
    if name in ("row_attn", "col_attn", "tri_attn_start", "tri_attn_end"):
        c_in = g("q_w").shape[0]
        pk["Wqkvg"] = _cat_cols(dev, act, c_in, [g("q_w"), g("k_w"), g("v_w"), g("gate_w")])
        hc = g("q_w").shape[1]
        zeros = torch.zeros(3 * hc, dtype=F32, device=dev)
        pk["bqkvg"] = _cat_vec(dev, [zeros, g("gate_b")])
        pk["Wo"] = _to_act(dev, act, g("out_w"))
        if name != "col_attn":
            pk["Wb"] = _to_act(dev, act, g("bias_w"))
    elif name in ("msa_transition", "pair_transition"):
        pk["W1"] = _to_act(dev, act, g("w1"))
        pk["W2"] = _to_act(dev, act, g("w2"))
        if act != F32 and SPLIT_TRANSITION:
            # [W_hi; W_hi; W_lo] for the 3-product first projection
            w1 = g("w1")
            cx, tc = w1.shape
            w3 = _empty((3 * cx, tc), act, dev)
            K.split_bf16(w1, cx, tc, w3, w3, h_rs=tc, l_rs=tc, hi2=w3, h2_rs=tc,
                         l_off=2 * cx * tc, h2_off=cx * tc)
            pk["W1x3"] = w3
    elif name == "opm":
        c_m = g("a_w").shape[0]
        pk["Wab"] = _cat_cols(dev, act, c_m, [g("a_w"), g("b_w")])
        pk["bab"] = _cat_vec(dev, [g("a_b"), g("b_b")])
        pk["Wo"] = _to_act(dev, act, g("out_w"))
    else:  # tri_mult_*
        c_z = g("a_w").shape[0]
        pk["Wp"] = _cat_cols(dev, act, c_z, [g("a_w"), g("b_w"), g("a_gate_w"),
                                             g("b_gate_w"), g("out_gate_w")])
        pk["bp"] = _cat_vec(dev, [g("a_b"), g("b_b"), g("a_gate_b"), g("b_gate_b"),
                                  g("out_gate_b")])
        pk["Wo"] = _to_act(dev, act, g("out_w"))
    return pk


def grad_views(name, cfg, bank: GradBank):
    """Packed fp32 gradient tensors of one sub-op plus the map from the
    reference's parameter suffixes to (strided) views of them."""
    cm, cz, h, hc, c, t = cfg.c_m, cfg.c_z, cfg.h, cfg.hc, cfg.c_opm, cfg.t_factor
    G, names = {}, {}
    if name in ("row_attn", "col_attn", "tri_attn_start", "tri_attn_end"):
        c_io = cm if name in ("row_attn", "col_attn") else cz
        G["ln_g"], G["ln_b"] = bank.take(c_io), bank.take(c_io)
        if name == "row_attn":
            G["lnz_g"], G["lnz_b"] = bank.take(cz), bank.take(cz)
        G["Wqkvg"] = bank.take(c_io, 4 * hc)
        G["gate_b"] = bank.take(hc)
        if name != "col_attn":
            G["Wb"] = bank.take(cz, h)
        G["Wo"], G["bo"] = bank.take(hc, c_io), bank.take(c_io)
        names.update(ln_g=G["ln_g"], ln_b=G["ln_b"], gate_b=G["gate_b"],
                     q_w=G["Wqkvg"][:, 0:hc], k_w=G["Wqkvg"][:, hc:2 * hc],
                     v_w=G["Wqkvg"][:, 2 * hc:3 * hc], gate_w=G["Wqkvg"][:, 3 * hc:],
                     out_w=G["Wo"], out_b=G["bo"])
        if name == "row_attn":
            names.update(lnz_g=G["lnz_g"], lnz_b=G["lnz_b"])
        if name != "col_attn":
            names["bias_w"] = G["Wb"]
    elif name in ("msa_transition", "pair_transition"):
        cx = cm if name == "msa_transition" else cz
        G["ln_g"], G["ln_b"] = bank.take(cx), bank.take(cx)
        G["W1"], G["b1"] = bank.take(cx, t * cx), bank.take(t * cx)
        G["W2"], G["b2"] = bank.take(t * cx, cx), bank.take(cx)
        names.update(ln_g=G["ln_g"], ln_b=G["ln_b"], w1=G["W1"], b1=G["b1"], w2=G["W2"],
                     b2=G["b2"])
    elif name == "opm":
        G["ln_g"], G["ln_b"] = bank.take(cm), bank.take(cm)
        G["Wab"], G["bab"] = bank.take(cm, 2 * c), bank.take(2 * c)
        G["Wo"], G["bo"] = bank.take(c * c, cz), bank.take(cz)
        names.update(ln_g=G["ln_g"], ln_b=G["ln_b"], a_w=G["Wab"][:, :c], b_w=G["Wab"][:, c:],
                     a_b=G["bab"][:c], b_b=G["bab"][c:], out_w=G["Wo"], out_b=G["bo"])
    else:
        G["ln_g"], G["ln_b"] = bank.take(cz), bank.take(cz)
        G["Wp"], G["bp"] = bank.take(cz, 4 * c + cz), bank.take(4 * c + cz)
        G["p_ln_g"], G["p_ln_b"] = bank.take(c), bank.take(c)
        G["Wo"], G["bo"] = bank.take(c, cz), bank.take(cz)
        Wp, bp = G["Wp"], G["bp"]
        names.update(ln_g=G["ln_g"], ln_b=G["ln_b"], a_w=Wp[:, 0:c], b_w=Wp[:, c:2 * c],
                     a_gate_w=Wp[:, 2 * c:3 * c], b_gate_w=Wp[:, 3 * c:4 * c],
                     out_gate_w=Wp[:, 4 * c:], a_b=bp[0:c], b_b=bp[c:2 * c],
                     a_gate_b=bp[2 * c:3 * c], b_gate_b=bp[3 * c:4 * c], out_gate_b=bp[4 * c:],
                     p_ln_g=G["p_ln_g"], p_ln_b=G["p_ln_b"], out_w=G["Wo"], out_b=G["bo"])
    return G, names


def subop_grad_numel(name, cfg) -> int:
    cm, cz, h, hc, c, t = cfg.c_m, cfg.c_z, cfg.h, cfg.hc, cfg.c_opm, cfg.t_factor
    if name in ("row_attn", "col_attn", "tri_attn_start", "tri_attn_end"):
        c_io = cm if name in ("row_attn", "col_attn") else cz
        n = 2 * c_io + c_io * 4 * hc + hc + hc * c_io + c_io
        if name == "row_attn":
            n += 2 * cz
        if name != "col_attn":
            n += cz * h
        return n
    if name in ("msa_transition", "pair_transition"):
        cx = cm if name == "msa_transition" else cz
        return 2 * cx + cx * t * cx + t * cx + t * cx * cx + cx
    if name == "opm":
        return 2 * cm + cm * 2 * c + 2 * c + c * c * cz + cz
    return 2 * cz + cz * (4 * c + cz) + 4 * c + cz + 2 * c + c * cz + cz


# ---------------------------------------------------------------------------
# gradient hand-off between consecutive sub-op backwards
# ---------------------------------------------------------------------------

def _ln_bwd_out(dy, x, rows, cols, mu, rs, gamma, dgamma, dbeta, dres, act, emit, dev):
    """LayerNorm backward producing a sub-op's input gradient dx (fp32).
    emit (a dict with the consumer's output-bias gradient slot under "bias",
    or None): when the layout allows, the same kernel also writes dx's bf16
    copy (emit["act"], the consumer's GEMM operand) and dx's column sums
    into emit["bias"] (emit["done"] = True), so the consumer skips its cast
    and its bias-gradient column sum."""
    dx = _empty((rows, cols), F32, dev)
    if (emit is not None and cols in (128, 256) and dy.dtype == F32 and dy.is_contiguous()
            and x.is_contiguous() and (dres is None or dres.is_contiguous())):
        dxa = _empty((rows, cols), act, dev) if act != F32 else None
        K.layernorm_bwd_ex(dy, x, rows, cols, mu, rs, gamma, dx, dgamma, dbeta, dres=dres,
                           dx_act=dxa, dx_colsum=emit["bias"])
        emit["act"] = dxa if dxa is not None else dx
        emit["done"] = True
        return dx
    K.layernorm_bwd(dy, x, rows, cols, mu, rs, gamma, dx, dgamma, dbeta, dres=dres)
    return dx


def _bias_fusable(cfg, act):
    """Pair-bias projection fused into the LayerNorm kernels (bf16 path)?"""
    return act != F32 and cfg.c_z == 128 and cfg.h <= 8


def _grad_in(dx_new, rows, cols, act, dev, handoff):
    """(bf16 operand copy of an incoming gradient, bias colsum already done?)"""
    if handoff is not None and handoff.get("act") is not None:
        return handoff["act"], bool(handoff.get("done"))
    if act == F32:
        return dx_new, False
    dxa = _empty((rows, cols), act, dev)
    K.copy2d(dx_new, rows, cols, dxa, s_rs=cols, d_rs=cols)
    return dxa, False


# ---------------------------------------------------------------------------
# geometry of the four attentions (rows of the position-major buffers)
# ---------------------------------------------------------------------------

def attn_geometry(name, cfg):
    """(nb, L, row stride of batch b, row stride of sequence l, rows)."""
    s, r = cfg.s, cfg.r
    if name == "row_attn":
        return s, r, r, 1, s * r
    if name == "col_attn":
        return r, s, 1, r, s * r
    if name == "tri_attn_start":
        return r, r, r, 1, r * r
    return r, r, 1, r, r * r      # tri_attn_end: attends over z^T


# ---------------------------------------------------------------------------
# gated attention sub-ops (row, col, tri start/end)
# ---------------------------------------------------------------------------

def attn_fwd(name, P, px, pk, x, z, cfg, act, resid=True, geom=None, bias_fn=None):
    """x_new = x + attn(x) (fp32 residual fused in the out-projection);
    resid=False returns the delta alone (the reference sub-op's value).
    DAP (dap.py): geom overrides attn_geometry (a row shard of the
    triangle attention: nb = local rows, L = r), and bias_fn maps the
    shard's pair-bias rows [h, rows] to the full [h, r*r] bias
    (the allgather of src/evoformer.py:406-407)."""
    dev = x.device
    h, hc, ch = cfg.h, cfg.hc, cfg.c_head
    nb, L, rb, rl, rows = geom if geom is not None else attn_geometry(name, cfg)
    c_io = x.shape[-1]
    r2 = cfg.r * cfg.r
    ctx = {}
    xh = _empty((rows, c_io), act, dev)
    mu, rs = _empty(rows, F32, dev), _empty(rows, F32, dev)
    K.layernorm(x, rows, c_io, P[f"{px}.ln_g"], P[f"{px}.ln_b"], xh, mu, rs, cfg.eps)
    # the pair-bias projection's backward fuses into the LayerNorm backward of
    # its input on the bf16 path (c_z = 128, h <= 8); in the forward the
    # separate projection kernel is faster than a fused LayerNorm
    # (evo_layernorm_fwd_proj: the per-row 8-way reduction costs occupancy)
    fuse_bias = name != "col_attn" and _bias_fusable(cfg, act)
    ctx.update(x=x, xh=xh, mu=mu, rs=rs, fuse_bias=fuse_bias)
    bias = None
    if name != "col_attn":
        if name == "row_attn":
            zh = _empty((r2, cfg.c_z), act, dev)
            zmu, zrs = _empty(r2, F32, dev), _empty(r2, F32, dev)
            K.layernorm(z, r2, cfg.c_z, P[f"{px}.lnz_g"], P[f"{px}.lnz_b"], zh, zmu, zrs,
                        cfg.eps)
            ctx.update(z=z, zh=zh, zmu=zmu, zrs=zrs)
            brows = r2
        else:
            zh = xh
            brows = rows
        bias = _empty((h, brows), F32, dev)
        # bias[hh, row] = zh[row] . Wb[:, hh]   (C(m=row, n=hh) at hh*brows + row)
        K.gemm(Mat(zh, cfg.c_z, 1), Mat(pk["Wb"], 1, h), Mat(bias, 1, brows), brows, h,
               cfg.c_z)
        if bias_fn is not None:
            bias = bias_fn(bias)
        ctx["bias"] = bias
    proj = _empty((rows, 4 * hc), act, dev)
    K.linear(xh, rows, c_io, pk["Wqkvg"], 4 * hc, 4 * hc, proj, 4 * hc, bias=pk["bqkvg"],
             epi=EPI_SIGMOID_FROM, col0=3 * hc)
    o = _empty((rows, hc), act, dev)
    gm = _empty((rows, hc), act, dev)
    lse = _empty((nb, h, L), F32, dev)
    bq, bk = (cfg.r, 1) if name != "tri_attn_end" else (1, cfg.r)
    # GEMM-composed path (bf16, L > 256 or c_head not 16 / 32): keep the
    # forward's probabilities for the backward instead of recomputing them,
    # when they fit the per-call byte cap (K.KEEP_P_MAX_BYTES)
    p_store = (_empty(K.long_p_elems(nb, h, L), act, dev)
               if K.use_long(act, L, ch) and K.keep_p(nb, h, L) else None)
    K.attention(proj=proj, hc=hc, nb=nb, H=h, L=L, D=ch, scale=ch ** -0.5,
                sb=rb * 4 * hc, sl=rl * 4 * hc, o=o, gm=gm, o_sb=rb * hc, o_sl=rl * hc,
                lse=lse, bias=bias, bh=r2, bq=bq, bk=bk, p_store=p_store)
    ctx["p_store"] = p_store
    x_new = _empty(x.shape, F32, dev)
    K.linear(gm, rows, hc, pk["Wo"], c_io, c_io, x_new, c_io, bias=P[f"{px}.out_b"],
             residual=x if resid else None)
    ctx.update(proj=proj, o=o, gm=gm, lse=lse, resid=resid, geom=(nb, L, rb, rl, rows))
    return x_new, ctx


def attn_bwd(name, P, px, pk, G, ctx, dx_new, cfg, act, handoff=None, emit=None, dz_res=None,
             join=None, dbias_fn=None):
    """Returns (dx [rows, c_io] fp32, dz_row or None).  handoff: the emit
    dict of the producer of dx_new (see _ln_bwd_out); emit: this sub-op's.
    dz_res (row attention, fused path only): added to dz_row inside its
    LayerNorm backward (the block join dz_in = dz_pair + dz_row, one fp32
    addition either way); returns (dx, dz_row + dz_res, True) then."""
    dev = dx_new.device
    h, hc, ch = cfg.h, cfg.hc, cfg.c_head
    nb, L, rb, rl, rows = ctx["geom"]
    c_io = dx_new.shape[-1]
    r2 = cfg.r * cfg.r
    dxa, bias_done = _grad_in(dx_new, rows, c_io, act, dev, handoff)
    off = OffPath()
    # out-projection
    with off.path():
        K.linear_dw(ctx["gm"], rows, hc, dxa, c_io, G["Wo"], c_io)
        if not bias_done:
            K.colsum(dx_new, rows, c_io, G["bo"])
    dgm = _empty((rows, hc), act, dev)
    K.linear_dx(dxa, rows, c_io, pk["Wo"], c_io, hc, dgm)
    # attention core (+ gate) backward
    dproj = _empty((rows, 4 * hc), act, dev)
    dbias = _empty((h, r2), F32, dev) if name != "col_attn" else None
    bq, bk = (cfg.r, 1) if name != "tri_attn_end" else (1, cfg.r)
    # the gate-bias gradient (column sums of dGpre) comes out of the
    # attention backward's prep pass
    K.attention(proj=ctx["proj"], hc=hc, nb=nb, H=h, L=L, D=ch, scale=ch ** -0.5,
                sb=rb * 4 * hc, sl=rl * 4 * hc, o=ctx["o"], gm=ctx["gm"], o_sb=rb * hc,
                o_sl=rl * hc, lse=ctx["lse"], bias=ctx.get("bias"), bh=r2, bq=bq, bk=bk,
                dgm=dgm, dproj=dproj, dbias=dbias, dgate_bias=G["gate_b"],
                p_store=ctx.get("p_store"))
    xh = ctx["xh"]
    with off.path():
        K.linear_dw(xh, rows, c_io, dproj, 4 * hc, G["Wqkvg"], 4 * hc)
    dxh = _empty((rows, c_io), F32, dev)
    K.linear_dx(dproj, rows, 4 * hc, pk["Wqkvg"], 4 * hc, c_io, dxh)
    # pair-bias gradient rows: r*r (row attention: the bias comes from all of
    # z), or this sub-op's rows (triangle attention; under DAP dbias_fn
    # turns the full dbias into the shard's rows: allreduce + own-row slice)
    bstride = r2 if name == "row_attn" else rows
    if dbias is not None and dbias_fn is not None:
        dbias = dbias_fn(dbias)
    dz_row = None
    if dbias is not None and ctx["fuse_bias"]:
        # the pair-bias projection's backward (dz += dbias Wb^T, dWb = LN(z)^T
        # dbias) fuses into the LayerNorm backward of its input
        if name == "row_attn":
            dz_row = _empty((r2, cfg.c_z), F32, dev)
            if join is not None and dz_res is not None:
                join()      # dz_res comes from the pair branch's stream
            K.layernorm_bwd_proj(None, ctx["z"], r2, ctx["zmu"], ctx["zrs"], P[f"{px}.lnz_g"],
                                 P[f"{px}.lnz_b"], dbias, r2, pk["Wb"], h, dz_row, G["lnz_g"],
                                 G["lnz_b"], G["Wb"], dres=dz_res)
        else:
            dres = dx_new if ctx["resid"] else None
            dx = _empty((rows, c_io), F32, dev)
            colsum = None
            dxa_out = None
            if emit is not None:
                dxa_out = _empty((rows, c_io), act, dev)
                colsum = emit["bias"]
            K.layernorm_bwd_proj(dxh, ctx["x"], rows, ctx["mu"], ctx["rs"], P[f"{px}.ln_g"],
                                 P[f"{px}.ln_b"], dbias, bstride, pk["Wb"], h, dx, G["ln_g"],
                                 G["ln_b"], G["Wb"], dres=dres, dx_act=dxa_out,
                                 dx_colsum=colsum)
            if emit is not None:
                emit["act"], emit["done"] = dxa_out, True
            off.join()
            return dx, None
    if dbias is not None and not ctx["fuse_bias"]:
        dbias_a = dbias if act == F32 else _empty((h, bstride), act, dev)
        if act != F32:
            K.copy2d(dbias, h, bstride, dbias_a, s_rs=bstride, d_rs=bstride)
        zh = ctx.get("zh", xh)
        # dWb[c, hh] = sum_row zh[row, c] dbias[hh, row]
        K.gemm(Mat(zh, 1, cfg.c_z), Mat(dbias_a, bstride, 1), Mat(G["Wb"], h, 1), cfg.c_z, h,
               bstride, split_k=K.pick_split(bstride, cfg.c_z, h))
        if name == "row_attn":
            dzh = _empty((r2, cfg.c_z), F32, dev)
            K.gemm(Mat(dbias_a, 1, r2), Mat(pk["Wb"], h, 1), Mat(dzh, cfg.c_z, 1), r2,
                   cfg.c_z, h)
            dz_row = _empty((r2, cfg.c_z), F32, dev)
            K.layernorm_bwd(dzh, ctx["z"], r2, cfg.c_z, ctx["zmu"], ctx["zrs"],
                            P[f"{px}.lnz_g"], dz_row, G["lnz_g"], G["lnz_b"])
        else:
            K.gemm(Mat(dbias_a, 1, bstride), Mat(pk["Wb"], h, 1), Mat(dxh, cfg.c_z, 1), bstride,
                   cfg.c_z, h, accumulate=True)
    dx = _ln_bwd_out(dxh, ctx["x"], rows, c_io, ctx["mu"], ctx["rs"], P[f"{px}.ln_g"],
                     G["ln_g"], G["ln_b"], dx_new if ctx["resid"] else None, act, emit, dev)
    off.join()
    if dz_res is not None:
        if ctx["fuse_bias"]:
            return dx, dz_row, True
        return dx, dz_row, False
    return dx, dz_row


# ---------------------------------------------------------------------------
# transitions (src/evoformer.py:314-329)
# ---------------------------------------------------------------------------

def transition_fwd(P, px, pk, x, cfg, act, resid=True):
    """relu(LN(x) W1 + b1) W2 + b2 (+ x).  On the bf16 path the first
    projection runs as a 3-product bf16 GEMM ([hi | lo | hi] LN(x) against
    [W_hi; W_hi; W_lo], K tripled): fp32-grade pre-activations, so the ReLU
    mask the backward applies is the reference's.  With plain bf16 operands
    near-zero pre-activations flip sign, and every flipped unit drops or
    adds a whole dhid entry in the cancellation-heavy column sums of the
    b1 / LN gradients (measured: the C3 extra stack's msa_transition
    gradients at 5e-2 rel-L2, the same as an oracle with bf16-rounded
    matmul operands; 1.3e-2 with this split)."""
    dev = x.device
    rows, cx = x.shape[0], x.shape[1]
    tc = cfg.t_factor * cx
    mu, rs = _empty(rows, F32, dev), _empty(rows, F32, dev)
    hid = _empty((rows, tc), act, dev)
    if "W1x3" in pk:
        xh = _empty((rows, 3 * cx), act, dev)      # [hi | lo | hi]
        if not K.layernorm_split(x, rows, cx, P[f"{px}.ln_g"], P[f"{px}.ln_b"], xh, mu, rs,
                                 cfg.eps):
            x32 = _empty((rows, cx), F32, dev)
            K.layernorm(x, rows, cx, P[f"{px}.ln_g"], P[f"{px}.ln_b"], x32, mu, rs, cfg.eps)
            K.split_bf16(x32, rows, cx, xh, xh, h_rs=3 * cx, l_rs=3 * cx, hi2=xh, h2_rs=3 * cx,
                         l_off=cx, h2_off=2 * cx)
            del x32
        xh_ld = 3 * cx
        K.linear(xh, rows, 3 * cx, pk["W1x3"], tc, tc, hid, tc, bias=P[f"{px}.b1"],
                 epi=EPI_RELU)
    else:
        xh = _empty((rows, cx), act, dev)
        K.layernorm(x, rows, cx, P[f"{px}.ln_g"], P[f"{px}.ln_b"], xh, mu, rs, cfg.eps)
        xh_ld = cx
        K.linear(xh, rows, cx, pk["W1"], tc, tc, hid, tc, bias=P[f"{px}.b1"], epi=EPI_RELU)
    x_new = _empty(x.shape, F32, dev)
    K.linear(hid, rows, tc, pk["W2"], cx, cx, x_new, cx, bias=P[f"{px}.b2"],
             residual=x if resid else None)
    return x_new, dict(x=x, xh=xh, xh_ld=xh_ld, mu=mu, rs=rs, hid=hid, resid=resid)


def transition_bwd(P, px, pk, G, ctx, dx_new, cfg, act, handoff=None, emit=None):
    dev = dx_new.device
    rows, cx = dx_new.shape[0], dx_new.shape[1]
    tc = cfg.t_factor * cx
    dxa, bias_done = _grad_in(dx_new, rows, cx, act, dev, handoff)
    off = OffPath()
    with off.path():
        K.linear_dw(ctx["hid"], rows, tc, dxa, cx, G["W2"], cx)
        if not bias_done:
            K.colsum(dx_new, rows, cx, G["b2"])
    dhid = _empty((rows, tc), act, dev)
    K.linear_dx(dxa, rows, cx, pk["W2"], cx, tc, dhid)
    if act != F32 and tc % 8 == 0:
        K.relu_bwd_colsum(dhid, ctx["hid"], dhid, rows, tc, G["b1"])
        with off.path():
            K.linear_dw(ctx["xh"], rows, cx, dhid, tc, G["W1"], tc, x_ld=ctx["xh_ld"])
    else:
        K.relu_bwd(dhid, ctx["hid"], dhid, rows * tc)
        with off.path():
            K.linear_dw(ctx["xh"], rows, cx, dhid, tc, G["W1"], tc, x_ld=ctx["xh_ld"])
            K.colsum(dhid, rows, tc, G["b1"])
    dxh = _empty((rows, cx), F32, dev)
    K.linear_dx(dhid, rows, tc, pk["W1"], tc, cx, dxh)
    dx = _ln_bwd_out(dxh, ctx["x"], rows, cx, ctx["mu"], ctx["rs"], P[f"{px}.ln_g"],
                     G["ln_g"], G["ln_b"], dx_new if ctx["resid"] else None, act, emit, dev)
    off.join()
    return dx


# ---------------------------------------------------------------------------
# outer product mean (src/evoformer.py:332-352)
# ---------------------------------------------------------------------------

def opm_fwd(P, px, pk, m, z_pair, cfg, act, s_norm=None, with_bias=True):
    """z_out = z_pair + opm(m): the block-end join (src/evoformer.py:460)
    fused as the out-projection's residual.  DAP (dap.py): m is an s-row
    shard (cfg.s = its rows), s_norm the full s of the mean, and only one
    rank of the group adds out_b before the partial sums are allreduced
    (src/evoformer.py:350-356)."""
    dev = m.device
    s, r, cm, c, cz = cfg.s, cfg.r, cfg.c_m, cfg.c_opm, cfg.c_z
    rows, rc = s * r, r * c
    mh = _empty((rows, cm), act, dev)
    mu, rs = _empty(rows, F32, dev), _empty(rows, F32, dev)
    K.layernorm(m, rows, cm, P[f"{px}.ln_g"], P[f"{px}.ln_b"], mh, mu, rs, cfg.eps)
    ab = _empty((2, rows, c), act, dev)       # a = ab[0] [s, r, c], b = ab[1]
    K.gemm(Mat(mh, cm, 1), Mat(pk["Wab"], 1, 2 * c), Mat(ab, c, rows * c, cdiv=c, cs0=1),
           rows, 2 * c, cm, bias=pk["bab"])
    # o[i,j,p,q] = (1/s) sum_s a[s,i,p] b[s,j,q];  m=(i,p), n=(j,q)
    o = _empty((r, r, c, c), act, dev)
    K.gemm(Mat(ab[0], 1, rc), Mat(ab[1], 1, rc),
           Mat(o, r * c * c, c * c, rdiv=c, rs0=c, cdiv=c, cs0=1), rc, rc, s,
           alpha=1.0 / (s_norm or s))
    z_out = _empty((r * r, cz), F32, dev)
    K.linear(o, r * r, c * c, pk["Wo"], cz, cz, z_out, cz,
             bias=P[f"{px}.out_b"] if with_bias else None,
             residual=z_pair)  # z_pair None => the delta alone
    return z_out, dict(m=m, mh=mh, mu=mu, rs=rs, ab=ab, o=o)


def opm_bwd(P, px, pk, G, ctx, dz_out, dz_out_act, dm_res, cfg, act, emit=None, s_norm=None):
    """Returns dm = dm_res + d(opm)/dm (s_norm: see opm_fwd)."""
    dev = dz_out.device
    s, r, cm, c, cz = cfg.s, cfg.r, cfg.c_m, cfg.c_opm, cfg.c_z
    rows, rc, r2 = s * r, r * c, r * r
    o, ab = ctx["o"], ctx["ab"]
    off = OffPath()
    with off.path():
        K.linear_dw(o, r2, c * c, dz_out_act, cz, G["Wo"], cz)
        K.colsum(dz_out, r2, cz, G["bo"])
    # do'[i,p,j,q] = (1/s) dz_out[(i,j)] . Wo[(p,q)]   (raw layout [(i,p),(j,q)])
    dor = _empty((rc, rc), act, dev)
    K.gemm(Mat(dz_out_act, cz, 1), Mat(pk["Wo"], cz, 1),
           Mat(dor, c * r * c, r * c, rdiv=r, rs0=c, cdiv=c, cs0=1), r2, c * c, cz,
           alpha=1.0 / (s_norm or s))
    dab = _empty((2, rows, c), act, dev)
    # da[s,(i,p)] = sum_(j,q) b[s,(j,q)] do'[(i,p),(j,q)]   (m = s: row-major
    # output for the TMA store; split-K fills the SMs: only s/128 x rc/128 tiles)
    sk = K.pick_split(rc, s, rc)
    K.gemm(Mat(ab[1], rc, 1), Mat(dor, rc, 1), Mat(dab[0], rc, 1), s, rc, rc, split_k=sk)
    # db[s,(j,q)] = sum_(i,p) a[s,(i,p)] do'[(i,p),(j,q)]
    K.gemm(Mat(ab[0], rc, 1), Mat(dor, 1, rc), Mat(dab[1], rc, 1), s, rc, rc, split_k=sk)
    mh = ctx["mh"]
    with off.path():
        # dWab[:, w*c:(w+1)*c] = mh^T dab[w]   (batched over w)
        K.gemm(Mat(mh, 1, cm, bs1=0), Mat(dab, 1, c, bs1=rows * c),
               Mat(G["Wab"], 2 * c, 1, bs1=c), cm, c, rows, B1=2,
               split_k=K.pick_split(rows, cm, c, 2))
        K.colsum(dab[0], rows, c, G["bab"][:c])
        K.colsum(dab[1], rows, c, G["bab"][c:])
    dmh = _empty((rows, cm), F32, dev)
    K.gemm(Mat(dab[0], c, 1), Mat(pk["Wab"], 2 * c, 1), Mat(dmh, cm, 1), rows, cm, c)
    K.gemm(Mat(dab[1], c, 1), Mat(pk["Wab"], 2 * c, 1, off=c), Mat(dmh, cm, 1), rows, cm, c,
           accumulate=True)
    dm = _ln_bwd_out(dmh, ctx["m"], rows, cm, ctx["mu"], ctx["rs"], P[f"{px}.ln_g"],
                     G["ln_g"], G["ln_b"], dm_res, act, emit, dev)
    off.join()
    return dm


# ---------------------------------------------------------------------------
# triangle multiplicative update (src/evoformer.py:359-397)
# ---------------------------------------------------------------------------

def _trimul_contract(incoming, a_cf, b_cf, out, r, c):
    """p[ch,i,j] = sum_k a[ch,i,k] b[ch,j,k] (out) | a[ch,k,i] b[ch,k,j] (in)."""
    r2 = r * r
    if not incoming:
        A, B = Mat(a_cf, r, 1, bs1=r2), Mat(b_cf, r, 1, bs1=r2)
    else:
        A, B = Mat(a_cf, 1, r, bs1=r2), Mat(b_cf, 1, r, bs1=r2)
    K.gemm(A, B, Mat(out, r, 1, bs1=r2), r, r, r, B1=c)


def trimul_fwd(name, P, px, pk, z, cfg, act, resid=True):
    dev = z.device
    r, c, cz = cfg.r, cfg.c_opm, cfg.c_z
    r2, ldp = r * r, 4 * c + cz
    incoming = name.endswith("_in")
    zh = _empty((r2, cz), act, dev)
    mu, rs = _empty(r2, F32, dev), _empty(r2, F32, dev)
    K.layernorm(z, r2, cz, P[f"{px}.ln_g"], P[f"{px}.ln_b"], zh, mu, rs, cfg.eps)
    proj = _empty((r2, ldp), act, dev)
    K.linear(zh, r2, cz, pk["Wp"], ldp, ldp, proj, ldp, bias=pk["bp"], epi=EPI_SIGMOID_FROM,
             col0=2 * c)
    a_cf = _empty((c, r, r), act, dev)
    b_cf = _empty((c, r, r), act, dev)
    K.trimul_gate_fwd(proj, r2, c, ldp, a_cf, b_cf)
    p_cf = _empty((c, r, r), F32, dev)
    _trimul_contract(incoming, a_cf, b_cf, p_cf, r, c)
    pn = _empty((r2, c), act, dev)
    pmu, prs = _empty(r2, F32, dev), _empty(r2, F32, dev)
    K.layernorm(p_cf, r2, c, P[f"{px}.p_ln_g"], P[f"{px}.p_ln_b"], pn, pmu, prs, cfg.eps,
                x_rs=1, x_cs=r2)
    o = _empty((r2, cz), act, dev)
    K.linear(pn, r2, c, pk["Wo"], cz, cz, o, cz, bias=P[f"{px}.out_b"])
    z_new = _empty(z.shape, F32, dev)
    if resid:
        K.outgate_fwd(z, r2, cz, proj, ldp, 4 * c, o, z_new)
    else:
        K.mul2d(proj, ldp, 4 * c, o, cz, z_new, r2, cz)
    return z_new, dict(z=z, zh=zh, mu=mu, rs=rs, proj=proj, a_cf=a_cf, b_cf=b_cf, p_cf=p_cf,
                       pn=pn, pmu=pmu, prs=prs, o=o, incoming=incoming, resid=resid)


def trimul_bwd(P, px, pk, G, ctx, dz_new, cfg, act):
    dev = dz_new.device
    r, c, cz = cfg.r, cfg.c_opm, cfg.c_z
    r2, ldp = r * r, 4 * c + cz
    proj = ctx["proj"]
    dproj = _empty((r2, ldp), act, dev)
    do = _empty((r2, cz), act, dev)
    # bf16: the out_b / out_gate_b / a,b value and gate bias gradients are
    # column sums of the fp32 values inside the gate kernels (not of the
    # bf16-rounded dproj / do: those sums cancel heavily at small widths)
    fused_cs = act != F32 and cz % 8 == 0 and ldp % 8 == 0
    if fused_cs:
        K.outgate_bwd(dz_new, r2, cz, proj, ldp, 4 * c, ctx["o"], do, dproj, ldp, 4 * c,
                      do_colsum=G["bo"], dg_colsum=G["bp"][4 * c:])
    else:
        K.outgate_bwd(dz_new, r2, cz, proj, ldp, 4 * c, ctx["o"], do, dproj, ldp, 4 * c)
    off = OffPath()
    with off.path():
        K.linear_dw(ctx["pn"], r2, c, do, cz, G["Wo"], cz)
        if not fused_cs:
            K.colsum(do, r2, cz, G["bo"])
    dpn = _empty((r2, c), F32, dev)
    K.linear_dx(do, r2, cz, pk["Wo"], cz, c, dpn)
    dp_cf = _empty((c, r, r), act, dev)
    K.layernorm_bwd(dpn, ctx["p_cf"], r2, c, ctx["pmu"], ctx["prs"], P[f"{px}.p_ln_g"], dp_cf,
                    G["p_ln_g"], G["p_ln_b"], x_rs=1, x_cs=r2, dx_rs=1, dx_cs=r2)
    a_cf, b_cf = ctx["a_cf"], ctx["b_cf"]
    da_cf = _empty((c, r, r), F32, dev)
    db_cf = _empty((c, r, r), F32, dev)
    if not ctx["incoming"]:
        # da[i,k] = sum_j dp[i,j] b[j,k];  db[j,k] = sum_i dp[i,j] a[i,k]
        K.gemm(Mat(dp_cf, r, 1, bs1=r2), Mat(b_cf, 1, r, bs1=r2), Mat(da_cf, r, 1, bs1=r2),
               r, r, r, B1=c)
        K.gemm(Mat(dp_cf, 1, r, bs1=r2), Mat(a_cf, 1, r, bs1=r2), Mat(db_cf, r, 1, bs1=r2),
               r, r, r, B1=c)
    else:
        # da[k,i] = sum_j b[k,j] dp[i,j];  db[k,j] = sum_i a[k,i] dp[i,j]
        K.gemm(Mat(b_cf, r, 1, bs1=r2), Mat(dp_cf, r, 1, bs1=r2), Mat(da_cf, r, 1, bs1=r2),
               r, r, r, B1=c)
        K.gemm(Mat(a_cf, r, 1, bs1=r2), Mat(dp_cf, 1, r, bs1=r2), Mat(db_cf, r, 1, bs1=r2),
               r, r, r, B1=c)
    K.trimul_gate_bwd(proj, r2, c, ldp, da_cf, db_cf, dproj, ldp,
                      colsum=G["bp"][:4 * c] if fused_cs else None)
    zh = ctx["zh"]
    with off.path():
        K.linear_dw(zh, r2, cz, dproj, ldp, G["Wp"], ldp)
        if not fused_cs:
            K.colsum(dproj, r2, ldp, G["bp"])
    dzh = _empty((r2, cz), F32, dev)
    K.linear_dx(dproj, r2, ldp, pk["Wp"], ldp, cz, dzh)
    dz = _empty((r2, cz), F32, dev)
    K.layernorm_bwd(dzh, ctx["z"], r2, cz, ctx["mu"], ctx["rs"], P[f"{px}.ln_g"], dz,
                    G["ln_g"], G["ln_b"], dres=dz_new if ctx["resid"] else None)
    off.join()
    return dz


# ---------------------------------------------------------------------------
# the parallel block (src/evoformer.py:456-461)
# ---------------------------------------------------------------------------

class BlockGrads:
    """Per-block, per-branch flat fp32 gradient buffers + reference names."""

    def __init__(self, blk, cfg, dev):
        self.msa = GradBank(sum(subop_grad_numel(n, cfg) for n in MSA_SUBOPS), dev)
        self.pair = GradBank(sum(subop_grad_numel(n, cfg) for n in PAIR_SUBOPS), dev)
        self.packed, self.names = {}, {}
        for n in MSA_SUBOPS + PAIR_SUBOPS:
            bank = self.msa if n in MSA_SUBOPS else self.pair
            G, names = grad_views(n, cfg, bank)
            self.packed[n] = G
            for suffix, v in names.items():
                self.names[f"blk{blk}.{n}.{suffix}"] = v


def pack_block(P, blk, cfg, act, dev, subops=MSA_SUBOPS + PAIR_SUBOPS):
    return {n: pack_subop(P, f"blk{blk}.{n}", n, cfg, act, dev) for n in subops}


def msa_branch_fwd(P, blk, pk, m, z, cfg, act):
    """MSA track + OPM operand state; returns (m_new, ctxs)."""
    s, r = cfg.s, cfg.r
    ctxs = {}
    m2 = m.reshape(s * r, cfg.c_m)
    m2, ctxs["row_attn"] = attn_fwd("row_attn", P, f"blk{blk}.row_attn", pk["row_attn"], m2,
                                    z.reshape(r * r, cfg.c_z), cfg, act)
    m2, ctxs["col_attn"] = attn_fwd("col_attn", P, f"blk{blk}.col_attn", pk["col_attn"], m2,
                                    None, cfg, act)
    m2, ctxs["msa_transition"] = transition_fwd(P, f"blk{blk}.msa_transition",
                                                pk["msa_transition"], m2, cfg, act)
    return m2, ctxs


def pair_branch_fwd(P, blk, pk, z, cfg, act):
    r = cfg.r
    ctxs = {}
    z2 = z.reshape(r * r, cfg.c_z)
    for n in ("tri_mult_out", "tri_mult_in"):
        z2, ctxs[n] = trimul_fwd(n, P, f"blk{blk}.{n}", pk[n], z2, cfg, act)
    for n in ("tri_attn_start", "tri_attn_end"):
        z2, ctxs[n] = attn_fwd(n, P, f"blk{blk}.{n}", pk[n], z2, None, cfg, act)
    z2, ctxs["pair_transition"] = transition_fwd(P, f"blk{blk}.pair_transition",
                                                 pk["pair_transition"], z2, cfg, act)
    return z2, ctxs


def pair_branch_bwd(P, blk, pk, G, ctxs, dz, cfg, act, dz_act=None):
    """dz: grad of the pair-track output (dz_act: its bf16 copy, if made);
    returns dz_pair (grad of z_in through the pair track, residual included).
    Each LayerNorm backward hands its output's bf16 copy and column sums to
    the next sub-op (_ln_bwd_out)."""
    h0 = None if dz_act is None else dict(act=dz_act, done=False)
    e1 = dict(bias=G["tri_attn_end"]["bo"])
    dz = transition_bwd(P, f"blk{blk}.pair_transition", pk["pair_transition"],
                        G["pair_transition"], ctxs["pair_transition"], dz, cfg, act,
                        handoff=h0, emit=e1)
    e2 = dict(bias=G["tri_attn_start"]["bo"])
    dz, _ = attn_bwd("tri_attn_end", P, f"blk{blk}.tri_attn_end", pk["tri_attn_end"],
                     G["tri_attn_end"], ctxs["tri_attn_end"], dz, cfg, act, handoff=e1, emit=e2)
    dz, _ = attn_bwd("tri_attn_start", P, f"blk{blk}.tri_attn_start", pk["tri_attn_start"],
                     G["tri_attn_start"], ctxs["tri_attn_start"], dz, cfg, act, handoff=e2)
    for n in ("tri_mult_in", "tri_mult_out"):
        dz = trimul_bwd(P, f"blk{blk}.{n}", pk[n], G[n], ctxs[n], dz, cfg, act)
    return dz


def msa_emit(G):
    """Hand-off slot for the OPM backward's output (-> msa_transition)."""
    return dict(bias=G["msa_transition"]["b2"])


def msa_branch_bwd(P, blk, pk, G, ctxs, dm, cfg, act, handoff=None, dz_pair=None, join=None):
    """dm: grad of the MSA-track output (incl. the OPM contribution; handoff:
    the OPM backward's emit dict); returns (dm_in, dz_row), or with dz_pair
    given (single-process block) (dm_in, dz_in = dz_pair + dz_row).  join:
    called right before the first launch that reads dz_pair (the pair
    branch's stream joins there)."""
    e1 = dict(bias=G["col_attn"]["bo"])
    dm = transition_bwd(P, f"blk{blk}.msa_transition", pk["msa_transition"],
                        G["msa_transition"], ctxs["msa_transition"], dm, cfg, act,
                        handoff=handoff, emit=e1)
    e2 = dict(bias=G["row_attn"]["bo"])
    dm, _ = attn_bwd("col_attn", P, f"blk{blk}.col_attn", pk["col_attn"], G["col_attn"],
                     ctxs["col_attn"], dm, cfg, act, handoff=e1, emit=e2)
    if dz_pair is None:
        dm, dz_row = attn_bwd("row_attn", P, f"blk{blk}.row_attn", pk["row_attn"],
                              G["row_attn"], ctxs["row_attn"], dm, cfg, act, handoff=e2)
        return dm, dz_row
    dm, dz, joined = attn_bwd("row_attn", P, f"blk{blk}.row_attn", pk["row_attn"],
                              G["row_attn"], ctxs["row_attn"], dm, cfg, act, handoff=e2,
                              dz_res=dz_pair, join=join)
    if not joined:
        if join is not None:
            join()
        dz_in = torch.empty_like(dz_pair)
        K.add(dz_pair, dz, dz_in)
        dz = dz_in
    return dm, dz


def block_fwd(P, blk, pk, m, z, cfg, act):
    """Parallel block: (m', z') with z' = pair_track(z) + opm(msa_track(m, z));
    the af2 / multimer wirings dispatch to variant_block_fwd."""
    if cfg.variant != "parallel":
        return variant_block_fwd(P, blk, pk, m, z, cfg, act)
    if BRANCH_STREAMS:
        # the two tracks are independent inside a parallel block (the premise
        # of branch parallelism): the pair track runs on a second stream of
        # this GPU while the MSA track runs here, joined before the OPM
        main, side = torch.cuda.current_stream(m.device), side_stream(m.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            z_pair, cp_ = pair_branch_fwd(P, blk, pk, z, cfg, act)
        m_new, cm_ = msa_branch_fwd(P, blk, pk, m, z, cfg, act)
        main.wait_stream(side)
    else:
        m_new, cm_ = msa_branch_fwd(P, blk, pk, m, z, cfg, act)
        z_pair, cp_ = pair_branch_fwd(P, blk, pk, z, cfg, act)
    z_new, co = opm_fwd(P, f"blk{blk}.opm", pk["opm"], m_new, z_pair, cfg, act)
    ctx = dict(msa=cm_, pair=cp_, opm=co)
    return m_new, z_new, ctx


def cast_act(x, act):
    if x.dtype == act:
        return x
    out = torch.empty(x.shape, dtype=act, device=x.device)
    K.copy2d(x, 1, x.numel(), out, s_rs=x.numel(), d_rs=x.numel())
    return out


def variant_block_fwd(P, blk, pk, m, z, cfg, act):
    """The serial wirings (src/evoformer.py:448-455), same native sub-op
    launches with every residual add fused into the producing GEMM:
      af2:      m' = msa_track(m, z); z1 = z + opm(m'); z' = pair_track(z1)
      multimer: z1 = z + opm(m);  m' = msa_track(m, z1); z' = pair_track(z1)"""
    if cfg.variant == "af2":
        m_new, cm_ = msa_branch_fwd(P, blk, pk, m, z, cfg, act)
        z1, co = opm_fwd(P, f"blk{blk}.opm", pk["opm"], m_new, z, cfg, act)
    else:
        z1, co = opm_fwd(P, f"blk{blk}.opm", pk["opm"], m, z, cfg, act)
        m_new, cm_ = msa_branch_fwd(P, blk, pk, m, z1, cfg, act)
    z_new, cp_ = pair_branch_fwd(P, blk, pk, z1, cfg, act)
    return m_new, z_new, dict(msa=cm_, pair=cp_, opm=co)


def variant_block_bwd(P, blk, pk, G, ctx, dm_out, dz_out, cfg, act):
    """VJP of variant_block_fwd; returns (dm_in, dz_in)."""
    dz1 = pair_branch_bwd(P, blk, pk, G, ctx["pair"], dz_out, cfg, act,
                          dz_act=cast_act(dz_out, act))
    if cfg.variant == "af2":
        e0 = msa_emit(G)
        dm1 = opm_bwd(P, f"blk{blk}.opm", pk["opm"], G["opm"], ctx["opm"], dz1,
                      cast_act(dz1, act), dm_out, cfg, act, emit=e0)
        # dz_in = dz1 (residual of z1 = z + opm) + dz_row (row attention's bias)
        return msa_branch_bwd(P, blk, pk, G, ctx["msa"], dm1, cfg, act, handoff=e0,
                              dz_pair=dz1)
    # multimer: the MSA track read z1, so its dz_row joins dz1 before the OPM
    dm1, dz1 = msa_branch_bwd(P, blk, pk, G, ctx["msa"], dm_out, cfg, act, dz_pair=dz1)
    dm = opm_bwd(P, f"blk{blk}.opm", pk["opm"], G["opm"], ctx["opm"], dz1, cast_act(dz1, act),
                 dm1, cfg, act)
    return dm, dz1


def block_bwd(P, blk, pk, G, ctx, dm_out, dz_out, cfg, act):
    """Returns (dm_in, dz_in) with dz_in = dz_pair + dz_row: the same two
    operands, in the same order, as the BP allreduce (src/comm.py:206-210)."""
    if cfg.variant != "parallel":
        return variant_block_bwd(P, blk, pk, G, ctx, dm_out, dz_out, cfg, act)
    dz_act = cast_act(dz_out, act)
    e0 = msa_emit(G)
    join = None
    if BRANCH_STREAMS:
        # pair-track backward on the second stream, concurrent with the OPM
        # and MSA-track backward; joined where dz_pair is consumed
        main, side = torch.cuda.current_stream(dz_out.device), side_stream(dz_out.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            dz_pair = pair_branch_bwd(P, blk, pk, G, ctx["pair"], dz_out, cfg, act,
                                      dz_act=dz_act)
        join = lambda: main.wait_stream(side)
        dm3 = opm_bwd(P, f"blk{blk}.opm", pk["opm"], G["opm"], ctx["opm"], dz_out, dz_act,
                      dm_out, cfg, act, emit=e0)
    else:
        dm3 = opm_bwd(P, f"blk{blk}.opm", pk["opm"], G["opm"], ctx["opm"], dz_out, dz_act,
                      dm_out, cfg, act, emit=e0)
        dz_pair = pair_branch_bwd(P, blk, pk, G, ctx["pair"], dz_out, cfg, act, dz_act=dz_act)
    # dz_in = dz_pair + dz_row (the BP allreduce's two operands), joined
    # inside the row attention's LayerNorm backward when fused
    dm_in, dz_in = msa_branch_bwd(P, blk, pk, G, ctx["msa"], dm3, cfg, act, handoff=e0,
                                  dz_pair=dz_pair, join=join)
    return dm_in, dz_in
