"""DAP: axial sharding of every sub-op over a group of ranks
(src/schedules.py:96-154, the shard hooks of src/evoformer.py:242-441).

Every rank of a DAP group holds the full m and z.  A sub-op computes the
delta of its own row shard (rows [lo, hi) of the axis the reference shards:
s for row attention, the MSA transition and the outer product mean, r for
column attention and every pair sub-op) on the native kernels of engine.py,
and the deltas are allgathered into the full tensor.  The backward follows
the reference's three shard primitives:

  enter(t)     its VJP allreduces the zero-padded shard gradient of t over
               the group (every sub-op input, the gathered partner
               projections of the triangle multiplication and the gathered
               pair-bias rows of triangle attention)
  gather(t)    allgather along the shard axis; its VJP keeps the rank's rows
  reduce_sum   the outer product mean's partial sums (fwd allreduce; the VJP
               passes the gradient through); out_b is added once and its
               gradient is replicated, not summed

so the collectives -- kinds, groups, element counts and phases -- are the
reference's one for one (expected_comm_volume's DAP rows).  Layouts in HBM
are engine.py's position-major ones; shard extraction, axis permutations and
the placement of gathered shards are batched strided copies (evo_copy3d),
the zero padding a memset (evo_zero).
"""

from __future__ import annotations

import dataclasses
import os

import torch

from . import engine as E
from . import kernels as K
from ._native import EPI_SIGMOID_FROM
from .errors import DimensionError
from .kernels import Mat

F32 = torch.float32
_DEBUG = os.environ.get("EVO_DAP_DEBUG") == "1"


def _chk(tag, t):
    """EVO_DAP_DEBUG=1: report non-finite sub-op results (diagnostics only)."""
    if _DEBUG and not bool(torch.isfinite(t).all()):
        print(f"[dap] non-finite {tag} {tuple(t.shape)}", flush=True)
    return t


class DapShard:
    """The DAP context of one rank (src/schedules.py:96-154) over a Comm."""

    def __init__(self, comm, group):
        self.comm = comm
        self.group = tuple(group)
        self.index = self.group.index(comm.rank)
        self.n = len(self.group)

    def bounds(self, size: int):
        if size % self.n != 0:
            raise DimensionError(f"axis of size {size} does not split over {self.n} shards")
        w = size // self.n
        return self.index * w, (self.index + 1) * w

    # -- collectives ---------------------------------------------------------
    def gather_rows(self, t, phase="fwd"):
        """Allgather of row shards [R, C] -> [n*R, C] (axis 0)."""
        out = torch.empty((self.n * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
        return self.comm.allgather(self.group, t, out, phase)

    def allreduce(self, t, phase):
        return self.comm.allreduce_sum(self.group, t, phase)

    def enter_rows(self, d_loc, total_rows, lo_row):
        """VJP of enter + row slice: the zero-padded [total_rows, C] gradient
        with rows [lo_row, lo_row + R) = d_loc, allreduced."""
        full = torch.empty((total_rows,) + tuple(d_loc.shape[1:]), dtype=F32,
                           device=d_loc.device)
        K.zero(full)
        cols = d_loc.numel() // d_loc.shape[0]
        K.copy2d(d_loc, d_loc.shape[0], cols, full, s_rs=cols, d_rs=cols, d_off=lo_row * cols)
        return self.allreduce(full, "bwd")


def _cfg(cfg, **kw):
    return dataclasses.replace(cfg, **kw)


def _add(a, b):
    out = torch.empty_like(a)
    K.add(a, b, out)
    return out


# ---------------------------------------------------------------------------
# axis-1 shards of [A, B, C] position-major tensors (col_attn, tri_attn_end)
# ---------------------------------------------------------------------------

def _cols(x, A, B, C, lo, w, transpose=False):
    """x [A, B, C] -> [A, w, C] = x[:, lo:lo+w] (transpose: [w, A, C])."""
    out = torch.empty((A * w, C) if not transpose else (w * A, C), dtype=x.dtype,
                      device=x.device)
    if not transpose:
        K.copy3d(x, A, w, C, out, s_bs=B * C, s_rs=C, d_bs=w * C, d_rs=C, s_off=lo * C)
    else:
        # out[j, a, :] = x[a, lo + j, :]
        K.copy3d(x, w, A, C, out, s_bs=C, s_rs=B * C, d_bs=A * C, d_rs=C, s_off=lo * C)
    return out


def _place_cols(buf, n, A, w, C, out, transpose=False):
    """Gathered axis-1 shards buf [n, A, w, C] (transpose: [n, w, A, C]) ->
    out [A, n*w, C]."""
    B = n * w
    for k in range(n):
        if not transpose:
            K.copy3d(buf, A, w, C, out, s_bs=w * C, s_rs=C, d_bs=B * C, d_rs=C,
                     s_off=k * A * w * C, d_off=k * w * C)
        else:
            # out[a, k*w + j, :] = buf[k, j, a, :]
            K.copy3d(buf, w, A, C, out, s_bs=A * C, s_rs=C, d_bs=C, d_rs=B * C,
                     s_off=k * w * A * C, d_off=k * w * C)
    return out


def _enter_cols(sh, d_loc, A, B, C, lo, w, transpose=False):
    """VJP of enter + axis-1 slice: zero [A, B, C] with columns lo:lo+w =
    d_loc ([A, w, C], transpose: [w, A, C]), allreduced."""
    full = torch.empty((A * B, C), dtype=F32, device=d_loc.device)
    K.zero(full)
    if not transpose:
        K.copy3d(d_loc, A, w, C, full, s_bs=w * C, s_rs=C, d_bs=B * C, d_rs=C, d_off=lo * C)
    else:
        K.copy3d(d_loc, w, A, C, full, s_bs=A * C, s_rs=C, d_bs=C, d_rs=B * C, d_off=lo * C)
    return sh.allreduce(full, "bwd")


# ---------------------------------------------------------------------------
# MSA track sub-ops
# ---------------------------------------------------------------------------

def row_attn_fwd(st, sh, blk, m, z):
    """src/evoformer.py:289-297: shard s; z whole (entered)."""
    cfg, act = st.cfg, st.act
    s, r = cfg.s, cfg.r
    lo, hi = sh.bounds(s)
    px = f"blk{blk}.row_attn"
    d, ctx = E.attn_fwd("row_attn", st.P, px, st.packs[blk]["row_attn"], m[lo * r:hi * r], z,
                        _cfg(cfg, s=hi - lo), act, resid=False)
    return _add(m, sh.gather_rows(_chk("row_attn", d))), (ctx, lo, hi)


def row_attn_bwd(st, sh, blk, c, dm):
    """Returns (dm_in, dz) -- both complete over the group."""
    cfg, act = st.cfg, st.act
    ctx, lo, hi = c
    r = cfg.r
    G = st.grads[blk].packed["row_attn"]
    dx, dz = E.attn_bwd("row_attn", st.P, f"blk{blk}.row_attn", st.packs[blk]["row_attn"], G,
                        ctx, dm[lo * r:hi * r].contiguous(), _cfg(cfg, s=hi - lo), act)
    dm_in = _add(dm, sh.enter_rows(dx, cfg.s * r, lo * r))
    return dm_in, sh.allreduce(dz, "bwd")


def col_attn_fwd(st, sh, blk, m):
    """src/evoformer.py:300-311: shard r (columns of m)."""
    cfg, act = st.cfg, st.act
    s, r, cm = cfg.s, cfg.r, cfg.c_m
    lo, hi = sh.bounds(r)
    w = hi - lo
    x = _cols(m, s, r, cm, lo, w)
    d, ctx = E.attn_fwd("col_attn", st.P, f"blk{blk}.col_attn", st.packs[blk]["col_attn"], x,
                        None, _cfg(cfg, r=w), act, resid=False)
    buf = sh.gather_rows(d)                        # [n, s, w, c_m]
    full = torch.empty_like(m)
    _place_cols(buf, sh.n, s, w, cm, full)
    return _add(m, full), (ctx, lo, w)


def col_attn_bwd(st, sh, blk, c, dm):
    cfg, act = st.cfg, st.act
    ctx, lo, w = c
    s, r, cm = cfg.s, cfg.r, cfg.c_m
    G = st.grads[blk].packed["col_attn"]
    dx, _ = E.attn_bwd("col_attn", st.P, f"blk{blk}.col_attn", st.packs[blk]["col_attn"], G,
                       ctx, _cols(dm, s, r, cm, lo, w), _cfg(cfg, r=w), act)
    return _add(dm, _enter_cols(sh, dx, s, r, cm, lo, w))


def transition_fwd(st, sh, blk, name, x, rows_axis):
    """src/evoformer.py:314-329: shard the leading axis (s or the first r)."""
    cfg, act = st.cfg, st.act
    R = x.shape[0] // rows_axis            # rows per leading index
    lo, hi = sh.bounds(rows_axis)
    d, ctx = E.transition_fwd(st.P, f"blk{blk}.{name}", st.packs[blk][name], x[lo * R:hi * R],
                              cfg, act, resid=False)
    return _add(x, sh.gather_rows(_chk(name, d))), (ctx, lo, hi, R)


def transition_bwd(st, sh, blk, name, c, dx_out):
    cfg, act = st.cfg, st.act
    ctx, lo, hi, R = c
    G = st.grads[blk].packed[name]
    dx = E.transition_bwd(st.P, f"blk{blk}.{name}", st.packs[blk][name], G, ctx,
                          dx_out[lo * R:hi * R].contiguous(), cfg, act)
    return _add(dx_out, sh.enter_rows(dx, dx_out.shape[0], lo * R))


def opm_fwd(st, sh, blk, m):
    """src/evoformer.py:332-356: shard s; partial sums reduce_sum'd, out_b once."""
    cfg, act = st.cfg, st.act
    s, r = cfg.s, cfg.r
    lo, hi = sh.bounds(s)
    o, ctx = E.opm_fwd(st.P, f"blk{blk}.opm", st.packs[blk]["opm"], m[lo * r:hi * r], None,
                       _cfg(cfg, s=hi - lo), act, s_norm=s, with_bias=sh.index == 0)
    _chk("opm part", o)
    sh.allreduce(o, "fwd")
    return o, (ctx, lo, hi)


def opm_bwd(st, sh, blk, c, d_o):
    """Returns the (complete) gradient of m through the OPM."""
    cfg, act = st.cfg, st.act
    ctx, lo, hi = c
    r = cfg.r
    G = st.grads[blk].packed["opm"]
    dm = E.opm_bwd(st.P, f"blk{blk}.opm", st.packs[blk]["opm"], G, ctx, d_o,
                   E.cast_act(d_o, act), None, _cfg(cfg, s=hi - lo), act, s_norm=cfg.s)
    return sh.enter_rows(dm, cfg.s * r, lo * r)


# ---------------------------------------------------------------------------
# pair track sub-ops
# ---------------------------------------------------------------------------

def _gather_cf(sh, loc, c, R, full_rows):
    """Channel-first shards loc [c, R] -> [c, n*R] (the allgather of
    src/evoformer.py:380, 386-387 on channel-first operands)."""
    buf = sh.gather_rows(loc)                                # [n*c, R]
    out = torch.empty((c, full_rows), dtype=loc.dtype, device=loc.device)
    K.copy3d(buf, sh.n, c, R, out, s_bs=c * R, s_rs=R, d_bs=R, d_rs=full_rows)
    return out


def _own_rows_cf(x, c, R, full_rows, lo_row, dtype):
    """[c, full_rows] -> [c, R] rows lo_row.. of every channel (gather VJP)."""
    out = torch.empty((c, R), dtype=dtype, device=x.device)
    K.copy2d(x, c, R, out, s_rs=full_rows, d_rs=R, s_off=lo_row)
    return out


def trimul_fwd(st, sh, blk, name, z):
    """src/evoformer.py:359-397 on rows [lo, hi) of z: the partner projections
    (b outgoing; a and b incoming) are allgathered channel-first."""
    cfg, act = st.cfg, st.act
    P, pk = st.P, st.packs[blk][name]
    px = f"blk{blk}.{name}"
    dev = z.device
    r, c, cz = cfg.r, cfg.c_opm, cfg.c_z
    r2, ldp = r * r, 4 * c + cz
    lo, hi = sh.bounds(r)
    w = hi - lo
    R = w * r
    incoming = name.endswith("_in")
    zl = z[lo * r:hi * r]
    zh = torch.empty((R, cz), dtype=act, device=dev)
    mu, rs = torch.empty(R, dtype=F32, device=dev), torch.empty(R, dtype=F32, device=dev)
    K.layernorm(zl, R, cz, P[f"{px}.ln_g"], P[f"{px}.ln_b"], zh, mu, rs, cfg.eps)
    proj = torch.empty((R, ldp), dtype=act, device=dev)
    K.linear(zh, R, cz, pk["Wp"], ldp, ldp, proj, ldp, bias=pk["bp"], epi=EPI_SIGMOID_FROM,
             col0=2 * c)
    a_cf = torch.empty((c, R), dtype=act, device=dev)
    b_cf = torch.empty((c, R), dtype=act, device=dev)
    K.trimul_gate_fwd(proj, R, c, ldp, a_cf, b_cf)
    b_full = _gather_cf(sh, b_cf, c, R, r2)
    a_full = _gather_cf(sh, a_cf, c, R, r2) if incoming else None
    p_cf = torch.empty((c, R), dtype=F32, device=dev)
    if not incoming:
        # p[ch, i, j] = sum_k a[ch, i, k] b[ch, j, k]   (i local)
        K.gemm(Mat(a_cf, r, 1, bs1=R), Mat(b_full, r, 1, bs1=r2), Mat(p_cf, r, 1, bs1=R),
               w, r, r, B1=c)
    else:
        # p[ch, i, j] = sum_k a[ch, k, lo + i] b[ch, k, j]
        K.gemm(Mat(a_full, 1, r, bs1=r2, off=lo), Mat(b_full, 1, r, bs1=r2),
               Mat(p_cf, r, 1, bs1=R), w, r, r, B1=c)
    pn = torch.empty((R, c), dtype=act, device=dev)
    pmu, prs = torch.empty(R, dtype=F32, device=dev), torch.empty(R, dtype=F32, device=dev)
    K.layernorm(p_cf, R, c, P[f"{px}.p_ln_g"], P[f"{px}.p_ln_b"], pn, pmu, prs, cfg.eps,
                x_rs=1, x_cs=R)
    o = torch.empty((R, cz), dtype=act, device=dev)
    K.linear(pn, R, c, pk["Wo"], cz, cz, o, cz, bias=P[f"{px}.out_b"])
    d = torch.empty((R, cz), dtype=F32, device=dev)
    K.mul2d(proj, ldp, 4 * c, o, cz, d, R, cz)
    _chk(name + " proj", proj)
    _chk(name + " p", p_cf)
    _chk(name, d)
    ctx = dict(zl=zl, zh=zh, mu=mu, rs=rs, proj=proj, a_cf=a_cf, b_cf=b_cf, a_full=a_full,
               b_full=b_full, p_cf=p_cf, pn=pn, pmu=pmu, prs=prs, o=o, lo=lo, w=w)
    return _add(z, sh.gather_rows(d)), ctx


def trimul_bwd(st, sh, blk, name, ctx, dz_out):
    cfg, act = st.cfg, st.act
    P, pk = st.P, st.packs[blk][name]
    G = st.grads[blk].packed[name]
    px = f"blk{blk}.{name}"
    dev = dz_out.device
    r, c, cz = cfg.r, cfg.c_opm, cfg.c_z
    r2, ldp = r * r, 4 * c + cz
    lo, w = ctx["lo"], ctx["w"]
    R = w * r
    incoming = name.endswith("_in")
    proj = ctx["proj"]
    dl = dz_out[lo * r:lo * r + R].contiguous()
    do = torch.empty((R, cz), dtype=act, device=dev)
    dproj = torch.empty((R, ldp), dtype=act, device=dev)
    fused_cs = act != F32 and cz % 8 == 0 and ldp % 8 == 0
    if fused_cs:
        K.outgate_bwd(dl, R, cz, proj, ldp, 4 * c, ctx["o"], do, dproj, ldp, 4 * c,
                      do_colsum=G["bo"], dg_colsum=G["bp"][4 * c:])
    else:
        K.outgate_bwd(dl, R, cz, proj, ldp, 4 * c, ctx["o"], do, dproj, ldp, 4 * c)
        K.colsum(do, R, cz, G["bo"])
    K.linear_dw(ctx["pn"], R, c, do, cz, G["Wo"], cz)
    dpn = torch.empty((R, c), dtype=F32, device=dev)
    K.linear_dx(do, R, cz, pk["Wo"], cz, c, dpn)
    dp_cf = torch.empty((c, R), dtype=act, device=dev)
    K.layernorm_bwd(dpn, ctx["p_cf"], R, c, ctx["pmu"], ctx["prs"], P[f"{px}.p_ln_g"], dp_cf,
                    G["p_ln_g"], G["p_ln_b"], x_rs=1, x_cs=R, dx_rs=1, dx_cs=R)
    a_cf, b_full, a_full = ctx["a_cf"], ctx["b_full"], ctx["a_full"]
    if not incoming:
        # da[ch, i, k] = sum_j dp[ch, i, j] b[ch, j, k]
        da_cf = torch.empty((c, R), dtype=F32, device=dev)
        K.gemm(Mat(dp_cf, r, 1, bs1=R), Mat(b_full, 1, r, bs1=r2), Mat(da_cf, r, 1, bs1=R),
               w, r, r, B1=c)
        # db_full[ch, j, k] = sum_i dp[ch, i, j] a[ch, i, k]  (partial over i)
        db_full = torch.empty((c, r2), dtype=F32, device=dev)
        K.gemm(Mat(dp_cf, 1, r, bs1=R), Mat(a_cf, 1, r, bs1=R), Mat(db_full, r, 1, bs1=r2),
               r, r, w, B1=c)
        sh.allreduce(db_full, "bwd")                         # enter(b)
        db_cf = _own_rows_cf(db_full, c, R, r2, lo * r, F32)  # gather VJP
    else:
        # da_full[ch, k, lo + i] = sum_j b[ch, k, j] dp[ch, i, j]  (zero elsewhere)
        da_full = torch.empty((c, r2), dtype=F32, device=dev)
        K.zero(da_full)
        K.gemm(Mat(b_full, r, 1, bs1=r2), Mat(dp_cf, r, 1, bs1=R),
               Mat(da_full, r, 1, bs1=r2, off=lo), r, w, r, B1=c)
        # db_full[ch, k, j] = sum_i a[ch, k, lo + i] dp[ch, i, j]
        db_full = torch.empty((c, r2), dtype=F32, device=dev)
        K.gemm(Mat(a_full, r, 1, bs1=r2, off=lo), Mat(dp_cf, 1, r, bs1=R),
               Mat(db_full, r, 1, bs1=r2), r, r, w, B1=c)
        sh.allreduce(da_full, "bwd")                         # enter(a)
        sh.allreduce(db_full, "bwd")                         # enter(b)
        da_cf = _own_rows_cf(da_full, c, R, r2, lo * r, F32)
        db_cf = _own_rows_cf(db_full, c, R, r2, lo * r, F32)
    K.trimul_gate_bwd(proj, R, c, ldp, da_cf, db_cf, dproj, ldp,
                      colsum=G["bp"][:4 * c] if fused_cs else None)
    K.linear_dw(ctx["zh"], R, cz, dproj, ldp, G["Wp"], ldp)
    if not fused_cs:
        K.colsum(dproj, R, ldp, G["bp"])
    dzh = torch.empty((R, cz), dtype=F32, device=dev)
    K.linear_dx(dproj, R, ldp, pk["Wp"], ldp, cz, dzh)
    dzl = torch.empty((R, cz), dtype=F32, device=dev)
    K.layernorm_bwd(dzh, ctx["zl"], R, cz, ctx["mu"], ctx["rs"], P[f"{px}.ln_g"], dzl,
                    G["ln_g"], G["ln_b"])
    return _add(dz_out, sh.enter_rows(dzl, r2, lo * r))


def _bias_fns(sh, h, R, r2, lo_row):
    """(gather of the shard's pair-bias rows [h, R] -> [h, r2]; its VJP with
    the enter: allreduce the full dbias, keep the shard's rows)."""
    def gather(b_loc):
        buf = sh.gather_rows(b_loc.reshape(h, R))             # [n*h, R]
        full = torch.empty((h, r2), dtype=b_loc.dtype, device=b_loc.device)
        K.copy3d(buf, sh.n, h, R, full, s_bs=h * R, s_rs=R, d_bs=R, d_rs=r2)
        return full

    def dgather(db_full):
        sh.allreduce(db_full, "bwd")
        return _own_rows_cf(db_full, h, R, r2, lo_row, F32)
    return gather, dgather


def tri_attn_fwd(st, sh, blk, name, z):
    """src/evoformer.py:400-420: shard the attended-row axis (rows of z for
    the start node, rows of z^T -- columns of z -- for the end node, whose
    whole computation runs in the transposed frame like the reference's)."""
    cfg, act = st.cfg, st.act
    r, cz, h = cfg.r, cfg.c_z, cfg.h
    lo, hi = sh.bounds(r)
    w = hi - lo
    R = w * r
    ending = name == "tri_attn_end"
    x = _cols(z, r, r, cz, lo, w, transpose=True) if ending else z[lo * r:hi * r]
    gather, dgather = _bias_fns(sh, h, R, r * r, lo * r)
    d, ctx = E.attn_fwd("tri_attn_start", st.P, f"blk{blk}.{name}", st.packs[blk][name], x,
                        None, cfg, act, resid=False, geom=(w, r, r, 1, R), bias_fn=gather)
    _chk(name, d)
    if not ending:
        return _add(z, sh.gather_rows(d)), (ctx, lo, w, dgather)
    buf = sh.gather_rows(d)                                  # [n, w, r, cz] (z^T rows)
    full = torch.empty_like(z)
    _place_cols(buf, sh.n, r, w, cz, full, transpose=True)
    return _add(z, full), (ctx, lo, w, dgather)


def tri_attn_bwd(st, sh, blk, name, c, dz_out):
    cfg, act = st.cfg, st.act
    ctx, lo, w, dgather = c
    r, cz = cfg.r, cfg.c_z
    R = w * r
    ending = name == "tri_attn_end"
    G = st.grads[blk].packed[name]
    dl = (_cols(dz_out, r, r, cz, lo, w, transpose=True) if ending
          else dz_out[lo * r:lo * r + R].contiguous())
    dx, _ = E.attn_bwd("tri_attn_start", st.P, f"blk{blk}.{name}", st.packs[blk][name], G,
                       ctx, dl, cfg, act, dbias_fn=dgather)
    if ending:
        return _add(dz_out, _enter_cols(sh, dx, r, r, cz, lo, w, transpose=True))
    return _add(dz_out, sh.enter_rows(dx, r * r, lo * r))


# ---------------------------------------------------------------------------
# tracks (src/evoformer.py:427-443)
# ---------------------------------------------------------------------------

def msa_track_fwd(st, sh, blk, m, z):
    cfg = st.cfg
    m, c1 = row_attn_fwd(st, sh, blk, m, z)
    m, c2 = col_attn_fwd(st, sh, blk, m)
    m, c3 = transition_fwd(st, sh, blk, "msa_transition", m, cfg.s)
    return m, (c1, c2, c3)


def msa_track_bwd(st, sh, blk, ctx, dm):
    """Returns (dm_in, dz_row)."""
    c1, c2, c3 = ctx
    dm = transition_bwd(st, sh, blk, "msa_transition", c3, dm)
    dm = col_attn_bwd(st, sh, blk, c2, dm)
    return row_attn_bwd(st, sh, blk, c1, dm)


def pair_track_fwd(st, sh, blk, z):
    cfg = st.cfg
    cs = []
    for name in ("tri_mult_out", "tri_mult_in"):
        z, c = trimul_fwd(st, sh, blk, name, z)
        cs.append(c)
    for name in ("tri_attn_start", "tri_attn_end"):
        z, c = tri_attn_fwd(st, sh, blk, name, z)
        cs.append(c)
    z, c = transition_fwd(st, sh, blk, "pair_transition", z, cfg.r)
    cs.append(c)
    return z, cs


def pair_track_bwd(st, sh, blk, cs, dz):
    dz = transition_bwd(st, sh, blk, "pair_transition", cs[4], dz)
    for i, name in ((3, "tri_attn_end"), (2, "tri_attn_start")):
        dz = tri_attn_bwd(st, sh, blk, name, cs[i], dz)
    for i, name in ((1, "tri_mult_in"), (0, "tri_mult_out")):
        dz = trimul_bwd(st, sh, blk, name, cs[i], dz)
    return dz


def replicated_slices(st, blk):
    """(offset, numel) of the MSA bank entries DAP must not sum: the outer
    product mean's out_b, computed whole on every rank (mark_replicated,
    src/evoformer.py:355)."""
    bank = st.grads[blk].msa.flat
    bo = st.grads[blk].packed["opm"]["bo"]
    return [((bo.data_ptr() - bank.data_ptr()) // bo.element_size(), bo.numel())]
