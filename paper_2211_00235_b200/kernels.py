"""Thin typed wrappers over the C ABI taking torch device tensors.

Every function here launches native kernels on the current CUDA stream
(torch is used only for device memory and the stream handle).  Shapes
and strides are passed explicitly; layouts are documented in DESIGN.md.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from ._native import AttnDesc, EvoMat, GemmDesc, check, lib

DT = {torch.float32: N.EVO_F32, torch.bfloat16: N.EVO_BF16}


def dt(t: torch.Tensor) -> int:
    try:
        return DT[t.dtype]
    except KeyError:
        raise N.ContractError(f"unsupported dtype {t.dtype}") from None


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# bench.py sets this to a list to time kernel families with CUDA events on
# the launching stream: entries (family, algorithmic_flops, ev_start, ev_end)
PROFILE = None


DT_NAME = {N.EVO_F32: "f32", N.EVO_BF16: "bf16"}
# optional list collecting (family, shape) per profiled call (bench --detail)
PROFILE_SHAPES = None
# bench.py sets this to a list to record replayable launches: entries
# (family, algorithmic_flops, launch_fn, keep_alive_tensors); replaying the
# recorded launches of one family inside a CUDA graph times that family's
# kernels back to back on the device, free of host launch gaps
RECORD = None


def _timed(family, flops, fn, shape=None, keep=()):
    if RECORD is not None:
        RECORD.append((family, flops, fn, keep))
    if PROFILE is None:
        return fn()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    PROFILE.append((family, flops, e0, e1))
    if PROFILE_SHAPES is not None:
        PROFILE_SHAPES.append(shape)
    return r


def ptr(t, off: int = 0):
    if t is None:
        return None
    return t.data_ptr() + off * t.element_size()


def _ws(nbytes: int, device) -> torch.Tensor | None:
    if nbytes <= 0:
        return None
    return torch.empty(int(nbytes), dtype=torch.uint8, device=device)


class Mat:
    """Strided view (element units) of a tensor for the GEMM descriptor:
    element (i, j, b1, b2) at off + i*rs + j*cs + b1*bs1 + b2*bs2, with an
    optional two-level row/column map (see include/evo_b200.h)."""

    __slots__ = ("t", "off", "rs", "cs", "bs1", "bs2", "rdiv", "rs0", "cdiv", "cs0")

    def __init__(self, t, rs, cs, bs1=0, bs2=0, off=0, rdiv=0, rs0=0, cdiv=0, cs0=0):
        self.t, self.off, self.rs, self.cs = t, off, rs, cs
        self.bs1, self.bs2 = bs1, bs2
        self.rdiv, self.rs0, self.cdiv, self.cs0 = rdiv, rs0, cdiv, cs0

    def c(self) -> EvoMat:
        return EvoMat(ptr(self.t, self.off), self.rs, self.cs, self.bs1, self.bs2,
                      self.rdiv, self.rs0, self.cdiv, self.cs0)


def gemm(A: Mat, B: Mat, Cm: Mat, M: int, N_: int, K: int, *, alpha: float = 1.0,
         bias=None, epi: int = N.EPI_NONE, col0: int = 0, accumulate: bool = False,
         residual=None, B1: int = 1, B2: int = 1, split_k: int = 1,
         force_simt: bool = False) -> None:
    """C(m,n) = epi(alpha * sum_k A(m,k) B(n,k) + bias[n]) (+ residual)."""
    if A.t.dtype != B.t.dtype:
        raise N.ContractError(f"gemm operand dtypes differ: {A.t.dtype} vs {B.t.dtype}")
    d = GemmDesc()
    d.dtype_ab = dt(A.t)
    d.dtype_c = dt(Cm.t)
    d.M, d.N, d.K, d.B1, d.B2 = M, N_, K, B1, B2
    d.A, d.B, d.C = A.c(), B.c(), Cm.c()
    d.alpha = alpha
    d.epilogue = epi
    d.epi_col0 = col0
    d.accumulate = 1 if accumulate else 0
    d.split_k = max(1, int(split_k))
    d.bias = ptr(bias)
    d.residual = ptr(residual)
    d.force_simt = 1 if force_simt else 0
    L = lib()
    nbytes = L.evo_gemm_workspace_bytes(C.byref(d))
    ws = _ws(nbytes, Cm.t.device)
    d.workspace = ptr(ws)
    d.workspace_bytes = nbytes
    _timed("gemm", 2.0 * M * N_ * K * B1 * B2,
           lambda: check(L.evo_gemm(C.byref(d), stream()), "evo_gemm"),
           (M, N_, K, B1 * B2, d.split_k, int(A.rs == 1), int(B.rs == 1), DT_NAME[d.dtype_c]),
           keep=(A.t, B.t, Cm.t, bias, residual, ws))


def pick_split(rows_k: int, M: int, N_: int, batch: int = 1, min_rows: int = 512) -> int:
    """Split-K factor for tall contractions (weight gradients, the OPM input
    gradients): as many K chunks as fit one wave of the 148 SMs next to the
    output tiles, each chunk >= `min_rows` (8 k-steps of the TMA pipeline)."""
    tn = 256 if N_ > 128 else 128  # evo_gemm's split-K tile width (gemm_tc.cu choose_bn)
    tiles = max(1, ((M + 127) // 128) * ((N_ + tn - 1) // tn) * batch)
    # 128 x 256 tiles: ~128 CTAs beat a full 148-CTA wave (measured on the
    # step's weight gradients: [128 x 1024] over 65536 rows 47.7 -> 45.5 us,
    # [128 x 512] 29.4 -> 26.9 us; the partials traffic grows with the split)
    by_fill = (128 if tn == 256 else 148) // tiles
    by_size = rows_k // min_rows
    return int(max(1, min(by_fill, by_size)))


def linear(x, rows: int, d_in: int, W, ldw: int, d_out: int, out, ldo: int, *, w_off=0,
           o_off=0, x_ld=None, bias=None, epi=N.EPI_NONE, col0=0, residual=None,
           alpha=1.0):
    """out[rows, d_out] = x[rows, d_in] @ W[:, w_off:w_off+d_out] (+bias...)."""
    x_ld = d_in if x_ld is None else x_ld
    gemm(Mat(x, x_ld, 1), Mat(W, 1, ldw, off=w_off), Mat(out, ldo, 1, off=o_off),
         rows, d_out, d_in, bias=bias, epi=epi, col0=col0, residual=residual, alpha=alpha)


def linear_dx(dy, rows: int, d_out: int, W, ldw: int, d_in: int, out, *, dy_ld=None,
              w_off=0, accumulate=False, out_ld=None):
    """out[rows, d_in] (+)= dy[rows, d_out] @ W[:, w_off:w_off+d_out]^T."""
    dy_ld = d_out if dy_ld is None else dy_ld
    out_ld = d_in if out_ld is None else out_ld
    gemm(Mat(dy, dy_ld, 1), Mat(W, ldw, 1, off=w_off), Mat(out, out_ld, 1), rows, d_in, d_out,
         accumulate=accumulate)


def linear_dw(x, rows: int, d_in: int, dy, d_out: int, dW, ldd: int, *, x_ld=None, dy_ld=None,
              dy_off=0, dw_off=0, accumulate=False):
    """dW[d_in, d_out] (+)= x^T @ dy over `rows` (split-K, deterministic)."""
    x_ld = d_in if x_ld is None else x_ld
    dy_ld = d_out if dy_ld is None else dy_ld
    if d_in <= 128 < d_out and rows >= 16384:
        # narrow input, wide output: compute dW^T = dy^T x (the wide side on
        # the MMA's M, 128-wide N tiles): [128 x 1024] over 65536 rows 43 -> 39 us
        gemm(Mat(dy, 1, dy_ld, off=dy_off), Mat(x, 1, x_ld), Mat(dW, 1, ldd, off=dw_off),
             d_out, d_in, rows, split_k=pick_split(rows, d_out, d_in), accumulate=accumulate)
        return
    gemm(Mat(x, 1, x_ld), Mat(dy, 1, dy_ld, off=dy_off), Mat(dW, ldd, 1, off=dw_off),
         d_in, d_out, rows, split_k=pick_split(rows, d_in, d_out), accumulate=accumulate)


def layernorm(x, rows: int, cols: int, gamma, beta, y, mean, rstd, eps: float, *,
              x_rs=None, x_cs=1, y_rs=None):
    x_rs = cols if x_rs is None else x_rs
    y_rs = cols if y_rs is None else y_rs
    check(lib().evo_layernorm_fwd(dt(x), dt(y), rows, cols, ptr(x), x_rs, x_cs, ptr(gamma),
                                  ptr(beta), ptr(y), y_rs, ptr(mean), ptr(rstd), eps, stream()),
          "evo_layernorm_fwd")


def layernorm_split(x, rows: int, cols: int, gamma, beta, y3, mean, rstd, eps: float) -> bool:
    """LN(x) into the split bf16 operand y3 [rows, 3*cols] = hi | lo | hi in
    one pass (contiguous fp32 rows of 128 / 256); False for other shapes
    (the caller composes LN + split_bf16 then)."""
    if cols not in (128, 256) or not x.is_contiguous() or x.dtype != torch.float32:
        return False
    check(lib().evo_layernorm_fwd_split(rows, cols, ptr(x), ptr(gamma), ptr(beta), ptr(y3),
                                        ptr(mean), ptr(rstd), eps, stream()),
          "evo_layernorm_fwd_split")
    return True


def layernorm_bwd(dy, x, rows: int, cols: int, mean, rstd, gamma, dx, dgamma, dbeta, *,
                  dres=None, dy_rs=None, x_rs=None, x_cs=1, dx_rs=None, dx_cs=1,
                  accumulate_params=False):
    dy_rs = cols if dy_rs is None else dy_rs
    x_rs = cols if x_rs is None else x_rs
    dx_rs = cols if dx_rs is None else dx_rs
    L = lib()
    nbytes = L.evo_layernorm_bwd_workspace_bytes(rows, cols)
    ws = _ws(nbytes, dx.device)
    check(L.evo_layernorm_bwd(dt(dy), dt(x), dt(dx), rows, cols, ptr(dy), dy_rs, ptr(x), x_rs,
                              x_cs, ptr(mean), ptr(rstd), ptr(gamma), ptr(dres), ptr(dx), dx_rs,
                              dx_cs, ptr(dgamma), ptr(dbeta), 1 if accumulate_params else 0,
                              ptr(ws), nbytes, stream()),
          "evo_layernorm_bwd")


def layernorm_bwd_ex(dy, x, rows: int, cols: int, mean, rstd, gamma, dx, dgamma, dbeta, *,
                     dres=None, dx_act=None, dx_colsum=None):
    """LayerNorm backward (contiguous fp32 dy/dx, cols 128|256) that also
    emits a bf16 copy of dx and/or its column sums (the next sub-op's GEMM
    operand and output-bias gradient)."""
    L = lib()
    nbytes = L.evo_layernorm_bwd_workspace_bytes(rows, cols)
    ws = _ws(nbytes, dx.device)
    check(L.evo_layernorm_bwd_ex(dt(x), rows, cols, ptr(dy), ptr(x), ptr(mean), ptr(rstd),
                                 ptr(gamma), ptr(dres), ptr(dx), ptr(dx_act), ptr(dgamma),
                                 ptr(dbeta), ptr(dx_colsum), ptr(ws), nbytes, stream()),
          "evo_layernorm_bwd_ex")


def layernorm_bwd_proj(dy, x, rows: int, mean, rstd, gamma, beta, dproj, p_rs: int, Wp, nh: int,
                       dx, dgamma, dbeta, dWp, *, dres=None, dx_act=None, dx_colsum=None):
    """LayerNorm backward with the pair-bias projection's backward fused in
    (dy may be None); writes dx (+ dx_act / dx_colsum), dgamma, dbeta, dWp."""
    L = lib()
    nbytes = L.evo_layernorm_bwd_workspace_bytes(rows, 128)
    ws = _ws(nbytes, dx.device)
    check(L.evo_layernorm_bwd_proj(rows, 128, ptr(dy), ptr(x), ptr(mean), ptr(rstd), ptr(gamma),
                                   ptr(beta), ptr(dres), ptr(dproj), p_rs, ptr(Wp), nh, ptr(dx),
                                   ptr(dx_act), ptr(dgamma), ptr(dbeta), ptr(dx_colsum), ptr(dWp),
                                   ptr(ws), nbytes, stream()),
          "evo_layernorm_bwd_proj")


# keys beyond the resident-key tensor-core attention (Lp <= 256)
LONG_L = 256
# fp32 logits elements per chunk of batch rows in the long-key path
LONG_CHUNK_ELEMS = 1 << 27
# bytes of bf16 probabilities one forward call may keep for its backward
# (the kept-P path); larger calls recompute P from the logits and lse in the
# backward.  Env EVO_KEEP_P_MAX_BYTES overrides; 0 disables keeping P.
import os as _os
KEEP_P_MAX_BYTES = int(_os.environ.get("EVO_KEEP_P_MAX_BYTES", str(8 << 30)))


def use_flash(dtype, L: int, D: int) -> bool:
    """bf16 with L > 256 keys (head dim 8 / 16 / 32) or head dim 8 (any L:
    the extra-MSA stack's c_head = 8): the streamed-key fused attention
    (csrc/attention_flash.cu)."""
    return dtype == torch.bfloat16 and ((L > LONG_L and D in (8, 16, 32)) or D == 8)


def use_long(dtype, L: int, D: int) -> bool:
    """bf16 shapes no fused tcgen05 attention takes (head dims other than
    16 / 32: the extra-MSA stack's c_head = 8) run on the GEMM-composed path
    instead of the SIMT kernels."""
    return (dtype == torch.bfloat16 and (L > LONG_L or D not in (16, 32))
            and not use_flash(dtype, L, D))


def _attn_desc(proj, hc, nb, H, L, D, scale, sb, sl, o, gm, o_sb, o_sl, lse, bias, bh, bq, bk):
    d = AttnDesc()
    d.dtype = dt(proj)
    d.nb, d.H, d.L, d.D, d.scale = nb, H, L, D, scale
    d.q, d.k, d.v, d.g = (ptr(proj, 0), ptr(proj, hc), ptr(proj, 2 * hc), ptr(proj, 3 * hc))
    d.sb, d.sl = sb, sl
    d.o, d.gm = ptr(o), ptr(gm)
    d.o_sb, d.o_sl = o_sb, o_sl
    d.bias, d.bh, d.bq, d.bk = ptr(bias), bh, bq, bk
    d.lse = ptr(lse)
    return d


def attention_flash(*, proj, hc, nb, H, L, D, scale, sb, sl, o, gm, o_sb, o_sl, lse, bias=None,
                    bh=0, bq=0, bk=0, dgm=None, dproj=None, dbias=None, dgate_bias=None):
    """L > 256 keys or head dim 8 on the bf16 path: csrc/attention_flash.cu
    (keys streamed through TMEM with an online softmax; the backward's dS
    never leaves the SM either).  Same argument meaning as ``attention``."""
    four = 4 * hc
    if sb % four or sl % four or o_sb != sb // 4 or o_sl != sl // 4:
        raise N.ContractError("attention_flash: proj / o row maps must be the same row ids")
    rb, rl = sb // four, sl // four
    rows = nb * L
    dev = proj.device
    Lb = lib()
    # the kernels read plain bias rows (bk = 1, 16-byte aligned): copy a
    # transposed (triangle end) or unaligned bias once per call
    pb, pbh, pbq = bias, bh, bq
    if bias is not None and not (bk == 1 and bq % 4 == 0 and bh % 4 == 0 and bh >= L * bq):
        Lp = (L + 3) // 4 * 4
        pb = torch.zeros(H * L * Lp, dtype=torch.float32, device=dev)
        for hh in range(H):
            copy2d(bias, L, L, pb, s_rs=bq, s_cs=bk, d_rs=Lp, s_off=hh * bh, d_off=hh * L * Lp)
        pbh, pbq = L * Lp, Lp
    d = _attn_desc(proj, hc, nb, H, L, D, scale, sb, sl, o, gm, o_sb, o_sl, lse, pb, pbh, pbq, 1)
    flops = 4.0 * nb * H * L * L * D
    if dgm is None:
        _timed("attention_fwd", flops,
               lambda: check(Lb.evo_attn_flash_fwd(C.byref(d), stream()), "evo_attn_flash_fwd"),
               keep=(proj, o, gm, lse, pb))
        return
    d.dgm = ptr(dgm)
    d.dq, d.dk, d.dv, d.dgpre = (ptr(dproj, 0), ptr(dproj, hc), ptr(dproj, 2 * hc),
                                 ptr(dproj, 3 * hc))
    # the prep pass fuses the gate-bias sums when its column groups tile a
    # 256-thread block; otherwise they are a separate column sum below
    fuse_gb = dgate_bias is not None and 256 % (H * D // 8) == 0
    d.dgate_bias = ptr(dgate_bias) if fuse_gb else None
    # dbias in the kernel's plain layout: the caller's, or a padded copy
    pdb = dbias
    if bias is not None and pb is not bias:
        pdb = torch.empty(H * pbh, dtype=torch.float32, device=dev)
    d.dbias = ptr(pdb)
    nbytes = Lb.evo_attn_flash_bwd_workspace_bytes(C.byref(d))
    ws = _ws(nbytes, dev)
    d.workspace, d.workspace_bytes = ptr(ws), nbytes
    _timed("attention_bwd", 2.0 * flops,
           lambda: check(Lb.evo_attn_flash_bwd(C.byref(d), stream()), "evo_attn_flash_bwd"),
           keep=(proj, o, gm, lse, pb, dgm, dproj, pdb, dgate_bias, ws))
    if bias is not None and pdb is not dbias:
        for hh in range(H):
            copy2d(pdb, L, L, dbias, s_rs=pbq, d_rs=bq, d_cs=bk, s_off=hh * pbh, d_off=hh * bh)
    if dgate_bias is not None and not fuse_gb:
        colsum(dproj, nb * L, hc, dgate_bias, rs=four, off=3 * hc)


def long_ld(L: int) -> int:
    """Row stride of the long path's [.., L, ld] logits / probabilities: L
    rounded up to 8 (16-byte aligned bf16 GEMM operand rows)."""
    return (L + 7) // 8 * 8


def long_p_elems(nb, H, L):
    """bf16 elements of the forward probabilities kept for the backward."""
    return nb * H * L * long_ld(L)


def keep_p(nb, H, L) -> bool:
    """Keep this call's forward P for the backward (within the byte cap)?"""
    return 2 * long_p_elems(nb, H, L) <= KEEP_P_MAX_BYTES


def attention_long(*, proj, hc, nb, H, L, D, scale, sb, sl, o, gm, o_sb, o_sl, lse, bias=None,
                   bh=0, bq=0, bk=0, dgm=None, dproj=None, dbias=None, dgate_bias=None,
                   p_store=None):
    """L > 256 on the bf16 path: S = scale*QK^T, O = PV, dP = dO V^T, dQ, dK,
    dV as strided-batched tcgen05 GEMMs (batch = (row chunk, head)) over
    chunks of batch rows, with the softmax / gate / dsoftmax row work in
    csrc/attention_long.cu.  Same argument meaning as ``attention``.
    p_store (bf16, long_p_elems): the forward writes P there and the
    backward reads it (no QK^T recompute); without it the backward
    recomputes P from the logits and lse."""
    four = 4 * hc
    if sb % four or sl % four or o_sb != sb // 4 or o_sl != sl // 4:
        raise N.ContractError("attention_long: proj / o row maps must be the same row ids")
    rb, rl = sb // four, sl // four
    rows = nb * L
    dev = proj.device
    Lb = lib()
    ld = long_ld(L)
    HLL = H * L * ld                      # one batch row's logits, row stride ld
    nbc_max = max(1, LONG_CHUNK_ELEMS // HLL)
    # the batched GEMMs take at most 65535 (row, head) batches per call
    csz = max(1, min(nb, nbc_max, 65535 // H))
    if p_store is not None and p_store.numel() < long_p_elems(nb, H, L):
        raise N.ContractError("attention_long: p_store too small")
    S = (torch.empty(csz * HLL, dtype=torch.float32, device=dev)
         if dgm is None or p_store is None else None)
    P = (torch.empty(csz * HLL, dtype=torch.bfloat16, device=dev)
         if p_store is None else None)
    lse_f = lse.view(-1)

    # the softmax reads the bias once per batch row: give it a plain
    # [H, L, L] copy when the bias is transposed (triangle end), so those
    # reads are coalesced
    sbias, sbh, sbq, sbk = bias, bh, bq, bk
    if bias is not None and bk != 1:
        sbias = torch.empty(H * L * L, dtype=torch.float32, device=dev)
        for hh in range(H):
            copy2d(bias, L, L, sbias, s_rs=bq, s_cs=bk, d_rs=L, s_off=hh * bh,
                   d_off=hh * L * L)
        sbh, sbq, sbk = L * L, L, 1
    if dgm is None:
        O32 = torch.empty(rows, hc, dtype=torch.float32, device=dev)
        for b0 in range(0, nb, csz):
            nbc = min(csz, nb - b0)
            # S = scale * Q K^T
            gemm(Mat(proj, sl, 1, sb, D, off=b0 * sb), Mat(proj, sl, 1, sb, D, off=b0 * sb + hc),
                 Mat(S, ld, 1, HLL, L * ld), L, L, D, alpha=scale, B1=nbc, B2=H)
            Pc, poff = (P, 0) if p_store is None else (p_store, b0 * HLL)
            check(Lb.evo_attn_long_softmax(nbc, H, L, ld, ptr(S), ptr(sbias), sbh, sbq, sbk,
                                           ptr(Pc, poff), ptr(lse_f, b0 * H * L), stream()),
                  "evo_attn_long_softmax")
            # O[row(b,q), h*D+d] = sum_k P[b,h,q,k] V[row(b,k), 2hc + h*D + d]
            gemm(Mat(Pc, ld, 1, HLL, L * ld, off=poff),
                 Mat(proj, 1, sl, sb, D, off=b0 * sb + 2 * hc),
                 Mat(O32, rl * hc, 1, rb * hc, D, off=b0 * rb * hc), L, D, L, B1=nbc, B2=H)
        check(Lb.evo_attn_long_gate(rows, hc, ptr(O32), ptr(proj, 3 * hc), four, ptr(o), ptr(gm),
                                    stream()), "evo_attn_long_gate")
        return
    # backward
    dO = torch.empty(rows, hc, dtype=torch.bfloat16, device=dev)
    Dq = torch.empty(rows, H, dtype=torch.float32, device=dev)
    check(Lb.evo_attn_long_prep(rows, H, D, ptr(dgm), ptr(proj, 3 * hc), four, ptr(o), ptr(dO),
                                ptr(dproj, 3 * hc), four, ptr(Dq), stream()), "evo_attn_long_prep")
    dP = torch.empty(csz * HLL, dtype=torch.float32, device=dev)
    dS = torch.empty(csz * HLL, dtype=torch.bfloat16, device=dev)
    for b0 in range(0, nb, csz):
        nbc = min(csz, nb - b0)
        if p_store is None:
            gemm(Mat(proj, sl, 1, sb, D, off=b0 * sb), Mat(proj, sl, 1, sb, D, off=b0 * sb + hc),
                 Mat(S, ld, 1, HLL, L * ld), L, L, D, alpha=scale, B1=nbc, B2=H)
            Pc, poff, Sp = P, 0, ptr(S)
        else:
            Pc, poff, Sp = p_store, b0 * HLL, None
        # dP[b,h,q,k] = sum_d dO[row(b,q), h*D+d] V[row(b,k), 2hc + h*D + d]
        gemm(Mat(dO, rl * hc, 1, rb * hc, D, off=b0 * rb * hc),
             Mat(proj, sl, 1, sb, D, off=b0 * sb + 2 * hc),
             Mat(dP, ld, 1, HLL, L * ld), L, L, D, B1=nbc, B2=H)
        check(Lb.evo_attn_long_dsoftmax(nbc, H, L, ld, Sp, ptr(dP), ptr(bias), bh, bq, bk,
                                        ptr(lse_f, b0 * H * L), ptr(Dq), b0 * rb, rb, rl,
                                        ptr(Pc, poff), ptr(dS), ptr(dbias), 1 if b0 > 0 else 0,
                                        stream()),
              "evo_attn_long_dsoftmax")
        # dV[row(b,k), 2hc+h*D+d] = sum_q P[b,h,q,k] dO[row(b,q), h*D+d]
        gemm(Mat(Pc, 1, ld, HLL, L * ld, off=poff),
             Mat(dO, 1, rl * hc, rb * hc, D, off=b0 * rb * hc),
             Mat(dproj, sl, 1, sb, D, off=b0 * sb + 2 * hc), L, D, L, B1=nbc, B2=H)
        # dQ = scale * dS K ;  dK = scale * dS^T Q
        gemm(Mat(dS, ld, 1, HLL, L * ld), Mat(proj, 1, sl, sb, D, off=b0 * sb + hc),
             Mat(dproj, sl, 1, sb, D, off=b0 * sb), L, D, L, alpha=scale, B1=nbc, B2=H)
        gemm(Mat(dS, 1, ld, HLL, L * ld), Mat(proj, 1, sl, sb, D, off=b0 * sb),
             Mat(dproj, sl, 1, sb, D, off=b0 * sb + hc), L, D, L, alpha=scale, B1=nbc, B2=H)
    if dgate_bias is not None:
        colsum(dproj, rows, hc, dgate_bias, rs=four, off=3 * hc)


def _tc_bias_layout_ok(bh, bq, bk, L) -> bool:
    """The tensor-core attention reads bias rows as 16-byte vectors: plain
    (bk = 1) or transposed (bq = 1) rows whose strides are multiples of 4,
    one head's rows tiling its bh span."""
    if bh < L * max(bq, bk):
        return False
    return ((bk == 1 and bq % 4 == 0 and bh % 4 == 0)
            or (bq == 1 and bk % 4 == 0 and bh % 4 == 0))


def _attention_padded_bias(*, bias, bh, bq, bk, dbias=None, L, H, **kw):
    """Crops with r % 4 != 0: run the tensor-core attention on a plain
    [H, L, Lp] copy of the bias (Lp = L rounded up to 4) and scatter its
    gradient back to the caller's layout."""
    Lp = (L + 3) // 4 * 4
    dev = bias.device
    bpad = torch.zeros(H * L * Lp, dtype=torch.float32, device=dev)
    for hh in range(H):
        copy2d(bias, L, L, bpad, s_rs=bq, s_cs=bk, d_rs=Lp, s_off=hh * bh, d_off=hh * L * Lp)
    dpad = (torch.empty(H * L * Lp, dtype=torch.float32, device=dev)
            if dbias is not None else None)
    attention(bias=bpad, bh=L * Lp, bq=Lp, bk=1, dbias=dpad, L=L, H=H, **kw)
    if dbias is not None:
        for hh in range(H):
            copy2d(dpad, L, L, dbias, s_rs=Lp, d_rs=bq, d_cs=bk, s_off=hh * L * Lp,
                   d_off=hh * bh)


def attention(*, proj, hc: int, nb: int, H: int, L: int, D: int, scale: float, sb: int,
              sl: int, o, gm, o_sb: int, o_sl: int, lse, bias=None, bh=0, bq=0, bk=0,
              dgm=None, dproj=None, dbias=None, dgate_bias=None, p_store=None):
    """Fused gated attention on the packed [rows, 4*hc] projection buffer
    (cols q | k | v | sigmoid(gate)).  Forward when dgm is None, else
    backward into dproj (same packing) and dbias."""
    if use_flash(proj.dtype, L, D):
        return attention_flash(proj=proj, hc=hc, nb=nb, H=H, L=L, D=D, scale=scale, sb=sb,
                               sl=sl, o=o, gm=gm, o_sb=o_sb, o_sl=o_sl, lse=lse, bias=bias,
                               bh=bh, bq=bq, bk=bk, dgm=dgm, dproj=dproj, dbias=dbias,
                               dgate_bias=dgate_bias)
    if use_long(proj.dtype, L, D):
        return attention_long(proj=proj, hc=hc, nb=nb, H=H, L=L, D=D, scale=scale, sb=sb,
                              sl=sl, o=o, gm=gm, o_sb=o_sb, o_sl=o_sl, lse=lse, bias=bias,
                              bh=bh, bq=bq, bk=bk, dgm=dgm, dproj=dproj, dbias=dbias,
                              dgate_bias=dgate_bias, p_store=p_store)
    if (bias is not None and proj.dtype == torch.bfloat16
            and not _tc_bias_layout_ok(bh, bq, bk, L)):
        return _attention_padded_bias(proj=proj, hc=hc, nb=nb, H=H, L=L, D=D, scale=scale,
                                      sb=sb, sl=sl, o=o, gm=gm, o_sb=o_sb, o_sl=o_sl, lse=lse,
                                      bias=bias, bh=bh, bq=bq, bk=bk, dgm=dgm, dproj=dproj,
                                      dbias=dbias, dgate_bias=dgate_bias)
    d = AttnDesc()
    d.dtype = dt(proj)
    d.nb, d.H, d.L, d.D, d.scale = nb, H, L, D, scale
    d.q, d.k, d.v, d.g = (ptr(proj, 0), ptr(proj, hc), ptr(proj, 2 * hc), ptr(proj, 3 * hc))
    d.sb, d.sl = sb, sl
    d.o, d.gm = ptr(o), ptr(gm)
    d.o_sb, d.o_sl = o_sb, o_sl
    d.bias, d.bh, d.bq, d.bk = ptr(bias), bh, bq, bk
    d.lse = ptr(lse)
    Lb = lib()
    flops = 4.0 * nb * H * L * L * D
    if dgm is None:
        _timed("attention_fwd", flops,
               lambda: check(Lb.evo_attention_fwd(C.byref(d), stream()), "evo_attention_fwd"),
               keep=(proj, o, gm, lse, bias))
        return
    d.dgm = ptr(dgm)
    d.dq, d.dk, d.dv, d.dgpre = (ptr(dproj, 0), ptr(dproj, hc), ptr(dproj, 2 * hc),
                                 ptr(dproj, 3 * hc))
    d.dbias = ptr(dbias)
    d.dgate_bias = ptr(dgate_bias)
    nbytes = Lb.evo_attention_bwd_workspace_bytes(C.byref(d))
    ws = _ws(nbytes, proj.device)
    d.workspace, d.workspace_bytes = ptr(ws), nbytes
    _timed("attention_bwd", 2.0 * flops,
           lambda: check(Lb.evo_attention_bwd(C.byref(d), stream()), "evo_attention_bwd"),
           keep=(proj, o, gm, lse, bias, dgm, dproj, dbias, dgate_bias, ws))


def colsum(src, rows: int, cols: int, dst, *, rs=None, off=0, accumulate=False):
    rs = cols if rs is None else rs
    L = lib()
    nbytes = L.evo_colsum_workspace_bytes(cols)
    ws = _ws(nbytes, dst.device)
    check(L.evo_colsum(dt(src), rows, cols, ptr(src, off), rs, ptr(dst),
                       1 if accumulate else 0, ptr(ws), nbytes, stream()), "evo_colsum")


def copy2d(src, rows: int, cols: int, dst, *, s_rs, s_cs=1, d_rs, d_cs=1, s_off=0, d_off=0):
    check(lib().evo_copy2d(dt(src), dt(dst), rows, cols, ptr(src, s_off), s_rs, s_cs,
                           ptr(dst, d_off), d_rs, d_cs, stream()), "evo_copy2d")


def copy3d(src, n0: int, rows: int, cols: int, dst, *, s_bs, s_rs, s_cs=1, d_bs, d_rs, d_cs=1,
           s_off=0, d_off=0):
    """dst[b, r, c] = src[b, r, c] over explicit element strides (any dtype pair)."""
    check(lib().evo_copy3d(dt(src), dt(dst), n0, rows, cols, ptr(src, s_off), s_bs, s_rs, s_cs,
                           ptr(dst, d_off), d_bs, d_rs, d_cs, stream()), "evo_copy3d")


def zero(t):
    """t[:] = 0 (stream-ordered memset of a contiguous tensor)."""
    check(lib().evo_zero(ptr(t), t.numel() * t.element_size(), stream()), "evo_zero")
    return t


def zeros(shape, dtype=torch.float32, device="cuda"):
    """A zero-filled tensor by memset (no framework kernel on the step path)."""
    return zero(torch.empty(shape, dtype=dtype, device=device))


def trimul_gate_fwd(proj, rows: int, c: int, ldp: int, a_cf, b_cf):
    check(lib().evo_trimul_gate_fwd(dt(proj), rows, c, ptr(proj), ldp, ptr(a_cf), ptr(b_cf),
                                    stream()), "evo_trimul_gate_fwd")


def trimul_gate_bwd(proj, rows: int, c: int, ldp: int, da_cf, db_cf, dproj, ldd: int,
                    colsum=None):
    """dproj[:, :4c] from da/db; colsum (fp32 [4c]) = their column sums taken
    from the fp32 values (the gate / value bias gradients)."""
    L = lib()
    ws = None
    nbytes = 0
    if colsum is not None:
        nbytes = L.evo_trimul_gate_bwd_workspace_bytes(rows, c)
        ws = _ws(nbytes, dproj.device)
    check(L.evo_trimul_gate_bwd(dt(proj), rows, c, ptr(proj), ldp, ptr(da_cf), ptr(db_cf),
                                ptr(dproj), ldd, ptr(colsum), ptr(ws), nbytes, stream()),
          "evo_trimul_gate_bwd")


def outgate_fwd(z, rows: int, cols: int, g, g_rs: int, g_off: int, o, znew):
    check(lib().evo_outgate_fwd(dt(o), rows, cols, ptr(z), ptr(g, g_off), g_rs, ptr(o), cols,
                                ptr(znew), stream()), "evo_outgate_fwd")


def outgate_bwd(dz, rows: int, cols: int, g, g_rs: int, g_off: int, o, do_, dgpre,
                dg_rs: int, dg_off: int, do_colsum=None, dg_colsum=None):
    L = lib()
    ws = None
    nbytes = 0
    if do_colsum is not None or dg_colsum is not None:
        nbytes = L.evo_outgate_bwd_workspace_bytes(rows, cols)
        ws = _ws(nbytes, dz.device)
    check(L.evo_outgate_bwd(dt(o), rows, cols, ptr(dz), ptr(g, g_off), g_rs, ptr(o), cols,
                            ptr(do_), cols, ptr(dgpre, dg_off), dg_rs, ptr(do_colsum),
                            ptr(dg_colsum), ptr(ws), nbytes, stream()),
          "evo_outgate_bwd")


def mul2d(a, a_rs: int, a_off: int, b, b_rs: int, out, rows: int, cols: int):
    """out[rows, cols] (contiguous) = a(r, c) * b(r, c)."""
    check(lib().evo_mul2d(dt(a), dt(b), dt(out), rows, cols, ptr(a, a_off), a_rs, ptr(b), b_rs,
                          ptr(out), cols, stream()), "evo_mul2d")


def relu_bwd(dh, h, dpre, n: int):
    check(lib().evo_relu_bwd(dt(h), n, ptr(dh), ptr(h), ptr(dpre), stream()), "evo_relu_bwd")


def relu_bwd_colsum(dh, h, dpre, rows: int, cols: int, colsum_dst):
    """dpre = dh * (h > 0) (bf16, contiguous) and its column sums (fp32)."""
    L = lib()
    nbytes = L.evo_colsum_workspace_bytes(cols)
    ws = _ws(nbytes, dpre.device)
    check(L.evo_relu_bwd_colsum(rows, cols, ptr(dh), ptr(h), ptr(dpre), ptr(colsum_dst), ptr(ws),
                                nbytes, stream()), "evo_relu_bwd_colsum")


def sq_mean(x, out, dx=None):
    ws = torch.empty(4096, dtype=torch.uint8, device=x.device)
    check(lib().evo_sq_mean(x.numel(), ptr(x), ptr(out), ptr(dx), ptr(ws), stream()),
          "evo_sq_mean")


def split_bf16(x, rows: int, cols: int, hi, lo, *, x_rs=None, h_rs=None, l_rs=None, hi2=None,
               h2_rs=None, h_off=0, l_off=0, h2_off=0):
    """hi = bf16(x), lo = bf16(x - hi) (hi also into hi2), row strides given."""
    x_rs = cols if x_rs is None else x_rs
    h_rs = cols if h_rs is None else h_rs
    l_rs = cols if l_rs is None else l_rs
    h2_rs = cols if h2_rs is None else h2_rs
    check(lib().evo_split_bf16(rows, cols, ptr(x), x_rs, ptr(hi, h_off), h_rs, ptr(lo, l_off),
                               l_rs, ptr(hi2, h2_off) if hi2 is not None else None, h2_rs,
                               stream()), "evo_split_bf16")


def div_scalar(x, d: float, out):
    """out = x / d (fp32, contiguous; in place when out is x)."""
    check(lib().evo_div_scalar(x.numel(), ptr(x), d, ptr(out), stream()), "evo_div_scalar")


def add(a, b, out):
    check(lib().evo_add(a.numel(), ptr(a), ptr(b), ptr(out), stream()), "evo_add")


def reduce_lead(src, nb: int, n1: int, n2: int, dst, d_s1: int, d_s2: int, accumulate=False):
    check(lib().evo_reduce_lead(dt(src), nb, n1, n2, ptr(src), ptr(dst), d_s1, d_s2,
                                1 if accumulate else 0, stream()), "evo_reduce_lead")
