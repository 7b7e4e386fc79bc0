/*
 * evo_b200.h -- C ABI of the B200-native Parallel Evoformer kernels.
 *
 * Plain C: raw device pointers, element strides, sizes, a cudaStream_t
 * passed as void*.  No torch types.  Every entry point returns 0 on
 * success or a negative EVO_E* status; evo_last_error() returns the
 * message of the last failure on the calling thread.  The host package
 * (paper_2211_00235_b200/_native.py) maps the statuses onto the
 * reference's error taxonomy (src/errors.py:9-38): EVO_EDIM ->
 * DimensionError, EVO_EARG -> ContractError, EVO_ECUDA/EVO_EUNSUP ->
 * NumericsError/RuntimeError.
 *
 * Citations: src/X.py:N = /root/reference/pkg/src/branchpar/X.py line N.
 * The reference has no FFI; each entry point replaces a numpy op of its
 * tape (src/tensor.py) or a fused group of them inside a sub-op
 * (src/evoformer.py), as noted per function.
 *
 * Kernels never allocate device memory: outputs and workspaces are
 * caller-owned.  All launches are stream-ordered on `stream`.
 */
#ifndef EVO_B200_H
#define EVO_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EVO_API __attribute__((visibility("default")))
#else
#define EVO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* element types */
#define EVO_F32 0
#define EVO_BF16 1

/* status codes */
#define EVO_OK 0
#define EVO_EARG -1    /* bad argument / null pointer / bad enum        */
#define EVO_EDIM -2    /* inconsistent or unsupported shape             */
#define EVO_ECUDA -3   /* CUDA launch or runtime error                  */
#define EVO_EUNSUP -4  /* valid request this build does not implement   */

/* GEMM epilogues (applied per output element, in this order:
 *   v = alpha * sum_k A(m,k) B(n,k)
 *   v += bias[n]                         (if bias)
 *   v = relu(v)                          (EVO_EPI_RELU)
 *   v = sigmoid(v) if n >= epi_col0      (EVO_EPI_SIGMOID_FROM)
 *   v += R(m,n)                          (if residual; F32, C's index map)
 *   C(m,n) = v  (or C(m,n) += v when accumulate)                      */
#define EVO_EPI_NONE 0
#define EVO_EPI_RELU 1
#define EVO_EPI_SIGMOID_FROM 2

/* A strided matrix view.  Element (i, j, b1, b2) lives at
 *   ptr + i*rs + j*cs + b1*bs1 + b2*bs2                (elements)
 * For GEMM outputs a two-level row map is allowed: if rdiv > 0 the row
 * term is (i / rdiv)*rs + (i % rdiv)*rs0, likewise cdiv/cs0 for columns
 * (used for the outer-product-mean [i,j,p,q] layout and the transposed
 * triangle-end bias).                                                  */
typedef struct evo_mat {
  void *ptr;
  int64_t rs, cs, bs1, bs2;
  int64_t rdiv, rs0, cdiv, cs0;
} evo_mat;

/* Strided batched GEMM   C(m,n) = epi( alpha * sum_k A(m,k) * B(n,k) ).
 * Replaces T.linear / T.matmul forward and both backward matmuls
 * (src/tensor.py:287-345): x@W is A=x (K contiguous), B(n,k)=W[k,n].
 * Dispatches to the tcgen05/TMA tensor-core kernel when dtype_ab is
 * EVO_BF16 and each operand has a unit stride along M/N or K with
 * 16-byte aligned rows, else to the SIMT FFMA kernel (the fp32 parity
 * path).  split_k > 1 partitions K and sums the fp32 partials in fixed
 * order (deterministic); it needs `workspace` of
 * evo_gemm_workspace_bytes() bytes.                                    */
typedef struct evo_gemm_desc {
  int32_t dtype_ab;      /* EVO_F32 | EVO_BF16 (A and B)                 */
  int32_t dtype_c;       /* EVO_F32 | EVO_BF16                           */
  int64_t M, N, K, B1, B2;
  evo_mat A, B, C;
  float alpha;
  int32_t epilogue;      /* EVO_EPI_*                                    */
  int32_t epi_col0;      /* first column for EVO_EPI_SIGMOID_FROM        */
  int32_t accumulate;    /* C += result (EVO_F32 C only)                 */
  int32_t split_k;       /* >= 1                                         */
  const float *bias;     /* [N] or NULL; shared over batches             */
  const float *residual; /* F32, indexed with C's map, or NULL           */
  int32_t force_simt;    /* 1: never use the tensor-core kernel          */
  void *workspace;
  size_t workspace_bytes;
} evo_gemm_desc;

EVO_API int evo_gemm(const evo_gemm_desc *d, void *stream);
EVO_API size_t evo_gemm_workspace_bytes(const evo_gemm_desc *d);

/* Row LayerNorm over the last axis (T.layer_norm forward,
 * src/tensor.py:366-381; eps from EvoConfig src/evoformer.py:56).
 * x: rows x cols, element (row, c) at x[row*x_rs + c*x_cs]
 * (x_cs = rows gives a channel-first input).  y[row*y_rs + c] =
 * xhat*gamma + beta.  mean/rstd: fp32 [rows] saved for the backward.  */
EVO_API int evo_layernorm_fwd(int dtype_x, int dtype_y, int64_t rows, int cols,
                      const void *x, int64_t x_rs, int64_t x_cs,
                      const float *gamma, const float *beta, void *y,
                      int64_t y_rs, float *mean, float *rstd, float eps,
                      void *stream);

/* LayerNorm backward (src/tensor.py:383-390):
 *   dx = rstd*(dxh - mean(dxh) - xhat*mean(dxh*xhat)),  dxh = dy*gamma
 *   dx_out(row,c) = (dres ? dres(row,c) : 0) + dx      (dx dtype_dx)
 *   dgamma = sum_rows dy*xhat, dbeta = sum_rows dy (fp32, deterministic,
 *   ADDED to existing contents when accumulate_params).
 * dy[row*dy_rs + c]; x as in the forward; dx at dx[row*dx_rs + c*dx_cs];
 * dres (fp32) shares dx's index map.  workspace: evo_layernorm_bwd_
 * workspace_bytes(rows, cols) bytes.                                   */
EVO_API int evo_layernorm_bwd(int dtype_dy, int dtype_x, int dtype_dx, int64_t rows,
                      int cols, const void *dy, int64_t dy_rs, const void *x,
                      int64_t x_rs, int64_t x_cs, const float *mean,
                      const float *rstd, const float *gamma, const float *dres,
                      void *dx, int64_t dx_rs, int64_t dx_cs, float *dgamma,
                      float *dbeta, int accumulate_params, void *workspace,
                      size_t workspace_bytes, void *stream);
EVO_API size_t evo_layernorm_bwd_workspace_bytes(int64_t rows, int cols);

/* LayerNorm backward of a contiguous [rows, cols] fp32 gradient (cols 128
 * or 256) with two by-products of its fp32 output dx fused in, for the
 * next sub-op's backward (src/evoformer.py:456-461 chains the sub-ops):
 *   dx_act    (bf16, may be NULL): a copy of dx, that sub-op's GEMM operand
 *   dx_colsum (fp32, may be NULL): sum over rows of dx, that sub-op's
 *             output-bias gradient (src/tensor.py:343), written
 * dgamma / dbeta are written (not accumulated); x is fp32 or bf16
 * (dtype_x); dres as in evo_layernorm_bwd.  Same workspace.            */
EVO_API int evo_layernorm_bwd_ex(int dtype_x, int64_t rows, int cols, const float *dy,
                                 const void *x, const float *mean, const float *rstd,
                                 const float *gamma, const float *dres, float *dx,
                                 void *dx_act, float *dgamma, float *dbeta,
                                 float *dx_colsum, void *workspace, size_t workspace_bytes,
                                 void *stream);

/* LayerNorm backward of a contiguous fp32 [rows, 128] input (c_z rows)
 * fused with the backward of the attention pair-bias projection that
 * consumed LN(x) (src/evoformer.py:279, bias = LN(z) Wb; Wp bf16 [128][nh],
 * nh <= 8):
 *   dy_tot = dy (fp32 [rows,128], may be NULL = 0) + sum_hh dproj[hh*p_rs+row] Wp[c*nh+hh]
 *   dx = LN_bwd(dy_tot) + dres;  dx_act / dx_colsum as evo_layernorm_bwd_ex;
 *   dgamma, dbeta, and dWp[c*nh + hh] = sum_rows bf16(LN(x))[row,c] * dproj[hh,row]
 *   (all written).  dproj fp32.  Workspace as evo_layernorm_bwd.        */
EVO_API int evo_layernorm_bwd_proj(int64_t rows, int cols, const float *dy, const float *x,
                                   const float *mean, const float *rstd, const float *gamma,
                                   const float *beta, const float *dres, const float *dproj,
                                   int64_t p_rs, const void *Wp, int nh, float *dx,
                                   void *dx_act, float *dgamma, float *dbeta,
                                   float *dx_colsum, float *dWp, void *workspace,
                                   size_t workspace_bytes, void *stream);

/* Fused gated attention forward over the middle axis
 * (_gated_attention core, src/evoformer.py:274-286):
 *   O[b,l,h,:] = softmax_k( scale*q.k + bias[h,l,k] ) v
 *   GM = G * O   (G = sigmoid gate, already activated)
 * q/k/v/g/o/gm element (b, l, h, d) at ptr + b*sb + l*sl + h*D + d.
 * lse fp32 [nb, H, L] saved for the backward.  L <= 256 keys resident;
 * bias(h,q,k) fp32 at bias[h*bh + q*bq + k*bk] (or NULL).                           */
typedef struct evo_attn_desc {
  int32_t dtype;           /* activations: EVO_F32 | EVO_BF16          */
  int64_t nb;              /* batch rows (B)                           */
  int32_t H, L, D;
  float scale;
  const void *q, *k, *v, *g;
  int64_t sb, sl;          /* shared strides of q/k/v/g (proj buffer)  */
  void *o, *gm;
  int64_t o_sb, o_sl;      /* strides of o and gm                      */
  const float *bias;
  int64_t bh, bq, bk;
  float *lse;
  /* backward only */
  const void *dgm;         /* grad of gm (o's strides)                 */
  void *dq, *dk, *dv, *dgpre; /* proj-gradient buffer (q's strides)    */
  float *dbias;            /* fp32 at h*bh+q*bq+k*bk (a dense [H,L,L] map); may be NULL */
  void *workspace;
  size_t workspace_bytes;
  float *dgate_bias;       /* backward, may be NULL: fp32 [H*D] column sums of
                              dGpre over all (b, l) (the gate bias gradient,
                              src/tensor.py:343), written */
} evo_attn_desc;

EVO_API int evo_attention_fwd(const evo_attn_desc *d, void *stream);
EVO_API int evo_attention_bwd(const evo_attn_desc *d, void *stream);
EVO_API size_t evo_attention_bwd_workspace_bytes(const evo_attn_desc *d);

/* Row work of the long-key (L > 256) bf16 attention, whose contractions run
 * as strided-batched evo_gemm calls over chunks of batch rows (the reference
 * op is the same _gated_attention, src/evoformer.py:268-286; softmax
 * src/tensor.py:352-361).  S/dP: fp32 [nbc, H, L, ld] (ld >= L, the row
 * stride: L rounded up to 8 so the GEMM operand rows stay 16-byte aligned);
 * P/dS: bf16, same shape; lse: fp32 [nbc, H, L]; bias/dbias: fp32 with the (bh, bq, bk) map
 * of evo_attn_desc; Dq: fp32 [rows, H] by activation row id
 * row0 + b*rb + q*rl.  dbias sums the chunk's batch rows in order and, with
 * acc, adds to the previous chunks' sum (deterministic).  dsoftmax with
 * S == NULL takes P as an input (the forward's probabilities) instead of
 * recomputing it from S, bias and lse.                                  */
EVO_API int evo_attn_long_softmax(int64_t nbc, int H, int L, int64_t ld, const float *S,
                                  const float *bias, int64_t bh, int64_t bq, int64_t bk, void *P,
                                  float *lse, void *stream);
EVO_API int evo_attn_long_gate(int64_t rows, int hc, const float *O, const void *g, int64_t g_rs,
                               void *o, void *gm, void *stream);
EVO_API int evo_attn_long_prep(int64_t rows, int H, int D, const void *dgm, const void *g,
                               int64_t g_rs, const void *o, void *dO, void *dgpre, int64_t dg_rs,
                               float *Dq, void *stream);
EVO_API int evo_attn_long_dsoftmax(int nbc, int H, int L, int64_t ld, const float *S,
                                   const float *dP,
                                   const float *bias, int64_t bh, int64_t bq, int64_t bk,
                                   const float *lse, const float *Dq, int64_t row0, int64_t rb,
                                   int64_t rl, void *P, void *dS, float *dbias, int acc,
                                   void *stream);

/* Long-key fused attention (tcgen05, keys streamed in 64-wide tiles with an
 * online softmax; no logits in HBM), bf16, head dim 16 / 32, any L: the same
 * op and descriptor as evo_attention_fwd/bwd (src/evoformer.py:268-286).
 * The bias (when present) must be plain rows: bk = 1, bq % 4 == 0,
 * bh >= L*bq; dbias is written in the same layout.  The backward runs the
 * prep pass (dO, dGpre, Dq, the gate-bias sums), the dq kernel (dbias as
 * fp32 partials over chunks of batch rows, summed in order) and the dk/dv
 * kernel; desc.workspace >= evo_attn_flash_bwd_workspace_bytes.          */
EVO_API int evo_attn_flash_fwd(const evo_attn_desc *d, void *stream);
EVO_API size_t evo_attn_flash_bwd_workspace_bytes(const evo_attn_desc *d);
EVO_API int evo_attn_flash_bwd(const evo_attn_desc *d, void *stream);

/* Deterministic reduction over the leading axis:
 * dst(i, j) (+)= sum_{b<nb} src[b*n1*n2 + i*n2 + j], dst at
 * dst[i*d_s1 + j*d_s2] fp32.  src dtype_src.  Replaces the bias-gradient
 * row sums of T.linear backward (src/tensor.py:343) and the pair-bias
 * gradient sum over the batch axis (_unbroadcast, src/tensor.py:194-203). */
EVO_API int evo_reduce_lead(int dtype_src, int64_t nb, int64_t n1, int64_t n2,
                    const void *src, float *dst, int64_t d_s1, int64_t d_s2,
                    int accumulate, void *stream);

/* Column sums of a tall matrix: dst[j] (+)= sum_i src[i*rs + j] (fp32
 * dst).  The bias gradient db = sum over rows of dy of T.linear
 * (src/tensor.py:343).  Deterministic two-stage reduction; workspace of
 * evo_colsum_workspace_bytes(cols) bytes.                               */
EVO_API int evo_colsum(int dtype_src, int64_t rows, int64_t cols, const void *src,
               int64_t rs, float *dst, int accumulate, void *workspace,
               size_t workspace_bytes, void *stream);
EVO_API size_t evo_colsum_workspace_bytes(int64_t cols);

/* 2-D strided copy with dtype conversion (weight packing, casts). */
EVO_API int evo_copy2d(int dtype_src, int dtype_dst, int64_t rows, int64_t cols,
               const void *src, int64_t s_rs, int64_t s_cs, void *dst,
               int64_t d_rs, int64_t d_cs, void *stream);

/* Batched 3-D strided copy with dtype conversion:
 * dst[b*d_bs + r*d_rs + c*d_cs] = src[b*s_bs + r*s_rs + c*s_cs].  The axis
 * permutations and shard placements of DAP (src/schedules.py:96-154:
 * allgather along an axis, the column shards of col_attn / tri_attn_end). */
EVO_API int evo_copy3d(int dtype_src, int dtype_dst, int64_t n0, int64_t rows, int64_t cols,
               const void *src, int64_t s_bs, int64_t s_rs, int64_t s_cs, void *dst,
               int64_t d_bs, int64_t d_rs, int64_t d_cs, void *stream);

/* bytes zero bytes at ptr, stream-ordered (the zero-padded shard gradients
 * DAP allreduces, src/schedules.py:122-128).                              */
EVO_API int evo_zero(void *ptr, size_t bytes, void *stream);

/* out(r,c) = a(r,c) * b(r,c); every operand 2-D strided, own dtype. */
EVO_API int evo_mul2d(int dtype_a, int dtype_b, int dtype_out, int64_t rows,
              int64_t cols, const void *a, int64_t a_rs, const void *b,
              int64_t b_rs, void *out, int64_t o_rs, void *stream);

/* Triangle-multiplication gating (src/evoformer.py:370-375).
 * proj rows (i,k) [r*r, ldp]: cols [0,c)=a value, [c,2c)=b value,
 * [2c,3c)=sigmoid(a gate), [3c,4c)=sigmoid(b gate).
 * fwd: a_cf[ch, row] = ga*a, b_cf[ch, row] = gb*b (channel-first).     */
EVO_API int evo_trimul_gate_fwd(int dtype, int64_t rows, int c, const void *proj,
                        int64_t ldp, void *a_cf, void *b_cf, void *stream);
/* bwd: from da_cf/db_cf (fp32, channel-first) write dproj[:, 0:4c]
 * (dvalue = d*g, dgate_pre = d*value*g*(1-g)).  colsum (fp32 [4c], may be
 * NULL): the column sums of those fp32 values before rounding to dtype (the
 * a_b | b_b | a_gate_b | b_gate_b gradients, deterministic order); needs
 * evo_trimul_gate_bwd_workspace_bytes of workspace.                     */
EVO_API size_t evo_trimul_gate_bwd_workspace_bytes(int64_t rows, int c);
EVO_API int evo_trimul_gate_bwd(int dtype, int64_t rows, int c, const void *proj,
                        int64_t ldp, const float *da_cf, const float *db_cf,
                        void *dproj, int64_t ldd, float *colsum, void *workspace,
                        size_t workspace_bytes, void *stream);

/* Output gate of the triangle multiplication (src/evoformer.py:394-396):
 * fwd: znew = z + g*o ;  bwd: do = dz*g, dgpre = dz*o*g*(1-g).
 * z, znew, dz fp32 [rows, cols] contiguous; g and o strided, dtype.     */
EVO_API int evo_outgate_fwd(int dtype, int64_t rows, int64_t cols, const float *z,
                    const void *g, int64_t g_rs, const void *o, int64_t o_rs,
                    float *znew, void *stream);
/* do_colsum / dg_colsum (fp32 [cols], both or neither; bf16, cols % 8 == 0):
 * column sums of do and dgpre from the fp32 values (the out_b and out_gate_b
 * gradients); workspace evo_outgate_bwd_workspace_bytes.                 */
EVO_API size_t evo_outgate_bwd_workspace_bytes(int64_t rows, int64_t cols);
EVO_API int evo_outgate_bwd(int dtype, int64_t rows, int64_t cols, const float *dz,
                    const void *g, int64_t g_rs, const void *o, int64_t o_rs,
                    void *do_, int64_t do_rs, void *dgpre, int64_t dg_rs,
                    float *do_colsum, float *dg_colsum, void *workspace,
                    size_t workspace_bytes, void *stream);

/* ReLU backward (src/tensor.py:274-280): dpre = dh * (pre > 0); `h` is
 * relu(pre) so h > 0 iff pre > 0.  Contiguous [n].                      */
EVO_API int evo_relu_bwd(int dtype, int64_t n, const void *dh, const void *h,
                 void *dpre, void *stream);

/* ReLU backward of a contiguous bf16 [rows, cols] (cols % 8 == 0) with the
 * column sums of its output fused in (the transition's first-layer bias
 * gradient, src/evoformer.py:314-329 / src/tensor.py:343):
 *   dpre = dh * (h > 0);  colsum_dst[c] = sum_rows dpre[:, c]  (fp32, written)
 * workspace: evo_colsum_workspace_bytes(cols).                          */
EVO_API int evo_relu_bwd_colsum(int64_t rows, int64_t cols, const void *dh, const void *h,
                                void *dpre, float *colsum_dst, void *workspace,
                                size_t workspace_bytes, void *stream);

/* Loss (src/schedules.py:194-195): out[0] += sum(x^2)/n (fp32,
 * deterministic two-pass); grad = 2*x/n written to dx (fp32, may be
 * NULL).  workspace >= 4 KiB.                                           */
EVO_API int evo_sq_mean(int64_t n, const float *x, float *out, float *dx,
                void *workspace, void *stream);

/* z_out = a + b elementwise (fp32), the block-end join z' = z_pair + o
 * (src/evoformer.py:460) when not fused into a GEMM epilogue.           */
EVO_API int evo_add(int64_t n, const float *a, const float *b, float *out,
            void *stream);

/* out = x / d (fp32, n elements; out may alias x): the division by dp of the
 * DP gradient mean (src/schedules.py:324-328).                           */
EVO_API int evo_div_scalar(int64_t n, const float *x, float d, float *out, void *stream);

/* LayerNorm forward of contiguous fp32 rows of 128 / 256 (c_z / c_m) into
 * the split bf16 operand y3 [rows, 3*cols] = hi | lo | hi (hi = bf16(y),
 * lo = bf16(y - hi)) of the 3-product transition projection; mean/rstd as
 * evo_layernorm_fwd.  EVO_EUNSUP for other shapes.                       */
EVO_API int evo_layernorm_fwd_split(int64_t rows, int cols, const float *x, const float *gamma,
                                    const float *beta, void *y3, float *mean, float *rstd,
                                    float eps, void *stream);

/* Split an fp32 [rows, cols] operand into bf16 hi = bf16(x) and
 * lo = bf16(x - hi) (hi also to hi2 when non-NULL), element strides per row.
 * Used for the 3-product bf16 GEMM (A3 = [hi | lo | hi], W3 = [W_hi; W_hi;
 * W_lo], K tripled) that gives the transitions' first projection fp32-grade
 * pre-activations, so the ReLU mask (src/tensor.py:274-280) matches the
 * reference's (src/evoformer.py:314-319).                                 */
EVO_API int evo_split_bf16(int64_t rows, int64_t cols, const float *x, int64_t x_rs, void *hi,
                           int64_t h_rs, void *lo, int64_t l_rs, void *hi2, int64_t h2_rs,
                           void *stream);

/* Library identity / diagnostics. */
EVO_API const char *evo_last_error(void);
EVO_API int evo_version(void);
/* Number of kernels this library has launched (all threads). */
EVO_API int64_t evo_launch_count(void);
/* 1 if the tcgen05 GEMM path is compiled in (the TMA encoder resolved). */
EVO_API int evo_tc_available(void);
/* Backend accounting: number of evo_gemm / evo_attention_* calls served by
 * each engine since load (EVO_BK_* below), and the engine of the last call
 * on this thread.  Tests assert the tensor-core path actually ran.        */
#define EVO_BK_GEMM_TC 0
#define EVO_BK_GEMM_SIMT 1
#define EVO_BK_GEMM_SKINNY 2
#define EVO_BK_ATTN_TC 3
#define EVO_BK_ATTN_SIMT 4
#define EVO_BK_ATTN_FLASH 5
#define EVO_BK_COUNT 6
EVO_API int64_t evo_backend_count(int backend);
EVO_API int evo_last_backend(void);
/* Strict tensor-core mode (default ON): a bf16 evo_gemm / evo_attention_*
 * call the tensor-core kernels do not take fails with EVO_EUNSUP instead of
 * running the SIMT kernels (the fp32 parity path is SIMT by design and is
 * unaffected).  0 = allow the SIMT fallback for bf16 (small test shapes). */
EVO_API void evo_set_strict_tc(int on);
EVO_API int evo_get_strict_tc(void);

#ifdef __cplusplus
}
#endif
#endif /* EVO_B200_H */
