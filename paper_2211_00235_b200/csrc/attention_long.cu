// Gated attention for L > 256 keys on the bf16 path (crop r = 384 row /
// triangle attention, the extra-MSA column attention over s_e = 1024): the
// four contractions (S = scale*QK^T, O = PV, dP = dO V^T, dQ/dK/dV) run as
// strided-batched tcgen05 GEMMs (evo_gemm) over chunks of batch rows, and
// these kernels do the row work between them:
//   softmax:   P = softmax(S + bias), lse           (src/tensor.py:352-357)
//   gate:      o = O, gm = sigmoid-gate * O         (src/evoformer.py:285)
//   prep:      dO = dGM*G, dGpre = dGM*O*G*(1-G), Dq = rowsum(dO*O)
//   dsoftmax:  P = exp(S + bias - lse), dS = P*(dP - Dq),
//              dbias[h,q,k] += sum over the chunk's batch rows of dS, in
//              batch order (deterministic; chunks accumulate in order)
// Orchestration: kernels.attention_long (Python, same descriptor meaning as
// evo_attention_fwd/bwd).
#include "common.cuh"

namespace evo {
namespace {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one warp per (b, h, q) logits row of S [nbc, H, L, L] fp32; the row
// (S + bias) stays in registers between the max, sum and normalise passes
// (L <= 32 * MAXJ; longer rows re-read S)
constexpr int MAXJ = 32;

template <int NJ>  // NJ > 0: row in NJ registers per lane (L <= 32 * NJ)
__global__ void long_softmax_kernel(int64_t nrows, int H, int L, int64_t ld,
                                    const float *__restrict__ S, const float *__restrict__ bias,
                                    int64_t bh, int64_t bq, int64_t bk, bf16 *__restrict__ P,
                                    float *__restrict__ lse) {
  evo_pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const int q = (int)(row % L);
  const int h = (int)((row / L) % H);
  const float *s = S + row * ld;
  const float *bb = bias ? bias + h * bh + q * bq : nullptr;
  bf16 *p = P + row * ld;
  float mx = -INFINITY, sum = 0.f;
  if constexpr (NJ > 0) {
    float v[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = j * 32 + lane;
      v[j] = k < L ? s[k] + (bb ? bb[k * bk] : 0.f) : -INFINITY;
      mx = fmaxf(mx, v[j]);
    }
    mx = warp_max(mx);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      v[j] = __expf(v[j] - mx);
      sum += v[j];
    }
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = j * 32 + lane;
      if (k < L) p[k] = __float2bfloat16(v[j] * inv);
    }
  } else {
    for (int k = lane; k < L; k += 32) mx = fmaxf(mx, s[k] + (bb ? bb[k * bk] : 0.f));
    mx = warp_max(mx);
    for (int k = lane; k < L; k += 32) sum += __expf(s[k] + (bb ? bb[k * bk] : 0.f) - mx);
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
    for (int k = lane; k < L; k += 32)
      p[k] = __float2bfloat16(__expf(s[k] + (bb ? bb[k * bk] : 0.f) - mx) * inv);
  }
  if (lane == 0) lse[row] = mx + logf(sum);
}

// [rows, hc]: o = O, gm = g * O (g = sigmoid(gate), already in proj)
__global__ void long_gate_kernel(int64_t n, int hc, const float *__restrict__ O,
                                 const bf16 *__restrict__ g, int64_t g_rs, bf16 *__restrict__ o,
                                 bf16 *__restrict__ gm) {
  evo_pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / hc;
    const int c = (int)(e - r * hc);
    const float ov = O[e];
    const bf16 ob = __float2bfloat16(ov);
    o[e] = ob;
    gm[e] = __float2bfloat16(__bfloat162float(g[r * g_rs + c]) * __bfloat162float(ob));
  }
}

// warp per (row, head): dO = dGM*G, dGpre = dGM*O*G*(1-G), Dq = sum_d dO*O
__global__ void long_prep_kernel(int64_t rows, int H, int D, const bf16 *__restrict__ dgm,
                                 const bf16 *__restrict__ g, int64_t g_rs,
                                 const bf16 *__restrict__ o, bf16 *__restrict__ dO,
                                 bf16 *__restrict__ dgpre, int64_t dg_rs,
                                 float *__restrict__ Dq) {
  evo_pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= rows * H) return;
  const int64_t r = w / H;
  const int h = (int)(w - r * H);
  const int hc = H * D;
  float acc = 0.f;
  for (int d = lane; d < D; d += 32) {
    const int c = h * D + d;
    const float gv = __bfloat162float(g[r * g_rs + c]);
    const float dg = __bfloat162float(dgm[r * hc + c]);
    const float ov = __bfloat162float(o[r * hc + c]);
    const bf16 dob = __float2bfloat16(dg * gv);
    dO[r * hc + c] = dob;
    dgpre[r * dg_rs + c] = __float2bfloat16(dg * ov * gv * (1.f - gv));
    acc += __bfloat162float(dob) * ov;
  }
  acc = warp_sum(acc);
  if (lane == 0) Dq[r * H + h] = acc;
}

// thread per (h, q, k) (consecutive threads along k: coalesced), batch rows
// of the chunk in order
__global__ void long_dsoftmax_kernel(int nbc, int H, int L, int64_t ld,
                                     const float *__restrict__ S,
                                     const float *__restrict__ dP,
                                     const float *__restrict__ bias, int64_t bh, int64_t bq,
                                     int64_t bk, const float *__restrict__ lse,
                                     const float *__restrict__ Dq, int64_t row0, int64_t rb,
                                     int64_t rl, bf16 *__restrict__ P, bf16 *__restrict__ dS,
                                     float *__restrict__ dbias, int acc) {
  evo_pdl_enter();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t LL = (int64_t)L * L;
  if (e >= H * LL) return;
  const int h = (int)(e / LL);
  const int q = (int)((e / L) % L), k = (int)(e % L);
  const float bv = (S && bias) ? bias[h * bh + q * bq + k * bk] : 0.f;
  float sum = 0.f;
#pragma unroll 4
  for (int b = 0; b < nbc; ++b) {
    const int64_t lrow = ((int64_t)b * H + h) * L + q;   // logits row in the chunk
    const int64_t arow = row0 + b * rb + q * rl;         // activation row id
    const int64_t ei = lrow * ld + k;
    float p;
    if (S) {  // recompute P from the logits and lse
      p = __expf(S[ei] + bv - lse[lrow]);
      P[ei] = __float2bfloat16(p);
    } else {  // the forward's P
      p = __bfloat162float(P[ei]);
    }
    const float ds = p * (dP[ei] - Dq[arow * H + h]);
    dS[ei] = __float2bfloat16(ds);
    sum += ds;
  }
  if (dbias) {
    float *db = dbias + h * bh + q * bq + k * bk;
    *db = acc ? *db + sum : sum;
  }
}

int warps_grid(int64_t warps, int wpb) { return (int)((warps + wpb - 1) / wpb); }

}  // namespace
}  // namespace evo

using namespace evo;

extern "C" {

EVO_API int evo_attn_long_softmax(int64_t nbc, int H, int L, int64_t ld, const float *S,
                                  const float *bias, int64_t bh, int64_t bq, int64_t bk, void *P,
                                  float *lse, void *stream) {
  EVO_REQUIRE(nbc >= 0 && H >= 1 && L >= 1 && ld >= L && S && P && lse, EVO_EARG,
              "attn_long_softmax: bad arguments");
  const int64_t rows = nbc * H * L;
  if (rows == 0) return EVO_OK;
#define EVO_LONG_SOFTMAX(NJ)                                                            \
  launch_k(long_softmax_kernel<NJ>, warps_grid(rows, 8), 256, 0, (cudaStream_t)stream, \
      rows, H, L, ld, S, bias, bh, bq, bk, reinterpret_cast<bf16 *>(P), lse)
  if (L <= 256) EVO_LONG_SOFTMAX(8);
  else if (L <= 512) EVO_LONG_SOFTMAX(16);
  else if (L <= 32 * MAXJ) EVO_LONG_SOFTMAX(32);
  else EVO_LONG_SOFTMAX(0);
#undef EVO_LONG_SOFTMAX
  EVO_LAUNCHED("long_softmax_kernel");
  return EVO_OK;
}

EVO_API int evo_attn_long_gate(int64_t rows, int hc, const float *O, const void *g, int64_t g_rs,
                               void *o, void *gm, void *stream) {
  EVO_REQUIRE(rows >= 0 && hc >= 1 && O && g && o && gm, EVO_EARG,
              "attn_long_gate: bad arguments");
  const int64_t n = rows * hc;
  if (n == 0) return EVO_OK;
  launch_k(long_gate_kernel, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, (cudaStream_t)stream, n, hc, O, reinterpret_cast<const bf16 *>(g), g_rs,
                                             reinterpret_cast<bf16 *>(o),
                                             reinterpret_cast<bf16 *>(gm));
  EVO_LAUNCHED("long_gate_kernel");
  return EVO_OK;
}

EVO_API int evo_attn_long_prep(int64_t rows, int H, int D, const void *dgm, const void *g,
                               int64_t g_rs, const void *o, void *dO, void *dgpre, int64_t dg_rs,
                               float *Dq, void *stream) {
  EVO_REQUIRE(rows >= 0 && H >= 1 && D >= 1 && dgm && g && o && dO && dgpre && Dq, EVO_EARG,
              "attn_long_prep: bad arguments");
  if (rows == 0) return EVO_OK;
  launch_k(long_prep_kernel, warps_grid(rows * H, 8), 256, 0, (cudaStream_t)stream, rows, H, D, reinterpret_cast<const bf16 *>(dgm), reinterpret_cast<const bf16 *>(g), g_rs,
      reinterpret_cast<const bf16 *>(o), reinterpret_cast<bf16 *>(dO),
      reinterpret_cast<bf16 *>(dgpre), dg_rs, Dq);
  EVO_LAUNCHED("long_prep_kernel");
  return EVO_OK;
}

EVO_API int evo_attn_long_dsoftmax(int nbc, int H, int L, int64_t ld, const float *S,
                                   const float *dP,
                                   const float *bias, int64_t bh, int64_t bq, int64_t bk,
                                   const float *lse, const float *Dq, int64_t row0, int64_t rb,
                                   int64_t rl, void *P, void *dS, float *dbias, int acc,
                                   void *stream) {
  EVO_REQUIRE(nbc >= 0 && H >= 1 && L >= 1 && ld >= L && dP && Dq && P && dS && (!S || lse),
              EVO_EARG,
              "attn_long_dsoftmax: bad arguments");
  if (nbc == 0) return EVO_OK;
  const int64_t n = (int64_t)H * L * L;
  launch_k(long_dsoftmax_kernel, (unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream, nbc, H, L, ld, S, dP, bias, bh, bq, bk, lse, Dq, row0, rb, rl, reinterpret_cast<bf16 *>(P),
      reinterpret_cast<bf16 *>(dS), dbias, acc);
  EVO_LAUNCHED("long_dsoftmax_kernel");
  return EVO_OK;
}

}  // extern "C"
