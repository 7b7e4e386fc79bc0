// SIMT (FFMA) strided batched GEMM: the fp32 parity path and the
// fallback for shapes the tcgen05 kernel does not take (tiny channel
// counts, non-unit strides).  C(m,n) = epi(alpha * sum_k A(m,k) B(n,k)).
//
// Replaces np.matmul in T.linear / T.matmul (src/tensor.py:299, 306-307,
// 325, 338-341).  Accumulation is two-level (per 16-wide K tile, then into
// the running sum) and split-K partials are summed in fixed order, so the
// result is deterministic and the fp32 error stays at BLAS level.
#include "common.cuh"
#include "gemm.cuh"
#include "gemm_epi.cuh"

namespace evo {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

struct SimtArgs {
  int64_t M, N, K, B1, B2;
  const void *A; int64_t a_rs, a_cs, a_b1, a_b2;
  const void *B; int64_t b_rs, b_cs, b_b1, b_b2;
  void *C; IdxMap cmap; int64_t c_b1, c_b2;
  float alpha;
  int epi, epi_col0, accumulate;
  const float *bias, *residual;
  int split_k; int64_t k_chunk;
  float *partial;  // split_k > 1: [split][B1*B2][M][N]
};

template <typename T>
__device__ __forceinline__ float ldg_f(const void *p, int64_t off) {
  return to_f(reinterpret_cast<const T *>(p)[off]);
}

template <typename TC>
__device__ __forceinline__ void epilogue_store(const SimtArgs &a, int64_t m, int64_t n,
                                               int64_t cbase, float v) {
  if (a.bias) v += a.bias[n];
  if (a.epi == EVO_EPI_RELU) v = fmaxf(v, 0.f);
  else if (a.epi == EVO_EPI_SIGMOID_FROM && n >= a.epi_col0) v = sigmoidf_stable(v);
  int64_t off = cbase + a.cmap.row(m) + a.cmap.col(n);
  if (a.residual) v += a.residual[off];
  TC *c = reinterpret_cast<TC *>(a.C);
  if (a.accumulate) v += to_f(c[off]);
  c[off] = from_f<TC>(v);
}

template <typename TA, typename TC>
__global__ void __launch_bounds__(NT) gemm_simt_kernel(SimtArgs a) {
  evo_pdl_enter();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  const int64_t n0 = (int64_t)blockIdx.x * BN, m0 = (int64_t)blockIdx.y * BM;
  const int64_t nbatch = a.B1 * a.B2;
  const int64_t z = blockIdx.z;
  const int64_t bidx = z % nbatch;
  const int split = (int)(z / nbatch);
  const int64_t b1 = bidx / a.B2, b2 = bidx % a.B2;
  const int64_t k_lo = split * a.k_chunk;
  const int64_t k_hi = min(a.K, k_lo + a.k_chunk);
  const int64_t abase = b1 * a.a_b1 + b2 * a.a_b2;
  const int64_t bbase = b1 * a.b_b1 + b2 * a.b_b2;
  const bool a_kc = (a.a_cs == 1);  // K contiguous
  const bool b_kc = (a.b_cs == 1);

  float acc[4][4], part[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = k_lo; k0 < k_hi; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = t + NT * i;
      int mm, kk;
      if (a_kc) { mm = e / BK; kk = e % BK; } else { mm = e % BM; kk = e / BM; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < a.M && gk < k_hi) v = ldg_f<TA>(a.A, abase + gm * a.a_rs + gk * a.a_cs);
      As[kk][mm] = v;
      int nn;
      if (b_kc) { nn = e / BK; kk = e % BK; } else { nn = e % BN; kk = e / BN; }
      int64_t gn = n0 + nn;
      gk = k0 + kk;
      v = 0.f;
      if (gn < a.N && gk < k_hi) v = ldg_f<TA>(a.B, bbase + gn * a.b_rs + gk * a.b_cs);
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) part[i][j] = 0.f;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 av = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
      float4 bv = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
      float ar[4] = {av.x, av.y, av.z, av.w};
      float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) part[i][j] = fmaf(ar[i], br[j], part[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += part[i][j];
    __syncthreads();
  }

  if (a.split_k > 1) {
    float *out = a.partial + ((int64_t)split * nbatch + bidx) * a.M * a.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t m = m0 + ty * 4 + i;
      if (m >= a.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int64_t n = n0 + tx * 4 + j;
        if (n < a.N) out[m * a.N + n] = acc[i][j];
      }
    }
    return;
  }
  const int64_t cbase = b1 * a.c_b1 + b2 * a.c_b2;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n < a.N) epilogue_store<TC>(a, m, n, cbase, a.alpha * acc[i][j]);
    }
  }
}

SimtArgs make_args(const evo_gemm_desc *d, int split, int64_t k_chunk) {
  SimtArgs a;
  a.M = d->M; a.N = d->N; a.K = d->K; a.B1 = d->B1; a.B2 = d->B2;
  a.A = d->A.ptr; a.a_rs = d->A.rs; a.a_cs = d->A.cs; a.a_b1 = d->A.bs1; a.a_b2 = d->A.bs2;
  a.B = d->B.ptr; a.b_rs = d->B.rs; a.b_cs = d->B.cs; a.b_b1 = d->B.bs1; a.b_b2 = d->B.bs2;
  a.C = d->C.ptr; a.cmap = idxmap_of(d->C); a.c_b1 = d->C.bs1; a.c_b2 = d->C.bs2;
  a.alpha = d->alpha; a.epi = d->epilogue; a.epi_col0 = d->epi_col0;
  a.accumulate = d->accumulate; a.bias = d->bias; a.residual = d->residual;
  a.split_k = split; a.k_chunk = k_chunk;
  a.partial = reinterpret_cast<float *>(d->workspace);
  return a;
}

// P consecutive outputs per block; the 256/P thread groups take partials
// g, g + 256/P, ... and the group sums are combined in order (fixed order:
// deterministic).  P = 8 when there are few outputs and many partials, so
// the reduction still spreads over every SM.
template <int P>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(EpiArgs e, int64_t M, int64_t N,
                                                            int64_t B2, int64_t nbatch, int split,
                                                            const float *partial) {
  evo_pdl_enter();
  constexpr int G = 256 / P;
  __shared__ float red[G][P + 1];
  const int o = threadIdx.x % P, grp = threadIdx.x / P;
  const int64_t total = nbatch * M * N;
  const int64_t idx = blockIdx.x * (int64_t)P + o;
  float v = 0.f;
  if (idx < total) {
#pragma unroll 4
    for (int s = grp; s < split; s += G) v += partial[(int64_t)s * total + idx];
  }
  red[grp][o] = v;
  __syncthreads();
  if (threadIdx.x < P && idx < total) {
    float t = red[0][o];
#pragma unroll 8
    for (int j = 1; j < G; ++j) t += red[j][o];
    const int64_t n = idx % N;
    const int64_t m = (idx / N) % M;
    const int64_t bidx = idx / (M * N);
    const int64_t b1 = bidx / B2, b2 = bidx % B2;
    const int64_t off = b1 * e.c_b1 + b2 * e.c_b2 + e.cmap.row(m) + e.cmap.col(n);
    epi_store(e, off, epi_value(e, n, t));
  }
}

// Few partials: one thread per 4 consecutive outputs (16-byte loads, the
// split loads independent and in flight), partials summed in split order.
__global__ void __launch_bounds__(256) splitk_reduce_vec_kernel(EpiArgs e, int64_t M, int64_t N,
                                                                int64_t B2, int64_t nbatch,
                                                                int split,
                                                                const float *__restrict__ partial) {
  evo_pdl_enter();
  const int64_t total = nbatch * M * N;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t idx = 4 * q;
  if (idx >= total) return;
  float4 v = __ldg(reinterpret_cast<const float4 *>(partial + idx));
#pragma unroll 4
  for (int s = 1; s < split; ++s) {
    const float4 w = __ldg(reinterpret_cast<const float4 *>(partial + (int64_t)s * total + idx));
    v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
  }
  const int64_t n = idx % N;
  const int64_t m = (idx / N) % M;
  const int64_t bidx = idx / (M * N);
  const int64_t b1 = bidx / B2, b2 = bidx % B2;
  const int64_t rb = b1 * e.c_b1 + b2 * e.c_b2 + e.cmap.row(m);
  const float t[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) epi_store(e, rb + e.cmap.col(n + j), epi_value(e, n + j, t[j]));
}

}  // namespace

int gemm_splitk_reduce(const evo_gemm_desc *d, int split, const float *partial,
                       cudaStream_t st) {
  const int64_t total = d->B1 * d->B2 * d->M * d->N;
  EVO_REQUIRE((total + 31) / 32 < (1ll << 31), EVO_EDIM, "evo_gemm: split-K output too large");
  if (split <= 32 && d->N % 4 == 0 && (reinterpret_cast<uintptr_t>(partial) & 15) == 0) {
    launch_k(splitk_reduce_vec_kernel, (unsigned)((total / 4 + 255) / 256), 256, 0, st, epi_args_of(d), d->M, d->N, d->B2, d->B1 * d->B2, split, partial);
  } else if (total / 32 < 2 * (int64_t)num_sms() && split > 32) {
    launch_k(splitk_reduce_kernel<8>, (unsigned)((total + 7) / 8), 256, 0, st, epi_args_of(d), d->M, d->N, d->B2, d->B1 * d->B2, split, partial);
  } else {
    launch_k(splitk_reduce_kernel<32>, (unsigned)((total + 31) / 32), 256, 0, st, epi_args_of(d), d->M, d->N, d->B2, d->B1 * d->B2, split, partial);
  }
  EVO_LAUNCHED("splitk_reduce_kernel");
  return EVO_OK;
}

size_t gemm_simt_workspace(const evo_gemm_desc *d) {
  if (d->split_k <= 1) return 0;
  return (size_t)d->split_k * d->B1 * d->B2 * d->M * d->N * sizeof(float);
}

int gemm_simt(const evo_gemm_desc *d, cudaStream_t st) {
  int split = d->split_k < 1 ? 1 : d->split_k;
  int64_t k_chunk = (d->K + split - 1) / split;
  k_chunk = ((k_chunk + BK - 1) / BK) * BK;
  if (k_chunk <= 0) k_chunk = BK;
  split = (int)((d->K + k_chunk - 1) / k_chunk);
  if (split < 1) split = 1;
  if (split > 1) {
    size_t need = (size_t)split * d->B1 * d->B2 * d->M * d->N * sizeof(float);
    EVO_REQUIRE(d->workspace && d->workspace_bytes >= need, EVO_EARG,
                "evo_gemm: split_k=%d needs %zu workspace bytes", split, need);
  }
  SimtArgs a = make_args(d, split, k_chunk);
  int64_t gz = d->B1 * d->B2 * split;
  EVO_REQUIRE(gz <= 65535 && (d->M + BM - 1) / BM <= 65535, EVO_EDIM,
              "evo_gemm: grid too large (batch*split=%lld, M=%lld)", (long long)gz,
              (long long)d->M);
  dim3 grid((unsigned)((d->N + BN - 1) / BN), (unsigned)((d->M + BM - 1) / BM), (unsigned)gz);
  if (d->K == 0) {
    // empty contraction: C = epi(0)
    split = 1;
  }
#define LAUNCH(TA, TCT)                                                        \
  launch_k(gemm_simt_kernel<TA, TCT>, grid, NT, 0, st, a);                          \
  EVO_LAUNCHED("gemm_simt_kernel");                                           \
  if (split > 1) return gemm_splitk_reduce(d, split, a.partial, st);
  if (d->dtype_ab == EVO_F32) {
    if (d->dtype_c == EVO_F32) { LAUNCH(float, float) } else { LAUNCH(float, bf16) }
  } else {
    if (d->dtype_c == EVO_F32) { LAUNCH(bf16, float) } else { LAUNCH(bf16, bf16) }
  }
#undef LAUNCH
  return EVO_OK;
}

}  // namespace evo
