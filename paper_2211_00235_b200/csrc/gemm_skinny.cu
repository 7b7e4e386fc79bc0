// Bandwidth-bound GEMM shapes that a 128-row tensor-core tile wastes:
//
//   rowdot  N <= 16, M large        (pair-bias projection  bias = LN(z) Wb,
//                                    src/evoformer.py:279: K = c_z, N = h)
//   expand  K <= 16, M large        (its input gradient    dz += dbias Wb^T)
//   tallk   min(M,N) <= 32, max <= 256, K huge  (weight gradients of the
//                                    narrow layers, dWb = LN(z)^T dbias over
//                                    the r*r pair rows)
//
// Each reads its operands once at HBM rate; tallk writes per-block partials
// that the split-K reducer sums in a fixed order (deterministic).  Same
// C(m,n) = epi(alpha * sum_k A(m,k) B(n,k)) contract as evo_gemm
// (include/evo_b200.h), any strides, bf16 or fp32 operands.
#include <algorithm>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "tc_common.cuh"

namespace evo {
namespace {
using namespace tc;

template <typename T>
__device__ __forceinline__ float ldf(const T *p, int64_t i) {
  if constexpr (std::is_same<T, float>::value) return __ldg(p + i);
  else return __bfloat162float(p[i]);
}

struct SkArgs {
  const void *A, *B;
  int64_t ars, acs, brs, bcs;
  int64_t M, N, K;
  int64_t a_b1, b_b1, nbatch;  // batch strides (B1 only)
  EpiArgs e;
  float *partial;
  int64_t kchunk;
};

// ---------------------------------------------------------------- rowdot
// One thread per output row; B staged in smem as fp32 [K][16].
template <typename T, int NMAX>
__global__ void __launch_bounds__(256) skinny_rowdot_kernel(const SkArgs a) {
  evo_pdl_enter();
  extern __shared__ float sB[];  // [K][NMAX]
  const T *A = reinterpret_cast<const T *>(a.A);
  const T *B = reinterpret_cast<const T *>(a.B);
  for (int64_t i = threadIdx.x; i < a.K * NMAX; i += blockDim.x) {
    const int64_t k = i / NMAX, n = i % NMAX;
    sB[i] = n < a.N ? ldf(B, n * a.brs + k * a.bcs) : 0.f;
  }
  __syncthreads();
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < a.M;
       m += (int64_t)gridDim.x * blockDim.x) {
    float acc[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) acc[n] = 0.f;
    const T *arow = A + m * a.ars;
    if constexpr (std::is_same<T, bf16>::value) {
      if (a.acs == 1 && (a.K & 7) == 0 && (reinterpret_cast<uintptr_t>(arow) & 15) == 0) {
#pragma unroll 4
        for (int64_t k0 = 0; k0 < a.K; k0 += 8) {
          const uint4 u = __ldg(reinterpret_cast<const uint4 *>(arow + k0));
          const __nv_bfloat162 *h2 = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(h2[j]);
            const float *b0 = sB + (k0 + 2 * j) * NMAX;
#pragma unroll
            for (int n = 0; n < NMAX; ++n) acc[n] = fmaf(f.x, b0[n], fmaf(f.y, b0[NMAX + n], acc[n]));
          }
        }
        goto store;
      }
    }
    for (int64_t k = 0; k < a.K; ++k) {
      const float x = ldf(A, m * a.ars + k * a.acs);
#pragma unroll
      for (int n = 0; n < NMAX; ++n) acc[n] = fmaf(x, sB[k * NMAX + n], acc[n]);
    }
  store:
    const int64_t rb = a.e.cmap.row(m);
#pragma unroll
    for (int n = 0; n < NMAX; ++n)
      if (n < a.N) epi_store(a.e, rb + a.e.cmap.col(n), epi_value(a.e, n, acc[n]));
  }
}

// ---------------------------------------------------------------- expand
// A warp owns 32 consecutive rows: lane l loads row m0+l's K <= 16 A values
// (coalesced when A is column-major, like dbias [h][r*r]), then for each of
// the 32 rows the values are broadcast by shuffles and every lane produces 4
// consecutive columns (B for those columns held in registers when N <= 128)
// and stores / reduce-adds them as one 16-byte vector: each output row is one
// fully coalesced 512-byte warp store.
template <typename T, int KK, bool NREG>
__global__ void __launch_bounds__(256) skinny_expand_kernel(const SkArgs a) {
  evo_pdl_enter();
  extern __shared__ float sB[];  // [KK][Np], Np = N rounded up to 4
  const T *A = reinterpret_cast<const T *>(a.A);
  const T *B = reinterpret_cast<const T *>(a.B);
  const int64_t Np = (a.N + 3) & ~int64_t(3);
  for (int64_t i = threadIdx.x; i < Np * KK; i += blockDim.x) {
    const int64_t k = i / Np, n = i % Np;
    sB[i] = (k < a.K && n < a.N) ? ldf(B, n * a.brs + k * a.bcs) : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const EpiArgs &e = a.e;
  const bool vec = e.dtype_c == EVO_F32 && e.cmap.cdiv == 0 && e.cmap.rdiv == 0 &&
                   e.cmap.cs == 1 && (e.cmap.rs & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(e.C) & 15) == 0 &&
                   (!e.residual || (reinterpret_cast<uintptr_t>(e.residual) & 15) == 0) &&
                   !e.bias && e.epi == EVO_EPI_NONE;
  float breg[NREG ? KK : 1][4];
  if constexpr (NREG) {
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      const float4 b = 4 * lane < Np ? *reinterpret_cast<const float4 *>(sB + k * Np + 4 * lane)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      breg[k][0] = b.x; breg[k][1] = b.y; breg[k][2] = b.z; breg[k][3] = b.w;
    }
  }
  const int64_t groups = (a.M + 31) / 32;
  const int64_t gw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t grp = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); grp < groups;
       grp += gw) {
    const int64_t m0 = grp * 32;
    const int64_t my = m0 + lane;
    float x[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k)
      x[k] = (my < a.M && k < a.K) ? ldf(A, my * a.ars + k * a.acs) : 0.f;
    const int rows = (int)std::min<int64_t>(32, a.M - m0);
    for (int r = 0; r < rows; ++r) {
      float xr[KK];
#pragma unroll
      for (int k = 0; k < KK; ++k) xr[k] = __shfl_sync(0xffffffffu, x[k], r);
      const int64_t m = m0 + r;
      const int64_t rb = e.cmap.row(m);
      for (int64_t n0 = 4 * lane; n0 < a.N; n0 += 128) {
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (NREG) {
#pragma unroll
          for (int k = 0; k < KK; ++k) {
#pragma unroll
            for (int u = 0; u < 4; ++u) o[u] = fmaf(xr[k], breg[k][u], o[u]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < KK; ++k) {
            const float4 b = *reinterpret_cast<const float4 *>(sB + k * Np + n0);
            o[0] = fmaf(xr[k], b.x, o[0]);
            o[1] = fmaf(xr[k], b.y, o[1]);
            o[2] = fmaf(xr[k], b.z, o[2]);
            o[3] = fmaf(xr[k], b.w, o[3]);
          }
        }
        if (vec && n0 + 4 <= a.N) {
          float4 v = make_float4(e.alpha * o[0], e.alpha * o[1], e.alpha * o[2], e.alpha * o[3]);
          float *dst = reinterpret_cast<float *>(e.C) + rb + n0;
          if (e.residual) {
            const float4 q = *reinterpret_cast<const float4 *>(e.residual + rb + n0);
            v.x += q.x; v.y += q.y; v.z += q.z; v.w += q.w;
          }
          if (e.accumulate) {
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x),
                         "f"(v.y), "f"(v.z), "f"(v.w)
                         : "memory");
          } else {
            *reinterpret_cast<float4 *>(dst) = v;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (n0 + u < a.N) epi_store(e, rb + e.cmap.col(n0 + u), epi_value(e, n0 + u, o[u]));
        }
      }
    }
  }
}

// ---------------------------------------------------------------- tallk
// C = sum_k A(:,k) B(:,k)^T with one "wide" operand (<= 256 wide, unit stride
// along its width) and one "narrow" operand (<= 32).  Thread w of a k-group
// owns wide index w and NN register accumulators; per k it loads one wide
// element (coalesced across the group) and reads the narrow values from a
// 64-k smem slab (broadcast).  Block (g, batch) covers k in
// [g*kchunk, (g+1)*kchunk); k-groups are combined in order, and the
// per-block partials [g][batch][M][N] go to the split-K reducer.
constexpr int TK_SLAB = 64;

template <typename T, int NN>
__global__ void __launch_bounds__(256) skinny_tallk_kernel(const SkArgs a, int wide_is_m) {
  evo_pdl_enter();
  extern __shared__ float sm[];
  float *sN = sm;  // [TK_SLAB][NN]
  const int W = (int)(wide_is_m ? a.M : a.N), Nn = (int)(wide_is_m ? a.N : a.M);
  const int Wp = (W + 31) & ~31;
  const int groups = 256 / Wp;
  const int tid = threadIdx.x, w = tid % Wp, kg = tid / Wp;
  const T *Aw = reinterpret_cast<const T *>(wide_is_m ? a.A : a.B) +
                blockIdx.y * (wide_is_m ? a.a_b1 : a.b_b1);
  const T *An = reinterpret_cast<const T *>(wide_is_m ? a.B : a.A) +
                blockIdx.y * (wide_is_m ? a.b_b1 : a.a_b1);
  const int64_t wks = wide_is_m ? a.acs : a.bcs;  // wide stride along k
  const int64_t nrs = wide_is_m ? a.brs : a.ars;  // narrow strides
  const int64_t nks = wide_is_m ? a.bcs : a.acs;
  const int64_t k_lo = blockIdx.x * a.kchunk;
  const int64_t k_hi = std::min(a.K, k_lo + a.kchunk);
  float acc[NN];
#pragma unroll
  for (int j = 0; j < NN; ++j) acc[j] = 0.f;
  const bool active = kg < groups && w < W;
  for (int64_t k0 = k_lo; k0 < k_hi; k0 += TK_SLAB) {
    const int rows = (int)std::min<int64_t>(TK_SLAB, k_hi - k0);
    __syncthreads();
    if (nks == 1) {  // narrow operand contiguous along k: k-fastest walk
      for (int i = tid; i < TK_SLAB * NN; i += 256) {
        const int kk = i % TK_SLAB, j = i / TK_SLAB;
        sN[kk * NN + j] = (kk < rows && j < Nn) ? ldf(An, j * nrs + (k0 + kk)) : 0.f;
      }
    } else {
      for (int i = tid; i < TK_SLAB * NN; i += 256) {
        const int kk = i / NN, j = i % NN;
        sN[i] = (kk < rows && j < Nn) ? ldf(An, j * nrs + (k0 + kk) * nks) : 0.f;
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll 4
      for (int kk = kg; kk < rows; kk += groups) {
        const float x = ldf(Aw, w + (k0 + kk) * wks);
        const float4 *nv = reinterpret_cast<const float4 *>(sN + kk * NN);
#pragma unroll
        for (int j = 0; j < NN / 4; ++j) {
          const float4 q = nv[j];
          acc[4 * j] = fmaf(x, q.x, acc[4 * j]);
          acc[4 * j + 1] = fmaf(x, q.y, acc[4 * j + 1]);
          acc[4 * j + 2] = fmaf(x, q.z, acc[4 * j + 2]);
          acc[4 * j + 3] = fmaf(x, q.w, acc[4 * j + 3]);
        }
      }
    }
  }
  // combine the k-groups in order (smem reuse: groups x Wp x NN floats)
  __syncthreads();
  float *red = sm;
  if (kg < groups) {
#pragma unroll
    for (int j = 0; j < NN; ++j) red[(kg * NN + j) * Wp + w] = acc[j];
  }
  __syncthreads();
  float *dst = a.partial + ((int64_t)blockIdx.x * a.nbatch + blockIdx.y) * a.M * a.N;
  for (int i = tid; i < Wp * NN; i += 256) {
    const int j = i / Wp, ww = i % Wp;
    if (ww >= W || j >= Nn) continue;
    float t = red[j * Wp + ww];
    for (int g2 = 1; g2 < groups; ++g2) t += red[(g2 * NN + j) * Wp + ww];
    const int64_t m = wide_is_m ? ww : j, n = wide_is_m ? j : ww;
    dst[m * a.N + n] = t;
  }
}

// ------------------------------------------------------------ tallk_bulk
// Same contraction when the wide operand is dense [K][W] and the narrow one
// dense [K][Nn] or k-contiguous [Nn][K]: one thread block per SM streams its
// k range through a 4-stage ring of bulk copies (tens of KB in flight per
// SM, the HBM-rate requirement), then each thread accumulates a 2-wide x NN
// block from smem (one 4-byte wide read + NN/8 16-byte broadcast reads per
// k).  Partials [g][batch][M][N] as above.
constexpr int TB_STAGES = 4;

struct BulkPlan {
  int kr;            // k rows per stage
  int narrow_kcont;  // narrow operand [Nn][K] (else dense [K][Nn])
  size_t stage_bytes, smem;
};

template <typename T, int NN>
__global__ void __launch_bounds__(256) skinny_tallk_bulk_kernel(const SkArgs a, int wide_is_m,
                                                                BulkPlan pl) {
  evo_pdl_enter();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int E = sizeof(T);
  const int W = (int)(wide_is_m ? a.M : a.N), Nn = (int)(wide_is_m ? a.N : a.M);
  const int KR = pl.kr;
  const size_t wbytes = (size_t)KR * W * E;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
  uint8_t *ring = smem_raw + 128;
  // narrow values of one stage as fp32 [KR][NN] (transposed/converted)
  float *sN = reinterpret_cast<float *>(ring + TB_STAGES * pl.stage_bytes);
  float *red = sN + KR * NN;

  const T *Aw = reinterpret_cast<const T *>(wide_is_m ? a.A : a.B) +
                blockIdx.y * (wide_is_m ? a.a_b1 : a.b_b1);
  const T *An = reinterpret_cast<const T *>(wide_is_m ? a.B : a.A) +
                blockIdx.y * (wide_is_m ? a.b_b1 : a.a_b1);
  const int64_t nrs = wide_is_m ? a.brs : a.ars;
  const int64_t k_lo = blockIdx.x * a.kchunk;
  const int64_t k_hi = std::min(a.K, k_lo + a.kchunk);
  const int nstage = (int)((k_hi - k_lo + KR - 1) / KR);
  const int tid = threadIdx.x;

  auto issue = [&](int st) {
    const int slot = st % TB_STAGES;
    const int64_t k0 = k_lo + (int64_t)st * KR;
    const int rows = (int)std::min<int64_t>(KR, k_hi - k0);
    uint8_t *dst = ring + slot * pl.stage_bytes;
    const uint32_t wb = (uint32_t)rows * W * E, nb = (uint32_t)rows * Nn * E;
    mbar_expect_tx(&bars[slot], wb + nb);
    bulk_load(dst, Aw + k0 * W, wb, &bars[slot]);
    if (pl.narrow_kcont) {
      for (int j = 0; j < Nn; ++j)
        bulk_load(dst + wbytes + (size_t)j * KR * E, An + j * nrs + k0, (uint32_t)rows * E,
                  &bars[slot]);
    } else {
      bulk_load(dst + wbytes, An + k0 * Nn, nb, &bars[slot]);
    }
  };
  if (tid == 0) {
    for (int i = 0; i < TB_STAGES; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < TB_STAGES && st < nstage; ++st) issue(st);
  }
  __syncthreads();

  const int Wh = W >> 1;  // wide pairs
  const int Whp = Wh <= 32 ? 32 : ((Wh + 31) & ~31);
  const int groups = 256 / Whp;
  const int wp = tid % Whp, kg = tid / Whp;
  const bool active = kg < groups && wp < Wh;
  float acc0[NN], acc1[NN];
#pragma unroll
  for (int j = 0; j < NN; ++j) acc0[j] = acc1[j] = 0.f;

  for (int st = 0; st < nstage; ++st) {
    const int slot = st % TB_STAGES;
    const int64_t k0 = k_lo + (int64_t)st * KR;
    const int rows = (int)std::min<int64_t>(KR, k_hi - k0);
    mbar_wait(&bars[slot], (uint32_t)((st / TB_STAGES) & 1));
    const uint8_t *buf = ring + slot * pl.stage_bytes;
    const T *sw = reinterpret_cast<const T *>(buf);
    const T *sn = reinterpret_cast<const T *>(buf + wbytes);
    // narrow -> fp32 [KR][NN] (zero-padded columns)
    for (int i = tid; i < KR * NN; i += 256) {
      const int kk = i / NN, j = i % NN;
      float v = 0.f;
      if (kk < rows && j < Nn) {
        const T t = pl.narrow_kcont ? sn[j * KR + kk] : sn[kk * Nn + j];
        if constexpr (sizeof(T) == 4) v = t; else v = __bfloat162float(t);
      }
      sN[i] = v;
    }
    __syncthreads();
    if (active) {
#pragma unroll 2
      for (int kk = kg; kk < rows; kk += groups) {
        float x0, x1;
        if constexpr (sizeof(T) == 4) {
          const float2 f = *reinterpret_cast<const float2 *>(sw + kk * W + 2 * wp);
          x0 = f.x; x1 = f.y;
        } else {
          const float2 f = __bfloat1622float2(
              *reinterpret_cast<const __nv_bfloat162 *>(sw + kk * W + 2 * wp));
          x0 = f.x; x1 = f.y;
        }
        const float4 *nv = reinterpret_cast<const float4 *>(sN + kk * NN);
#pragma unroll
        for (int q = 0; q < NN / 4; ++q) {
          const float4 v = nv[q];
          acc0[4 * q] = fmaf(x0, v.x, acc0[4 * q]);
          acc0[4 * q + 1] = fmaf(x0, v.y, acc0[4 * q + 1]);
          acc0[4 * q + 2] = fmaf(x0, v.z, acc0[4 * q + 2]);
          acc0[4 * q + 3] = fmaf(x0, v.w, acc0[4 * q + 3]);
          acc1[4 * q] = fmaf(x1, v.x, acc1[4 * q]);
          acc1[4 * q + 1] = fmaf(x1, v.y, acc1[4 * q + 1]);
          acc1[4 * q + 2] = fmaf(x1, v.z, acc1[4 * q + 2]);
          acc1[4 * q + 3] = fmaf(x1, v.w, acc1[4 * q + 3]);
        }
      }
    }
    __syncthreads();  // slot and sN free
    if (tid == 0 && st + TB_STAGES < nstage) issue(st + TB_STAGES);
  }
  // combine the k-groups in order: red[g][j][w]
  if (kg < groups && wp < Wh) {
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      red[(kg * NN + j) * W + 2 * wp] = acc0[j];
      red[(kg * NN + j) * W + 2 * wp + 1] = acc1[j];
    }
  }
  __syncthreads();
  float *dst = a.partial + ((int64_t)blockIdx.x * a.nbatch + blockIdx.y) * a.M * a.N;
  for (int i = tid; i < W * Nn; i += 256) {
    const int j = i / W, ww = i % W;
    float t = red[j * W + ww];
    for (int g2 = 1; g2 < groups; ++g2) t += red[(g2 * NN + j) * W + ww];
    const int64_t m = wide_is_m ? ww : j, n = wide_is_m ? j : ww;
    dst[m * a.N + n] = t;
  }
}

enum Kind { SK_NONE = 0, SK_ROWDOT, SK_EXPAND, SK_TALLK };

// wide operand (the larger of M, N) must have unit stride along its width
bool tallk_ok(const evo_gemm_desc *d, bool &wide_is_m) {
  if (d->B2 != 1 || d->K < 8192 || d->B1 > 64) return false;
  wide_is_m = d->M >= d->N;
  const int64_t W = wide_is_m ? d->M : d->N, Nn = wide_is_m ? d->N : d->M;
  const int64_t wrs = wide_is_m ? d->A.rs : d->B.rs;
  // Nn > 16 makes the SIMT FMA work (M*N*K) outgrow the bytes: TC + split-K
  return W <= 256 && Nn <= 16 && wrs == 1;
}

Kind classify(const evo_gemm_desc *d) {
  if (d->K < 1) return SK_NONE;
  const int64_t nb = d->B1 * d->B2;
  // any M: a narrow side (N <= 16 outputs, or K <= 16) would waste most of a
  // 128-wide tensor-core tile, and N < 8 does not fit the TMA operand maps
  if (nb == 1 && d->N <= 16 && d->K <= 2048) return SK_ROWDOT;
  if (nb == 1 && d->K <= 16 && d->N >= 32 && d->N <= 2048) return SK_EXPAND;
  bool wm;
  if (tallk_ok(d, wm)) return SK_TALLK;
  return SK_NONE;
}

// bulk-copy plan for tallk, or false when the layouts do not allow it
bool bulk_plan(const evo_gemm_desc *d, bool wide_is_m, int64_t kchunk, BulkPlan &pl) {
  const int64_t E = d->dtype_ab == EVO_BF16 ? 2 : 4;
  const int64_t W = wide_is_m ? d->M : d->N, Nn = wide_is_m ? d->N : d->M;
  const evo_mat &w = wide_is_m ? d->A : d->B;
  const evo_mat &n = wide_is_m ? d->B : d->A;
  auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(w.ptr) || !al(n.ptr) || (W & 1) || d->K % 16 || kchunk % 16) return false;
  if (w.rs != 1 || w.cs != W || (W * E) % 16 || (w.bs1 * E) % 16 || (n.bs1 * E) % 16)
    return false;
  if (n.rs == 1 && n.cs == Nn && (Nn * E) % 16 == 0) {
    pl.narrow_kcont = 0;
  } else if (n.cs == 1 && (n.rs * E) % 16 == 0) {
    pl.narrow_kcont = 1;
  } else {
    return false;
  }
  int kr = (int)(40960 / ((W + Nn) * E));
  kr = std::min<int>(kr & ~15, 256);
  if (kr < 16) return false;
  pl.kr = kr;
  pl.stage_bytes = (((size_t)kr * (W + Nn) * E) + 127) & ~size_t(127);
  const int nn = Nn <= 8 ? 8 : Nn <= 16 ? 16 : 32;
  const size_t red = std::max<size_t>((size_t)kr * nn, (size_t)8 * nn * W) * sizeof(float);
  pl.smem = 128 + TB_STAGES * pl.stage_bytes + (size_t)kr * nn * sizeof(float) + red;
  return pl.smem <= 200 * 1024;
}

int tallk_blocks(const evo_gemm_desc *d, int64_t &kchunk) {
  // one block per SM (the bulk ring keeps each SM's HBM share in flight)
  int64_t g = std::max<int64_t>(1, num_sms() / d->B1);
  g = std::min<int64_t>(g, (d->K + 255) / 256);
  kchunk = (d->K + g - 1) / g;
  kchunk = ((kchunk + TK_SLAB - 1) / TK_SLAB) * TK_SLAB;
  return (int)((d->K + kchunk - 1) / kchunk);
}

SkArgs args_of(const evo_gemm_desc *d) {
  SkArgs a;
  a.A = d->A.ptr; a.B = d->B.ptr;
  a.ars = d->A.rs; a.acs = d->A.cs; a.brs = d->B.rs; a.bcs = d->B.cs;
  a.M = d->M; a.N = d->N; a.K = d->K;
  a.a_b1 = d->A.bs1; a.b_b1 = d->B.bs1; a.nbatch = d->B1;
  a.e = epi_args_of(d);
  a.partial = nullptr;
  a.kchunk = 0;
  return a;
}

template <typename T>
int run(const evo_gemm_desc *d, Kind kind, cudaStream_t st) {
  SkArgs a = args_of(d);
  if (kind == SK_ROWDOT) {
    const size_t smem = (size_t)d->K * 16 * sizeof(float);
    EVO_MAX_SMEM_ONCE((skinny_rowdot_kernel<T, 16>));
    EVO_MAX_SMEM_ONCE((skinny_rowdot_kernel<T, 8>));
    const int blocks = (int)std::min<int64_t>((d->M + 255) / 256, (int64_t)num_sms() * 4);
    if (d->N <= 8) {
      launch_k(skinny_rowdot_kernel<T, 8>, blocks, 256, (size_t)d->K * 8 * sizeof(float), st, a);
    } else {
      launch_k(skinny_rowdot_kernel<T, 16>, blocks, 256, smem, st, a);
    }
    EVO_LAUNCHED("skinny_rowdot_kernel");
    return EVO_OK;
  }
  if (kind == SK_EXPAND) {
    const int kk = d->K <= 8 ? 8 : 16;
    const size_t smem = (size_t)((d->N + 3) & ~int64_t(3)) * kk * sizeof(float);
    const int64_t groups = (d->M + 31) / 32;
    const int blocks = (int)std::min<int64_t>((groups + 7) / 8, (int64_t)num_sms() * 8);
    const bool nreg = d->N <= 128;
#define EXPAND(KK, NR)                                                   \
  EVO_MAX_SMEM_ONCE((skinny_expand_kernel<T, KK, NR>));                  \
  launch_k(skinny_expand_kernel<T, KK, NR>, blocks, 256, smem, st, a);
    if (kk == 8) {
      if (nreg) { EXPAND(8, true) } else { EXPAND(8, false) }
    } else {
      if (nreg) { EXPAND(16, true) } else { EXPAND(16, false) }
    }
#undef EXPAND
    EVO_LAUNCHED("skinny_expand_kernel");
    return EVO_OK;
  }
  int64_t kc;
  const int g = tallk_blocks(d, kc);
  const size_t need = (size_t)g * d->B1 * d->M * d->N * sizeof(float);
  EVO_REQUIRE(d->workspace && d->workspace_bytes >= need, EVO_EARG,
              "evo_gemm(skinny): needs %zu workspace bytes", need);
  a.partial = reinterpret_cast<float *>(d->workspace);
  a.kchunk = kc;
  bool wm = true;
  tallk_ok(d, wm);
  const int64_t Nn = wm ? d->N : d->M;
  const dim3 grid((unsigned)g, (unsigned)d->B1);
  BulkPlan pl;
  if (bulk_plan(d, wm, kc, pl)) {
    EVO_MAX_SMEM_ONCE((skinny_tallk_bulk_kernel<T, 8>));
    EVO_MAX_SMEM_ONCE((skinny_tallk_bulk_kernel<T, 16>));
    EVO_MAX_SMEM_ONCE((skinny_tallk_bulk_kernel<T, 32>));
    if (Nn <= 8)
      launch_k(skinny_tallk_bulk_kernel<T, 8>, grid, 256, pl.smem, st, a, wm ? 1 : 0, pl);
    else if (Nn <= 16)
      launch_k(skinny_tallk_bulk_kernel<T, 16>, grid, 256, pl.smem, st, a, wm ? 1 : 0, pl);
    else
      launch_k(skinny_tallk_bulk_kernel<T, 32>, grid, 256, pl.smem, st, a, wm ? 1 : 0, pl);
    EVO_LAUNCHED("skinny_tallk_bulk_kernel");
    return gemm_splitk_reduce(d, g, a.partial, st);
  }
  const size_t smem = (size_t)256 * 32 * sizeof(float);  // >= slab and k-group combine
  if (Nn <= 8) {
    launch_k(skinny_tallk_kernel<T, 8>, grid, 256, smem, st, a, wm ? 1 : 0);
  } else if (Nn <= 16) {
    launch_k(skinny_tallk_kernel<T, 16>, grid, 256, smem, st, a, wm ? 1 : 0);
  } else {
    launch_k(skinny_tallk_kernel<T, 32>, grid, 256, smem, st, a, wm ? 1 : 0);
  }
  EVO_LAUNCHED("skinny_tallk_kernel");
  return gemm_splitk_reduce(d, g, a.partial, st);
}

}  // namespace

bool gemm_skinny_accepts(const evo_gemm_desc *d) { return classify(d) != SK_NONE; }

size_t gemm_skinny_workspace(const evo_gemm_desc *d) {
  if (classify(d) != SK_TALLK) return 0;
  int64_t kc;
  const int g = tallk_blocks(d, kc);
  return (size_t)g * d->B1 * d->M * d->N * sizeof(float);
}

int gemm_skinny(const evo_gemm_desc *d, cudaStream_t st) {
  const Kind kind = classify(d);
  if (kind == SK_NONE) return EVO_EUNSUP;
  return d->dtype_ab == EVO_BF16 ? run<bf16>(d, kind, st) : run<float>(d, kind, st);
}

}  // namespace evo
