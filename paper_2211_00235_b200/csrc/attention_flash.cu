// Gated attention over any number of keys on 5th-gen tensor cores: the
// long-key path (L > 256: crop r = 384 row / triangle attention, the MSA
// column attention over s = 512 or the extra-MSA s_e = 1024 / 5120
// sequences).  Same op as attention_tc.cu (src/evoformer.py:268-286, softmax
// src/tensor.py:352-361), with the keys streamed in tiles of KT = 64 so no
// logit ever reaches HBM:
//
// forward  (grid: 128-query tiles x H x nb; 8 softmax warps + 1 issuer warp)
//   S_j = Q K_j^T (TMEM), online softmax in the log2 domain with a lazily
//   updated running max (a row's max moves only when the tile max exceeds it
//   by more than 8: P <= 2^8 keeps bf16 P and the fp32 row sum exact enough,
//   and O in TMEM is rescaled only then), P_j (bf16 pairs) -> TMEM,
//   O += P_j V_j (TS MMA).  Epilogue O / l, gate, o, gm, lse.
// dq       (grid: q-tiles x H x chunks of batch rows)
//   S_j, dP_j = dO V_j^T;  P = exp2(S*c + bias*log2e - lse*log2e),
//   dS = P (dP - Dq) -> TMEM;  dQ += dS K_j (TS MMA);  dbias: each thread
//   adds its dS values into the chunk's fp32 partial (one owner thread per
//   element, batch rows in order: deterministic), chunks reduced in order.
// dkv      (grid: 128-key tiles x H x nb)
//   S^T_j = K Q_j^T, dP^T_j = V dO_j^T;  P^T, dS^T -> TMEM;
//   dV += P^T dO_j, dK += dS^T Q_j (TS MMAs).
// The prep pass (dO = dGM G, dGpre, Dq = rowsum(dO O)) is attention_long's.
// Bias: plain [H][L][bq] fp32 (the caller copies a transposed bias plain).
#include "common.cuh"
#include "tc_common.cuh"

namespace evo {
void note_backend(int b);
namespace {
using namespace tc;

constexpr float LOG2E_F = 1.4426950408889634f;
constexpr int QT = 128;    // queries (fwd / dq) or keys (dkv) per CTA = UMMA M
constexpr int KT = 64;     // streamed tile (keys, or queries in dkv) = UMMA N
constexpr int NEW = 8;     // elementwise warps: two threads per TMEM lane (row)
constexpr int NTH = (NEW + 1) * 32;
constexpr uint32_t BIAS_TILE = 2 * 16384;  // two [128 x 32] fp32 SW128 boxes

struct FlashArgs {
  int64_t nb;
  int H, L, D;
  float scale;
  const bf16 *g;            // sigmoid gate (proj cols 3hc), q's strides
  int64_t sb, sl;           // proj row strides (elements) of batch b / position l
  bf16 *o, *gm;             // [rows, hc] with o_sb / o_sl
  int64_t o_sb, o_sl;
  float *lse;               // [nb, H, L]
  const float *Dq;          // [rows, H] by activation row id
  int64_t rb, rl;           // activation row id = b*rb + l*rl
  bf16 *dq, *dk, *dv;       // proj-gradient columns (q's strides)
  float *dbias_part;        // [chunks][H][L][L] (dq kernel)
  int64_t chunk;
};

// swizzle of a [rows x D] bf16 tile with 2D-byte rows (TMA: 32B / 64B)
template <int D> struct Sw {
  static constexpr uint32_t bytes = 2 * D;
  static constexpr uint32_t layout = D == 32 ? 4 : 6;
  static constexpr uint32_t sbo = 8 * bytes;
};
template <int D>
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int ks) {
  return umma_desc(base + ks * 32, 16, Sw<D>::sbo, Sw<D>::layout);
}
template <int D>
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int ks) {
  return umma_desc(base + ks * 16 * Sw<D>::bytes, 16, Sw<D>::sbo, Sw<D>::layout);
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pk2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float2 upk2(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162 *>(&u);
  return __bfloat1622float2(h);
}
template <int N>
__device__ __forceinline__ void tld(uint32_t taddr, uint32_t (&v)[N]) {
  static_assert(N == 8 || N == 16 || N == 32, "tmem load width");
  if constexpr (N == 32) {
    tmem_ld32_nw(taddr, v);
  } else if constexpr (N == 16) {
    tmem_ld16_nw(taddr, v);
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
  }
}
template <int N>
__device__ __forceinline__ void tst(uint32_t taddr, const uint32_t (&v)[N]) {
  static_assert(N == 8 || N == 16, "tmem store width");
  if constexpr (N == 16) {
    tmem_st16(taddr, v);
  } else {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
        : "memory");
  }
}

// 32 bias values of query row `row` (keys kk*32 .. +31 of the tile) from a
// [128 rows x 32] fp32 SW128 box
__device__ __forceinline__ void bias_row(const uint8_t *box, int row, float (&out)[32]) {
  const uint8_t *base = box + row * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 v = *reinterpret_cast<const float4 *>(base + ((c ^ (row & 7)) << 4));
    out[4 * c] = v.x; out[4 * c + 1] = v.y; out[4 * c + 2] = v.z; out[4 * c + 3] = v.w;
  }
}
// element (q, k) of a [KT q rows x 32 k] fp32 SW128 box (dkv: read by column)
__device__ __forceinline__ float bias_at(const uint8_t *box, int q, int kk) {
  return *reinterpret_cast<const float *>(box + q * 128 + ((((kk >> 2) ^ (q & 7))) << 4) +
                                          (kk & 3) * 4);
}

// ======================================================================= fwd
// TMEM: buffer i at 96 i: S (64 fp32) | P (32 bf16 pairs);  O at 192.
template <int D, bool BIAS>
__global__ void __launch_bounds__(NTH, 1)
attn_flash_fwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                      const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mB,
                      const FlashArgs a) {
  constexpr int NS = 2;                                // K/V(/bias) stages
  constexpr uint32_t QB = QT * Sw<D>::bytes, KB = KT * Sw<D>::bytes;
  constexpr uint32_t STG = (BIAS ? BIAS_TILE : 0) + 2 * KB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sStage = smem_raw;                          // NS x [bias | K | V]
  uint8_t *sQ = sStage + NS * STG;
  float *sX = reinterpret_cast<float *>(sQ + QB);      // [2 parity][2 half][128] max exchange
  float *sL = sX + 2 * 2 * 128;                        // [2 half][128] row sums
  // 0 Q, 1-2 stage full, 3-4 S done, 5-6 P packed (8 warps), 7-8 PV done
  uint64_t *bars = reinterpret_cast<uint64_t *>(sL + 2 * 128);
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 9);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int L = a.L;
  const int T = (L + KT - 1) / KT;

  if (tid == NEW * 32) {
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], (i == 5 || i == 6) ? NEW : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == NEW) {
    // ------------------------------------------------------------ issuer
    auto load_tile = [&](int j) {
      uint8_t *st = sStage + (j % NS) * STG;
      uint64_t *bar = &bars[1 + (j % NS)];
      if (lane == 0) {
        mbar_expect_tx(bar, STG);
        if (BIAS) {
          tma_load_3d(st, &mB, bar, j * KT, q0, h);
          tma_load_3d(st + 16384, &mB, bar, j * KT + 32, q0, h);
        }
        uint8_t *kv = st + (BIAS ? BIAS_TILE : 0);
        tma_load_4d(kv, &mK, bar, 0, j * KT, (int)b, h);
        tma_load_4d(kv + KB, &mV, bar, 0, j * KT, (int)b, h);
      }
      __syncwarp();
    };
    if (lane == 0) {
      mbar_expect_tx(&bars[0], QB);
      tma_load_4d(sQ, &mQ, &bars[0], 0, q0, (int)b, h);
    }
    __syncwarp();
    for (int j = 0; j < NS && j < T; ++j) load_tile(j);
    const uint32_t idesc_s = idesc_bf16(128, KT, false, false);
    const uint32_t idesc_o = idesc_bf16(128, D, false, true);
    const uint32_t sQa = smem_u32(sQ);
    mbar_wait(&bars[0], 0);
    for (int j = 0; j <= T; ++j) {
      if (j < T) {
        const int st = j % NS;
        mbar_wait(&bars[1 + st], (uint32_t)((j / NS) & 1));
        fence_after();
        const uint32_t sK = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0);
        const uint32_t d = tmem + (j & 1) * 96;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_bf16_el(d, desc_k<D>(sQa, ks), desc_k<D>(sK, ks), idesc_s, ks > 0);
        umma_commit_el(&bars[3 + (j & 1)]);
      }
      if (j >= 1) {
        const int i = j - 1, bi = i & 1, st = i % NS;
        mbar_wait(&bars[5 + bi], (uint32_t)((i >> 1) & 1));   // P_i packed
        fence_after();
        const uint32_t sV = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0) + KB;
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(tmem + 192, tmem + bi * 96 + 64 + 8 * ks, desc_mn<D>(sV, ks), idesc_o,
                          (i > 0 || ks > 0) ? 1u : 0u);
        umma_commit_el(&bars[7 + bi]);
        if (i + NS < T) {
          mbar_wait(&bars[7 + bi], (uint32_t)((i >> 1) & 1));  // stage of tile i free
          load_tile(i + NS);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int quad = warp & 3, hf = warp >> 2;
    const int t = quad * 32 + lane;
    const int q = q0 + t;
    const bool qv = q < L;
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const float sc_l2 = a.scale * LOG2E_F;
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j < T; ++j) {
      const int bi = j & 1, st = j % NS;
      const int kb = j * KT + hf * 32;          // first key of this thread's 32
      if (BIAS) mbar_wait(&bars[1 + st], (uint32_t)((j / NS) & 1));  // bias tile landed
      mbar_wait(&bars[3 + bi], (uint32_t)((j >> 1) & 1));
      fence_after();
      uint32_t sv[32];
      tld<32>(lane_addr + bi * 96 + hf * 32, sv);
      float bb[32];
      if (BIAS) bias_row(sStage + st * STG + hf * 16384, t, bb);
      tmem_wait_ld();
      float x[32];
      float mt = -INFINITY;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        float v = __uint_as_float(sv[k]) * sc_l2;
        if (BIAS) v = fmaf(bb[k], LOG2E_F, v);
        x[k] = (kb + k < L) ? v : -INFINITY;
        mt = fmaxf(mt, x[k]);
      }
      float *sx = sX + bi * 256;
      sx[hf * 128 + t] = mt;
      named_bar_sync(1 + quad, 64);             // the row's two halves
      mt = fmaxf(sx[t], sx[128 + t]);
      const bool grow = mt > m_run + 8.f;
      float alpha = 1.f;
      if (grow) {
        alpha = ex2f(m_run - mt);               // 0 on the first tile
        m_run = mt;
      }
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
        // rescale this row's half of O once PV of the previous tile is done
        const int i = j - 1;
        mbar_wait(&bars[7 + (i & 1)], (uint32_t)((i >> 1) & 1));
        fence_after();
        constexpr int HD = D / 2;
        uint32_t ov[HD];
        tld<HD>(lane_addr + 192 + hf * HD, ov);
        tmem_wait_ld();
        if (grow) {
#pragma unroll
          for (int c = 0; c < HD; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha);
        }
        tst<HD>(lane_addr + 192 + hf * HD, ov);
      }
      l *= alpha;
      uint32_t pk[16];
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        const float p0 = ex2f(x[k] - m_run), p1 = ex2f(x[k + 1] - m_run);
        l += p0 + p1;
        pk[k >> 1] = pk2(p0, p1);
      }
      tst<16>(lane_addr + bi * 96 + 64 + hf * 16, pk);
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[5 + bi]);
    }
    // epilogue: O / l, gate, lse
    const int i = T - 1;
    mbar_wait(&bars[7 + (i & 1)], (uint32_t)((i >> 1) & 1));
    fence_after();
    sL[hf * 128 + t] = l;
    named_bar_sync(1 + quad, 64);
    const float lt = sL[t] + sL[128 + t];
    constexpr int HD = D / 2;
    uint32_t ov[HD];
    tld<HD>(lane_addr + 192 + hf * HD, ov);
    tmem_wait_ld();
    if (qv) {
      const float inv = 1.f / lt;
      const int64_t ooff = b * a.o_sb + (int64_t)q * a.o_sl + h * D + hf * HD;
      const bf16 *gp = a.g + b * a.sb + (int64_t)q * a.sl + h * D + hf * HD;
      uint32_t o2[HD / 2], g2[HD / 2];
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        const uint4 gq = *reinterpret_cast<const uint4 *>(gp + 8 * c);
        const uint32_t gw[4] = {gq.x, gq.y, gq.z, gq.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float v0 = __uint_as_float(ov[8 * c + 2 * e]) * inv;
          const float v1 = __uint_as_float(ov[8 * c + 2 * e + 1]) * inv;
          const float2 gg = upk2(gw[e]);
          o2[4 * c + e] = pk2(v0, v1);
          g2[4 * c + e] = pk2(gg.x * v0, gg.y * v1);
        }
      }
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        *reinterpret_cast<uint4 *>(a.o + ooff + 8 * c) =
            make_uint4(o2[4 * c], o2[4 * c + 1], o2[4 * c + 2], o2[4 * c + 3]);
        *reinterpret_cast<uint4 *>(a.gm + ooff + 8 * c) =
            make_uint4(g2[4 * c], g2[4 * c + 1], g2[4 * c + 2], g2[4 * c + 3]);
      }
      if (hf == 0) a.lse[(b * a.H + h) * (int64_t)L + q] = m_run * (1.f / LOG2E_F) + logf(lt);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// ======================================================================== dq
// TMEM: buffer i at 160 i: S (64) | dP (64) | dS (32 bf16 pairs); dQ at 320.
template <int D, bool BIAS>
__global__ void __launch_bounds__(NTH, 1)
attn_flash_dq_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                     const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mdO,
                     const __grid_constant__ CUtensorMap mB, const FlashArgs a) {
  constexpr int NS = 2;
  constexpr uint32_t QB = QT * Sw<D>::bytes, KB = KT * Sw<D>::bytes;
  constexpr uint32_t STG = (BIAS ? BIAS_TILE : 0) + 2 * KB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sStage = smem_raw;
  uint8_t *sQ = sStage + NS * STG;                     // Q | dO of the current row
  // 0 row Q/dO, 1-2 stage full, 3-4 S/dP done, 5-6 dS packed (8 warps),
  // 7-8 dQ MMA done, 9 row's dQ read back (8 warps)
  uint64_t *bars = reinterpret_cast<uint64_t *>(sQ + 2 * QB);
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 10);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L;
  const int T = (L + KT - 1) / KT;
  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  const int nrows = b_hi > b_lo ? (int)(b_hi - b_lo) : 0;
  const int G = nrows * T;                             // tiles over the chunk

  if (tid == NEW * 32) {
    for (int i = 0; i < 10; ++i)
      mbar_init(&bars[i], (i == 5 || i == 6 || i == 9) ? NEW : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == NEW) {
    auto load_tile = [&](int g) {
      const int64_t b = b_lo + g / T;
      const int j = g % T;
      uint8_t *st = sStage + (g % NS) * STG;
      uint64_t *bar = &bars[1 + (g % NS)];
      if (lane == 0) {
        mbar_expect_tx(bar, STG);
        if (BIAS) {
          tma_load_3d(st, &mB, bar, j * KT, q0, h);
          tma_load_3d(st + 16384, &mB, bar, j * KT + 32, q0, h);
        }
        uint8_t *kv = st + (BIAS ? BIAS_TILE : 0);
        tma_load_4d(kv, &mK, bar, 0, j * KT, (int)b, h);
        tma_load_4d(kv + KB, &mV, bar, 0, j * KT, (int)b, h);
      }
      __syncwarp();
    };
    auto load_row = [&](int64_t b) {
      if (lane == 0) {
        mbar_expect_tx(&bars[0], 2 * QB);
        tma_load_4d(sQ, &mQ, &bars[0], 0, q0, (int)b, h);
        tma_load_4d(sQ + QB, &mdO, &bars[0], 0, q0, (int)b, h);
      }
      __syncwarp();
    };
    if (G > 0) {
      load_row(b_lo);
      for (int g = 0; g < NS && g < G; ++g) load_tile(g);
    }
    const uint32_t idesc_s = idesc_bf16(128, KT, false, false);
    const uint32_t idesc_o = idesc_bf16(128, D, false, true);
    const uint32_t sQa = smem_u32(sQ), sdOa = sQa + QB;
    for (int g = 0; g <= G; ++g) {
      if (g < G) {
        const int64_t r = g / T;
        const int j = g % T;
        if (j == 0) mbar_wait(&bars[0], (uint32_t)(r & 1));   // row's Q / dO landed
        const int st = g % NS;
        mbar_wait(&bars[1 + st], (uint32_t)((g / NS) & 1));
        fence_after();
        const uint32_t sK = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0), sV = sK + KB;
        const uint32_t d = tmem + (g & 1) * 160;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_bf16_el(d, desc_k<D>(sQa, ks), desc_k<D>(sK, ks), idesc_s, ks > 0);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_bf16_el(d + 64, desc_k<D>(sdOa, ks), desc_k<D>(sV, ks), idesc_s, ks > 0);
        umma_commit_el(&bars[3 + (g & 1)]);
        if (j == T - 1 && r + 1 < nrows) {
          // the row's last S/dP MMAs read Q / dO: reload them for the next row
          mbar_wait(&bars[3 + (g & 1)], (uint32_t)((g >> 1) & 1));
          load_row(b_lo + r + 1);
        }
      }
      if (g >= 1) {
        const int i = g - 1, bi = i & 1, st = i % NS;
        const int ji = i % T;
        mbar_wait(&bars[5 + bi], (uint32_t)((i >> 1) & 1));   // dS_i packed
        if (ji == 0 && i > 0) mbar_wait(&bars[9], (uint32_t)(((i / T) - 1) & 1));  // dQ read
        fence_after();
        const uint32_t sK = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0);
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(tmem + 320, tmem + bi * 160 + 128 + 8 * ks, desc_mn<D>(sK, ks), idesc_o,
                          (ji > 0 || ks > 0) ? 1u : 0u);
        umma_commit_el(&bars[7 + bi]);
        if (i + NS < G) {
          mbar_wait(&bars[7 + bi], (uint32_t)((i >> 1) & 1));  // stage of tile i free
          load_tile(i + NS);
        }
      }
    }
  } else {
    const int quad = warp & 3, hf = warp >> 2;
    const int t = quad * 32 + lane;
    const int q = q0 + t;
    const bool qv = q < L;
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const float sc_l2 = a.scale * LOG2E_F;
    float lse_l2 = 0.f, dq_ = 0.f;
    float *part = BIAS ? a.dbias_part + (int64_t)blockIdx.z * a.H * L * (int64_t)L +
                             ((int64_t)h * L + q) * L
                       : nullptr;
    for (int g = 0; g < G; ++g) {
      const int r = g / T, j = g % T, bi = g & 1, st = g % NS;
      const int64_t b = b_lo + r;
      if (j == 0) {
        lse_l2 = qv ? a.lse[(b * a.H + h) * (int64_t)L + q] * LOG2E_F : 0.f;
        dq_ = qv ? a.Dq[(b * a.rb + (int64_t)q * a.rl) * a.H + h] : 0.f;
      }
      const int kb = j * KT + hf * 32;
      if (BIAS) mbar_wait(&bars[1 + st], (uint32_t)((g / NS) & 1));  // bias tile landed
      mbar_wait(&bars[3 + bi], (uint32_t)((g >> 1) & 1));
      fence_after();
      uint32_t sv[32], dv[32];
      tld<32>(lane_addr + bi * 160 + hf * 32, sv);
      tld<32>(lane_addr + bi * 160 + 64 + hf * 32, dv);
      float bb[32];
      if (BIAS) bias_row(sStage + st * STG + hf * 16384, t, bb);
      tmem_wait_ld();
      uint32_t pk[16];
      float ds[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        float x = fmaf(__uint_as_float(sv[k]), sc_l2, -lse_l2);
        if (BIAS) x = fmaf(bb[k], LOG2E_F, x);
        const float p = (qv && kb + k < L) ? ex2f(x) : 0.f;
        ds[k] = p * (__uint_as_float(dv[k]) - dq_);
      }
#pragma unroll
      for (int k = 0; k < 32; k += 2) pk[k >> 1] = pk2(ds[k], ds[k + 1]);
      tst<16>(lane_addr + bi * 160 + 128 + hf * 16, pk);
      if (BIAS && qv) {
        float *dst = part + kb;
        if (kb + 32 <= L && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float4 v = make_float4(ds[4 * c], ds[4 * c + 1], ds[4 * c + 2], ds[4 * c + 3]);
            if (r > 0) {
              const float4 o = *reinterpret_cast<const float4 *>(dst + 4 * c);
              v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
            }
            *reinterpret_cast<float4 *>(dst + 4 * c) = v;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (kb + k < L) dst[k] = r > 0 ? dst[k] + ds[k] : ds[k];
        }
      }
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[5 + bi]);
      if (j == T - 1) {
        // the row's dQ: wait for its last dQ MMA, scale, store
        mbar_wait(&bars[7 + bi], (uint32_t)((g >> 1) & 1));
        fence_after();
        constexpr int HD = D / 2;
        uint32_t v[HD];
        tld<HD>(lane_addr + 320 + hf * HD, v);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[9]);
        if (qv) {
          bf16 *dst = a.dq + b * a.sb + (int64_t)q * a.sl + h * D + hf * HD;
#pragma unroll
          for (int c = 0; c < HD / 8; ++c) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              w[e] = pk2(__uint_as_float(v[8 * c + 2 * e]) * a.scale,
                         __uint_as_float(v[8 * c + 2 * e + 1]) * a.scale);
            *reinterpret_cast<uint4 *>(dst + 8 * c) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ======================================================================= dkv
// CTA = 128 keys; the queries stream in tiles of 64.  TMEM: buffer i at
// 192 i: S^T (64) | dP^T (64) | P^T (32 pairs) | dS^T (32 pairs);
// dK at 384, dV at 384 + D.
template <int D, bool BIAS>
__global__ void __launch_bounds__(NTH, 1)
attn_flash_dkv_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                      const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mdO,
                      const __grid_constant__ CUtensorMap mB, const FlashArgs a) {
  constexpr int NS = 2;
  constexpr uint32_t KB = QT * Sw<D>::bytes, QB = KT * Sw<D>::bytes;
  // stage: bias [64 q x 128 k] as four [64 x 32] SW128 boxes | Q | dO | lse | Dq
  constexpr uint32_t BT = BIAS ? 4 * 8192 : 0;
  constexpr uint32_t STG = (BT + 2 * QB + 2 * KT * 4 + 1023) / 1024 * 1024;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sStage = smem_raw;
  uint8_t *sK = sStage + NS * STG;                     // K | V of the CTA's keys
  // 0 K/V, 1-2 stage TMA full, 3-4 stage lse/Dq staged, 5-6 S/dP done,
  // 7-8 P/dS packed (8 warps), 9-10 dK/dV MMAs done
  uint64_t *bars = reinterpret_cast<uint64_t *>(sK + 2 * KB);
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 11);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k0 = blockIdx.x * QT, h = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int L = a.L;
  const int T = (L + KT - 1) / KT;

  if (tid == NEW * 32) {
    for (int i = 0; i < 11; ++i) mbar_init(&bars[i], (i == 7 || i == 8) ? NEW : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == NEW) {
    auto load_tile = [&](int j) {
      uint8_t *st = sStage + (j % NS) * STG;
      uint64_t *bar = &bars[1 + (j % NS)];
      if (lane == 0) {
        mbar_expect_tx(bar, BT + 2 * QB);
        if (BIAS) {
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_3d(st + c * 8192, &mB, bar, k0 + 32 * c, j * KT, h);
        }
        tma_load_4d(st + BT, &mQ, bar, 0, j * KT, (int)b, h);
        tma_load_4d(st + BT + QB, &mdO, bar, 0, j * KT, (int)b, h);
      }
      // lse (log2 units) and Dq of the tile's 64 queries
      float *sl = reinterpret_cast<float *>(st + BT + 2 * QB), *sd = sl + KT;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int qi = lane + 32 * e, q = j * KT + qi;
        sl[qi] = q < L ? a.lse[(b * a.H + h) * (int64_t)L + q] * LOG2E_F : 0.f;
        sd[qi] = q < L ? a.Dq[(b * a.rb + (int64_t)q * a.rl) * a.H + h] : 0.f;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[3 + (j % NS)]);
      __syncwarp();
    };
    if (lane == 0) {
      mbar_expect_tx(&bars[0], 2 * KB);
      tma_load_4d(sK, &mK, &bars[0], 0, k0, (int)b, h);
      tma_load_4d(sK + KB, &mV, &bars[0], 0, k0, (int)b, h);
    }
    __syncwarp();
    for (int j = 0; j < NS && j < T; ++j) load_tile(j);
    const uint32_t idesc_s = idesc_bf16(128, KT, false, false);
    const uint32_t idesc_o = idesc_bf16(128, D, false, true);
    const uint32_t sKa = smem_u32(sK), sVa = sKa + KB;
    mbar_wait(&bars[0], 0);
    for (int j = 0; j <= T; ++j) {
      if (j < T) {
        const int st = j % NS;
        mbar_wait(&bars[1 + st], (uint32_t)((j / NS) & 1));
        fence_after();
        const uint32_t sQ = smem_u32(sStage + st * STG) + BT, sdO = sQ + QB;
        const uint32_t d = tmem + (j & 1) * 192;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_bf16_el(d, desc_k<D>(sKa, ks), desc_k<D>(sQ, ks), idesc_s, ks > 0);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_bf16_el(d + 64, desc_k<D>(sVa, ks), desc_k<D>(sdO, ks), idesc_s, ks > 0);
        umma_commit_el(&bars[5 + (j & 1)]);
      }
      if (j >= 1) {
        const int i = j - 1, bi = i & 1, st = i % NS;
        mbar_wait(&bars[7 + bi], (uint32_t)((i >> 1) & 1));   // P^T / dS^T packed
        fence_after();
        const uint32_t sQ = smem_u32(sStage + st * STG) + BT, sdO = sQ + QB;
        const uint32_t base = tmem + bi * 192;
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(tmem + 384 + D, base + 128 + 8 * ks, desc_mn<D>(sdO, ks), idesc_o,
                          (i > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(tmem + 384, base + 160 + 8 * ks, desc_mn<D>(sQ, ks), idesc_o,
                          (i > 0 || ks > 0) ? 1u : 0u);
        umma_commit_el(&bars[9 + bi]);
        if (i + NS < T) {
          mbar_wait(&bars[9 + bi], (uint32_t)((i >> 1) & 1));
          load_tile(i + NS);
        }
      }
    }
  } else {
    const int quad = warp & 3, hf = warp >> 2;
    const int t = quad * 32 + lane;                    // key row of the tile
    const int k = k0 + t;
    const bool kv = k < L;
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const float sc_l2 = a.scale * LOG2E_F;
    for (int j = 0; j < T; ++j) {
      const int bi = j & 1, st = j % NS;
      const int qb = j * KT + hf * 32;          // first query of this thread's 32
      mbar_wait(&bars[3 + st], (uint32_t)((j / NS) & 1));
      if (BIAS) mbar_wait(&bars[1 + st], (uint32_t)((j / NS) & 1));  // bias tile landed
      mbar_wait(&bars[5 + bi], (uint32_t)((j >> 1) & 1));
      fence_after();
      uint32_t sv[32], dv[32];
      tld<32>(lane_addr + bi * 192 + hf * 32, sv);
      tld<32>(lane_addr + bi * 192 + 64 + hf * 32, dv);
      const uint8_t *stg = sStage + st * STG;
      const float *sl = reinterpret_cast<const float *>(stg + BT + 2 * QB) + hf * 32;
      const float *sd = sl + KT;
      tmem_wait_ld();
      uint32_t pp[16], pd[16];
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 l4 = *reinterpret_cast<const float4 *>(sl + c);
        const float4 d4 = *reinterpret_cast<const float4 *>(sd + c);
        const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dq4[4] = {d4.x, d4.y, d4.z, d4.w};
        float p[4], ds[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int qq = c + e;
          float x = fmaf(__uint_as_float(sv[qq]), sc_l2, -lv[e]);
          if (BIAS) x = fmaf(bias_at(stg + (t >> 5) * 8192, hf * 32 + qq, t & 31), LOG2E_F, x);
          p[e] = (kv && qb + qq < L) ? ex2f(x) : 0.f;
          ds[e] = p[e] * (__uint_as_float(dv[qq]) - dq4[e]);
        }
        pp[c >> 1] = pk2(p[0], p[1]);
        pp[(c >> 1) + 1] = pk2(p[2], p[3]);
        pd[c >> 1] = pk2(ds[0], ds[1]);
        pd[(c >> 1) + 1] = pk2(ds[2], ds[3]);
      }
      tst<16>(lane_addr + bi * 192 + 128 + hf * 16, pp);
      tst<16>(lane_addr + bi * 192 + 160 + hf * 16, pd);
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[7 + bi]);
    }
    // dK = scale * acc, dV = acc
    const int i = T - 1;
    mbar_wait(&bars[9 + (i & 1)], (uint32_t)((i >> 1) & 1));
    fence_after();
    constexpr int HD = D / 2;
    uint32_t vk[HD], vv[HD];
    tld<HD>(lane_addr + 384 + hf * HD, vk);
    tld<HD>(lane_addr + 384 + D + hf * HD, vv);
    tmem_wait_ld();
    if (kv) {
      bf16 *dk = a.dk + b * a.sb + (int64_t)k * a.sl + h * D + hf * HD;
      bf16 *dvp = a.dv + b * a.sb + (int64_t)k * a.sl + h * D + hf * HD;
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        uint32_t wk[4], wv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          wk[e] = pk2(__uint_as_float(vk[8 * c + 2 * e]) * a.scale,
                      __uint_as_float(vk[8 * c + 2 * e + 1]) * a.scale);
          wv[e] = pk2(__uint_as_float(vv[8 * c + 2 * e]), __uint_as_float(vv[8 * c + 2 * e + 1]));
        }
        *reinterpret_cast<uint4 *>(dk + 8 * c) = make_uint4(wk[0], wk[1], wk[2], wk[3]);
        *reinterpret_cast<uint4 *>(dvp + 8 * c) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ====================================================================== host
bool flash_head_map(CUtensorMap *m, const void *base, int D, int L, int64_t nb, int H, int64_t sl,
                    int64_t sb, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)L, (cuuint64_t)nb, (cuuint64_t)H};
  cuuint64_t strides[3] = {(cuuint64_t)sl * 2, (cuuint64_t)sb * 2, (cuuint64_t)D * 2};
  cuuint32_t box[4] = {(cuuint32_t)D, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMapSwizzle sw = D == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// plain fp32 bias [H][L rows (q)][row stride bq] read as boxes {32 k, rows q}
bool flash_bias_map(CUtensorMap *m, const float *bias, int L, int H, int64_t bq, int64_t bh,
                    int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)L, (cuuint64_t)H};
  cuuint64_t strides[2] = {(cuuint64_t)bq * 4, (cuuint64_t)bh * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1}, es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(bias), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

FlashArgs flash_args(const evo_attn_desc *d) {
  FlashArgs a;
  a.nb = d->nb; a.H = d->H; a.L = d->L; a.D = d->D; a.scale = d->scale;
  a.g = reinterpret_cast<const bf16 *>(d->g);
  a.sb = d->sb; a.sl = d->sl;
  a.o = reinterpret_cast<bf16 *>(d->o); a.gm = reinterpret_cast<bf16 *>(d->gm);
  a.o_sb = d->o_sb; a.o_sl = d->o_sl;
  a.lse = d->lse;
  a.Dq = nullptr; a.rb = 0; a.rl = 0;
  a.dq = reinterpret_cast<bf16 *>(d->dq); a.dk = reinterpret_cast<bf16 *>(d->dk);
  a.dv = reinterpret_cast<bf16 *>(d->dv);
  a.dbias_part = nullptr; a.chunk = 1;
  return a;
}

bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_flash(const evo_attn_desc *d, bool bwd) {
  EVO_REQUIRE(d && d->dtype == EVO_BF16 && (d->D == 16 || d->D == 32) && d->L >= 1 &&
                  d->nb >= 1 && d->nb <= 65535 && d->H >= 1 && d->H <= 65535,
              EVO_EUNSUP, "attention_flash: bf16, head dim 16 / 32, nb <= 65535 (D=%d L=%d nb=%lld)",
              d ? d->D : -1, d ? d->L : -1, d ? (long long)d->nb : -1ll);
  EVO_REQUIRE(d->sb % 8 == 0 && d->sl % 8 == 0 && d->o_sb % 8 == 0 && d->o_sl % 8 == 0 &&
                  al16(d->q) && al16(d->k) && al16(d->v) && al16(d->g) && al16(d->o),
              EVO_EUNSUP, "attention_flash: 16-byte aligned rows required");
  EVO_REQUIRE(!d->bias || (d->bk == 1 && d->bq % 4 == 0 && d->bh % 4 == 0 && al16(d->bias)),
              EVO_EUNSUP, "attention_flash: plain bias rows (bk = 1, bq %% 4 == 0) required");
  if (bwd)
    EVO_REQUIRE(al16(d->dq) && al16(d->dk) && al16(d->dv) && al16(d->dgm), EVO_EUNSUP,
                "attention_flash: 16-byte aligned gradient rows required");
  return EVO_OK;
}

template <int D, bool BIAS>
int flash_fwd(const evo_attn_desc *d, cudaStream_t st) {
  FlashArgs a = flash_args(d);
  CUtensorMap mq, mk, mv, mb;
  if (!flash_head_map(&mq, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !flash_head_map(&mk, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, KT) ||
      !flash_head_map(&mv, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, KT))
    return EVO_EUNSUP;
  if (BIAS) {
    if (!flash_bias_map(&mb, d->bias, d->L, d->H, d->bq, d->bh, QT)) return EVO_EUNSUP;
  } else {
    mb = mq;
  }
  constexpr uint32_t STG = (BIAS ? BIAS_TILE : 0) + 2 * KT * 2 * D;
  const size_t smem = 2 * STG + QT * 2 * D + (4 * 128 + 2 * 128) * 4 + 9 * 8 + 16;
  auto kfn = attn_flash_fwd_kernel<D, BIAS>;
  EVO_MAX_SMEM_ONCE(kfn);
  dim3 grid((d->L + QT - 1) / QT, d->H, (unsigned)d->nb);
  kfn<<<grid, NTH, smem, st>>>(mq, mk, mv, mb, a);
  EVO_LAUNCHED("attn_flash_fwd_kernel");
  return EVO_OK;
}

template <int D, bool BIAS>
int flash_bwd(const evo_attn_desc *d, const void *dO, const float *Dq, int64_t rb, int64_t rl,
              float *dbias_part, int64_t chunk, cudaStream_t st) {
  FlashArgs a = flash_args(d);
  a.Dq = Dq; a.rb = rb; a.rl = rl;
  a.dbias_part = dbias_part;
  a.chunk = chunk;
  const int64_t hc = (int64_t)d->H * D;
  CUtensorMap mq, mk, mv, mdo, mb, mq2, mdo2, mk2, mv2, mb2;
  // dq kernel: Q / dO tiles of 128 queries, K / V tiles of 64 keys
  if (!flash_head_map(&mq, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !flash_head_map(&mdo, dO, D, d->L, d->nb, d->H, rl * hc, rb * hc, QT) ||
      !flash_head_map(&mk, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, KT) ||
      !flash_head_map(&mv, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, KT))
    return EVO_EUNSUP;
  // dkv kernel: K / V tiles of 128 keys, Q / dO tiles of 64 queries
  if (!flash_head_map(&mk2, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !flash_head_map(&mv2, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !flash_head_map(&mq2, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, KT) ||
      !flash_head_map(&mdo2, dO, D, d->L, d->nb, d->H, rl * hc, rb * hc, KT))
    return EVO_EUNSUP;
  if (BIAS) {
    if (!flash_bias_map(&mb, d->bias, d->L, d->H, d->bq, d->bh, QT) ||
        !flash_bias_map(&mb2, d->bias, d->L, d->H, d->bq, d->bh, KT))
      return EVO_EUNSUP;
  } else {
    mb = mq;
    mb2 = mq;
  }
  {
    constexpr uint32_t STG = (BIAS ? BIAS_TILE : 0) + 2 * KT * 2 * D;
    const size_t smem = 2 * STG + 2 * QT * 2 * D + 10 * 8 + 16;
    auto kfn = attn_flash_dq_kernel<D, BIAS>;
    EVO_MAX_SMEM_ONCE(kfn);
    const int64_t nch = (d->nb + chunk - 1) / chunk;
    dim3 grid((d->L + QT - 1) / QT, d->H, (unsigned)nch);
    kfn<<<grid, NTH, smem, st>>>(mq, mk, mv, mdo, mb, a);
    EVO_LAUNCHED("attn_flash_dq_kernel");
  }
  {
    constexpr uint32_t BT = BIAS ? 4 * 8192 : 0;
    constexpr uint32_t STG = (BT + 2 * KT * 2 * D + 2 * KT * 4 + 1023) / 1024 * 1024;
    const size_t smem = 2 * STG + 2 * QT * 2 * D + 11 * 8 + 16;
    auto kfn = attn_flash_dkv_kernel<D, BIAS>;
    EVO_MAX_SMEM_ONCE(kfn);
    dim3 grid((d->L + QT - 1) / QT, d->H, (unsigned)d->nb);
    kfn<<<grid, NTH, smem, st>>>(mq2, mk2, mv2, mdo2, mb2, a);
    EVO_LAUNCHED("attn_flash_dkv_kernel");
  }
  return EVO_OK;
}

}  // namespace
}  // namespace evo

using namespace evo;

extern "C" {

EVO_API int evo_attn_flash_fwd(const evo_attn_desc *d, void *stream) {
  int rc = check_flash(d, false);
  if (rc != EVO_OK) return rc;
  cudaStream_t st = as_stream(stream);
  note_backend(EVO_BK_ATTN_FLASH);
  if (d->D == 32) return d->bias ? flash_fwd<32, true>(d, st) : flash_fwd<32, false>(d, st);
  return d->bias ? flash_fwd<16, true>(d, st) : flash_fwd<16, false>(d, st);
}

EVO_API int evo_attn_flash_bwd(const evo_attn_desc *d, const void *dO, const float *Dq,
                               int64_t rb, int64_t rl, float *dbias_part, int64_t chunk,
                               void *stream) {
  int rc = check_flash(d, true);
  if (rc != EVO_OK) return rc;
  EVO_REQUIRE(dO && Dq && al16(dO) && chunk >= 1, EVO_EARG, "attn_flash_bwd: bad arguments");
  EVO_REQUIRE(!d->bias || dbias_part, EVO_EARG, "attn_flash_bwd: bias needs dbias partials");
  cudaStream_t st = as_stream(stream);
  note_backend(EVO_BK_ATTN_FLASH);
  if (d->D == 32)
    return d->bias ? flash_bwd<32, true>(d, dO, Dq, rb, rl, dbias_part, chunk, st)
                   : flash_bwd<32, false>(d, dO, Dq, rb, rl, dbias_part, chunk, st);
  return d->bias ? flash_bwd<16, true>(d, dO, Dq, rb, rl, dbias_part, chunk, st)
                 : flash_bwd<16, false>(d, dO, Dq, rb, rl, dbias_part, chunk, st);
}

}  // extern "C"
