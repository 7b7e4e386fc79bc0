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
// dq       (grid: q-tiles x H x chunks of batch rows; rows in groups of 4)
//   S_j, dP_j = dO V_j^T;  P = exp2(S*c + bias*log2e - lse*log2e),
//   dS = P (dP - Dq) -> TMEM;  dQ += dS K_j (TS MMA);  dbias: a group's dS
//   summed in TMEM, then added by its one owner thread into the chunk's fp32
//   partial (groups in order: deterministic), chunks reduced in order.
// dkv      (grid: 128-key tiles x H x nb)
//   S^T_j = K Q_j^T, dP^T_j = V dO_j^T;  P^T, dS^T -> TMEM;
//   dV += P^T dO_j, dK += dS^T Q_j (TS MMAs).
// The prep pass (dO = dGM G, dGpre, Dq = rowsum(dO O), lse in log2 units) is
// attention_tc's.
// Bias: plain [H][L][bq] fp32 (the caller copies a transposed bias plain).
#include <algorithm>

#include "common.cuh"
#include "tc_common.cuh"

namespace evo {
void note_backend(int b);
int attn_prep_run(const evo_attn_desc *d, void *dO_out, float *Dq, float *gpart, float *lse2,
                  cudaStream_t st);
int reduce_lead(int, int64_t, int64_t, int64_t, const void *, float *, int64_t, int64_t, int,
                cudaStream_t);
namespace {
using namespace tc;

constexpr float LOG2E_F = 1.4426950408889634f;
constexpr int QT = 128;    // queries (fwd / dq) or keys (dkv) per CTA = UMMA M
constexpr int KT = 64;     // streamed tile (keys, or queries in dkv) = UMMA N
// each kernel: TPR elementwise threads per TMEM lane (row), EPT = KT / TPR
// elements each, NEW = 4 TPR elementwise warps + 1 issuer warp
constexpr int TPR_FWD = 2, TPR_DQ = 2, TPR_DKV = 4;  // fwd: 2 CTAs / SM; dq, dkv: 1 (512 TMEM cols)
constexpr int NS_FWD = 2, NS_BWD = 4;     // streamed-tile stages
// forward stages: two with a bias tile (40 KB each, two CTAs per SM), four
// without one (the K/V tiles alone are small): the extra depth hides the
// TMA latency of the next tiles behind the softmax
template <bool BIAS> constexpr int ns_fwd() { return BIAS ? NS_FWD : 4; }
constexpr int nth_of(int tpr) { return (4 * tpr + 1) * 32; }
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
  const float *Dq;          // [nb, H, L]
  bf16 *dq, *dk, *dv;       // proj-gradient columns (q's strides)
  float *dbias_part;        // [chunks][H][L][L] (dq kernel)
  int64_t chunk;
  int group;                // dq kernel: batch rows per group (1, 2 or 4; bias)
};

// swizzle of a [rows x D] bf16 tile with 2D-byte rows (TMA: none / 32B / 64B)
template <int D> struct Sw {
  static constexpr uint32_t bytes = 2 * D;
  static constexpr uint32_t layout = D == 32 ? 4 : (D == 16 ? 6 : 0);
  static constexpr uint32_t sbo = 8 * bytes;
};
// K steps (16 wide) of a head-dim contraction; D = 8 runs one step whose
// upper 8 columns come from a zero region (c_head = 8: the extra-MSA stack)
template <int D> constexpr int ksteps() { return D < 16 ? 1 : D / 16; }
// accumulator width (UMMA N >= 16): D = 8 accumulates 16 columns, the upper
// 8 of which are never read
template <int D> constexpr int dacc() { return D < 16 ? 16 : D; }
// K-major [rows x D] operand, K step ks.  D = 8 (no swizzle, 16-byte rows):
// the second 8-column core matrix sits `zlbo` bytes on (a zero region for the
// padded operand, 0 = itself for the other one)
template <int D>
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int ks, uint32_t zlbo = 0) {
  if constexpr (D == 8) return umma_desc(base, zlbo, 128, 0);
  return umma_desc(base + ks * 32, 16, Sw<D>::sbo, Sw<D>::layout);
}
// MN-major B(n = d, k = row) from a [rows x D] tile, K step ks (16 rows).
// D = 8: core matrices of 8 rows x 16 B, K groups 128 B apart; the second N
// group (columns 8..15) repeats the first (never read)
template <int D>
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int ks) {
  if constexpr (D == 8) return umma_desc(base + ks * 256, 128, 0, 0);
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
  static_assert(N == 4 || N == 8 || N == 16 || N == 32 || N == 64, "tmem load width");
  if constexpr (N == 64) {
    uint32_t (&lo)[32] = *reinterpret_cast<uint32_t(*)[32]>(&v[0]);
    uint32_t (&hi)[32] = *reinterpret_cast<uint32_t(*)[32]>(&v[32]);
    tmem_ld32_nw(taddr, lo);
    tmem_ld32_nw(taddr + 32, hi);
  } else if constexpr (N == 32) {
    tmem_ld32_nw(taddr, v);
  } else if constexpr (N == 16) {
    tmem_ld16_nw(taddr, v);
  } else if constexpr (N == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
  }
}
template <int N>
__device__ __forceinline__ void tst(uint32_t taddr, const uint32_t (&v)[N]) {
  static_assert(N == 4 || N == 8 || N == 16 || N == 32, "tmem store width");
  if constexpr (N == 32) {
    tmem_st32(taddr, v);
  } else if constexpr (N == 16) {
    tmem_st16(taddr, v);
  } else if constexpr (N == 8) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
        : "memory");
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
                 : "memory");
  }
}

// EPT bias values of query row `row`, tile keys k0 .. k0+EPT-1 (k0 % EPT ==
// 0), from the stage's two [128 rows x 32] fp32 SW128 boxes
template <int EPT>
__device__ __forceinline__ void bias_row(const uint8_t *tile, int row, int k0, float (&out)[EPT]) {
#pragma unroll
  for (int c = 0; c < EPT / 4; ++c) {
    const int kk = k0 + 4 * c;   // box kk / 32, 16-byte chunk (kk % 32) / 4
    const uint8_t *base = tile + (kk >> 5) * 16384 + row * 128;
    const float4 v = *reinterpret_cast<const float4 *>(base + ((((kk & 31) >> 2) ^ (row & 7)) << 4));
    out[4 * c] = v.x; out[4 * c + 1] = v.y; out[4 * c + 2] = v.z; out[4 * c + 3] = v.w;
  }
}
// element (q, k) of a [KT q rows x 32 k] fp32 SW128 box (dkv: read by column)
__device__ __forceinline__ float bias_at(const uint8_t *box, int q, int kk) {
  return *reinterpret_cast<const float *>(box + q * 128 + ((((kk >> 2) ^ (q & 7))) << 4) +
                                          (kk & 3) * 4);
}

// ======================================================================= fwd
// Persistent over a chunk of batch rows: tile g = (row r, key tile j), the
// K/V(/bias) stage ring and the S/P double buffer run continuously across
// rows; Q tiles and the O accumulators are double-buffered by row parity so
// a row's epilogue overlaps the next row's MMAs.
// TMEM (256): S/P buffer g&1 at 96 (g&1): S (64 fp32) | P (32 bf16 pairs);
// O of row parity p at 192 + D p.
// Softmax warp w: lane quadrant w & 3 (rows), part w >> 2 (EPT keys).
// two CTAs per SM: 18 warps over 4 SMSPs put 5 on one, so <= 96 registers
template <int D, bool BIAS>
__global__ void __maxnreg__(96)
attn_flash_fwd_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                      const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mB,
                      const FlashArgs a) {
  evo_pdl_enter();
  constexpr int TPR = TPR_FWD, EPT = KT / TPR, NEW = 4 * TPR;
  constexpr int NS = ns_fwd<BIAS>();
  constexpr uint32_t QB = QT * Sw<D>::bytes, KB = KT * Sw<D>::bytes;
  constexpr uint32_t STG = (BIAS ? BIAS_TILE : 0) + 2 * KB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sStage = smem_raw;                          // NS x [bias | K | V]
  uint8_t *sQ = sStage + NS * STG;                     // 2 x Q (row parity)
  float *sX = reinterpret_cast<float *>(sQ + 2 * QB);  // [2 parity][TPR][128] max exchange
  float *sL = sX + 2 * TPR * 128;                      // [TPR][128] row sums
  uint64_t *bars = reinterpret_cast<uint64_t *>(sL + TPR * 128);
  uint64_t *qfull = bars, *fullb = qfull + 2, *sdone = fullb + NS, *pp = sdone + 2,
           *pvd = pp + 2, *ord = pvd + 2;
  constexpr int NBAR = 2 + NS + 8;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + NBAR);
  // 2 KB of zeros above every operand: the padded head-dim half (D = 8)
  uint8_t *sZ = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(tslot + 4) + 1023) & ~static_cast<uintptr_t>(1023));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L;
  const int T = (L + KT - 1) / KT;
  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  const int nrows = b_hi > b_lo ? (int)(b_hi - b_lo) : 0;
  const int G = nrows * T;

  if (tid == NEW * 32) {
    for (int i = 0; i < NBAR; ++i) {
      uint64_t *bb = &bars[i];
      const bool warps = bb == &pp[0] || bb == &pp[1] || bb == &ord[0] || bb == &ord[1];
      mbar_init(bb, warps ? NEW : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (D == 8) {
    for (int i = tid; i < 512; i += blockDim.x) reinterpret_cast<uint32_t *>(sZ)[i] = 0u;
    fence_proxy_async_smem();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == NEW) {
    // ------------------------------------------------------------ issuer
    auto load_tile = [&](int g) {
      const int64_t b = b_lo + g / T;
      const int j = g % T;
      uint8_t *st = sStage + (g % NS) * STG;
      uint64_t *bar = &fullb[g % NS];
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
    auto load_q = [&](int r) {
      if (lane == 0) {
        mbar_expect_tx(&qfull[r & 1], QB);
        tma_load_4d(sQ + (r & 1) * QB, &mQ, &qfull[r & 1], 0, q0, (int)(b_lo + r), h);
      }
      __syncwarp();
    };
    for (int r = 0; r < 2 && r < nrows; ++r) load_q(r);
    for (int g = 0; g < NS && g < G; ++g) load_tile(g);
    const uint32_t idesc_s = idesc_bf16(128, KT, false, false);
    const uint32_t idesc_o = idesc_bf16(128, dacc<D>(), false, true);
    int r = 0, j = 0;          // coordinates of tile g
    int ri = 0, ji = -1;       // coordinates of tile g - 1
    for (int g = 0; g <= G; ++g) {
      if (g < G) {
        if (j == 0) mbar_wait(&qfull[r & 1], (uint32_t)((r >> 1) & 1));
        const int st = g % NS;
        mbar_wait(&fullb[st], (uint32_t)((g / NS) & 1));
        fence_after();
        const uint32_t sK = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0);
        const uint32_t sQa = smem_u32(sQ) + (r & 1) * QB;
        const uint32_t d = tmem + (g & 1) * 96;
#pragma unroll
        for (int ks = 0; ks < ksteps<D>(); ++ks)
          umma_bf16_el(d, desc_k<D>(sQa, ks, smem_u32(sZ) - sQa), desc_k<D>(sK, ks), idesc_s,
                       ks > 0);
        umma_commit_el(&sdone[g & 1]);
        if (j == T - 1 && r + 2 < nrows) {
          mbar_wait(&sdone[g & 1], (uint32_t)((g >> 1) & 1));   // row r's S MMAs read Q
          load_q(r + 2);
        }
      }
      if (g >= 1) {
        const int i = g - 1, bi = i & 1, st = i % NS;
        mbar_wait(&pp[bi], (uint32_t)((i >> 1) & 1));   // P_i packed
        if (ji == 0 && ri >= 2) mbar_wait(&ord[ri & 1], (uint32_t)(((ri >> 1) - 1) & 1));
        fence_after();
        const uint32_t sV = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0) + KB;
        const uint32_t oc = tmem + 192 + dacc<D>() * (ri & 1);
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(oc, tmem + bi * 96 + 64 + 8 * ks, desc_mn<D>(sV, ks), idesc_o,
                          (ji > 0 || ks > 0) ? 1u : 0u);
        umma_commit_el(&pvd[bi]);
        if (i + NS < G) {
          mbar_wait(&pvd[bi], (uint32_t)((i >> 1) & 1));  // stage of tile i free
          load_tile(i + NS);
        }
      }
      ri = r;
      ji = j;
      if (++j == T) {
        j = 0;
        ++r;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int quad = warp & 3, part = warp >> 2;
    const int t = quad * 32 + lane;
    const int q = q0 + t;
    const bool qv = q < L;
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const float sc_l2 = a.scale * LOG2E_F;
    constexpr int OD = D / TPR < 4 ? 4 : D / TPR;   // epilogue columns per thread
    float m_run = -INFINITY, l = 0.f;
    int r = 0, j = 0;
    for (int g = 0; g < G; ++g) {
      const int bi = g & 1, st = g % NS;
      const int kb = j * KT + part * EPT;        // first key of this thread's EPT
      const uint32_t oc = lane_addr + 192 + dacc<D>() * (r & 1) + part * OD;
      if (j == 0) {
        m_run = -INFINITY;
        l = 0.f;
      }
      if (BIAS) mbar_wait(&fullb[st], (uint32_t)((g / NS) & 1));  // bias tile landed
      mbar_wait(&sdone[bi], (uint32_t)((g >> 1) & 1));
      fence_after();
      uint32_t sv[EPT];
      tld<EPT>(lane_addr + bi * 96 + part * EPT, sv);
      float bb[EPT];
      if (BIAS) bias_row(sStage + st * STG, t, part * EPT, bb);
      tmem_wait_ld();
      float x[EPT];
      float mt = -INFINITY;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        x[k] = BIAS ? fmaf(bb[k], LOG2E_F, __uint_as_float(sv[k]) * sc_l2)
                    : __uint_as_float(sv[k]) * sc_l2;
        mt = fmaxf(mt, x[k]);
      }
      if (kb + EPT > L) {  // the last key tile: mask keys beyond L
        mt = -INFINITY;
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          if (kb + k >= L) x[k] = -INFINITY;
          mt = fmaxf(mt, x[k]);
        }
      }
      float *sx = sX + bi * (TPR * 128);
      sx[part * 128 + t] = mt;
      if (TPR > 1) named_bar_sync(1 + quad, 32 * TPR);   // the row's TPR parts
#pragma unroll
      for (int p2 = 0; p2 < TPR; ++p2) mt = fmaxf(mt, sx[p2 * 128 + t]);
      const bool grow = mt > m_run + 8.f;
      float alpha = 1.f;
      if (grow) {
        alpha = ex2f(m_run - mt);               // 0 on the row's first tile
        m_run = mt;
      }
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
        // rescale this row's part of O once PV of the previous tile is done
        mbar_wait(&pvd[(g - 1) & 1], (uint32_t)(((g - 1) >> 1) & 1));
        fence_after();
        uint32_t ov[OD];
        tld<OD>(oc, ov);
        tmem_wait_ld();
        if (grow) {
#pragma unroll
          for (int c = 0; c < OD; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha);
        }
        tst<OD>(oc, ov);
      }
      l *= alpha;
      uint32_t pk[EPT / 2];
#pragma unroll
      for (int k = 0; k < EPT; k += 2) {
        const float p0 = ex2f(x[k] - m_run), p1 = ex2f(x[k + 1] - m_run);
        l += p0 + p1;
        pk[k >> 1] = pk2(p0, p1);
      }
      tst<EPT / 2>(lane_addr + bi * 96 + 64 + part * (EPT / 2), pk);
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pp[bi]);
      if (j == T - 1) {
        // epilogue of row r: O / l, gate, lse (overlaps the next row's MMAs)
        const int64_t b = b_lo + r;
        mbar_wait(&pvd[bi], (uint32_t)((g >> 1) & 1));
        fence_after();
        uint32_t ov[OD];
        tld<OD>(oc, ov);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ord[r & 1]);
        sL[part * 128 + t] = l;
        if (TPR > 1) named_bar_sync(1 + quad, 32 * TPR);
        float lt = 0.f;
#pragma unroll
        for (int p2 = 0; p2 < TPR; ++p2) lt += sL[p2 * 128 + t];
        if (qv && part * OD < D) {
          const float inv = 1.f / lt;
          const int64_t ooff = b * a.o_sb + (int64_t)q * a.o_sl + h * D + part * OD;
          const bf16 *gp = a.g + b * a.sb + (int64_t)q * a.sl + h * D + part * OD;
          // OD = D / TPR consecutive columns: 16-byte chunks (OD % 8 == 0) or
          // one 8-byte chunk (OD == 4)
          constexpr int CW = OD % 8 == 0 ? 8 : 4;
#pragma unroll
          for (int c0 = 0; c0 < OD; c0 += CW) {
            uint32_t gw[CW / 2], o2[CW / 2], g2[CW / 2];
            if constexpr (CW == 8) {
              const uint4 gq = *reinterpret_cast<const uint4 *>(gp + c0);
              gw[0] = gq.x; gw[1] = gq.y; gw[2] = gq.z; gw[3] = gq.w;
            } else {
              const uint2 gq = *reinterpret_cast<const uint2 *>(gp + c0);
              gw[0] = gq.x; gw[1] = gq.y;
            }
#pragma unroll
            for (int e = 0; e < CW / 2; ++e) {
              const float v0 = __uint_as_float(ov[c0 + 2 * e]) * inv;
              const float v1 = __uint_as_float(ov[c0 + 2 * e + 1]) * inv;
              const float2 gg = upk2(gw[e]);
              o2[e] = pk2(v0, v1);
              g2[e] = pk2(gg.x * v0, gg.y * v1);
            }
            if constexpr (CW == 8) {
              *reinterpret_cast<uint4 *>(a.o + ooff + c0) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
              *reinterpret_cast<uint4 *>(a.gm + ooff + c0) = make_uint4(g2[0], g2[1], g2[2], g2[3]);
            } else {
              *reinterpret_cast<uint2 *>(a.o + ooff + c0) = make_uint2(o2[0], o2[1]);
              *reinterpret_cast<uint2 *>(a.gm + ooff + c0) = make_uint2(g2[0], g2[1]);
            }
          }
          if (part == 0) a.lse[(b * a.H + h) * (int64_t)L + q] = m_run * (1.f / LOG2E_F) + logf(lt);
        }
      }
      if (++j == T) {
        j = 0;
        ++r;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// store OD fp32 TMEM values (x scale) as bf16 at dst (16-byte or 8-byte chunks)
template <int OD>
__device__ __forceinline__ void store_row_bf16(bf16 *dst, const uint32_t (&v)[OD], float scale) {
  constexpr int CW = OD % 8 == 0 ? 8 : 4;
#pragma unroll
  for (int c0 = 0; c0 < OD; c0 += CW) {
    uint32_t w[CW / 2];
#pragma unroll
    for (int e = 0; e < CW / 2; ++e)
      w[e] = pk2(__uint_as_float(v[c0 + 2 * e]) * scale,
                 __uint_as_float(v[c0 + 2 * e + 1]) * scale);
    if constexpr (CW == 8)
      *reinterpret_cast<uint4 *>(dst + c0) = make_uint4(w[0], w[1], w[2], w[3]);
    else
      *reinterpret_cast<uint2 *>(dst + c0) = make_uint2(w[0], w[1]);
  }
}

// N consecutive fp32 values at p: 16-byte loads when aligned, else scalar
template <int N>
__device__ __forceinline__ void load_f32(const float *p, bool vec, float (&out)[N]) {
  if (vec) {
#pragma unroll
    for (int c = 0; c < N / 4; ++c) {
      const float4 v = *reinterpret_cast<const float4 *>(p + 4 * c);
      out[4 * c] = v.x; out[4 * c + 1] = v.y; out[4 * c + 2] = v.z; out[4 * c + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int c = 0; c < N; ++c) out[c] = p[c];
  }
}

// ======================================================================== dq
// Persistent over a chunk of batch rows.  With a pair bias the rows run in
// GROUPS of a.group (4), tile by tile: (row pb, key tile j), (pb+1, j), ...,
// (pb+3, j), (pb, j+1), ..., so a thread meets the group's dS tiles of the
// same keys back to back; their sum (parked in TMEM) is the one dbias
// reduction: a quarter of the L2 reduction traffic of one reduction per row,
// which bounds this kernel with a bias (nb H L^2 fp32 reductions per call).
// Q / dO in four row buffers (row mod 4: the next group's rows load as this
// group's rows finish), dQ in four accumulators (row mod 4).
// TMEM: buffer g&1 at 160 (g&1): S (64) | dP (64) | dS (32 bf16 pairs);
// dQ of row r at 320 + dacc (r mod 4); the parked dS sum past them.
constexpr int DQ_QBUF = 4, DQ_ACC = 4, DQ_GROUP = 4;

template <int D, bool BIAS>
__global__ void __launch_bounds__(nth_of(TPR_DQ), 1)
attn_flash_dq_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                     const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mdO,
                     const __grid_constant__ CUtensorMap mB, const FlashArgs a) {
  evo_pdl_enter();
  constexpr int TPR = TPR_DQ, EPT = KT / TPR, NEW = 4 * TPR;
  constexpr int NS = NS_BWD, NQB = DQ_QBUF;
  constexpr uint32_t QB = QT * Sw<D>::bytes, KB = KT * Sw<D>::bytes;
  constexpr uint32_t STG = (BIAS ? BIAS_TILE : 0) + 2 * KB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sStage = smem_raw;
  uint8_t *sQ = sStage + NS * STG;                     // NQB x [Q | dO] (row mod NQB)
  uint64_t *bars = reinterpret_cast<uint64_t *>(sQ + NQB * 2 * QB);
  uint64_t *qfull = bars, *fullb = qfull + NQB, *sdone = fullb + NS, *dsp = sdone + 2,
           *dqd = dsp + 2, *dqr = dqd + 2;               // dqr: DQ_ACC
  constexpr int NBAR = NQB + NS + 6 + DQ_ACC;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + NBAR);
  // 2 KB of zeros above every operand: the padded head-dim half (D = 8)
  uint8_t *sZ = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(tslot + 4) + 1023) & ~static_cast<uintptr_t>(1023));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L;
  const int T = (L + KT - 1) / KT;
  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  const int nrows = b_hi > b_lo ? (int)(b_hi - b_lo) : 0;
  const int G = nrows * T;                             // tiles over the chunk
  // the tile order, stepped incrementally (no divisions on the issue path):
  // (row r, key tile j, first row pb and size gs of r's group; the last
  // group may be short, a.group 1 = one row at a time)
  struct TIt { int r, j, pb, gs; };
  const int GR = a.group;
  auto first_it = [&]() { return TIt{0, 0, 0, min(GR, nrows)}; };
  auto adv = [&](TIt &t) {
    if (t.r + 1 < t.pb + t.gs) {
      ++t.r;
    } else {
      t.r = t.pb;
      if (++t.j == T) {
        t.j = 0;
        t.pb += t.gs;
        t.gs = min(GR, nrows - t.pb);
        t.r = t.pb;
      }
    }
  };

  if (tid == NEW * 32) {
    for (int i = 0; i < NBAR; ++i) {
      uint64_t *bb = &bars[i];
      const bool warps = bb == &dsp[0] || bb == &dsp[1] || (bb >= dqr && bb < dqr + DQ_ACC);
      mbar_init(bb, warps ? NEW : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (D == 8) {
    for (int i = tid; i < 512; i += blockDim.x) reinterpret_cast<uint32_t *>(sZ)[i] = 0u;
    fence_proxy_async_smem();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t DQC = 320;                        // dQ accumulators
  constexpr uint32_t PARK = DQC + DQ_ACC * dacc<D>();  // parked dS sums

  if (warp == NEW) {
    auto load_tile = [&](int g, const TIt &it) {
      const int r = it.r, j = it.j;
      const int64_t b = b_lo + r;
      uint8_t *st = sStage + (g % NS) * STG;
      uint64_t *bar = &fullb[g % NS];
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
    auto load_row = [&](int r) {
      if (lane == 0) {
        uint8_t *dst = sQ + (r % NQB) * 2 * QB;
        mbar_expect_tx(&qfull[r % NQB], 2 * QB);
        tma_load_4d(dst, &mQ, &qfull[r % NQB], 0, q0, (int)(b_lo + r), h);
        tma_load_4d(dst + QB, &mdO, &qfull[r % NQB], 0, q0, (int)(b_lo + r), h);
      }
      __syncwarp();
    };
    for (int r = 0; r < NQB && r < nrows; ++r) load_row(r);
    TIt tl = first_it(), ts = first_it(), tq = first_it();   // next load, S/dP, dQ tiles
    for (int g = 0; g < NS && g < G; ++g) {
      load_tile(g, tl);
      adv(tl);
    }
    const uint32_t idesc_s = idesc_bf16(128, KT, false, false);
    const uint32_t idesc_o = idesc_bf16(128, dacc<D>(), false, true);
    for (int g = 0; g <= G; ++g) {
      if (g < G) {
        const int r = ts.r, j = ts.j;
        adv(ts);
        if (j == 0) mbar_wait(&qfull[r % NQB], (uint32_t)((r / NQB) & 1));   // row's Q / dO
        const int st = g % NS;
        mbar_wait(&fullb[st], (uint32_t)((g / NS) & 1));
        fence_after();
        const uint32_t sK = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0), sV = sK + KB;
        const uint32_t sQa = smem_u32(sQ) + (r % NQB) * 2 * QB, sdOa = sQa + QB;
        const uint32_t d = tmem + (g & 1) * 160;
#pragma unroll
        for (int ks = 0; ks < ksteps<D>(); ++ks)
          umma_bf16_el(d, desc_k<D>(sQa, ks, smem_u32(sZ) - sQa), desc_k<D>(sK, ks), idesc_s,
                       ks > 0);
#pragma unroll
        for (int ks = 0; ks < ksteps<D>(); ++ks)
          umma_bf16_el(d + 64, desc_k<D>(sdOa, ks, smem_u32(sZ) - sdOa), desc_k<D>(sV, ks),
                       idesc_s, ks > 0);
        umma_commit_el(&sdone[g & 1]);
        if (j == T - 1 && r + NQB < nrows) {
          // row r's last S/dP MMAs read Q / dO: load row r + NQB into its buffer
          mbar_wait(&sdone[g & 1], (uint32_t)((g >> 1) & 1));
          load_row(r + NQB);
        }
      }
      if (g >= 1) {
        const int i = g - 1, bi = i & 1, st = i % NS;
        const int ri = tq.r, ji = tq.j;
        adv(tq);
        mbar_wait(&dsp[bi], (uint32_t)((i >> 1) & 1));   // dS_i packed
        // row ri's accumulator was read out (row ri - DQ_ACC)
        if (ji == 0 && ri >= DQ_ACC)
          mbar_wait(&dqr[ri % DQ_ACC], (uint32_t)(((ri / DQ_ACC) - 1) & 1));
        fence_after();
        const uint32_t sK = smem_u32(sStage + st * STG) + (BIAS ? BIAS_TILE : 0);
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(tmem + DQC + dacc<D>() * (ri % DQ_ACC), tmem + bi * 160 + 128 + 8 * ks,
                          desc_mn<D>(sK, ks), idesc_o, (ji > 0 || ks > 0) ? 1u : 0u);
        umma_commit_el(&dqd[bi]);
      }
      // refill the stage of tile g - 2 (see the dk/dv kernel)
      if (g >= 2 && g - 2 + NS < G) {
        const int i2 = g - 2;
        mbar_wait(&dqd[i2 & 1], (uint32_t)((i2 >> 1) & 1));  // stage of tile g - 2 free
        load_tile(i2 + NS, tl);
        adv(tl);
      }
    }
  } else {
    const int quad = warp & 3, part = warp >> 2;
    const int t = quad * 32 + lane;
    const int q = q0 + t;
    const bool qv = q < L;
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const float sc_l2 = a.scale * LOG2E_F;
    constexpr int OD = D / TPR < 4 ? 4 : D / TPR;   // epilogue columns per thread
    float *prow = BIAS ? a.dbias_part + (int64_t)blockIdx.z * a.H * L * (int64_t)L +
                             ((int64_t)h * L + q) * L
                       : nullptr;
    // lse / Dq of this thread's query row for the pair's rows (slot 0 / 1),
    // the next pair's fetched one pair ahead
    auto fetch = [&](int r, float &l, float &d) {
      if (qv && r < nrows) {
        l = a.lse[((b_lo + r) * a.H + h) * (int64_t)L + q];
        d = a.Dq[((b_lo + r) * a.H + h) * (int64_t)L + q];
      } else {
        l = 0.f;
        d = 0.f;
      }
    };
    float lse_n[DQ_GROUP], dq_n[DQ_GROUP], lse_l2[DQ_GROUP], dq_[DQ_GROUP];
#pragma unroll
    for (int u = 0; u < DQ_GROUP; ++u) {
      fetch(u < GR ? u : nrows, lse_n[u], dq_n[u]);
      lse_l2[u] = dq_[u] = 0.f;
    }
    // the running dS sum of a group's rows parks in TMEM past the dQ
    // accumulators until the group's last row: registers would spill
    const uint32_t park = lane_addr + PARK + part * EPT;
    TIt te = first_it();
    for (int g = 0; g < G; ++g) {
      const int bi = g & 1, st = g % NS;
      const int r = te.r, j = te.j, pb = te.pb, gs = te.gs;
      adv(te);
      const int slot = r - pb;
      if (j == 0 && slot == 0) {                     // a new group: its rows' lse / Dq
#pragma unroll
        for (int u = 0; u < DQ_GROUP; ++u) {
          lse_l2[u] = lse_n[u] * LOG2E_F;
          dq_[u] = dq_n[u];
        }
        const int nx = pb + gs;                      // the next group's first row
        const int ngs = min(GR, nrows - nx);
#pragma unroll
        for (int u = 0; u < DQ_GROUP; ++u)           // (past the group: zeros)
          fetch(u < ngs ? nx + u : nrows, lse_n[u], dq_n[u]);
      }
      const int64_t b = b_lo + r;
      const int kb = j * KT + part * EPT;
      float *dst = prow + kb;
      const bool full_k = kb + EPT <= L;
      const bool vec = full_k && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
      if (BIAS) mbar_wait(&fullb[st], (uint32_t)((g / NS) & 1));  // bias tile landed
      mbar_wait(&sdone[bi], (uint32_t)((g >> 1) & 1));
      fence_after();
      uint32_t sv[EPT], dv[EPT];
      tld<EPT>(lane_addr + bi * 160 + part * EPT, sv);
      tld<EPT>(lane_addr + bi * 160 + 64 + part * EPT, dv);
      float bb[EPT];
      if (BIAS) bias_row(sStage + st * STG, t, part * EPT, bb);
      tmem_wait_ld();
      uint32_t pk[EPT / 2];
      float ds[EPT];
      // selects, not an indexed load: a runtime index would put the arrays
      // in local memory
      const float ll = slot < 2 ? (slot ? lse_l2[1] : lse_l2[0]) : (slot == 2 ? lse_l2[2] : lse_l2[3]);
      const float dqv = slot < 2 ? (slot ? dq_[1] : dq_[0]) : (slot == 2 ? dq_[2] : dq_[3]);
      if (qv && full_k) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          float x = fmaf(__uint_as_float(sv[k]), sc_l2, -ll);
          if (BIAS) x = fmaf(bb[k], LOG2E_F, x);
          ds[k] = ex2f(x) * (__uint_as_float(dv[k]) - dqv);
        }
      } else {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          float x = fmaf(__uint_as_float(sv[k]), sc_l2, -ll);
          if (BIAS) x = fmaf(bb[k], LOG2E_F, x);
          const float p = (qv && kb + k < L) ? ex2f(x) : 0.f;
          ds[k] = p * (__uint_as_float(dv[k]) - dqv);
        }
      }
#pragma unroll
      for (int k = 0; k < EPT; k += 2) pk[k >> 1] = pk2(ds[k], ds[k + 1]);
      tst<EPT / 2>(lane_addr + bi * 160 + 128 + part * (EPT / 2), pk);
      if (BIAS && qv) {
        // the chunk's dbias partial: the group's rows summed (parked in
        // TMEM), then the chunk's first group stores and later groups add
        // with fire-and-forget reductions (one owner thread per element,
        // program order per address: the sum runs over the groups in order)
        const bool emit = slot == gs - 1;            // the group's last row
        if (gs > 1) {
          uint32_t u[EPT];
          if (slot > 0) {                            // add the parked sum
            tld<EPT>(park, u);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < EPT; ++k) ds[k] += __uint_as_float(u[k]);
          }
          if (!emit) {                               // park the running sum
#pragma unroll
            for (int k = 0; k < EPT; ++k) u[k] = __float_as_uint(ds[k]);
            tst<EPT>(park, u);
          }
        }
        const bool first = pb == 0;
        if (emit && vec) {
#pragma unroll
          for (int c = 0; c < EPT / 4; ++c) {
            float *d4 = dst + 4 * c;
            if (first) {
              *reinterpret_cast<float4 *>(d4) =
                  make_float4(ds[4 * c], ds[4 * c + 1], ds[4 * c + 2], ds[4 * c + 3]);
            } else {
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d4),
                           "f"(ds[4 * c]), "f"(ds[4 * c + 1]), "f"(ds[4 * c + 2]),
                           "f"(ds[4 * c + 3])
                           : "memory");
            }
          }
        } else if (emit) {
#pragma unroll
          for (int k2 = 0; k2 < EPT; ++k2) {
            if (kb + k2 >= L) continue;
            if (first) dst[k2] = ds[k2];
            else asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + k2), "f"(ds[k2]) : "memory");
          }
        }
      }
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dsp[bi]);
      if (j == T - 1) {
        // the row's dQ: wait for its last dQ MMA, scale, store
        mbar_wait(&dqd[bi], (uint32_t)((g >> 1) & 1));
        fence_after();
        uint32_t v[OD];
        tld<OD>(lane_addr + DQC + dacc<D>() * (r % DQ_ACC) + part * OD, v);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dqr[r % DQ_ACC]);
        if (qv && part * OD < D)
          store_row_bf16<OD>(a.dq + b * a.sb + (int64_t)q * a.sl + h * D + part * OD, v, a.scale);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ======================================================================= dkv
// CTA = 128 keys x a chunk of batch rows; the queries stream in tiles of 64
// (tile g = (row r, query tile j)); K / V and the dK / dV accumulators are
// double-buffered by row parity.  TMEM: buffer g&1 at 192 (g&1): S^T (64) |
// dP^T (64) | P^T (32 pairs) | dS^T (32 pairs); dK / dV of row parity p at
// 384 + 2 D p (+ D).  lse / Dq of the thread's queries: global loads, one
// tile ahead.
template <int D, bool BIAS>
__global__ void __launch_bounds__(nth_of(TPR_DKV), 1)
attn_flash_dkv_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                      const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mdO,
                      const __grid_constant__ CUtensorMap mB, const FlashArgs a) {
  evo_pdl_enter();
  constexpr int TPR = TPR_DKV, EPT = KT / TPR, NEW = 4 * TPR;
  constexpr int NS = NS_BWD;
  constexpr uint32_t KB = QT * Sw<D>::bytes, QB = KT * Sw<D>::bytes;
  // stage: bias [64 q x 128 k] as four [64 x 32] SW128 boxes | Q | dO |
  // lse [64] | Dq [64] (fp32, by cp.async: any L)
  constexpr uint32_t BT = BIAS ? 4 * 8192 : 0;
  constexpr uint32_t STG = (BT + 2 * QB + 2 * KT * 4 + 1023) / 1024 * 1024;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sStage = smem_raw;
  uint8_t *sK = sStage + NS * STG;                     // 2 x [K | V] (row parity)
  uint64_t *bars = reinterpret_cast<uint64_t *>(sK + 4 * KB);
  uint64_t *kvfull = bars, *fullb = kvfull + 2, *sdone = fullb + NS, *pp2 = sdone + 2,
           *mmd = pp2 + 2, *accr = mmd + 2;
  constexpr int NBAR = 2 + NS + 8;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + NBAR);
  // 2 KB of zeros above every operand: the padded head-dim half (D = 8)
  uint8_t *sZ = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(tslot + 4) + 1023) & ~static_cast<uintptr_t>(1023));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L;
  const int T = (L + KT - 1) / KT;
  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  const int nrows = b_hi > b_lo ? (int)(b_hi - b_lo) : 0;
  const int G = nrows * T;

  if (tid == NEW * 32) {
    for (int i = 0; i < NBAR; ++i) {
      uint64_t *bb = &bars[i];
      const bool warps = bb == &pp2[0] || bb == &pp2[1] || bb == &accr[0] || bb == &accr[1];
      const bool stage = bb >= fullb && bb < fullb + NS;   // TMA + 32 cp.async lanes
      mbar_init(bb, warps ? NEW : (stage ? 33 : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (D == 8) {
    for (int i = tid; i < 512; i += blockDim.x) reinterpret_cast<uint32_t *>(sZ)[i] = 0u;
    fence_proxy_async_smem();
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
      uint64_t *bar = &fullb[g % NS];
      if (lane == 0) {
        mbar_expect_tx(bar, BT + 2 * QB);
        if (BIAS) {
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_3d(st + c * 8192, &mB, bar, k0 + 32 * c, j * KT, h);
        }
        tma_load_4d(st + BT, &mQ, bar, 0, j * KT, (int)b, h);
        tma_load_4d(st + BT + QB, &mdO, bar, 0, j * KT, (int)b, h);
      }
      // lse / Dq of the tile's 64 queries (zero past L)
      const int64_t rowo = (b * a.H + h) * (int64_t)L;
      float *sl = reinterpret_cast<float *>(st + BT + 2 * QB);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int qi = lane + 32 * e, q = j * KT + qi;
        const uint32_t n = q < L ? 4u : 0u;
        const float *src1 = a.lse + rowo + (q < L ? q : 0);
        const float *src2 = a.Dq + rowo + (q < L ? q : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(sl + qi)),
                     "l"(src1), "r"(n)
                     : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(sl + KT + qi)),
                     "l"(src2), "r"(n)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                   : "memory");
      __syncwarp();
    };
    auto load_kv = [&](int r) {
      if (lane == 0) {
        uint8_t *dst = sK + (r & 1) * 2 * KB;
        mbar_expect_tx(&kvfull[r & 1], 2 * KB);
        tma_load_4d(dst, &mK, &kvfull[r & 1], 0, k0, (int)(b_lo + r), h);
        tma_load_4d(dst + KB, &mV, &kvfull[r & 1], 0, k0, (int)(b_lo + r), h);
      }
      __syncwarp();
    };
    for (int r = 0; r < 2 && r < nrows; ++r) load_kv(r);
    for (int g = 0; g < NS && g < G; ++g) load_tile(g);
    const uint32_t idesc_s = idesc_bf16(128, KT, false, false);
    const uint32_t idesc_o = idesc_bf16(128, dacc<D>(), false, true);
    int r = 0, j = 0, ri = 0, ji = -1;
    for (int g = 0; g <= G; ++g) {
      if (g < G) {
        if (j == 0) mbar_wait(&kvfull[r & 1], (uint32_t)((r >> 1) & 1));
        const int st = g % NS;
        mbar_wait(&fullb[st], (uint32_t)((g / NS) & 1));
        fence_after();
        const uint32_t sQ = smem_u32(sStage + st * STG) + BT, sdO = sQ + QB;
        const uint32_t sKa = smem_u32(sK) + (r & 1) * 2 * KB, sVa = sKa + KB;
        const uint32_t d = tmem + (g & 1) * 192;
#pragma unroll
        for (int ks = 0; ks < ksteps<D>(); ++ks)
          umma_bf16_el(d, desc_k<D>(sKa, ks, smem_u32(sZ) - sKa), desc_k<D>(sQ, ks), idesc_s,
                       ks > 0);
#pragma unroll
        for (int ks = 0; ks < ksteps<D>(); ++ks)
          umma_bf16_el(d + 64, desc_k<D>(sVa, ks, smem_u32(sZ) - sVa), desc_k<D>(sdO, ks),
                       idesc_s, ks > 0);
        umma_commit_el(&sdone[g & 1]);
        if (j == T - 1 && r + 2 < nrows) {
          mbar_wait(&sdone[g & 1], (uint32_t)((g >> 1) & 1));   // row r's K / V read
          load_kv(r + 2);
        }
      }
      if (g >= 1) {
        const int i = g - 1, bi = i & 1, st = i % NS;
        mbar_wait(&pp2[bi], (uint32_t)((i >> 1) & 1));   // P^T / dS^T packed
        if (ji == 0 && ri >= 2) mbar_wait(&accr[ri & 1], (uint32_t)(((ri >> 1) - 1) & 1));
        fence_after();
        const uint32_t sQ = smem_u32(sStage + st * STG) + BT, sdO = sQ + QB;
        const uint32_t base = tmem + bi * 192;
        const uint32_t acc = tmem + 384 + 2 * dacc<D>() * (ri & 1);
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(acc + dacc<D>(), base + 128 + 8 * ks, desc_mn<D>(sdO, ks), idesc_o,
                          (ji > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < KT / 16; ++ks)
          umma_bf16_ts_el(acc, base + 160 + 8 * ks, desc_mn<D>(sQ, ks), idesc_o,
                          (ji > 0 || ks > 0) ? 1u : 0u);
        umma_commit_el(&mmd[bi]);
      }
      // refill the stage of tile g - 2 (its dV/dK MMAs were issued an
      // iteration ago: by now they are usually done, so this wait no longer
      // sits between the tile's dV/dK MMAs and the next S MMA)
      if (g >= 2 && g - 2 + NS < G) {
        const int i2 = g - 2;
        mbar_wait(&mmd[i2 & 1], (uint32_t)((i2 >> 1) & 1));
        load_tile(i2 + NS);
      }
      ri = r;
      ji = j;
      if (++j == T) {
        j = 0;
        ++r;
      }
    }
  } else {
    const int quad = warp & 3, part = warp >> 2;
    const int t = quad * 32 + lane;                    // key row of the tile
    const int k = k0 + t;
    const bool kv = k < L;
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    const float sc_l2 = a.scale * LOG2E_F;
    constexpr int OD = D / TPR < 4 ? 4 : D / TPR;   // epilogue columns per thread
    // transposed bias reads: element (q, kk = t & 31) of a [64 q x 32 k]
    // SW128 box sits at q*128 + ((kk/4 ^ q%8) << 4) + (kk%4)*4; q % 8 is the
    // compile-time qq % 8 (part*EPT is a multiple of 8)
    uint32_t boff[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) boff[e] = ((((t & 31) >> 2) ^ e) << 4) + (t & 3) * 4;
    int r = 0, j = 0;
    for (int g = 0; g < G; ++g) {
      const int bi = g & 1, st = g % NS;
      const int qb = j * KT + part * EPT;        // first query of this thread's EPT
      mbar_wait(&fullb[st], (uint32_t)((g / NS) & 1));   // bias, lse, Dq landed
      mbar_wait(&sdone[bi], (uint32_t)((g >> 1) & 1));
      fence_after();
      uint32_t sv[EPT], dv[EPT];
      tld<EPT>(lane_addr + bi * 192 + part * EPT, sv);
      tld<EPT>(lane_addr + bi * 192 + 64 + part * EPT, dv);
      const uint8_t *stg = sStage + st * STG;
      const float *sl = reinterpret_cast<const float *>(stg + BT + 2 * QB) + part * EPT;
      const float *sd = sl + KT;
      const uint8_t *bx = stg + (t >> 5) * 8192 + part * EPT * 128;
      float lq[EPT], dq[EPT], bq[EPT];
#pragma unroll
      for (int c = 0; c < EPT; c += 4) {
        const float4 l4 = *reinterpret_cast<const float4 *>(sl + c);
        const float4 d4 = *reinterpret_cast<const float4 *>(sd + c);
        lq[c] = l4.x; lq[c + 1] = l4.y; lq[c + 2] = l4.z; lq[c + 3] = l4.w;  // log2 units
        dq[c] = d4.x; dq[c + 1] = d4.y; dq[c + 2] = d4.z; dq[c + 3] = d4.w;
      }
      if (BIAS) {
#pragma unroll
        for (int qq = 0; qq < EPT; ++qq)
          bq[qq] = *reinterpret_cast<const float *>(bx + qq * 128 + boff[qq & 7]);
      }
      tmem_wait_ld();
      uint32_t pp[EPT / 2], pd[EPT / 2];
      const bool full = kv && qb + EPT <= L;
      if (full) {  // interior tiles: no per-element mask
#pragma unroll
        for (int c = 0; c < EPT; c += 2) {
          float p[2], ds[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int qq = c + e;
            float x = fmaf(__uint_as_float(sv[qq]), sc_l2, -lq[qq]);
            if (BIAS) x = fmaf(bq[qq], LOG2E_F, x);
            p[e] = ex2f(x);
            ds[e] = p[e] * (__uint_as_float(dv[qq]) - dq[qq]);
          }
          pp[c >> 1] = pk2(p[0], p[1]);
          pd[c >> 1] = pk2(ds[0], ds[1]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < EPT; c += 2) {
          float p[2], ds[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int qq = c + e;
            float x = fmaf(__uint_as_float(sv[qq]), sc_l2, -lq[qq]);
            if (BIAS) x = fmaf(bq[qq], LOG2E_F, x);
            p[e] = (kv && qb + qq < L) ? ex2f(x) : 0.f;
            ds[e] = p[e] * (__uint_as_float(dv[qq]) - dq[qq]);
          }
          pp[c >> 1] = pk2(p[0], p[1]);
          pd[c >> 1] = pk2(ds[0], ds[1]);
        }
      }
      tst<EPT / 2>(lane_addr + bi * 192 + 128 + part * (EPT / 2), pp);
      tst<EPT / 2>(lane_addr + bi * 192 + 160 + part * (EPT / 2), pd);
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pp2[bi]);
      if (j == T - 1) {
        // dK = scale * acc, dV = acc of row r
        mbar_wait(&mmd[bi], (uint32_t)((g >> 1) & 1));
        fence_after();
        const uint32_t acc = lane_addr + 384 + 2 * dacc<D>() * (r & 1);
        uint32_t vk[OD], vv[OD];
        tld<OD>(acc + part * OD, vk);
        tld<OD>(acc + dacc<D>() + part * OD, vv);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&accr[r & 1]);
        if (kv && part * OD < D) {
          const int64_t off = (b_lo + r) * a.sb + (int64_t)k * a.sl + h * D + part * OD;
          store_row_bf16<OD>(a.dk + off, vk, a.scale);
          store_row_bf16<OD>(a.dv + off, vv, 1.f);
        }
      }
      if (++j == T) {
        j = 0;
        ++r;
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
  CUtensorMapSwizzle sw = D == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : (D == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE);
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

// EVO_FLASH_DQ_GROUP=1/2/4 forces the dq kernel's rows per group (default 4:
// with a bias a quarter of the dbias reductions; without one, measured
// 1.53 -> 1.41 ms at 1024 keys, D = 8, too)
static const int g_dq_group = [] {
  const char *e = getenv("EVO_FLASH_DQ_GROUP");
  const int v = e ? atoi(e) : 0;
  return (v == 1 || v == 2 || v == 4) ? v : 0;
}();

FlashArgs flash_args(const evo_attn_desc *d) {
  FlashArgs a;
  a.nb = d->nb; a.H = d->H; a.L = d->L; a.D = d->D; a.scale = d->scale;
  a.g = reinterpret_cast<const bf16 *>(d->g);
  a.sb = d->sb; a.sl = d->sl;
  a.o = reinterpret_cast<bf16 *>(d->o); a.gm = reinterpret_cast<bf16 *>(d->gm);
  a.o_sb = d->o_sb; a.o_sl = d->o_sl;
  a.lse = d->lse;
  a.Dq = nullptr;
  a.dq = reinterpret_cast<bf16 *>(d->dq); a.dk = reinterpret_cast<bf16 *>(d->dk);
  a.dv = reinterpret_cast<bf16 *>(d->dv);
  a.dbias_part = nullptr; a.chunk = 1;
  a.group = 1;
  return a;
}

bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_flash(const evo_attn_desc *d, bool bwd) {
  EVO_REQUIRE(d && d->dtype == EVO_BF16 && (d->D == 8 || d->D == 16 || d->D == 32) && d->L >= 1 &&
                  d->nb >= 1 && d->nb <= 65535 && d->H >= 1 && d->H <= 65535,
              EVO_EUNSUP, "attention_flash: bf16, head dim 8 / 16 / 32, nb <= 65535 (D=%d L=%d nb=%lld)",
              d ? d->D : -1, d ? d->L : -1, d ? (long long)d->nb : -1ll);
  EVO_REQUIRE(d->sb % 8 == 0 && d->sl % 8 == 0 && d->o_sb % 8 == 0 && d->o_sl % 8 == 0 &&
                  al16(d->q) && al16(d->k) && al16(d->v) && al16(d->g) && al16(d->o),
              EVO_EUNSUP, "attention_flash: 16-byte aligned rows required");
  EVO_REQUIRE(!d->bias || (d->bk == 1 && d->bq % 4 == 0 && d->bh % 4 == 0 &&
                           d->bh >= (int64_t)d->L * d->bq && al16(d->bias)),
              EVO_EUNSUP, "attention_flash: plain bias rows (bk = 1, bq %% 4 == 0) required");
  if (bwd)
    EVO_REQUIRE(al16(d->dq) && al16(d->dk) && al16(d->dv) && al16(d->dgm), EVO_EUNSUP,
                "attention_flash: 16-byte aligned gradient rows required");
  return EVO_OK;
}

// batch rows per persistent CTA: `per_sm` CTAs per SM over (tiles x heads x
// chunks)
int64_t flash_chunk(const evo_attn_desc *d, int per_sm, int64_t &nch) {
  const int64_t qt = (d->L + QT - 1) / QT;
  nch = std::max<int64_t>(1, std::min<int64_t>(d->nb, (int64_t)per_sm * num_sms() /
                                                          std::max<int64_t>(1, qt * d->H)));
  const int64_t chunk = (d->nb + nch - 1) / nch;
  nch = (d->nb + chunk - 1) / chunk;
  return chunk;
}

struct FlashWs {
  size_t dO, Dq, lse2, gate, part, total;
};
FlashWs flash_ws(const evo_attn_desc *d) {
  FlashWs w;
  auto pad = [](size_t x) { return (x + 255) / 256 * 256; };
  const int64_t span = (d->nb - 1) * d->o_sb + (int64_t)(d->L - 1) * d->o_sl + (int64_t)d->H * d->D;
  w.dO = 0;
  w.Dq = pad((size_t)span * 2);
  w.lse2 = w.Dq + pad((size_t)d->nb * d->H * d->L * 4);   // lse in log2 units (dk/dv)
  w.gate = w.lse2 + pad((size_t)d->nb * d->H * d->L * 4);
  w.part = w.gate + pad((size_t)num_sms() * 8 * d->H * d->D * 4);
  int64_t nch;
  flash_chunk(d, 1, nch);
  w.total = w.part + (d->bias ? pad((size_t)nch * d->H * d->L * d->L * 4) : 0);
  return w;
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
  const size_t smem = ns_fwd<BIAS>() * STG + 2 * QT * 2 * D + (3 * TPR_FWD * 128) * 4 +
                      (2 + ns_fwd<BIAS>() + 8) * 8 + 16 + 1024 + 2048;
  auto kfn = attn_flash_fwd_kernel<D, BIAS>;
  EVO_MAX_SMEM_ONCE(kfn);
  // one batch row per CTA (measured faster than persistent chunks: the
  // softmax warps' per-row epilogue would serialise with the next row)
  const int64_t nch = d->nb;
  a.chunk = 1;
  dim3 grid((d->L + QT - 1) / QT, d->H, (unsigned)nch);
  launch_k(kfn, grid, nth_of(TPR_FWD), smem, st, mq, mk, mv, mb, a);
  EVO_LAUNCHED("attn_flash_fwd_kernel");
  return EVO_OK;
}

template <int D, bool BIAS>
int flash_bwd(const evo_attn_desc *d, cudaStream_t st) {
  FlashArgs a = flash_args(d);
  const FlashWs w = flash_ws(d);
  EVO_REQUIRE(d->workspace && d->workspace_bytes >= w.total, EVO_EARG,
              "attention_flash bwd: workspace needs %zu bytes", w.total);
  uint8_t *ws = reinterpret_cast<uint8_t *>(d->workspace);
  bf16 *dO = reinterpret_cast<bf16 *>(ws + w.dO);
  float *Dq = reinterpret_cast<float *>(ws + w.Dq);
  float *lse2 = reinterpret_cast<float *>(ws + w.lse2);
  int rc = attn_prep_run(d, dO, Dq, reinterpret_cast<float *>(ws + w.gate), lse2, st);
  if (rc != EVO_OK) return rc;
  int64_t nch;
  a.chunk = flash_chunk(d, 1, nch);
  a.Dq = Dq;
  a.dbias_part = BIAS ? reinterpret_cast<float *>(ws + w.part) : nullptr;
  a.group = g_dq_group ? g_dq_group : DQ_GROUP;
  CUtensorMap mq, mk, mv, mdo, mb, mq2, mdo2, mk2, mv2, mb2;
  // dq kernel: Q / dO tiles of 128 queries, K / V tiles of 64 keys
  if (!flash_head_map(&mq, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !flash_head_map(&mdo, dO, D, d->L, d->nb, d->H, d->o_sl, d->o_sb, QT) ||
      !flash_head_map(&mk, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, KT) ||
      !flash_head_map(&mv, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, KT))
    return EVO_EUNSUP;
  // dkv kernel: K / V tiles of 128 keys, Q / dO tiles of 64 queries
  if (!flash_head_map(&mk2, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !flash_head_map(&mv2, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !flash_head_map(&mq2, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, KT) ||
      !flash_head_map(&mdo2, dO, D, d->L, d->nb, d->H, d->o_sl, d->o_sb, KT))
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
    // (the 2 KiB zero block and its alignment only for D = 8)
    const size_t smem = NS_BWD * STG + DQ_QBUF * 2 * QT * 2 * D +
                        (DQ_QBUF + NS_BWD + 6 + DQ_ACC) * 8 + 16 + (D == 8 ? 1024 + 2048 : 0);
    auto kfn = attn_flash_dq_kernel<D, BIAS>;
    EVO_MAX_SMEM_ONCE(kfn);
    dim3 grid((d->L + QT - 1) / QT, d->H, (unsigned)nch);
    launch_k(kfn, grid, nth_of(TPR_DQ), smem, st, mq, mk, mv, mdo, mb, a);
    EVO_LAUNCHED("attn_flash_dq_kernel");
  }
  {
    constexpr uint32_t BT = BIAS ? 4 * 8192 : 0;
    constexpr uint32_t STG = (BT + 2 * KT * 2 * D + 2 * KT * 4 + 1023) / 1024 * 1024;
    const size_t smem = NS_BWD * STG + 4 * QT * 2 * D + (2 + NS_BWD + 8) * 8 + 16 + 1024 + 2048;
    auto kfn = attn_flash_dkv_kernel<D, BIAS>;
    EVO_MAX_SMEM_ONCE(kfn);
    dim3 grid((d->L + QT - 1) / QT, d->H, (unsigned)nch);
    FlashArgs a2 = a;
    a2.lse = lse2;      // staged as log2 units: no per-logit rescale in the dk/dv pass
    launch_k(kfn, grid, nth_of(TPR_DKV), smem, st, mq2, mk2, mv2, mdo2, mb2, a2);
    EVO_LAUNCHED("attn_flash_dkv_kernel");
  }
  if (BIAS) {
    // dbias = sum of the chunk partials in chunk order, into the plain layout
    return reduce_lead(EVO_F32, nch, (int64_t)d->H * d->L, d->L, a.dbias_part, d->dbias,
                       d->bq, 1, 0, st);
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
  if (d->D == 16) return d->bias ? flash_fwd<16, true>(d, st) : flash_fwd<16, false>(d, st);
  return d->bias ? flash_fwd<8, true>(d, st) : flash_fwd<8, false>(d, st);
}

EVO_API size_t evo_attn_flash_bwd_workspace_bytes(const evo_attn_desc *d) {
  if (check_flash(d, false) != EVO_OK) return 0;
  return flash_ws(d).total;
}

EVO_API int evo_attn_flash_bwd(const evo_attn_desc *d, void *stream) {
  int rc = check_flash(d, true);
  if (rc != EVO_OK) return rc;
  EVO_REQUIRE(!d->bias || d->dbias, EVO_EARG, "attn_flash_bwd: bias needs dbias");
  cudaStream_t st = as_stream(stream);
  note_backend(EVO_BK_ATTN_FLASH);
  if (d->D == 32) return d->bias ? flash_bwd<32, true>(d, st) : flash_bwd<32, false>(d, st);
  if (d->D == 16) return d->bias ? flash_bwd<16, true>(d, st) : flash_bwd<16, false>(d, st);
  return d->bias ? flash_bwd<8, true>(d, st) : flash_bwd<8, false>(d, st);
}

}  // extern "C"
