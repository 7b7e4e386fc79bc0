// Fused gated attention with pair bias on 5th-gen tensor cores (sm_100a).
//
// Same contract as attention_simt.cu (src/evoformer.py:268-286): per
// (batch row b, head h) Q,K,V [L, D] live in the packed projection buffer,
// O = softmax(scale*QK^T + bias[h]) V, GM = G*O, lse saved.  L <= 256 keys
// are resident, so the softmax is exact (one pass over TMEM for the max,
// one for exp/sum); logits never leave the SM.
//
// Forward (grid: q-tiles x H x nb, 128 threads, thread t owns query row t):
//   TMA: Q tile [128 x D], K, V [Lp x D] (swizzle = 2D bytes)
//   tcgen05.mma  S = Q K^T        -> TMEM [128 x Lp] fp32
//   softmax rows in registers (bias added from L2), P (bf16) -> smem
//   tcgen05.mma  O = P V          -> TMEM [128 x D]  (V as MN-major B)
//   epilogue: O/sum, gate, store o, gm, lse
// Backward (deterministic, no atomics):
//   prep:  dO = dGM*G, dGpre = dGM*O*G*(1-G), Dq = rowsum(dO*O)
//   dq kernel (grid q-tiles x H x chunks; loops the chunk's batch rows):
//     S = QK^T, P = exp(S + bias - lse) -> smem;  dP = dO V^T;
//     dS = P*(dP - Dq) -> smem; dbias partial += dS (TMEM accumulator);
//     dq = scale * dS K
//   dkv kernel (grid k-tiles x H x nb): S^T = K Q^T, dP^T = V dO^T,
//     P^T, dS^T -> smem; dv = P^T dO; dk = scale * dS^T Q
//   dbias = ordered sum of the chunk partials.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace evo {

int colsum_partials(int nblk, int64_t cols, const float *part, float *dst, int acc,
                    cudaStream_t st);
int reduce_lead(int, int64_t, int64_t, int64_t, const void *, float *, int64_t, int64_t, int,
                cudaStream_t);

namespace {
using namespace tc;

constexpr float LOG2E = 1.4426950408889634f;
constexpr int QT = 128;      // query (or key) rows per CTA = UMMA M
constexpr int PBYTES = 128 * 256 * 2;  // P / dS staging, [128 x 256] bf16 SW128

struct AttnTcArgs {
  int64_t nb;
  int H, L, Lp, D;
  float scale;
  const bf16 *g;
  int64_t sb, sl;
  bf16 *o, *gm;
  int64_t o_sb, o_sl;
  const float *bias;
  int64_t bh, bq, bk;
  float *lse;
  // backward
  const bf16 *dO;   // prep output, o's strides
  const float *Dq;  // [nb, H, L]
  bf16 *dq, *dk, *dv;  // proj-gradient buffer (q's strides)
  float *dbias_part;
  int64_t chunk;
};


__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Load D consecutive fp32 TMEM columns of this thread's lane into out[].
template <int D>
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&out)[D]) {
  if constexpr (D == 16) {
    uint32_t v[16];
    tmem_ld16(taddr, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = __uint_as_float(v[j]);
  } else {
#pragma unroll
    for (int c = 0; c < D; c += 32) {
      uint32_t v[32];
      tmem_ld32(taddr + c, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) out[c + j] = __uint_as_float(v[j]);
    }
  }
}

// swizzle code / atom for a [rows x D] bf16 tile with 2D-byte rows
template <int D> struct Sw {
  static constexpr uint32_t bytes = 2 * D;                      // row pitch
  static constexpr uint32_t layout = D == 64 ? 2 : (D == 32 ? 4 : 6);
  static constexpr uint32_t sbo = 8 * bytes;                    // 8-row group
};

// K-major descriptor of a [rows x D] tile, K slice ks (16 wide).
template <int D>
__device__ __forceinline__ uint64_t desc_kmajor_tile(uint32_t base, int ks) {
  return umma_desc(base + ks * 32, 16, Sw<D>::sbo, Sw<D>::layout);
}
// MN-major descriptor of a [keys x D] tile used as B(n=d, k=key); K slice ks.
template <int D>
__device__ __forceinline__ uint64_t desc_mnmajor_tile(uint32_t base, int ks) {
  // N = D is exactly one swizzle-atom wide, so LBO (MN-chunk stride) is unused
  return umma_desc(base + ks * 16 * Sw<D>::bytes, 16, Sw<D>::sbo, Sw<D>::layout);
}
// K-major SW128 descriptor of the [128 x 256] P/dS staging buffer, K slice ks.
__device__ __forceinline__ uint64_t desc_pbuf(uint32_t base, int ks) {
  return umma_desc(base + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024, 2);
}
// Write 8 bf16 (one 16-byte chunk: keys k8*8 .. k8*8+7) of row `row` into
// the swizzled P buffer.
__device__ __forceinline__ void pbuf_store8(uint8_t *pbuf, int row, int k8, uint4 val) {
  const int atom = k8 >> 3, chunk = k8 & 7;
  uint8_t *dst = pbuf + atom * 16384 + row * 128 + ((chunk ^ (row & 7)) << 4);
  *reinterpret_cast<uint4 *>(dst) = val;
}
__device__ __forceinline__ uint4 pbuf_load8(const uint8_t *pbuf, int row, int k8) {
  const int atom = k8 >> 3, chunk = k8 & 7;
  return *reinterpret_cast<const uint4 *>(pbuf + atom * 16384 + row * 128 +
                                          ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float2 unpack2(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162 *>(&u);
  return __bfloat1622float2(h);
}

__device__ __forceinline__ float bias_at(const AttnTcArgs &a, int h, int q, int k) {
  return a.bias[(int64_t)h * a.bh + (int64_t)q * a.bq + (int64_t)k * a.bk];
}

// ====================================================================== fwd
// Pair-bias tile of one (head, 128-query tile) for all Lp keys, fp32,
// resident in smem for the CTA's whole batch-row chunk:
//   plain  (bk == 1): Lp/32 TMA boxes [128 q x 32 k], 128B-swizzled rows
//   trans. (bq == 1): Lp/32 TMA boxes [32 k x 128 q] (q contiguous)
constexpr uint32_t BIAS_BYTES = 128 * 256 * 4;
// A/B switch for the pipelined backward kernels (EVO_ATTN_NO_PIPE=1 in the
// environment selects the previous one-row-at-a-time kernels)
static const bool g_attn_no_pipe = [] {
  const char *e = getenv("EVO_ATTN_NO_PIPE");
  return e && e[0] == '1';
}();
// elementwise warps of the pipelined dq kernel (EVO_DQ_EWW=16: the previous
// 8-keys-per-thread layout; default 8 warps, 16 keys per thread per unit)
static const int g_dq_eww = [] {
  const char *e = getenv("EVO_DQ_EWW");
  return e && atoi(e) == 16 ? 16 : 8;
}();

template <bool TBIAS>
__device__ __forceinline__ float bias_smem(const uint8_t *sb, int row, int k) {
  if constexpr (TBIAS) {
    return reinterpret_cast<const float *>(sb)[k * 128 + row];
  } else {
    const int box = k >> 5, kk = k & 31, chunk = kk >> 2;
    const float *p = reinterpret_cast<const float *>(
        sb + box * 16384 + row * 128 + ((chunk ^ (row & 7)) << 4));
    return p[kk & 3];
  }
}
// 32 consecutive keys [k0, k0+32) of one row (k0 % 32 == 0)
template <bool TBIAS>
__device__ __forceinline__ void bias_row32(const uint8_t *sb, int row, int k0, float (&out)[32]) {
  if constexpr (TBIAS) {
    const float *p = reinterpret_cast<const float *>(sb) + k0 * 128 + row;
#pragma unroll
    for (int j = 0; j < 32; ++j) out[j] = p[j * 128];
  } else {
    const uint8_t *base = sb + (k0 >> 5) * 16384 + row * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float4 v = *reinterpret_cast<const float4 *>(base + ((c ^ (row & 7)) << 4));
      out[4 * c] = v.x; out[4 * c + 1] = v.y; out[4 * c + 2] = v.z; out[4 * c + 3] = v.w;
    }
  }
}

// Load the bias tile (h, q0 .. q0+127, all keys) with TMA.
template <bool TBIAS>
__device__ __forceinline__ void load_bias_tile(uint8_t *sb, const CUtensorMap *map, uint64_t *bar,
                                               int h, int q0, int Lp) {
  const int nbox = (Lp + 31) / 32;
  mbar_expect_tx(bar, (uint32_t)nbox * 16384u);
  for (int j = 0; j < nbox; ++j) {
    if constexpr (TBIAS)
      tma_load_3d(sb + j * 16384, map, bar, q0, 32 * j, h);
    else
      tma_load_3d(sb + j * 16384, map, bar, 32 * j, q0, h);
  }
}

// Two warpgroups ping-pong over the batch rows of the CTA's chunk; WG w
// owns TMEM columns [256w, 256w+256): S (fp32) -> P (bf16 pairs, in place,
// cols [0, Lp/2)) -> O (cols [128, 128+D)).
template <int D, int BIASMODE>  // 0 none, 1 plain, 2 transposed
__global__ void __launch_bounds__(256)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                   const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mB,
                   const AttnTcArgs a) {
  evo_pdl_enter();
  constexpr uint32_t TILE = QT * Sw<D>::bytes;
  constexpr uint32_t FULL = 256 * Sw<D>::bytes;
  constexpr uint32_t WGB = TILE + 2 * FULL;  // per-warpgroup Q | K | V
  constexpr bool TB = BIASMODE == 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                            ~uintptr_t(1023));
  uint8_t *sBias = sm;
  uint8_t *sWG = sBias + (BIASMODE ? BIAS_BYTES : 0);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sWG + 2 * WGB);  // 0 bias, 1-2 qk, 3-4 mma, 5-6 v
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 7);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int w = tid >> 7, t = tid & 127;
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L, Lp = a.Lp;
  const int q = q0 + t;
  const bool qv = q < L;
  uint8_t *sQ = sWG + w * WGB;
  uint8_t *sK = sQ + TILE;
  uint8_t *sV = sK + FULL;
  uint64_t *tbar = &bars[1 + w];
  uint64_t *mbar = &bars[3 + w];

  if (tid == 0) {
    for (int i = 0; i < 7; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (BIASMODE) load_bias_tile<TB>(sBias, &mB, &bars[0], h, q0, Lp);
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tslot + 256u * w;                       // lane 0, WG columns
  const uint32_t lane_addr = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  if (BIASMODE) mbar_wait(&bars[0], 0);

  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  uint32_t ph_qk = 0, ph_v = 0, ph_m = 0;
  const uint32_t idesc_s = idesc_bf16(128, Lp, false, false);
  const uint32_t idesc_o = idesc_bf16(128, D, false, true);
  const uint32_t kv_bytes = (uint32_t)Lp * Sw<D>::bytes;
  uint64_t *qkbar = tbar, *vbar = &bars[5 + w];
  // prologue: loads for the WG's first row
  if (t == 0 && b_lo + w < b_hi) {
    const int b0 = (int)(b_lo + w);
    mbar_expect_tx(qkbar, TILE + kv_bytes);
    tma_load_4d(sQ, &mQ, qkbar, 0, q0, b0, h);
    tma_load_4d(sK, &mK, qkbar, 0, 0, b0, h);
    mbar_expect_tx(vbar, kv_bytes);
    tma_load_4d(sV, &mV, vbar, 0, 0, b0, h);
  }
  for (int64_t b = b_lo + w; b < b_hi; b += 2) {
    const bool has_next = b + 2 < b_hi;
    if (t == 0) {
      mbar_wait(qkbar, ph_qk);
      fence_after();
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        umma_bf16(tbase, desc_kmajor_tile<D>(smem_u32(sQ), ks),
                  desc_kmajor_tile<D>(smem_u32(sK), ks), idesc_s, ks > 0);
      umma_commit(mbar);
    }
    ph_qk ^= 1;
    // gate row prefetch (consumed in the epilogue)
    uint4 graw[D / 8];
    if (qv) {
      const bf16 *gp = a.g + b * a.sb + (int64_t)q * a.sl + h * D;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) graw[i] = *reinterpret_cast<const uint4 *>(gp + 8 * i);
    }
    mbar_wait(mbar, ph_m);
    ph_m ^= 1;
    fence_after();
    if (t == 0 && has_next) {  // Q, K consumed by the S MMA: prefetch the next row's
      mbar_expect_tx(qkbar, TILE + kv_bytes);
      tma_load_4d(sQ, &mQ, qkbar, 0, q0, (int)(b + 2), h);
      tma_load_4d(sK, &mK, qkbar, 0, 0, (int)(b + 2), h);
    }
    // pass 1: s = scale*acc + bias (masked keys -> -inf), row max, write back
    float mx = -INFINITY;
    for (int c0 = 0; c0 < Lp; c0 += 64) {
      uint32_t v[2][32];
      tmem_ld32_nw(lane_addr + c0, v[0]);
      tmem_ld32_nw(lane_addr + c0 + 32, v[1]);
      tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        float bb[32];
        if (BIASMODE) bias_row32<TB>(sBias, t, c0 + 32 * u, bb);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float s = __uint_as_float(v[u][j]) * a.scale;
          if (BIASMODE) s += bb[j];
          s = (c0 + 32 * u + j < L) ? s : -INFINITY;
          mx = fmaxf(mx, s);
          v[u][j] = __float_as_uint(s);
        }
        tmem_st32(lane_addr + c0 + 32 * u, v[u]);
      }
    }
    tmem_st_wait();
    // pass 2: p = exp(s - max) -> bf16 pairs in place (cols c0/2 ..), row sum
    float sum = 0.f;
    const float mxl = mx * LOG2E;
    for (int c0 = 0; c0 < Lp; c0 += 64) {
      uint32_t v[2][32];
      tmem_ld32_nw(lane_addr + c0, v[0]);
      tmem_ld32_nw(lane_addr + c0 + 32, v[1]);
      tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float p0 = ex2(__uint_as_float(v[u][2 * j]) * LOG2E - mxl);
          float p1 = ex2(__uint_as_float(v[u][2 * j + 1]) * LOG2E - mxl);
          sum += p0 + p1;
          pk[j] = pack2(p0, p1);
        }
        tmem_st16(lane_addr + ((c0 + 32 * u) >> 1), pk);
      }
    }
    tmem_st_wait();
    fence_before();
    named_bar_sync(1 + w, 128);
    if (t == 0) {
      mbar_wait(vbar, ph_v);
      fence_after();
      for (int ks = 0; ks < Lp / 16; ++ks)
        umma_bf16_ts(tbase + 128, tbase + ks * 8, desc_mnmajor_tile<D>(smem_u32(sV), ks),
                     idesc_o, ks > 0);
      umma_commit(mbar);
    }
    ph_v ^= 1;
    mbar_wait(mbar, ph_m);
    ph_m ^= 1;
    fence_after();
    if (t == 0 && has_next) {  // V consumed: prefetch the next row's
      mbar_expect_tx(vbar, kv_bytes);
      tma_load_4d(sV, &mV, vbar, 0, 0, (int)(b + 2), h);
    }
    float o[D];
    tmem_ld_row<D>(lane_addr + 128, o);
    if (qv) {
      const float inv = 1.f / sum;
      const int64_t ooff = b * a.o_sb + (int64_t)q * a.o_sl + h * D;
#pragma unroll
      for (int d8 = 0; d8 < D; d8 += 8) {
        const uint32_t *gw = reinterpret_cast<const uint32_t *>(&graw[d8 / 8]);
        uint32_t ov[4], gv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float o0 = o[d8 + 2 * j] * inv, o1 = o[d8 + 2 * j + 1] * inv;
          float2 g2 = unpack2(gw[j]);
          ov[j] = pack2(o0, o1);
          gv[j] = pack2(g2.x * o0, g2.y * o1);
        }
        *reinterpret_cast<uint4 *>(a.o + ooff + d8) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
        *reinterpret_cast<uint4 *>(a.gm + ooff + d8) = make_uint4(gv[0], gv[1], gv[2], gv[3]);
      }
      a.lse[(b * a.H + h) * (int64_t)L + q] = mx + logf(sum);
    }
    fence_before();
    named_bar_sync(1 + w, 128);  // TMEM of this WG free for the next row
    fence_after();
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(*tslot, 512);
}

// ===================================================================== prep
// dO = dGM*G (bf16, o's layout), dGpre = dGM*O*G*(1-G) (proj gate cols),
// Dq[b,h,q] = sum_d dO*O.  One thread per 8-column chunk of a (row, head)
// (consecutive lanes read consecutive 16-byte chunks); the D/8 chunk
// threads of a head reduce Dq with shuffles.
// gpart (may be NULL; needs 256 % (H*CH) == 0 so a thread's column group is
// fixed across the grid stride): per-block column sums of dGpre,
// [gridDim.x][H*D], reduced over blocks afterwards (fixed order).
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_prep_kernel(const AttnTcArgs a, const bf16 *dgm,
                                                            bf16 *dO_out, bf16 *dgpre, float *Dq,
                                                            float *gpart, float *lse2) {
  evo_pdl_enter();
  constexpr int CH = D / 8;  // chunks per head (1, 2 or 4)
  // 32-bit index math (the host checks total < 2^31): the per-element
  // 64-bit divisions by H and L were the kernel's issue bottleneck
  const uint32_t HC = (uint32_t)a.H * CH, L = (uint32_t)a.L;
  const uint32_t total = (uint32_t)(a.nb * (int64_t)a.L) * HC;
  const int lane = threadIdx.x & 31;
  float gacc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  // warp-uniform trip count (the shuffles below need every lane)
  for (uint32_t e0 = blockIdx.x * blockDim.x + (threadIdx.x - lane); e0 < total;
       e0 += gridDim.x * blockDim.x) {
    const uint32_t e = e0 + lane;
    const bool ok = e < total;
    const uint32_t r = e / HC, hc = e - r * HC;
    const int c = (int)(hc % CH);
    const int h = (int)(hc / CH);
    const uint32_t b32 = r / L;
    const int l = (int)(r - b32 * L);
    const int64_t b = b32;
    const int64_t ooff = b * a.o_sb + (int64_t)l * a.o_sl + h * D + 8 * c;
    const int64_t goff = b * a.sb + (int64_t)l * a.sl + h * D + 8 * c;
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
    const uint4 graw = ok ? __ldg(reinterpret_cast<const uint4 *>(a.g + goff)) : z4;
    const uint4 oraw = ok ? __ldg(reinterpret_cast<const uint4 *>(a.o + ooff)) : z4;
    const uint4 draw = ok ? __ldg(reinterpret_cast<const uint4 *>(dgm + ooff)) : z4;
    const uint32_t *gw = reinterpret_cast<const uint32_t *>(&graw);
    const uint32_t *ow = reinterpret_cast<const uint32_t *>(&oraw);
    const uint32_t *dw = reinterpret_cast<const uint32_t *>(&draw);
    uint32_t dov[4], dgv[4];
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 g2 = unpack2(gw[j]), o2 = unpack2(ow[j]), d2 = unpack2(dw[j]);
      float do0 = d2.x * g2.x, do1 = d2.y * g2.y;
      acc += do0 * o2.x + do1 * o2.y;
      dov[j] = pack2(do0, do1);
      dgv[j] = pack2(d2.x * o2.x * g2.x * (1.f - g2.x), d2.y * o2.y * g2.y * (1.f - g2.y));
    }
    if (ok) {
      *reinterpret_cast<uint4 *>(dO_out + ooff) = make_uint4(dov[0], dov[1], dov[2], dov[3]);
      *reinterpret_cast<uint4 *>(dgpre + goff) = make_uint4(dgv[0], dgv[1], dgv[2], dgv[3]);
      if (gpart) {  // the gate-bias gradient sums the bf16 values stored
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack2(dgv[j]);
          gacc[2 * j] += f.x;
          gacc[2 * j + 1] += f.y;
        }
      }
    }
    // fixed-order reduction over the CH chunk lanes (aligned groups of CH)
#pragma unroll
    for (int off = 1; off < CH; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (ok && c == 0) {
      const int64_t i = (b * a.H + h) * (int64_t)a.L + l;
      Dq[i] = acc;
      if (lse2) lse2[i] = a.lse[i] * LOG2E;  // the streamed-key dk/dv stages log2 units
    }
  }
  if (gpart) {
    // threads t, t + G, t + 2G, ... (G = H*CH column groups) share columns
    __shared__ float red[256][9];
#pragma unroll
    for (int j = 0; j < 8; ++j) red[threadIdx.x][j] = gacc[j];
    __syncthreads();
    const int G = a.H * CH;
    for (int i = threadIdx.x; i < G * 8; i += blockDim.x) {
      const int grp = i / 8, j = i % 8;
      float t = 0.f;
      for (int k = grp; k < (int)blockDim.x; k += G) t += red[k][j];
      gpart[(int64_t)blockIdx.x * (a.H * D) + grp * 8 + j] = t;
    }
  }
}

// ============================================================ bwd helpers
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
// 16 consecutive bias values of one row from a smem tile; ROWBOX: tile is
// 32-key boxes of 128B-swizzled rows (read along the row), else a
// [key][128 rows] tile read by column.
template <bool ROWBOX>
__device__ __forceinline__ void bias_row16(const uint8_t *sb, int row, int k0, float (&out)[16]) {
  if constexpr (ROWBOX) {
    const uint8_t *base = sb + (k0 >> 5) * 16384 + row * 128;
    const int c0 = (k0 & 31) >> 2;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float4 v = *reinterpret_cast<const float4 *>(base + (((c0 + c) ^ (row & 7)) << 4));
      out[4 * c] = v.x; out[4 * c + 1] = v.y; out[4 * c + 2] = v.z; out[4 * c + 3] = v.w;
    }
  } else {
    const float *p = reinterpret_cast<const float *>(sb) + k0 * 128 + row;
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = p[j * 128];
  }
}
// Fold log2(e) into a resident bias tile once per CTA.
__device__ __forceinline__ void scale_tile(uint8_t *sb, int nfloat4, int nthreads = 0) {
  float4 *p = reinterpret_cast<float4 *>(sb);
  const int stride = nthreads ? nthreads : (int)blockDim.x;
  for (int i = threadIdx.x; i < nfloat4; i += stride) {
    float4 v = p[i];
    v.x *= LOG2E; v.y *= LOG2E; v.z *= LOG2E; v.w *= LOG2E;
    p[i] = v;
  }
}
// A bias tile whose rows run along the thread's index (boxes of [32 outer][128
// inner] plain floats, outer = the index a thread iterates) rewritten in
// place, box by box, into the 128B-swizzled [128 inner][32 outer] box layout
// the row-box readers use, scaled by log2(e): the backward kernels then read
// a thread's consecutive bias values as 16-byte vectors instead of one
// strided scalar per element (once per CTA; the tile serves every batch row).
// All 512 elementwise threads call it (named barrier 1).
template <int NT = 512>
__device__ __forceinline__ void transpose_scale_bias_boxes(uint8_t *sb, int nbox, int tid) {
  constexpr int PER = 4096 / NT;
  for (int j = 0; j < nbox; ++j) {
    float *box = reinterpret_cast<float *>(sb + j * 16384);
    float v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) v[i] = box[tid + NT * i] * LOG2E;
    named_bar_sync(1, NT);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + NT * i, o = e >> 7, in = e & 127;
      *reinterpret_cast<float *>(sb + j * 16384 + in * 128 + ((((o >> 2) ^ (in & 7))) << 4) +
                                 (o & 3) * 4) = v[i];
    }
    named_bar_sync(1, NT);
  }
}

// TMEM column of the 16-wide K slice `ks` of bf16-pair data written in place
// into quarters: keys [i*KQ, (i+1)*KQ) -> cols [i*KQ, i*KQ + KQ/2).
__device__ __forceinline__ uint32_t quarter_col(int ks, int KQ) {
  const int k = 16 * ks;
  return (uint32_t)((k / KQ) * KQ + (k % KQ) / 2);
}

// ================================================================= fwd, v2
// Lp = 128 or 256.  Four threads per query row (warps w, w+4, w+8, w+12 share the
// row's TMEM lane; quarter qr owns keys [64qr, 64qr+64)), so each thread
// keeps its 64 logits x = S*scale*log2e + bias*log2e in registers between
// the max and the exp pass: one TMEM read and one bias read per element.
// Two TMEM row slots [256s, 256s+256) hold S, then P (bf16 pairs, packed in
// place into each quarter's first 32 columns), then O at col 32.  Warp 16
// issues: the PV MMA of row b once all 16 warps packed P(b), the S MMA of
// row b+2 once row b's epilogue has read O, the TMA loads of row b+2 once
// PV(b) completed.  Row b's epilogue runs between row b+1's two passes, so
// the PV MMA of b and the S MMA of b+2 overlap elementwise work.
template <int D, int BIASMODE, int LPC>
__global__ void __launch_bounds__(544, 1)
attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                    const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mB,
                    const AttnTcArgs a) {
  evo_pdl_enter();
  constexpr uint32_t TILE = QT * Sw<D>::bytes;
  // LPC = Lp (128 or 256): each thread owns KQ = LPC/4 keys; O sits in
  // quarter 0's freed half (Lp 256) or past S (Lp 128)
  constexpr int KQ = LPC / 4;
  constexpr uint32_t OCOL = LPC == 256 ? 32 : 128;
  constexpr uint32_t FULL = LPC * Sw<D>::bytes;
  constexpr uint32_t ROWB = TILE + 2 * FULL;  // Q | K | V of one batch row
  constexpr bool TB = BIASMODE == 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sBias = smem_raw;
  uint8_t *sRow = sBias + (BIASMODE ? BIAS_BYTES : 0);
  float *sMax = reinterpret_cast<float *>(sRow + 2 * ROWB);  // [parity][quarter][128]
  float *sSum = sMax + 2 * 4 * 128;
  // 0 bias, 1-2 row Q|K, 3-4 S MMA done, 5-6 PV MMA done, 7-8 P packed
  // (16 warps), 9-10 epilogue read O (16 warps), 11-12 row V  [by row parity]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sSum + 2 * 4 * 128);
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 13);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = (warp & 3) * 32 + lane;  // query row (TMEM lane)
  const int qr = (warp >> 2) & 3;        // key quarter
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L;
  const int q = q0 + t;
  const bool qv = q < L;
  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);

  if (tid == 512) {
    for (int i = 0; i < 13; ++i) mbar_init(&bars[i], (i >= 7 && i < 11) ? 16 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (BIASMODE) load_bias_tile<TB>(sBias, &mB, &bars[0], h, q0, LPC);
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  auto rowbuf = [&](int64_t r) -> uint8_t * { return sRow + ((r - b_lo) & 1) * ROWB; };

  if (warp == 16) {
    // ------------------------------------------------------------ issuer
    {
    const uint32_t idesc_s = idesc_bf16(128, LPC, false, false);
    const uint32_t idesc_o = idesc_bf16(128, D, false, true);
    // Q|K and V of a row load separately: Q|K of row r+2 as soon as S(r)
    // is done (its S MMA then waits on nothing but the epilogue of row r),
    // V of row r+2 once PV(r) has read row r's V
    auto load_qk = [&](int64_t r) {
      uint8_t *rb = rowbuf(r);
      uint64_t *bar = &bars[1 + ((r - b_lo) & 1)];
      mbar_expect_tx(bar, TILE + FULL);
      tma_load_4d(rb, &mQ, bar, 0, q0, (int)r, h);
      tma_load_4d(rb + TILE, &mK, bar, 0, 0, (int)r, h);
    };
    auto load_v = [&](int64_t r) {
      uint8_t *rb = rowbuf(r);
      uint64_t *bar = &bars[11 + ((r - b_lo) & 1)];
      mbar_expect_tx(bar, FULL);
      tma_load_4d(rb + TILE + FULL, &mV, bar, 0, 0, (int)r, h);
    };
    auto issue_s = [&](int64_t r) {
      const int p = (int)((r - b_lo) & 1);
      const uint32_t ph = (uint32_t)(((r - b_lo) >> 1) & 1);
      mbar_wait(&bars[1 + p], ph);
      fence_after();
      const uint32_t sQ = smem_u32(rowbuf(r)), sK = sQ + TILE;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        umma_bf16_el(tmem + 256 * p, desc_kmajor_tile<D>(sQ, ks), desc_kmajor_tile<D>(sK, ks),
                     idesc_s, ks > 0);
      umma_commit_el(&bars[3 + p]);
    };
    if (b_lo < b_hi) {
      if (lane == 0) {
        load_qk(b_lo);
        load_v(b_lo);
        if (b_lo + 1 < b_hi) {
          load_qk(b_lo + 1);
          load_v(b_lo + 1);
        }
      }
      __syncwarp();
      issue_s(b_lo);
      if (b_lo + 1 < b_hi) issue_s(b_lo + 1);
      for (int64_t r = b_lo; r < b_hi; ++r) {
        const int p = (int)((r - b_lo) & 1);
        const uint32_t ph = (uint32_t)(((r - b_lo) >> 1) & 1);
        if (r + 2 < b_hi) {
          mbar_wait(&bars[3 + p], ph);  // S(r) done: row r's Q|K is free
          if (lane == 0) load_qk(r + 2);
          __syncwarp();
        }
        mbar_wait(&bars[7 + p], ph);  // P(r) packed by all 16 warps
        mbar_wait(&bars[11 + p], ph);  // V(r) landed
        fence_after();
        const uint32_t sV = smem_u32(rowbuf(r)) + TILE + FULL;
        const uint32_t slot = tmem + 256 * p;
        constexpr int SPQ = KQ / 16;  // K slices per quarter
#pragma unroll
        for (int ks = 0; ks < LPC / 16; ++ks)
          umma_bf16_ts_el(slot + OCOL, slot + KQ * (ks / SPQ) + 8 * (ks % SPQ),
                          desc_mnmajor_tile<D>(sV, ks), idesc_o, ks > 0);
        umma_commit_el(&bars[5 + p]);
        if (r + 2 < b_hi) {
          mbar_wait(&bars[5 + p], ph);  // PV(r) done: row r's V is free
          if (lane == 0) load_v(r + 2);
          __syncwarp();
          mbar_wait(&bars[9 + p], ph);  // epilogue(r) read O: slot p is free
          fence_after();
          issue_s(r + 2);
        }
      }
    }
    __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ softmax
    const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    if (BIASMODE) {
      mbar_wait(&bars[0], 0);
      scale_tile(sBias, 8 * 16384 / 16, 512);
      named_bar_sync(1, 512);
    }
    const float sc_l2 = a.scale * LOG2E;
    uint4 gq_prev = make_uint4(0u, 0u, 0u, 0u);
    float mx_prev = 0.f;
    auto epilogue = [&](int64_t rr) {  // O of batch row rr -> o, gm, lse
      const int p = (int)((rr - b_lo) & 1);
      mbar_wait(&bars[5 + p], (uint32_t)(((rr - b_lo) >> 1) & 1));
      fence_after();
      uint32_t ov[8];
      constexpr int QD = D / 4;
      if constexpr (QD == 8) {
        tmem_ld8_nw(lane_addr + 256 * p + OCOL + 8 * qr, ov);
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(ov[0]), "=r"(ov[1]), "=r"(ov[2]), "=r"(ov[3])
                     : "r"(lane_addr + 256 * p + OCOL + 4 * qr));
      }
      tmem_wait_ld();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[9 + p]);  // slot p's O read
      const float *ss = sSum + p * 512;
      const float sum = (ss[t] + ss[128 + t]) + (ss[256 + t] + ss[384 + t]);
      if (qv) {
        const float inv = 1.f / sum;
        const int64_t ooff = rr * a.o_sb + (int64_t)q * a.o_sl + h * D + qr * QD;
        const uint32_t *gw = reinterpret_cast<const uint32_t *>(&gq_prev);
        uint32_t o2[4], g2v[4];
#pragma unroll
        for (int j = 0; j < QD / 2; ++j) {
          const float o0 = __uint_as_float(ov[2 * j]) * inv;
          const float o1 = __uint_as_float(ov[2 * j + 1]) * inv;
          const float2 g2 = unpack2(gw[j]);
          o2[j] = pack2(o0, o1);
          g2v[j] = pack2(g2.x * o0, g2.y * o1);
        }
        if constexpr (QD == 8) {
          *reinterpret_cast<uint4 *>(a.o + ooff) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
          *reinterpret_cast<uint4 *>(a.gm + ooff) = make_uint4(g2v[0], g2v[1], g2v[2], g2v[3]);
        } else {
          *reinterpret_cast<uint2 *>(a.o + ooff) = make_uint2(o2[0], o2[1]);
          *reinterpret_cast<uint2 *>(a.gm + ooff) = make_uint2(g2v[0], g2v[1]);
        }
        if (qr == 0) a.lse[(rr * a.H + h) * (int64_t)L + q] = mx_prev * (1.f / LOG2E) + logf(sum);
      }
    };
    for (int64_t r = b_lo; r < b_hi; ++r) {
      const int p = (int)((r - b_lo) & 1);
      const uint32_t ph = (uint32_t)(((r - b_lo) >> 1) & 1);
      const uint32_t slot = lane_addr + 256 * p;
      const int kb = KQ * qr;
      // gate slice of this row (consumed by its epilogue, one row later)
      // (volatile: issued here, a row ahead of its use, not sunk to the use)
      uint4 gq = make_uint4(0u, 0u, 0u, 0u);
      if (qv) {
        const bf16 *gp = a.g + r * a.sb + (int64_t)q * a.sl + h * D + qr * (D / 4);
        if constexpr (D == 32) {
          asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(gq.x), "=r"(gq.y), "=r"(gq.z), "=r"(gq.w)
                       : "l"(gp));
        } else {
          asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(gq.x), "=r"(gq.y) : "l"(gp));
        }
      }
      mbar_wait(&bars[3 + p], ph);
      fence_after();
      // pass 1: logits of this thread's KQ keys -> registers, local max
      float x[KQ];
      float mx = -INFINITY;
      const bool kfull = kb + KQ <= L;  // interior key slices skip the mask
#pragma unroll
      for (int c = 0; c < KQ / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(slot + kb + 32 * c, v);
        float bb[32];
        if (BIASMODE) bias_row32<TB>(sBias, t, kb + 32 * c, bb);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float xx = __uint_as_float(v[j]) * sc_l2;
          if (BIASMODE) xx += bb[j];
          x[32 * c + j] = xx;
        }
        if (!kfull) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (kb + 32 * c + j >= L) x[32 * c + j] = -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, x[32 * c + j]);
      }
      float *sm_ = sMax + p * 512;
      sm_[qr * 128 + t] = mx;
      named_bar_sync(2 + (warp & 3), 128);  // the row's four quarters
      mx = fmaxf(fmaxf(sm_[t], sm_[128 + t]), fmaxf(sm_[256 + t], sm_[384 + t]));
      // the previous row's epilogue (its PV MMA overlapped pass 1)
      if (r > b_lo) epilogue(r - 1);
      // pass 2: p = exp2(x - max) -> bf16 pairs in this quarter's first 32 cols
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < KQ / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float p0 = ex2(x[32 * c + 2 * j] - mx);
          const float p1 = ex2(x[32 * c + 2 * j + 1] - mx);
          sum += p0 + p1;
          pk[j] = pack2(p0, p1);
        }
        tmem_st16(slot + kb + 16 * c, pk);
      }
      sSum[p * 512 + qr * 128 + t] = sum;
      gq_prev = gq;
      mx_prev = mx;
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[7 + p]);
    }
    if (b_lo < b_hi) epilogue(b_hi - 1);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ======================================================================= dq
// CTA = (128-query tile, head, chunk of batch rows), 512 threads: 4 threads
// per query row, thread quarter `qr` owns keys [qr*KQ, (qr+1)*KQ) (KQ=Lp/4)
// and keeps that slice of the dbias partial in REGISTERS across the chunk.
// TMEM: S [0, Lp) and dP [256, 256+Lp) from back-to-back MMAs; one pass
// computes P, dS, dbias and writes dS (bf16 pairs) in place into the
// thread's own S columns; dq = scale * dS K as a TS MMA into [256, 256+D).
template <int D, int BIASMODE>
__global__ void __launch_bounds__(512, 1)
attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                      const __grid_constant__ CUtensorMap mV,
                      const __grid_constant__ CUtensorMap mdO,
                      const __grid_constant__ CUtensorMap mB, const AttnTcArgs a) {
  evo_pdl_enter();
  constexpr uint32_t TILE = QT * Sw<D>::bytes;
  constexpr uint32_t FULL = 256 * Sw<D>::bytes;
  constexpr bool TB = BIASMODE == 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                            ~uintptr_t(1023));
  uint8_t *sBias = sm;
  uint8_t *sQ = sBias + (BIASMODE ? BIAS_BYTES : 0);
  uint8_t *sdO = sQ + TILE;
  uint8_t *sV = sdO + TILE;
  uint8_t *sK2 = sV + FULL;  // two K buffers (K of row b+1 streams in during row b)
  uint64_t *bars = reinterpret_cast<uint64_t *>(sK2 + 2 * FULL);  // 0 bias, 1 q/dO/V, 2-3 K, 4 mma
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 5);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = (warp & 3) * 32 + lane;  // query row in the tile
  const int qr = warp >> 2;              // key quarter
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L, Lp = a.Lp, KQ = Lp / 4;
  const int q = q0 + t;
  const bool qv = q < L;
  const bool want_bias = a.dbias_part != nullptr;

  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (BIASMODE) load_bias_tile<TB>(sBias, &mB, &bars[0], h, q0, Lp);
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  if (BIASMODE) {
    mbar_wait(&bars[0], 0);
    scale_tile(sBias, ((Lp + 31) / 32) * 16384 / 16);
    __syncthreads();
  }

  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  uint32_t ph_a = 0, ph_m = 0, ph_k2 = 0;  // ph_k2: bit i = phase of K buffer i
  const uint32_t kv_bytes = (uint32_t)Lp * Sw<D>::bytes;
  auto load_qdv = [&](int64_t bb) {
    mbar_expect_tx(&bars[1], 2 * TILE + kv_bytes);
    tma_load_4d(sQ, &mQ, &bars[1], 0, q0, (int)bb, h);
    tma_load_4d(sdO, &mdO, &bars[1], 0, q0, (int)bb, h);
    tma_load_4d(sV, &mV, &bars[1], 0, 0, (int)bb, h);
  };
  auto load_k = [&](int64_t bb) {
    const int kb = (int)((bb - b_lo) & 1);
    mbar_expect_tx(&bars[2 + kb], kv_bytes);
    tma_load_4d(sK2 + kb * FULL, &mK, &bars[2 + kb], 0, 0, (int)bb, h);
  };
  if (tid == 0 && b_lo < b_hi) {
    load_qdv(b_lo);
    load_k(b_lo);
  }
  const uint32_t idesc_s = idesc_bf16(128, Lp, false, false);
  const uint32_t idesc_o = idesc_bf16(128, D, false, true);
  const float sc_l2 = a.scale * LOG2E;
  float acc[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) acc[j] = 0.f;
  float lse_n = 0.f, Dq_n = 0.f;
  if (qv && b_lo < b_hi) {
    lse_n = a.lse[(b_lo * a.H + h) * (int64_t)L + q];
    Dq_n = a.Dq[(b_lo * a.H + h) * (int64_t)L + q];
  }

  for (int64_t b = b_lo; b < b_hi; ++b) {
    const bool has_next = b + 1 < b_hi;
    const int kb = (int)((b - b_lo) & 1);
    uint8_t *sK = sK2 + kb * FULL;
    const float lse_l2 = lse_n * LOG2E;
    const float Dq = Dq_n;
    if (qv && has_next) {
      lse_n = a.lse[((b + 1) * a.H + h) * (int64_t)L + q];
      Dq_n = a.Dq[((b + 1) * a.H + h) * (int64_t)L + q];
    }
    if (tid == 0) {
      if (has_next) load_k(b + 1);  // the other K buffer is idle since row b-1
      mbar_wait(&bars[1], ph_a);
      mbar_wait(&bars[2 + kb], (ph_k2 >> kb) & 1);
      fence_after();
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        umma_bf16(tmem, desc_kmajor_tile<D>(smem_u32(sQ), ks),
                  desc_kmajor_tile<D>(smem_u32(sK), ks), idesc_s, ks > 0);
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        umma_bf16(tmem + 256, desc_kmajor_tile<D>(smem_u32(sdO), ks),
                  desc_kmajor_tile<D>(smem_u32(sV), ks), idesc_s, ks > 0);
      umma_commit(&bars[4]);
    }
    ph_a ^= 1;
    ph_k2 ^= 1u << kb;
    mbar_wait(&bars[4], ph_m);
    ph_m ^= 1;
    fence_after();
    if (tid == 0 && has_next) load_qdv(b + 1);  // Q, dO, V consumed
    // one pass: P, dS, dbias for this thread's keys
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (16 * s < KQ) {
        const int k0 = qr * KQ + 16 * s;
        uint32_t sv[16], dv[16];
        tmem_ld16_nw(lane_addr + k0, sv);
        tmem_ld16_nw(lane_addr + 256 + k0, dv);
        tmem_wait_ld();
        float bb[16];
        if (BIASMODE) bias_row16<!TB>(sBias, t, k0, bb);
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          float ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            float x = __uint_as_float(sv[j + u]) * sc_l2 - lse_l2;
            if (BIASMODE) x += bb[j + u];
            float p = (qv && k0 + j + u < L) ? ex2(x) : 0.f;
            ds[u] = p * (__uint_as_float(dv[j + u]) - Dq);
            acc[16 * s + j + u] += ds[u];
          }
          pk[j >> 1] = pack2(ds[0], ds[1]);
        }
        tmem_st8(lane_addr + qr * KQ + 8 * s, pk);
      }
    }
    tmem_st_wait();
    fence_before();
    __syncthreads();
    if (tid == 0) {
      fence_after();
      for (int ks = 0; ks < Lp / 16; ++ks)
        umma_bf16_ts(tmem + 256, tmem + quarter_col(ks, KQ),
                     desc_mnmajor_tile<D>(smem_u32(sK), ks), idesc_o, ks > 0);
      umma_commit(&bars[4]);
    }
    mbar_wait(&bars[4], ph_m);
    ph_m ^= 1;
    fence_after();
    {  // dq row: 4 threads x D/4 columns
      constexpr int QD = D / 4;
      uint32_t v[8];
      if constexpr (QD == 8) {
        tmem_ld8_nw(lane_addr + 256 + qr * 8, v);
      } else {  // D == 16: 4 columns each
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(lane_addr + 256 + qr * 4));
      }
      tmem_wait_ld();
      if (qv) {
        bf16 *dst = a.dq + b * a.sb + (int64_t)q * a.sl + h * D + qr * QD;
        if constexpr (QD == 8) {
          uint32_t w4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            w4[j] = pack2(__uint_as_float(v[2 * j]) * a.scale,
                          __uint_as_float(v[2 * j + 1]) * a.scale);
          *reinterpret_cast<uint4 *>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        } else {
          uint32_t w2[2];
#pragma unroll
          for (int j = 0; j < 2; ++j)
            w2[j] = pack2(__uint_as_float(v[2 * j]) * a.scale,
                          __uint_as_float(v[2 * j + 1]) * a.scale);
          *reinterpret_cast<uint2 *>(dst) = make_uint2(w2[0], w2[1]);
        }
      }
    }
    fence_before();
    __syncthreads();  // TMEM + smem free for the next row
    fence_after();
  }
  if (want_bias && qv) {
    float *dst = a.dbias_part + (int64_t)blockIdx.z * a.H * a.bh +
                 (int64_t)h * a.bh + (int64_t)q * a.bq;
    const int kbase = qr * KQ;
    if (a.bk == 1 && kbase + KQ <= L && ((reinterpret_cast<uintptr_t>(dst + kbase) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 64; j += 4)
        if (j < KQ)
          *reinterpret_cast<float4 *>(dst + kbase + j) =
              make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (j < KQ && kbase + j < L) dst[(int64_t)(kbase + j) * a.bk] = acc[j];
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ====================================================================== dkv
// CTA = (128-key tile, head, chunk of batch rows), 512 threads, 4 per key
// row; quarter qr owns queries [qr*QQ, (qr+1)*QQ).  TMEM: S^T [0, Lp),
// dP^T [256, 256+Lp); P^T and dS^T written in place (bf16 pairs) into each
// thread's own columns; dv = P^T dO and dk = scale * dS^T Q as TS MMAs.
template <bool TBK>  // keys contiguous in the smem tile (plain bias)?
__device__ __forceinline__ void load_bias_tile_k(uint8_t *sb, const CUtensorMap *map,
                                                 uint64_t *bar, int h, int k0, int Lp) {
  const int nbox = (Lp + 31) / 32;
  mbar_expect_tx(bar, (uint32_t)nbox * 16384u);
  for (int j = 0; j < nbox; ++j) {
    if constexpr (TBK)
      tma_load_3d(sb + j * 16384, map, bar, k0, 32 * j, h);   // {k inner 128, 32 q}
    else
      tma_load_3d(sb + j * 16384, map, bar, 32 * j, k0, h);   // {32 q inner, 128 k}
  }
}

template <int D, int BIASMODE>
__global__ void __launch_bounds__(512, 1)
attn_bwd_dkv_tc_kernel(const __grid_constant__ CUtensorMap mKt, const __grid_constant__ CUtensorMap mVt,
                       const __grid_constant__ CUtensorMap mQa,
                       const __grid_constant__ CUtensorMap mdOa,
                       const __grid_constant__ CUtensorMap mB, const AttnTcArgs a) {
  evo_pdl_enter();
  constexpr uint32_t TILE = QT * Sw<D>::bytes;
  constexpr uint32_t FULL = 256 * Sw<D>::bytes;
  // plain bias (bk == 1): smem [q][128 k], read by column;
  // transposed (bq == 1): 32-query boxes [k][32 q], 128B-swizzled rows
  constexpr bool KCONTIG = BIASMODE == 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                            ~uintptr_t(1023));
  uint8_t *sBias = sm;
  uint8_t *sQ2 = sBias + (BIASMODE ? BIAS_BYTES : 0);  // two (Q | dO) buffers
  uint8_t *sK = sQ2 + 4 * FULL;
  uint8_t *sV = sK + TILE;
  float *sLse = reinterpret_cast<float *>(sV + TILE);
  float *sDq = sLse + 256;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sDq + 256);  // 0 bias, 1 K/V, 2-3 Q/dO, 4 mma
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 5);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = (warp & 3) * 32 + lane;  // key row in the tile
  const int qr = warp >> 2;              // query quarter
  const int k0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L, Lp = a.Lp, QQ = Lp / 4;
  const int k = k0 + t;
  const bool kv = k < L;

  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (BIASMODE) load_bias_tile_k<KCONTIG>(sBias, &mB, &bars[0], h, k0, Lp);
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  if (BIASMODE) {
    mbar_wait(&bars[0], 0);
    scale_tile(sBias, ((Lp + 31) / 32) * 16384 / 16);
    __syncthreads();
  }
  // free columns for dV / dK after the in-place P^T / dS^T packing
  const uint32_t DVC = Lp >= 256 ? (uint32_t)(QQ / 2) : (uint32_t)Lp;

  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  uint32_t ph_kv = 0, ph_q2 = 0, ph_m = 0;
  const uint32_t all_bytes = (uint32_t)Lp * Sw<D>::bytes;
  auto load_kv = [&](int64_t bb) {
    mbar_expect_tx(&bars[1], 2 * TILE);
    tma_load_4d(sK, &mKt, &bars[1], 0, k0, (int)bb, h);
    tma_load_4d(sV, &mVt, &bars[1], 0, k0, (int)bb, h);
  };
  auto load_q = [&](int64_t bb) {
    const int qb = (int)((bb - b_lo) & 1);
    mbar_expect_tx(&bars[2 + qb], 2 * all_bytes);
    tma_load_4d(sQ2 + qb * 2 * FULL, &mQa, &bars[2 + qb], 0, 0, (int)bb, h);
    tma_load_4d(sQ2 + qb * 2 * FULL + FULL, &mdOa, &bars[2 + qb], 0, 0, (int)bb, h);
  };
  if (tid == 0 && b_lo < b_hi) {
    load_kv(b_lo);
    load_q(b_lo);
  }
  const uint32_t idesc_s = idesc_bf16(128, Lp, false, false);
  const uint32_t idesc_o = idesc_bf16(128, D, false, true);
  const float sc_l2 = a.scale * LOG2E;
  float lse_n = 0.f, Dq_n = 0.f;
  if (tid < L && b_lo < b_hi) {
    lse_n = a.lse[(b_lo * a.H + h) * (int64_t)L + tid] * LOG2E;
    Dq_n = a.Dq[(b_lo * a.H + h) * (int64_t)L + tid];
  }

  for (int64_t b = b_lo; b < b_hi; ++b) {
    const bool has_next = b + 1 < b_hi;
    const int qb = (int)((b - b_lo) & 1);
    uint8_t *sQ = sQ2 + qb * 2 * FULL;
    uint8_t *sdO = sQ + FULL;
    if (tid < Lp) {
      sLse[tid] = lse_n;
      sDq[tid] = Dq_n;
    }
    if (tid < L && has_next) {
      lse_n = a.lse[((b + 1) * a.H + h) * (int64_t)L + tid] * LOG2E;
      Dq_n = a.Dq[((b + 1) * a.H + h) * (int64_t)L + tid];
    } else {
      lse_n = 0.f;
      Dq_n = 0.f;
    }
    if (tid == 0) {
      if (has_next) load_q(b + 1);  // the other Q/dO buffer is idle since row b-1
      mbar_wait(&bars[1], ph_kv);
      mbar_wait(&bars[2 + qb], (ph_q2 >> qb) & 1);
      fence_after();
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        umma_bf16(tmem, desc_kmajor_tile<D>(smem_u32(sK), ks),
                  desc_kmajor_tile<D>(smem_u32(sQ), ks), idesc_s, ks > 0);
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        umma_bf16(tmem + 256, desc_kmajor_tile<D>(smem_u32(sV), ks),
                  desc_kmajor_tile<D>(smem_u32(sdO), ks), idesc_s, ks > 0);
      umma_commit(&bars[4]);
    }
    ph_kv ^= 1;
    ph_q2 ^= 1u << qb;
    mbar_wait(&bars[4], ph_m);
    ph_m ^= 1;
    fence_after();
    __syncthreads();  // lse / Dq of this row visible
    if (tid == 0 && has_next) load_kv(b + 1);  // K, V tiles consumed
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (16 * s < QQ) {
        const int c0 = qr * QQ + 16 * s;
        uint32_t sv[16], dv[16];
        tmem_ld16_nw(lane_addr + c0, sv);
        tmem_ld16_nw(lane_addr + 256 + c0, dv);
        tmem_wait_ld();
        float bb[16];
        if (BIASMODE) bias_row16<!KCONTIG>(sBias, t, c0, bb);
        uint32_t pk[8], dk8[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          float p[2], ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int qq = c0 + j + u;
            float x = __uint_as_float(sv[j + u]) * sc_l2 - sLse[qq];
            if (BIASMODE) x += bb[j + u];
            p[u] = (kv && qq < L) ? ex2(x) : 0.f;
            ds[u] = p[u] * (__uint_as_float(dv[j + u]) - sDq[qq]);
          }
          pk[j >> 1] = pack2(p[0], p[1]);
          dk8[j >> 1] = pack2(ds[0], ds[1]);
        }
        tmem_st8(lane_addr + qr * QQ + 8 * s, pk);
        tmem_st8(lane_addr + 256 + qr * QQ + 8 * s, dk8);
      }
    }
    tmem_st_wait();
    fence_before();
    __syncthreads();
    if (tid == 0) {
      fence_after();
      for (int ks = 0; ks < Lp / 16; ++ks)
        umma_bf16_ts(tmem + DVC, tmem + quarter_col(ks, QQ),
                     desc_mnmajor_tile<D>(smem_u32(sdO), ks), idesc_o, ks > 0);
      for (int ks = 0; ks < Lp / 16; ++ks)
        umma_bf16_ts(tmem + 256 + DVC, tmem + 256 + quarter_col(ks, QQ),
                     desc_mnmajor_tile<D>(smem_u32(sQ), ks), idesc_o, ks > 0);
      umma_commit(&bars[4]);
    }
    mbar_wait(&bars[4], ph_m);
    ph_m ^= 1;
    fence_after();
    {  // dv, dk rows: 4 threads x D/4 columns
      constexpr int QD = D / 4;
      uint32_t v1[8], v2[8];
      if constexpr (QD == 8) {
        tmem_ld8_nw(lane_addr + DVC + qr * 8, v1);
        tmem_ld8_nw(lane_addr + 256 + DVC + qr * 8, v2);
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v1[0]), "=r"(v1[1]), "=r"(v1[2]), "=r"(v1[3])
                     : "r"(lane_addr + DVC + qr * 4));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v2[0]), "=r"(v2[1]), "=r"(v2[2]), "=r"(v2[3])
                     : "r"(lane_addr + 256 + DVC + qr * 4));
      }
      tmem_wait_ld();
      if (kv) {
        const int64_t off = b * a.sb + (int64_t)k * a.sl + h * D + qr * QD;
        if constexpr (QD == 8) {
          uint32_t w1[4], w2[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            w1[j] = pack2(__uint_as_float(v1[2 * j]), __uint_as_float(v1[2 * j + 1]));
            w2[j] = pack2(__uint_as_float(v2[2 * j]) * a.scale,
                          __uint_as_float(v2[2 * j + 1]) * a.scale);
          }
          *reinterpret_cast<uint4 *>(a.dv + off) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
          *reinterpret_cast<uint4 *>(a.dk + off) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
        } else {
          uint32_t w1[2], w2[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            w1[j] = pack2(__uint_as_float(v1[2 * j]), __uint_as_float(v1[2 * j + 1]));
            w2[j] = pack2(__uint_as_float(v2[2 * j]) * a.scale,
                          __uint_as_float(v2[2 * j + 1]) * a.scale);
          }
          *reinterpret_cast<uint2 *>(a.dv + off) = make_uint2(w1[0], w1[1]);
          *reinterpret_cast<uint2 *>(a.dk + off) = make_uint2(w2[0], w2[1]);
        }
      }
    }
    fence_before();
    __syncthreads();
    fence_after();
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ============================================================ dkv, pipelined
// Lp == 256.  Units of 64 queries (four per batch row) flow through three
// TMEM regions [S^T 64 | dP^T 64] at 128*(u%3); the S^T / dP^T MMAs of unit
// u+2 are issued while the threads run the elementwise pass of unit u, so
// the tensor core and the CUDA cores overlap instead of taking turns.  P^T
// and dS^T are packed in place into each thread's own columns (a 16-query
// K slice = one thread quarter = 8 packed columns), dV / dK accumulate in
// TMEM across the row's four units (row-parity accumulators [dV 32 | dK 32]
// at 384 + 64*(r&1)) and are read back one unit into the next row, and the
// TMA loads of row r+1 go out as soon as row r-1's accumulators are read.
// Warps 0-15 run the elementwise passes (4 lane quadrants x 4 query
// quarters); warps 16 and 17 only issue (16: the S^T/dP^T MMAs, each as soon
// as its region's previous dV/dK MMAs completed; 17: the dV/dK MMAs and the
// TMA loads), so no elementwise warp ever waits on issue latency.
// smem: bias 128 KiB + two rows of K|V|Q|dO (96 KiB) + lse/Dq: no 1 KiB
// alignment slack, the dynamic smem base is 1 KiB aligned (checked).
template <int D, int BIASMODE, int NU>
__global__ void __launch_bounds__(576, 1)
attn_bwd_dkv_pipe_kernel(const __grid_constant__ CUtensorMap mKt,
                         const __grid_constant__ CUtensorMap mVt,
                         const __grid_constant__ CUtensorMap mQa,
                         const __grid_constant__ CUtensorMap mdOa,
                         const __grid_constant__ CUtensorMap mB, const AttnTcArgs a) {
  evo_pdl_enter();
  constexpr int UW = 64, LPC = NU * UW;           // Lp = 64 NU (128 or 256)
  constexpr uint32_t TILE = QT * Sw<D>::bytes;
  constexpr uint32_t FULL = LPC * Sw<D>::bytes;
  constexpr uint32_t ROWB = 2 * TILE + 2 * FULL;  // K | V | Q | dO of one batch row
  // row buffers: with no bias tile the smem takes a third, so row r+2's
  // loads go out at row r's first unit (short rows still hide TMA latency)
  constexpr int NBUF = BIASMODE ? 2 : 3;
  constexpr bool KCONTIG = BIASMODE == 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sBias = smem_raw;
  uint8_t *sRow = sBias + (BIASMODE ? BIAS_BYTES : 0);
  float *sLse = reinterpret_cast<float *>(sRow + NBUF * ROWB);
  float *sDq = sLse + 256;
  // 0 bias, 1-2 row data (row parity), 3-5 S^T/dP^T MMAs (region),
  // 6-7 the row's last dV/dK MMAs (row parity), 8-9 and 13 unit's
  // elementwise pass done (one arrival per warp; by region u % 3, see
  // ewdone below), 10-12 a unit's dV/dK MMAs done (region):
  // the region is rewritten by the S^T MMA two units later only after its
  // packed P^T / dS^T were consumed
  // (row-data barriers 1..NBUF; the others shifted by 1 when NBUF == 3)
  uint64_t *bars_all = reinterpret_cast<uint64_t *>(sDq + 256);
  uint64_t *rowbar = bars_all + 1;
  uint64_t *bars = bars_all + (NBUF - 2);  // bars[3..13] as documented above
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars_all + 15);
  // unit-done barriers by REGION (u % 3): unit u+3's arrivals need unit u+3's
  // S^T MMA, which waits for unit u's dV/dK MMAs, which wait for unit u's
  // arrivals -- so a barrier never completes twice before its waiter looked
  // (two per-parity barriers could: u+2's S^T MMA only waits for u-1)
  auto ewdone = [&](int rg) -> uint64_t * { return rg < 2 ? &bars[8 + rg] : &bars[13]; };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = (warp & 3) * 32 + lane;  // key row in the tile
  const int qr = warp >> 2;              // 16-query quarter of each unit
  const int k0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L;
  const int k = k0 + t;
  const bool kv = k < L;
  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  const int64_t nrows = b_hi - b_lo;
  const int64_t U = nrows > 0 ? nrows * NU : 0;

  constexpr int ISSUER = 512;
  const bool ew = tid < 512;  // elementwise warps
  if (tid == ISSUER) {
    for (int i = 0; i < 15; ++i) {
      const bool ewd = &bars_all[i] == ewdone(0) || &bars_all[i] == ewdone(1) ||
                       &bars_all[i] == ewdone(2);
      mbar_init(&bars_all[i], ewd ? 16 : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (BIASMODE) load_bias_tile_k<KCONTIG>(sBias, &mB, &bars_all[0], h, k0, LPC);
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);

  auto rowbuf = [&](int64_t r) -> uint8_t * { return sRow + ((r - b_lo) % NBUF) * ROWB; };
  auto load_row = [&](int64_t r) {
    uint8_t *rb = rowbuf(r);
    uint64_t *bar = &rowbar[(r - b_lo) % NBUF];
    mbar_expect_tx(bar, ROWB);
    tma_load_4d(rb, &mKt, bar, 0, k0, (int)r, h);
    tma_load_4d(rb + TILE, &mVt, bar, 0, k0, (int)r, h);
    tma_load_4d(rb + 2 * TILE, &mQa, bar, 0, 0, (int)r, h);
    tma_load_4d(rb + 2 * TILE + FULL, &mdOa, bar, 0, 0, (int)r, h);
  };
  const uint32_t idesc_s = idesc_bf16(128, UW, false, false);
  const uint32_t idesc_o = idesc_bf16(128, D, false, true);
  auto issue_mma1 = [&](int u, int reg) {  // warp-collective (issuer warp)
    const int64_t r = b_lo + u / NU;
    const int ui = u % NU;
    if (ui == 0) mbar_wait(&rowbar[(r - b_lo) % NBUF], (uint32_t)(((r - b_lo) / NBUF) & 1));
    fence_after();
    const uint32_t sK = smem_u32(rowbuf(r)), sV = sK + TILE;
    const uint32_t sQ = sK + 2 * TILE + ui * UW * Sw<D>::bytes;
    const uint32_t sdO = sQ + FULL;
    const uint32_t d = tmem + reg * 128;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks)
      umma_bf16_el(d, desc_kmajor_tile<D>(sK, ks), desc_kmajor_tile<D>(sQ, ks), idesc_s, ks > 0);
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks)
      umma_bf16_el(d + 64, desc_kmajor_tile<D>(sV, ks), desc_kmajor_tile<D>(sdO, ks), idesc_s,
                   ks > 0);
    umma_commit_el(&bars[3 + reg]);
  };
  auto readout = [&](int64_t rr) {  // dV, dK rows of batch row rr -> global
    const int pp = (int)((rr - b_lo) & 1);
    mbar_wait(&bars[6 + pp], (uint32_t)(((rr - b_lo) >> 1) & 1));
    fence_after();
    constexpr int QD = D / 4;
    const uint32_t acc = lane_addr + 384 + pp * 64;
    uint32_t v1[8], v2[8];
    if constexpr (QD == 8) {
      tmem_ld8_nw(acc + qr * 8, v1);
      tmem_ld8_nw(acc + 32 + qr * 8, v2);
    } else {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v1[0]), "=r"(v1[1]), "=r"(v1[2]), "=r"(v1[3])
                   : "r"(acc + qr * 4));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v2[0]), "=r"(v2[1]), "=r"(v2[2]), "=r"(v2[3])
                   : "r"(acc + 32 + qr * 4));
    }
    tmem_wait_ld();
    if (kv) {
      const int64_t off = rr * a.sb + (int64_t)k * a.sl + h * D + qr * QD;
      if constexpr (QD == 8) {
        uint32_t w1[4], w2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          w1[j] = pack2(__uint_as_float(v1[2 * j]), __uint_as_float(v1[2 * j + 1]));
          w2[j] = pack2(__uint_as_float(v2[2 * j]) * a.scale,
                        __uint_as_float(v2[2 * j + 1]) * a.scale);
        }
        *reinterpret_cast<uint4 *>(a.dv + off) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
        *reinterpret_cast<uint4 *>(a.dk + off) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
      } else {
        uint32_t w1[2], w2[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          w1[j] = pack2(__uint_as_float(v1[2 * j]), __uint_as_float(v1[2 * j + 1]));
          w2[j] = pack2(__uint_as_float(v2[2 * j]) * a.scale,
                        __uint_as_float(v2[2 * j + 1]) * a.scale);
        }
        *reinterpret_cast<uint2 *>(a.dv + off) = make_uint2(w1[0], w1[1]);
        *reinterpret_cast<uint2 *>(a.dk + off) = make_uint2(w2[0], w2[1]);
      }
    }
  };

  if (!ew) {
    // ------------------------------------------------------------ issuer
    if (warp == 16 && nrows > 0) {
      // S^T/dP^T MMAs: unit v into region v%3 once unit v-3's dV/dK MMAs
      // (the region's previous readers) completed
      if (lane == 0)
        for (int i = 0; i < NBUF && i < nrows; ++i) load_row(b_lo + i);
      __syncwarp();
      int reg = 0;
      uint32_t ph3 = 0;
      for (int v = 0; v < (int)U; ++v) {
        if (v >= 3) {
          mbar_wait(&bars[10 + reg], (ph3 >> reg) & 1u);
          ph3 ^= 1u << reg;
        }
        issue_mma1(v, reg);
        reg = reg == 2 ? 0 : reg + 1;
      }
    } else if (warp == 17 && nrows > 0) {
      int reg = 0;
      for (int u = 0; u < (int)U; ++u) {
        const int64_t r = b_lo + u / NU;
        const int ui = u % NU;
        const int rp = (int)((r - b_lo) & 1);
        mbar_wait(ewdone((int)(u % 3)), (uint32_t)((u / 3) & 1));  // all 16 warps packed unit u
        fence_after();
        // at a row's first unit the warps have read row r-1's accumulators,
        // so row r-1's smem buffer is free for row r-1+NBUF
        if (ui == 0 && r > b_lo && r - 1 + NBUF < b_hi) {
          if (lane == 0) load_row(r - 1 + NBUF);
          __syncwarp();
        }
        const uint32_t acc = tmem + 384 + rp * 64;
        const uint32_t sQ = smem_u32(rowbuf(r)) + 2 * TILE, sdO = sQ + FULL;
        const uint32_t reg_col = tmem + reg * 128;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_bf16_ts_el(acc, reg_col + ks * 16, desc_mnmajor_tile<D>(sdO, ui * 4 + ks), idesc_o,
                          (ui > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_bf16_ts_el(acc + 32, reg_col + 64 + ks * 16, desc_mnmajor_tile<D>(sQ, ui * 4 + ks),
                          idesc_o, (ui > 0 || ks > 0) ? 1u : 0u);
        if (ui == NU - 1) umma_commit_el(&bars[6 + rp]);
        umma_commit_el(&bars[10 + reg]);
        reg = reg == 2 ? 0 : reg + 1;
      }
    }
    __syncwarp();
  } else {
  // ------------------------------------------------------------ elementwise
  float lse_n = 0.f, Dq_n = 0.f;
  if (tid < L && nrows > 0) {
    lse_n = a.lse[(b_lo * a.H + h) * (int64_t)L + tid] * LOG2E;
    Dq_n = a.Dq[(b_lo * a.H + h) * (int64_t)L + tid];
  }
  if (BIASMODE) {
    mbar_wait(&bars_all[0], 0);
    if constexpr (KCONTIG) transpose_scale_bias_boxes(sBias, LPC / 32, tid);
    else scale_tile(sBias, (LPC / 32) * 16384 / 16, 512);
  }
  const float sc_l2 = a.scale * LOG2E;

  int reg = 0;
  uint32_t ph3 = 0;  // bit i: parity of region i's S^T/dP^T barrier
  for (int u = 0; u < (int)U; ++u) {
    const int64_t r = b_lo + u / NU;
    const int ui = u % NU;
    if (ui == 0) {  // this row's lse / Dq into smem; prefetch the next row's
      if (r > b_lo) named_bar_sync(1, 512);  // every warp is done with row r-1's lse / Dq
      if (tid < 256) {
        sLse[tid] = lse_n;
        sDq[tid] = Dq_n;
      }
      if (tid < L && r + 1 < b_hi) {
        lse_n = a.lse[((r + 1) * a.H + h) * (int64_t)L + tid] * LOG2E;
        Dq_n = a.Dq[((r + 1) * a.H + h) * (int64_t)L + tid];
      } else {
        lse_n = 0.f;
        Dq_n = 0.f;
      }
      named_bar_sync(1, 512);
    }
    mbar_wait(&bars[3 + reg], (ph3 >> reg) & 1u);
    ph3 ^= 1u << reg;
    fence_after();
    const uint32_t rb = lane_addr + reg * 128;
    const int c0 = qr * 16;
    const int qb = ui * UW + c0;  // first query of this thread's 16
    uint32_t sv[16], dv[16];
    tmem_ld16_nw(rb + c0, sv);
    tmem_ld16_nw(rb + 64 + c0, dv);
    tmem_wait_ld();
    float bb[16], ls[16], dq[16];
    if (BIASMODE) bias_row16<true>(sBias, t, qb, bb);  // row boxes in both modes (see above)
#pragma unroll
    for (int j = 0; j < 16; j += 4) {  // warp-uniform 16-byte broadcasts
      const float4 l4 = *reinterpret_cast<const float4 *>(sLse + qb + j);
      const float4 d4 = *reinterpret_cast<const float4 *>(sDq + qb + j);
      ls[j] = l4.x; ls[j + 1] = l4.y; ls[j + 2] = l4.z; ls[j + 3] = l4.w;
      dq[j] = d4.x; dq[j + 1] = d4.y; dq[j + 2] = d4.z; dq[j + 3] = d4.w;
    }
    const bool full = kv && qb + 16 <= L;
    uint32_t pk[8], dk8[8];
    if (full) {  // interior units: no per-element mask
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        float pp2[2], ds[2];
#pragma unroll
        for (int w2 = 0; w2 < 2; ++w2) {
          float x = fmaf(__uint_as_float(sv[j + w2]), sc_l2, -ls[j + w2]);
          if (BIASMODE) x += bb[j + w2];
          pp2[w2] = ex2(x);
          ds[w2] = pp2[w2] * (__uint_as_float(dv[j + w2]) - dq[j + w2]);
        }
        pk[j >> 1] = pack2(pp2[0], pp2[1]);
        dk8[j >> 1] = pack2(ds[0], ds[1]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        float pp2[2], ds[2];
#pragma unroll
        for (int w2 = 0; w2 < 2; ++w2) {
          float x = fmaf(__uint_as_float(sv[j + w2]), sc_l2, -ls[j + w2]);
          if (BIASMODE) x += bb[j + w2];
          const float e = ex2(x);
          pp2[w2] = (kv && qb + j + w2 < L) ? e : 0.f;
          ds[w2] = pp2[w2] * (__uint_as_float(dv[j + w2]) - dq[j + w2]);
        }
        pk[j >> 1] = pack2(pp2[0], pp2[1]);
        dk8[j >> 1] = pack2(ds[0], ds[1]);
      }
    }
    tmem_st8(rb + c0, pk);
    tmem_st8(rb + 64 + c0, dk8);
    if (ui == 0 && r > b_lo) readout(r - 1);
    tmem_st_wait();
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(ewdone(reg));
    reg = reg == 2 ? 0 : reg + 1;
  }
  if (nrows > 0) readout(b_hi - 1);
  }  // elementwise warps
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ============================================================= dq, pipelined
// Lp == 256.  Units of 32 keys (eight per batch row) flow through three TMEM
// regions [S 32 | dP 32] at 64*(u%3); the S/dP MMAs run two units ahead of
// the elementwise pass.  dS (bf16 pairs) is packed into the region's first
// 16 columns (a per-lane-quadrant named barrier separates the loads from the
// in-place stores of the four warps sharing those TMEM lanes), then:
//   dQ   += dS K_u          (TS MMA; row-parity accumulators at 192 + 32*(r&1))
//   dbias[ui] += dS I_32    (TS MMA against a 32x32 identity in smem: the
//                            batch-row sum of dS accumulates in TMEM cols
//                            256 + 32*ui for the whole chunk)
// so no thread keeps a dbias partial in registers and two dedicated issuer
// warps fit the register budget: warp 16 issues the S/dP MMAs (each one as
// soon as its region's previous dQ/dbias MMAs completed), warp 17 the
// dQ/dbias MMAs and the TMA loads (warp-collective, one elected lane).
// dbias sums bf16-rounded dS (the values the dQ MMA consumes).
template <bool ROWBOX>
__device__ __forceinline__ void bias_row8(const uint8_t *sb, int row, int k0, float (&out)[8]) {
  if constexpr (ROWBOX) {
    const uint8_t *base = sb + (k0 >> 5) * 16384 + row * 128;
    const int c0 = (k0 & 31) >> 2;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float4 v = *reinterpret_cast<const float4 *>(base + (((c0 + c) ^ (row & 7)) << 4));
      out[4 * c] = v.x; out[4 * c + 1] = v.y; out[4 * c + 2] = v.z; out[4 * c + 3] = v.w;
    }
  } else {
    const float *p = reinterpret_cast<const float *>(sb) + k0 * 128 + row;
#pragma unroll
    for (int j = 0; j < 8; ++j) out[j] = p[j * 128];
  }
}

template <int D, int BIASMODE, int NU, int EWW>
__global__ void __launch_bounds__(32 * EWW + 64, 1)
attn_bwd_dq_pipe_kernel(const __grid_constant__ CUtensorMap mQ,
                        const __grid_constant__ CUtensorMap mK,
                        const __grid_constant__ CUtensorMap mV,
                        const __grid_constant__ CUtensorMap mdO,
                        const __grid_constant__ CUtensorMap mB, const AttnTcArgs a) {
  evo_pdl_enter();
  constexpr int UW = 32, LPC = NU * UW;           // Lp = 32 NU (128 or 256)
  constexpr int QW = EWW / 4;                     // elementwise warps per lane quadrant
  constexpr int KPT = UW / QW;                    // keys per thread per unit
  constexpr int NEW = 32 * EWW;                   // elementwise threads
  constexpr uint32_t TILE = QT * Sw<D>::bytes;
  constexpr uint32_t FULL = LPC * Sw<D>::bytes;
  constexpr uint32_t ROWB = 2 * TILE + 2 * FULL;  // Q | dO | K | V of one batch row
  constexpr int NBUF = BIASMODE ? 2 : 3;          // see the dk/dv kernel
  constexpr bool TB = BIASMODE == 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t *sBias = smem_raw;
  uint8_t *sRow = sBias + (BIASMODE ? BIAS_BYTES : 0);
  uint8_t *sI = sRow + NBUF * ROWB;  // 32 x 32 bf16 identity, K-major SW64
  // 0 bias, 1-2 row data (row parity), 3-5 S/dP MMAs (region), 6-7 row's
  // last dQ MMAs (row parity), 8-9 and 14 unit packed (16 warp arrivals, by
  // region u % 3), 10-12 unit's MMAs done (region), 13 chunk's last MMAs
  // (row-data barriers 1..NBUF; the others shifted by 1 when NBUF == 3)
  uint64_t *bars_all = reinterpret_cast<uint64_t *>(sI + 2048);
  uint64_t *rowbar = bars_all + 1;
  uint64_t *bars = bars_all + (NBUF - 2);
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars_all + 16);
  // unit-done barriers by region (u % 3), see the dk/dv kernel
  auto ewdone = [&](int rg) -> uint64_t * { return rg < 2 ? &bars[8 + rg] : &bars[14]; };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = (warp & 3) * 32 + lane;  // query row in the tile
  const int qr = warp >> 2;              // KPT-key slice of each unit
  const int q0 = blockIdx.x * QT, h = blockIdx.y;
  const int L = a.L;
  const int q = q0 + t;
  const bool qv = q < L;
  const int64_t b_lo = blockIdx.z * a.chunk;
  const int64_t b_hi = min(a.nb, b_lo + a.chunk);
  const int64_t nrows = b_hi - b_lo;
  const int64_t U = nrows > 0 ? nrows * NU : 0;

  if (tid == NEW) {
    for (int i = 0; i < 16; ++i) {
      const bool ewd = &bars_all[i] == ewdone(0) || &bars_all[i] == ewdone(1) ||
                       &bars_all[i] == ewdone(2);
      mbar_init(&bars_all[i], ewd ? EWW : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (BIASMODE) load_bias_tile<TB>(sBias, &mB, &bars_all[0], h, q0, LPC);
  }
  // identity: row n has bf16 1.0 at column n (SW64: 16-byte chunk c of row n
  // sits at chunk c ^ ((n >> 1) & 3))
  for (int i = tid; i < 2048 / 16; i += blockDim.x) {
    const int n = i >> 2, c = i & 3;  // physical chunk c of row n
    uint4 z = make_uint4(0u, 0u, 0u, 0u);
    const int lc = c ^ ((n >> 1) & 3);  // logical chunk stored here
    if (lc == (n >> 3)) {
      const int pos = n & 7;  // bf16 slot within the chunk
      uint32_t w = 0x3f80u << (16 * (pos & 1));
      if ((pos >> 1) == 0) z.x = w; else if ((pos >> 1) == 1) z.y = w;
      else if ((pos >> 1) == 2) z.z = w; else z.w = w;
    }
    *reinterpret_cast<uint4 *>(sI + n * 64 + c * 16) = z;
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(tslot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  auto rowbuf = [&](int64_t r) -> uint8_t * { return sRow + ((r - b_lo) % NBUF) * ROWB; };

  if (warp >= EWW) {
    // ------------------------------------------------------------ issuers
    const uint32_t idesc_s = idesc_bf16(128, UW, false, false);
    const uint32_t idesc_o = idesc_bf16(128, D, false, true);
    const uint32_t idesc_i = idesc_bf16(128, 32, false, false);
    auto load_row = [&](int64_t r) {
      uint8_t *rb = rowbuf(r);
      uint64_t *bar = &rowbar[(r - b_lo) % NBUF];
      mbar_expect_tx(bar, ROWB);
      tma_load_4d(rb, &mQ, bar, 0, q0, (int)r, h);
      tma_load_4d(rb + TILE, &mdO, bar, 0, q0, (int)r, h);
      tma_load_4d(rb + 2 * TILE, &mK, bar, 0, 0, (int)r, h);
      tma_load_4d(rb + 2 * TILE + FULL, &mV, bar, 0, 0, (int)r, h);
    };
    if (warp == EWW && nrows > 0) {
      // S/dP MMAs: unit v into region v%3 once unit v-3's dQ/dbias MMAs
      // (the region's previous readers) completed
      if (lane == 0)
        for (int i = 0; i < NBUF && i < nrows; ++i) load_row(b_lo + i);
      __syncwarp();
      int reg = 0;
      uint32_t ph3 = 0;  // bit i: parity of region i's dQ/dbias-done barrier
      for (int v = 0; v < (int)U; ++v) {
        const int64_t r = b_lo + v / NU;
        const int ui = v % NU;
        if (v >= 3) {
          mbar_wait(&bars[10 + reg], (ph3 >> reg) & 1u);
          ph3 ^= 1u << reg;
        }
        if (ui == 0) mbar_wait(&rowbar[(r - b_lo) % NBUF], (uint32_t)(((r - b_lo) / NBUF) & 1));
        fence_after();
        const uint32_t sQ = smem_u32(rowbuf(r)), sdO = sQ + TILE;
        const uint32_t sK = sQ + 2 * TILE + ui * UW * Sw<D>::bytes, sV = sK + FULL;
        const uint32_t d = tmem + reg * 64;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_bf16_el(d, desc_kmajor_tile<D>(sQ, ks), desc_kmajor_tile<D>(sK, ks), idesc_s,
                       ks > 0);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_bf16_el(d + 32, desc_kmajor_tile<D>(sdO, ks), desc_kmajor_tile<D>(sV, ks),
                       idesc_s, ks > 0);
        umma_commit_el(&bars[3 + reg]);
        reg = reg == 2 ? 0 : reg + 1;
      }
    } else if (warp == EWW + 1 && nrows > 0) {
      // dQ / dbias MMAs of unit u once all EWW warps packed its dS
      const uint32_t sIa = smem_u32(sI);
      int reg = 0;
      for (int u = 0; u < (int)U; ++u) {
        const int64_t r = b_lo + u / NU;
        const int ui = u % NU;
        const int rp = (int)((r - b_lo) & 1);
        mbar_wait(ewdone((int)(u % 3)), (uint32_t)((u / 3) & 1));
        fence_after();
        if (ui == 0 && r > b_lo && r - 1 + NBUF < b_hi) {  // row r-1 read back: buffer free
          if (lane == 0) load_row(r - 1 + NBUF);
          __syncwarp();
        }
        const uint32_t sK = smem_u32(rowbuf(r)) + 2 * TILE;
        const uint32_t reg_col = tmem + reg * 64;
        const uint32_t acc = tmem + 192 + rp * 32;
        const uint32_t dba = tmem + 256 + ui * 32;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
          umma_bf16_ts_el(acc, reg_col + ks * 8, desc_mnmajor_tile<D>(sK, ui * 2 + ks), idesc_o,
                          (ui > 0 || ks > 0) ? 1u : 0u);
        if (BIASMODE) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            umma_bf16_ts_el(dba, reg_col + ks * 8, desc_kmajor_tile<32>(sIa, ks), idesc_i,
                            (r > b_lo || ks > 0) ? 1u : 0u);
        }
        if (ui == NU - 1) umma_commit_el(&bars[6 + rp]);
        umma_commit_el(&bars[10 + reg]);
        reg = reg == 2 ? 0 : reg + 1;
      }
      umma_commit_el(&bars[13]);  // every MMA of the chunk (dbias sums) done
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ elementwise
    auto readout = [&](int64_t rr) {  // dq row of batch row rr -> global
      const int pp = (int)((rr - b_lo) & 1);
      mbar_wait(&bars[6 + pp], (uint32_t)(((rr - b_lo) >> 1) & 1));
      fence_after();
      constexpr int QD = D / QW;
      const uint32_t acc = lane_addr + 192 + pp * 32;
      uint32_t v[16];
      if constexpr (QD == 16) {
        tmem_ld16_nw(acc + qr * 16, v);
      } else if constexpr (QD == 8) {
        tmem_ld8_nw(acc + qr * 8, *reinterpret_cast<uint32_t(*)[8]>(v));
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(acc + qr * 4));
      }
      tmem_wait_ld();
      if (qv) {
        bf16 *dst = a.dq + rr * a.sb + (int64_t)q * a.sl + h * D + qr * QD;
        if constexpr (QD == 16) {
          uint32_t w8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            w8[j] = pack2(__uint_as_float(v[2 * j]) * a.scale,
                          __uint_as_float(v[2 * j + 1]) * a.scale);
          *reinterpret_cast<uint4 *>(dst) = make_uint4(w8[0], w8[1], w8[2], w8[3]);
          *reinterpret_cast<uint4 *>(dst + 8) = make_uint4(w8[4], w8[5], w8[6], w8[7]);
        } else if constexpr (QD == 8) {
          uint32_t w4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            w4[j] = pack2(__uint_as_float(v[2 * j]) * a.scale,
                          __uint_as_float(v[2 * j + 1]) * a.scale);
          *reinterpret_cast<uint4 *>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        } else {
          uint32_t w2[2];
#pragma unroll
          for (int j = 0; j < 2; ++j)
            w2[j] = pack2(__uint_as_float(v[2 * j]) * a.scale,
                          __uint_as_float(v[2 * j + 1]) * a.scale);
          *reinterpret_cast<uint2 *>(dst) = make_uint2(w2[0], w2[1]);
        }
      }
    };
    if (BIASMODE) {
      mbar_wait(&bars_all[0], 0);
      if constexpr (TB) transpose_scale_bias_boxes<NEW>(sBias, LPC / 32, tid);
      else scale_tile(sBias, (LPC / 32) * 16384 / 16, NEW);
      named_bar_sync(1, NEW);
    }
    const float sc_l2 = a.scale * LOG2E;
    float lse_n = 0.f, Dq_n = 0.f;
    if (qv && nrows > 0) {
      lse_n = a.lse[(b_lo * a.H + h) * (int64_t)L + q];
      Dq_n = a.Dq[(b_lo * a.H + h) * (int64_t)L + q];
    }
    float lse_l2 = 0.f, Dq = 0.f;
    int reg = 0;
    uint32_t ph3 = 0;  // bit i: parity of region i's S/dP barrier
    const int U32 = (int)U;
    for (int u = 0; u < U32; ++u) {
      const int64_t r = b_lo + u / NU;
      const int ui = u % NU;
      if (ui == 0) {
        lse_l2 = lse_n * LOG2E;
        Dq = Dq_n;
        if (qv && r + 1 < b_hi) {
          lse_n = a.lse[((r + 1) * a.H + h) * (int64_t)L + q];
          Dq_n = a.Dq[((r + 1) * a.H + h) * (int64_t)L + q];
        }
      }
      mbar_wait(&bars[3 + reg], (ph3 >> reg) & 1u);
      ph3 ^= 1u << reg;
      fence_after();
      const uint32_t rb = lane_addr + reg * 64;
      const int c0 = qr * KPT;
      const int kb = ui * UW + c0;  // first key of this thread's KPT
      uint32_t sv[KPT], dv[KPT];
      float bb[KPT];
      if constexpr (KPT == 16) {
        tmem_ld16_nw(rb + c0, sv);
        tmem_ld16_nw(rb + 32 + c0, dv);
        tmem_wait_ld();
        if (BIASMODE) bias_row16<true>(sBias, t, kb, bb);  // row boxes in both modes
      } else {
        tmem_ld8_nw(rb + c0, sv);
        tmem_ld8_nw(rb + 32 + c0, dv);
        tmem_wait_ld();
        if (BIASMODE) bias_row8<true>(sBias, t, kb, bb);
      }
      const bool full = qv && kb + KPT <= L;
      uint32_t pk[KPT / 2];
      if (full) {  // interior units: no per-element mask
#pragma unroll
        for (int j = 0; j < KPT; j += 2) {
          float ds[2];
#pragma unroll
          for (int w2 = 0; w2 < 2; ++w2) {
            float x = fmaf(__uint_as_float(sv[j + w2]), sc_l2, -lse_l2);
            if (BIASMODE) x += bb[j + w2];
            ds[w2] = ex2(x) * (__uint_as_float(dv[j + w2]) - Dq);
          }
          pk[j >> 1] = pack2(ds[0], ds[1]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < KPT; j += 2) {
          float ds[2];
#pragma unroll
          for (int w2 = 0; w2 < 2; ++w2) {
            float x = fmaf(__uint_as_float(sv[j + w2]), sc_l2, -lse_l2);
            if (BIASMODE) x += bb[j + w2];
            const float e = ex2(x);
            const float p = (qv && kb + j + w2 < L) ? e : 0.f;
            ds[w2] = p * (__uint_as_float(dv[j + w2]) - Dq);
          }
          pk[j >> 1] = pack2(ds[0], ds[1]);
        }
      }
      // the QW warps of this lane quadrant have loaded the region's S
      // columns before any of them overwrites them with packed dS
      named_bar_sync(2 + (warp & 3), 32 * QW);
      if constexpr (KPT == 16) {
        tmem_st8(rb + qr * 8, pk);
      } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                         rb + qr * 4),
                     "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3])
                     : "memory");
      }
      if (ui == 0 && r > b_lo) readout(r - 1);
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ewdone(reg));
      reg = reg == 2 ? 0 : reg + 1;
    }
    if (nrows > 0) {
      readout(b_hi - 1);
      // dbias partial of this chunk: TMEM cols 256 + key -> global
      mbar_wait(&bars[13], 0);
      fence_after();
      if (a.dbias_part != nullptr) {
        float *dst = a.dbias_part + (int64_t)blockIdx.z * a.H * a.bh +
                     (int64_t)h * a.bh + (int64_t)q * a.bq;
#pragma unroll
        for (int c = 0; c < 8 / QW; ++c) {
          const int kb = qr * (256 / QW) + 32 * c;
          uint32_t v[32];
          tmem_ld32(lane_addr + 256 + kb, v);
          if (qv) {
            if (a.bk == 1 && kb + 32 <= L && ((reinterpret_cast<uintptr_t>(dst + kb) & 15) == 0)) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4 *>(dst + kb + j) =
                    make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (kb + j < L) dst[(int64_t)(kb + j) * a.bk] = __uint_as_float(v[j]);
            }
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ===================================================================== host
// 4-D map over a (b, l, h, d) strided bf16 buffer: dims {D, L, nb, H}.
bool head_map(CUtensorMap *m, const void *base, int D, int L, int64_t nb, int H, int64_t sl,
              int64_t sb, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)L, (cuuint64_t)nb, (cuuint64_t)H};
  cuuint64_t strides[3] = {(cuuint64_t)sl * 2, (cuuint64_t)sb * 2, (cuuint64_t)D * 2};
  cuuint32_t box[4] = {(cuuint32_t)D, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMapSwizzle sw = D == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : (D == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

AttnTcArgs make_args(const evo_attn_desc *d) {
  AttnTcArgs a;
  a.nb = d->nb; a.H = d->H; a.L = d->L; a.Lp = (d->L + 15) / 16 * 16; a.D = d->D;
  a.scale = d->scale;
  a.g = reinterpret_cast<const bf16 *>(d->g);
  a.sb = d->sb; a.sl = d->sl;
  a.o = reinterpret_cast<bf16 *>(d->o); a.gm = reinterpret_cast<bf16 *>(d->gm);
  a.o_sb = d->o_sb; a.o_sl = d->o_sl;
  a.bias = d->bias; a.bh = d->bh; a.bq = d->bq; a.bk = d->bk;
  a.lse = d->lse;
  a.dO = nullptr; a.Dq = nullptr;
  a.dq = reinterpret_cast<bf16 *>(d->dq); a.dk = reinterpret_cast<bf16 *>(d->dk);
  a.dv = reinterpret_cast<bf16 *>(d->dv);
  a.dbias_part = nullptr; a.chunk = 1;
  return a;
}


// 3-D map over the fp32 bias buffer: plain {k, q, h} / transposed {q, k, h}
bool bias_map(CUtensorMap *m, const evo_attn_desc *d, bool transposed) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const int L = d->L;
  cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)L, (cuuint64_t)d->H};
  cuuint64_t strides[2];
  cuuint32_t box[3], es[3] = {1, 1, 1};
  if (!transposed) {  // inner = k (stride 1), outer = q (stride bq)
    strides[0] = (cuuint64_t)d->bq * 4;
    box[0] = 32; box[1] = 128;
  } else {            // inner = q (stride 1), outer = k (stride bk)
    strides[0] = (cuuint64_t)d->bk * 4;
    box[0] = 128; box[1] = 32;
  }
  strides[1] = (cuuint64_t)d->bh * 4;
  box[2] = 1;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(d->bias), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            transposed ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The per-chunk dbias partials are [H][bh] images of the bias layout (the
// reducer writes H*bh elements, padding between rows included), so the
// rows must tile one head's span: bh >= L * (row stride).
int bias_mode(const evo_attn_desc *d) {
  if (!d->bias) return 0;
  if (d->bh < (int64_t)d->L * std::max(d->bq, d->bk)) return -1;
  if (d->bk == 1 && d->bq % 4 == 0 && d->bh % 4 == 0) return 1;
  if (d->bq == 1 && d->bk % 4 == 0 && d->bh % 4 == 0) return 2;
  return -1;
}

// Batch-row chunks per (tile, head) so the whole grid is ONE wave of
// one-CTA-per-SM blocks (a 149th CTA would double the kernel time).
int64_t row_chunks(const evo_attn_desc *d) {
  int64_t tiles = (int64_t)d->H * ((d->L + QT - 1) / QT);
  int64_t want = (int64_t)num_sms() / tiles;
  return std::max<int64_t>(1, std::min<int64_t>(d->nb, want));
}

// byte offset of the gate-bias partials in the backward workspace (after
// dO, Dq and the dbias chunk partials); sized for SMs*8 prep blocks
size_t gate_part_offset(const evo_attn_desc *d) {
  const int64_t span = (d->nb - 1) * d->o_sb + (int64_t)(d->L - 1) * d->o_sl + (int64_t)d->H * d->D;
  const size_t dO_pad = ((size_t)span * 2 + 255) / 256 * 256;
  const size_t Dq_pad = ((size_t)d->nb * d->H * d->L * 4 + 255) / 256 * 256;
  size_t part = 0;
  if (d->dbias) {
    int64_t nch = row_chunks(d);
    int64_t chunk = (d->nb + nch - 1) / nch;
    nch = (d->nb + chunk - 1) / chunk;
    part = ((size_t)nch * d->H * d->bh * 4 + 255) / 256 * 256;
  }
  return dO_pad + Dq_pad + part;
}

template <int D, int BM_>
int fwd_launch_mode(const evo_attn_desc *d, cudaStream_t st) {
  AttnTcArgs a = make_args(d);
  a.Lp = (d->L + 63) / 64 * 64;  // softmax passes take 64-key steps (masked beyond L)
  CUtensorMap mq, mk, mv, mb;
  if (!head_map(&mq, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !head_map(&mk, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, a.Lp) ||
      !head_map(&mv, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, a.Lp))
    return EVO_EUNSUP;
  if (BM_) {
    if (!bias_map(&mb, d, BM_ == 2)) return EVO_EUNSUP;
  } else {
    mb = mq;  // unused
  }
  int64_t nch = row_chunks(d);
  a.chunk = (d->nb + nch - 1) / nch;
  nch = (d->nb + a.chunk - 1) / a.chunk;
  const size_t smem = 1024 + (BM_ ? BIAS_BYTES : 0) +
                      2 * ((size_t)QT * 2 * D + 2 * 256 * 2 * D) + 128;
  dim3 grid((d->L + QT - 1) / QT, d->H, (unsigned)nch);
  if ((a.Lp == 256 || a.Lp == 128) && D <= 32 && !g_attn_no_pipe) {
    const size_t smem2 = (BM_ ? BIAS_BYTES : 0) + 2 * ((size_t)QT * 2 * D + 2 * (size_t)a.Lp * 2 * D) +
                         2 * 2 * 4 * 128 * 4 + 13 * 8 + 16;
    if (a.Lp == 256) {
      EVO_MAX_SMEM_ONCE((attn_fwd_tc2_kernel<D, BM_, 256>));
      launch_k(attn_fwd_tc2_kernel<D, BM_, 256>, grid, 544, smem2, st, mq, mk, mv, mb, a);
    } else {
      EVO_MAX_SMEM_ONCE((attn_fwd_tc2_kernel<D, BM_, 128>));
      launch_k(attn_fwd_tc2_kernel<D, BM_, 128>, grid, 544, smem2, st, mq, mk, mv, mb, a);
    }
    EVO_LAUNCHED("attn_fwd_tc2_kernel");
    return EVO_OK;
  }
  EVO_MAX_SMEM_ONCE((attn_fwd_tc_kernel<D, BM_>));
  launch_k(attn_fwd_tc_kernel<D, BM_>, grid, 256, smem, st, mq, mk, mv, mb, a);
  EVO_LAUNCHED("attn_fwd_tc_kernel");
  return EVO_OK;
}

template <int D>
int fwd_launch(const evo_attn_desc *d, cudaStream_t st) {
  switch (bias_mode(d)) {
    case 0: return fwd_launch_mode<D, 0>(d, st);
    case 1: return fwd_launch_mode<D, 1>(d, st);
    case 2: return fwd_launch_mode<D, 2>(d, st);
  }
  return EVO_EUNSUP;
}

// bias map for the dk/dv kernel: tiles over (all queries) x (128 keys)
bool bias_map_k(CUtensorMap *m, const evo_attn_desc *d, bool kcontig) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const int L = d->L;
  cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)L, (cuuint64_t)d->H};
  cuuint64_t strides[2];
  cuuint32_t box[3], es[3] = {1, 1, 1};
  if (kcontig) {  // plain: inner = k (stride 1), outer = q (stride bq); box {128 k, 32 q}
    strides[0] = (cuuint64_t)d->bq * 4;
    box[0] = 128; box[1] = 32;
  } else {        // transposed: inner = q (stride 1), outer = k (stride bk); box {32 q, 128 k}
    strides[0] = (cuuint64_t)d->bk * 4;
    box[0] = 32; box[1] = 128;
  }
  strides[1] = (cuuint64_t)d->bh * 4;
  box[2] = 1;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(d->bias), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            kcontig ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, int BM_>
int bwd_launch_mode(const evo_attn_desc *d, cudaStream_t st) {
  AttnTcArgs a = make_args(d);
  a.Lp = (d->L + 63) / 64 * 64;  // the backward works in 64-key granules
  const int Lp = a.Lp;
  // workspace: dO (o's strides) | Dq [nb, H, L] | dbias chunk partials
  const int64_t span = (d->nb - 1) * d->o_sb + (int64_t)(d->L - 1) * d->o_sl + (int64_t)d->H * D;
  const size_t dO_pad = ((size_t)span * 2 + 255) / 256 * 256;
  const size_t Dq_pad = ((size_t)d->nb * d->H * d->L * 4 + 255) / 256 * 256;
  int64_t nch = row_chunks(d);
  const int64_t chunk = (d->nb + nch - 1) / nch;
  nch = (d->nb + chunk - 1) / chunk;
  uint8_t *ws = reinterpret_cast<uint8_t *>(d->workspace);
  bf16 *dObuf = reinterpret_cast<bf16 *>(ws);
  float *Dq = reinterpret_cast<float *>(ws + dO_pad);
  float *part = d->dbias ? reinterpret_cast<float *>(ws + dO_pad + Dq_pad) : nullptr;
  {
    int64_t total = d->nb * (int64_t)d->L * d->H * (D / 8);
    const bool fuse_gb = d->dgate_bias && (256 % (d->H * (D / 8)) == 0);
    int blocks = (int)std::min<int64_t>((total + 255) / 256,
                                        (int64_t)num_sms() * (fuse_gb ? 8 : 32));
    float *gpart = fuse_gb ? reinterpret_cast<float *>(ws + gate_part_offset(d)) : nullptr;
    launch_k(attn_bwd_prep_kernel<D>, blocks, 256, 0, st, a, reinterpret_cast<const bf16 *>(d->dgm),
                                                     dObuf, reinterpret_cast<bf16 *>(d->dgpre), Dq,
                                                     gpart, static_cast<float *>(nullptr));
    EVO_LAUNCHED("attn_bwd_prep_kernel");
    if (d->dgate_bias) {
      if (fuse_gb) {
        const int rc = colsum_partials(blocks, (int64_t)d->H * D, gpart, d->dgate_bias, 0, st);
        if (rc != EVO_OK) return rc;
      } else {
        EVO_REQUIRE(false, EVO_EUNSUP, "attention bwd: gate-bias sums need 256 %% (H*D/8) == 0");
      }
    }
  }
  a.dO = dObuf;
  a.Dq = Dq;
  a.dbias_part = part;
  a.chunk = chunk;
  CUtensorMap mq, mk, mv, mdo, mqa, mdoa, mkt, mvt, mb, mbk;
  if (!head_map(&mq, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !head_map(&mk, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, Lp) ||
      !head_map(&mv, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, Lp) ||
      !head_map(&mdo, dObuf, D, d->L, d->nb, d->H, d->o_sl, d->o_sb, QT) ||
      !head_map(&mqa, d->q, D, d->L, d->nb, d->H, d->sl, d->sb, Lp) ||
      !head_map(&mdoa, dObuf, D, d->L, d->nb, d->H, d->o_sl, d->o_sb, Lp) ||
      !head_map(&mkt, d->k, D, d->L, d->nb, d->H, d->sl, d->sb, QT) ||
      !head_map(&mvt, d->v, D, d->L, d->nb, d->H, d->sl, d->sb, QT))
    return EVO_EUNSUP;
  if (BM_) {
    if (!bias_map(&mb, d, BM_ == 2) || !bias_map_k(&mbk, d, BM_ == 1)) return EVO_EUNSUP;
  } else {
    mb = mq;
    mbk = mq;
  }
  const int tiles = (d->L + QT - 1) / QT;
  const bool pipe = (Lp == 256 || Lp == 128) && !g_attn_no_pipe;
  const size_t nbuf = BM_ ? 2 : 3;
  if (pipe) {
    const size_t smem = (BM_ ? BIAS_BYTES : 0) +
                        nbuf * (2 * (size_t)QT * 2 * D + 2 * (size_t)Lp * 2 * D) + 2048 + 16 * 8 +
                        16;
    dim3 grid(tiles, d->H, (unsigned)nch);
    if (g_dq_eww == 16) {
      if (Lp == 256) {
        EVO_MAX_SMEM_ONCE((attn_bwd_dq_pipe_kernel<D, BM_, 8, 16>));
        launch_k(attn_bwd_dq_pipe_kernel<D, BM_, 8, 16>, grid, 576, smem, st, mq, mk, mv, mdo, mb, a);
      } else {
        EVO_MAX_SMEM_ONCE((attn_bwd_dq_pipe_kernel<D, BM_, 4, 16>));
        launch_k(attn_bwd_dq_pipe_kernel<D, BM_, 4, 16>, grid, 576, smem, st, mq, mk, mv, mdo, mb, a);
      }
    } else {
      if (Lp == 256) {
        EVO_MAX_SMEM_ONCE((attn_bwd_dq_pipe_kernel<D, BM_, 8, 8>));
        launch_k(attn_bwd_dq_pipe_kernel<D, BM_, 8, 8>, grid, 320, smem, st, mq, mk, mv, mdo, mb, a);
      } else {
        EVO_MAX_SMEM_ONCE((attn_bwd_dq_pipe_kernel<D, BM_, 4, 8>));
        launch_k(attn_bwd_dq_pipe_kernel<D, BM_, 4, 8>, grid, 320, smem, st, mq, mk, mv, mdo, mb, a);
      }
    }
    EVO_LAUNCHED("attn_bwd_dq_pipe_kernel");
  } else {
    const size_t smem = 1024 + (BM_ ? BIAS_BYTES : 0) + 2 * (size_t)QT * 2 * D +
                        3 * 256 * 2 * D + 128;
    EVO_MAX_SMEM_ONCE((attn_bwd_dq_tc_kernel<D, BM_>));
    dim3 grid(tiles, d->H, (unsigned)nch);
    launch_k(attn_bwd_dq_tc_kernel<D, BM_>, grid, 512, smem, st, mq, mk, mv, mdo, mb, a);
    EVO_LAUNCHED("attn_bwd_dq_tc_kernel");
  }
  if (pipe) {
    const size_t smem = (BM_ ? BIAS_BYTES : 0) +
                        nbuf * (2 * (size_t)QT * 2 * D + 2 * (size_t)Lp * 2 * D) + 2 * 256 * 4 +
                        15 * 8 + 16;
    dim3 grid(tiles, d->H, (unsigned)nch);
    if (Lp == 256) {
      EVO_MAX_SMEM_ONCE((attn_bwd_dkv_pipe_kernel<D, BM_, 4>));
      launch_k(attn_bwd_dkv_pipe_kernel<D, BM_, 4>, grid, 576, smem, st, mkt, mvt, mqa, mdoa, mbk, a);
    } else {
      EVO_MAX_SMEM_ONCE((attn_bwd_dkv_pipe_kernel<D, BM_, 2>));
      launch_k(attn_bwd_dkv_pipe_kernel<D, BM_, 2>, grid, 576, smem, st, mkt, mvt, mqa, mdoa, mbk, a);
    }
    EVO_LAUNCHED("attn_bwd_dkv_pipe_kernel");
  } else {
    const size_t smem = 1024 + (BM_ ? BIAS_BYTES : 0) + 4 * 256 * 2 * D +
                        2 * (size_t)QT * 2 * D + 2 * 256 * 4 + 128;
    EVO_MAX_SMEM_ONCE((attn_bwd_dkv_tc_kernel<D, BM_>));
    dim3 grid(tiles, d->H, (unsigned)nch);
    launch_k(attn_bwd_dkv_tc_kernel<D, BM_>, grid, 512, smem, st, mkt, mvt, mqa, mdoa, mbk, a);
    EVO_LAUNCHED("attn_bwd_dkv_tc_kernel");
  }
  if (d->dbias)
    return reduce_lead(EVO_F32, nch, 1, (int64_t)d->H * d->bh, part, d->dbias, 0, 1, 0, st);
  return EVO_OK;
}

template <int D>
int bwd_launch(const evo_attn_desc *d, cudaStream_t st) {
  switch (bias_mode(d)) {
    case 0: return bwd_launch_mode<D, 0>(d, st);
    case 1: return bwd_launch_mode<D, 1>(d, st);
    case 2: return bwd_launch_mode<D, 2>(d, st);
  }
  return EVO_EUNSUP;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

bool attention_tc_accepts(const evo_attn_desc *d) {
  if (d->dtype != EVO_BF16) return false;
  if (bias_mode(d) < 0) return false;
  // D=64 would need 229 KB of smem in the dk/dv kernel: SIMT path
  if (!(d->D == 16 || d->D == 32)) return false;
  if (d->L < 1 || d->L > 256 || d->nb < 1 || d->nb > 65535) return false;
  if (d->sl % 8 || d->sb % 8 || d->o_sl % 8 || d->o_sb % 8) return false;
  if (!aligned16(d->q) || !aligned16(d->k) || !aligned16(d->v) || !aligned16(d->g) ||
      !aligned16(d->o))
    return false;
  if (d->gm && !aligned16(d->gm)) return false;
  if (d->dq && !(aligned16(d->dq) && aligned16(d->dk) && aligned16(d->dv) && aligned16(d->dgpre)))
    return false;
  if (d->dgm && !aligned16(d->dgm)) return false;
  return tc::encode_fn() != nullptr;
}

size_t attention_tc_bwd_ws(const evo_attn_desc *d) {
  if (!attention_tc_accepts(d)) return 0;
  if (d->dgate_bias)
    return gate_part_offset(d) + (size_t)num_sms() * 8 * d->H * d->D * 4;
  // dO uses o's strides: size it by the extent those strides span.
  const int64_t span = (d->nb - 1) * d->o_sb + (int64_t)(d->L - 1) * d->o_sl + (int64_t)d->H * d->D;
  const size_t dO_pad = ((size_t)span * 2 + 255) / 256 * 256;
  const size_t Dq_pad = ((size_t)d->nb * d->H * d->L * 4 + 255) / 256 * 256;
  size_t part = 0;
  if (d->dbias) {
    int64_t nch = row_chunks(d);
    int64_t chunk = (d->nb + nch - 1) / nch;
    nch = (d->nb + chunk - 1) / chunk;
    part = (size_t)nch * d->H * d->bh * 4;
  }
  return dO_pad + Dq_pad + part;
}

int attention_tc_fwd(const evo_attn_desc *d, cudaStream_t st) {
  switch (d->D) {
    case 16: return fwd_launch<16>(d, st);
    case 32: return fwd_launch<32>(d, st);
    case 64: return fwd_launch<64>(d, st);
  }
  return EVO_EUNSUP;
}

// The backward's prep pass for other kernels (attention_flash.cu): dO (o's
// strides) -> dO_out, dGpre -> d->dgpre, Dq [nb, H, L]; the gate-bias sums
// into d->dgate_bias when set (gpart: SMs*8*H*D fp32 of workspace).
int attn_prep_run(const evo_attn_desc *d, void *dO_out, float *Dq, float *gpart, float *lse2,
                  cudaStream_t st) {
  if (d->D != 8 && d->D != 16 && d->D != 32) return EVO_EUNSUP;
  AttnTcArgs a = make_args(d);
  int64_t total = d->nb * (int64_t)d->L * d->H * (d->D / 8);
  EVO_REQUIRE(total + 256LL * num_sms() * 32 < (1LL << 31), EVO_EUNSUP,
              "attention bwd prep: more than 2^31 chunks");
  const bool fuse_gb = d->dgate_bias && (256 % (d->H * (d->D / 8)) == 0);
  EVO_REQUIRE(!d->dgate_bias || fuse_gb, EVO_EUNSUP,
              "attention bwd: gate-bias sums need 256 %% (H*D/8) == 0");
  int blocks = (int)std::min<int64_t>((total + 255) / 256,
                                      (int64_t)num_sms() * (fuse_gb ? 8 : 32));
  bf16 *dO = reinterpret_cast<bf16 *>(dO_out);
  const bf16 *dgm = reinterpret_cast<const bf16 *>(d->dgm);
  bf16 *dgp = reinterpret_cast<bf16 *>(d->dgpre);
  float *gp = fuse_gb ? gpart : nullptr;
  if (d->D == 32)
    launch_k(attn_bwd_prep_kernel<32>, blocks, 256, 0, st, a, dgm, dO, dgp, Dq, gp, lse2);
  else if (d->D == 16)
    launch_k(attn_bwd_prep_kernel<16>, blocks, 256, 0, st, a, dgm, dO, dgp, Dq, gp, lse2);
  else
    launch_k(attn_bwd_prep_kernel<8>, blocks, 256, 0, st, a, dgm, dO, dgp, Dq, gp, lse2);
  EVO_LAUNCHED("attn_bwd_prep_kernel");
  if (fuse_gb) return colsum_partials(blocks, (int64_t)d->H * d->D, gp, d->dgate_bias, 0, st);
  return EVO_OK;
}

int attention_tc_bwd(const evo_attn_desc *d, cudaStream_t st) {
  EVO_REQUIRE(d->workspace && d->workspace_bytes >= attention_tc_bwd_ws(d), EVO_EARG,
              "attention bwd (tc): workspace too small");
  switch (d->D) {
    case 16: return bwd_launch<16>(d, st);
    case 32: return bwd_launch<32>(d, st);
    case 64: return bwd_launch<64>(d, st);
  }
  return EVO_EUNSUP;
}

}  // namespace evo
