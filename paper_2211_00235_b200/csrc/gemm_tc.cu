// tcgen05 / TMA / TMEM GEMM for sm_100a (bf16 operands, fp32 accumulate).
//
// C(m,n) = epi(alpha * sum_k A(m,k) B(n,k)) for strided, batched operands
// whose unit stride runs along K ("K-major") or along M/N ("MN-major").
// Every projection, weight-gradient, outer-product-mean and triangle
// contraction of the bf16 path goes through here (src/tensor.py:287-345
// and the einsums of src/evoformer.py:343-392).
//
// Structure (one CTA per SM, persistent, warp-specialised, 192 threads):
//   warp 0      TMA producer: 128B-swizzled A/B tiles -> smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused epilogue
//               (bias / relu / sigmoid / residual / strided or two-level
//               stores) -> global
// Pipelines: smem full/empty mbarriers (TMA <-> MMA) and a double-buffered
// TMEM accumulator with full/empty mbarriers (MMA <-> epilogue), so the
// epilogue of tile i overlaps the main loop of tile i+1.
#include <cuda.h>

#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "tc_common.cuh"
#include <cstdlib>

namespace evo {
namespace tc {
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}
}  // namespace tc

namespace {
using namespace tc;

constexpr int BM = 128;
constexpr int BK = 64;           // one 128-byte swizzle atom of bf16
constexpr int EPI_WARPS = 8;
constexpr int NTHREADS = 64 + 32 * EPI_WARPS;  // TMA warp, MMA warp, epilogue warps
constexpr int SMEM_A = BM * BK * 2;  // 16 KiB

struct TcParams {
  int64_t M, N, K, B2, nbatch;
  int c_aligned;
  int64_t tiles_m, tiles_n, num_tiles;
  int64_t k_chunk;
  int split;
  int a_kmajor, b_kmajor;
  int a_bat1, a_bat2, b_bat1, b_bat2;  // batch coordinate used by the map?
  uint32_t idesc;
  EpiArgs epi;
  float *partial;
  int store_mode;  // 0: thread stores, 1: TMA 2-D, 2: TMA {cdiv, N/cdiv, M}, 3: TMA 4-D
  int64_t cdiv, rdiv;
  int bias_smem;   // bias[0..N) staged in smem by the epilogue warps
  int box_w;       // TMA store box width in columns (64: bf16, 128-byte rows;
                   // 65: 64 columns as two 64-byte SW64 rows per output row)
  int res_tma;     // fp32 residual TMA-loaded into the staging boxes
};
constexpr int BIAS_SMEM_MAX = 2048;

// 32-bit index math (num_tiles < 2^31, checked on the host): the 64-bit
// divisions cost the epilogue warps ~300 instructions per tile
__device__ __forceinline__ void decode_tile(const TcParams &p, int64_t t64, int64_t &bidx,
                                            int &sp, int64_t &mt, int64_t &nt) {
  const uint32_t t = (uint32_t)t64, tn = (uint32_t)p.tiles_n, tm = (uint32_t)p.tiles_m;
  uint32_t ntl = t % tn;
  uint32_t r = t / tn;
  const uint32_t mtl = r % tm;
  // rotate n per m-row: consecutive tiles still share the A rows, but a CTA
  // striding by the grid size no longer always lands on the same n-tile
  // (148 % tiles_n == 0 would pin e.g. all sigmoid columns to 1/4 of the SMs)
  ntl = (ntl + mtl) % tn;
  r /= tm;
  sp = (int)(r % (uint32_t)p.split);
  bidx = (int64_t)(r / (uint32_t)p.split);
  mt = mtl;
  nt = ntl;
}


// Compile-time epilogue kinds (runtime residual/accumulate stay per chunk).
// EK_SPLIT: split-K partial writer (no store staging boxes, so the smem
// goes to a deeper TMA ring: the weight-gradient GEMMs are bound by the
// bytes in flight per SM, ring depth x stage size / memory latency).
enum { EK_NONE = 0, EK_BIAS = 1, EK_BIAS_RELU = 2, EK_BIAS_SIGMOID = 3, EK_SPLIT = 4 };

// sigmoid(x) = 0.5 + 0.5 tanh(x/2): one MUFU op (tanh.approx, rel. error
// ~2^-11, below the bf16 rounding of the stored gate) instead of ex2 + rcp;
// the gate columns made the epilogue MUFU-bound.  Saturates to exactly 0/1.
__device__ __forceinline__ float fast_sigmoid(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
  return fmaf(0.5f, t, 0.5f);
}

// Finish one 32-column chunk of one output row: alpha, bias, activation,
// residual, store.  Fully unrolled; vector stores when the chunk's 32
// destination elements are contiguous and aligned.
// alpha, bias and activation of one 32-column chunk (thread-per-row)
template <int EPI>
__device__ __forceinline__ void epi_math(const TcParams &p, const EpiArgs &e, const uint32_t (&v)[32],
                                         int64_t nb, float (&x)[32], const float *bias) {
  const bool full = nb + 32 <= p.N;
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = e.alpha * __uint_as_float(v[j]);
  if constexpr (EPI == EK_BIAS || EPI == EK_BIAS_RELU || EPI == EK_BIAS_SIGMOID) {
    if (full && ((reinterpret_cast<uintptr_t>(bias + nb) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 b4 = reinterpret_cast<const float4 *>(bias + nb)[j];
        x[4 * j] += b4.x; x[4 * j + 1] += b4.y; x[4 * j + 2] += b4.z; x[4 * j + 3] += b4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] += (nb + j < p.N) ? bias[nb + j] : 0.f;
    }
  }
  if constexpr (EPI == EK_BIAS_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fmaxf(x[j], 0.f);
  }
  if constexpr (EPI == EK_BIAS_SIGMOID) {
    if (nb >= e.epi_col0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = fast_sigmoid(x[j]);
    } else if (nb + 32 > e.epi_col0) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (nb + j >= e.epi_col0) x[j] = fast_sigmoid(x[j]);
    }
  }
}

template <int EPI>
__device__ __forceinline__ void epi_chunk(const TcParams &p, const EpiArgs &e, const uint32_t (&v)[32],
                                          int64_t rbase, int64_t nb, bool row_ok_g, float *stage) {
  float x[32];
  const bool full = nb + 32 <= p.N;
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = e.alpha * __uint_as_float(v[j]);
  if constexpr (EPI == EK_BIAS || EPI == EK_BIAS_RELU || EPI == EK_BIAS_SIGMOID) {
    if (full && ((reinterpret_cast<uintptr_t>(e.bias + nb) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 b4 = reinterpret_cast<const float4 *>(e.bias + nb)[j];
        x[4 * j] += b4.x; x[4 * j + 1] += b4.y; x[4 * j + 2] += b4.z; x[4 * j + 3] += b4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] += (nb + j < p.N) ? e.bias[nb + j] : 0.f;
    }
  }
  if constexpr (EPI == EK_BIAS_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fmaxf(x[j], 0.f);
  }
  if constexpr (EPI == EK_BIAS_SIGMOID) {
    if (nb >= e.epi_col0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = fast_sigmoid(x[j]);
    } else if (nb + 32 > e.epi_col0) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (nb + j >= e.epi_col0) x[j] = fast_sigmoid(x[j]);
    }
  }
  // destination: contiguous if plain unit-stride columns, or a two-level
  // column map whose inner block is a multiple of 32 with unit stride
  const IdxMap &cm = e.cmap;
  const bool contig = full && ((cm.cdiv == 0 && cm.cs == 1) ||
                               (cm.cdiv > 0 && (cm.cdiv % 32) == 0 && cm.cs0 == 1));
  const int64_t base = rbase + cm.col(nb);
  // Every lane must take the same path through the staged store (shuffles).
  const bool lane_ok = contig && p.c_aligned &&
                       ((e.dtype_c == EVO_BF16 && (base & 7) == 0 && !e.residual && !e.accumulate) ||
                        (e.dtype_c == EVO_F32 && (base & 3) == 0));
  if (__all_sync(0xffffffffu, lane_ok || !row_ok_g)) {
    // Stage the warp's 32 rows x 32 columns through padded smem, then write
    // whole contiguous row segments per store instruction.
    const int lane = threadIdx.x & 31;
    if (e.dtype_c == EVO_BF16) {
      // packed bf16 pairs, row pitch 17 words (conflict-free both ways)
      uint32_t *st32 = reinterpret_cast<uint32_t *>(stage);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
        st32[lane * 17 + j] = *reinterpret_cast<uint32_t *>(&h2);
      }
      __syncwarp();
      const int c = lane & 3;  // 8-column group
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 8 * i + (lane >> 2);
        const int64_t rb = __shfl_sync(0xffffffffu, base, r);
        const bool ok = __shfl_sync(0xffffffffu, row_ok_g ? 1 : 0, r);
        const uint32_t *src = st32 + r * 17 + 4 * c;
        if (ok)
          *reinterpret_cast<uint4 *>(reinterpret_cast<bf16 *>(e.C) + rb + 8 * c) =
              make_uint4(src[0], src[1], src[2], src[3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) stage[lane * 33 + j] = x[j];
      __syncwarp();
      const int c = lane & 7;  // 4-column group
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + (lane >> 3);
        const int64_t rb = __shfl_sync(0xffffffffu, base, r);
        const bool ok = __shfl_sync(0xffffffffu, row_ok_g ? 1 : 0, r);
        const float *src = stage + r * 33 + 4 * c;
        float4 o = make_float4(src[0], src[1], src[2], src[3]);
        if (ok) {
          float *dst = reinterpret_cast<float *>(e.C) + rb + 4 * c;
          if (e.residual) {
            float4 q = *reinterpret_cast<const float4 *>(e.residual + rb + 4 * c);
            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
          }
          if (e.accumulate) {
            float4 q = *reinterpret_cast<const float4 *>(dst);
            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
          }
          *reinterpret_cast<float4 *>(dst) = o;
        }
      }
    }
    __syncwarp();
    return;
  }
  if (!row_ok_g) return;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int64_t n = nb + j;
    if (n < p.N) epi_store(e, rbase + cm.col(n), x[j]);
  }
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(NTHREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
               const TcParams p) {
  evo_pdl_enter();
  constexpr int SMEM_B = BN * BK * 2;
  constexpr uint32_t STAGE_BYTES = SMEM_A + SMEM_B;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered accumulator
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + STAGES * SMEM_A;
  constexpr int SW_BYTES = EPI == EK_SPLIT ? 0 : EPI_WARPS * 8192;
  uint8_t *sW = sB + STAGES * SMEM_B;  // EPI_WARPS x 8 KiB, 1 KiB aligned
  uint64_t *full = reinterpret_cast<uint64_t *>(sW + SW_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  // residual boxes: per epilogue warp, one mbarrier per staging box
  uint64_t *rbar = reinterpret_cast<uint64_t *>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    prefetch_map(&tmA);
    prefetch_map(&tmB);
    if (p.store_mode >= 1 && p.store_mode <= 3) prefetch_map(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);
    }
    for (int i = 0; i < 2 * EPI_WARPS; ++i) mbar_init(&rbar[i], 1);
    if (p.res_tma) prefetch_map(&tmR);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int64_t bidx, mt, nt;
        int sp;
        decode_tile(p, t, bidx, sp, mt, nt);
        const int b1 = (int)(bidx / p.B2), b2 = (int)(bidx % p.B2);
        const int ab1 = p.a_bat1 ? b1 : 0, ab2 = p.a_bat2 ? b2 : 0;
        const int bb1 = p.b_bat1 ? b1 : 0, bb2 = p.b_bat2 ? b2 : 0;
        const int64_t k_lo = sp * p.k_chunk;
        const int64_t k_hi = min(p.K, k_lo + p.k_chunk);
        const int m0 = (int)(mt * BM), n0 = (int)(nt * BN);
        for (int64_t k = k_lo; k < k_hi; k += BK) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          uint8_t *a_dst = sA + stage * SMEM_A;
          uint8_t *b_dst = sB + stage * SMEM_B;
          if (p.a_kmajor) {
            tma_load_4d(a_dst, &tmA, &full[stage], (int)k, m0, ab1, ab2);
          } else {
#pragma unroll
            for (int h = 0; h < BM / 64; ++h)
              tma_load_4d(a_dst + h * 8192, &tmA, &full[stage], m0 + 64 * h, (int)k, ab1, ab2);
          }
          if (p.b_kmajor) {
            tma_load_4d(b_dst, &tmB, &full[stage], (int)k, n0, bb1, bb2);
          } else {
#pragma unroll
            for (int h = 0; h < BN / 64; ++h)
              tma_load_4d(b_dst + h * 8192, &tmB, &full[stage], n0 + 64 * h, (int)k, bb1, bb2);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      const uint32_t a_lbo = p.a_kmajor ? 16u : 8192u;
      const uint32_t b_lbo = p.b_kmajor ? 16u : 8192u;
      const uint32_t a_kstep = p.a_kmajor ? 32u : 2048u;  // bytes per 16-wide K slice
      const uint32_t b_kstep = p.b_kmajor ? 32u : 2048u;
      for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int64_t bidx, mt, nt;
        int sp;
        decode_tile(p, t, bidx, sp, mt, nt);
        const int64_t k_lo = sp * p.k_chunk;
        const int64_t k_hi = min(p.K, k_lo + p.k_chunk);
        mbar_wait(&tempty[acc], aphase ^ 1);
        fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        uint32_t first = 1;
        for (int64_t k = k_lo; k < k_hi; k += BK) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * SMEM_A);
          const uint32_t b_addr = smem_u32(sB + stage * SMEM_B);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            uint64_t ad = sw128_desc(a_addr + ks * a_kstep, a_lbo, 1024);
            uint64_t bd = sw128_desc(b_addr + ks * b_kstep, b_lbo, 1024);
            umma_bf16(d_tmem, ad, bd, p.idesc, first ? 0u : 1u);
            first = 0;
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    // EPI_WARPS warps; warps w and w+4 share TMEM lane quadrant w%4 and
    // split the 32-column chunks of the tile between them.
    const int ew = warp - 2;
    const int q = warp & 3;
    // per-warp 8 KiB region (derived from the __shared__ array so accesses
    // stay LDS/STS): two 4 KiB TMA-store boxes, or the padded staging tile
    uint8_t *wreg = smem_raw + ((sW - smem_raw) + ew * 8192);
    float *stage = reinterpret_cast<float *>(wreg);
    uint32_t chunk_ctr = 0;
    uint32_t rph = 0;  // residual box mbarrier parities
    const int half = ew >> 2;  // 0 or 1
    int acc = 0;
    uint32_t aphase = 0;
    const EpiArgs &e = p.epi;
    const float *bias = e.bias;
    if (p.bias_smem) {
      // after the slot (16 B) and the residual mbarriers (128 B), 16-B aligned
      float *sb = reinterpret_cast<float *>(smem_raw + ((reinterpret_cast<uint8_t *>(tmem_slot) -
                                                         smem_raw) + 160));
      for (int64_t i = threadIdx.x - 64; i < p.N; i += 32 * EPI_WARPS) sb[i] = e.bias[i];
      named_bar_sync(1, 32 * EPI_WARPS);
      bias = sb;
    }
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int64_t bidx, mt, nt;
      int sp;
      decode_tile(p, t, bidx, sp, mt, nt);
      mbar_wait(&tfull[acc], aphase);
      fence_after();
      const int64_t m = mt * BM + q * 32 + lane;
      const int64_t n0 = nt * BN;
      const bool row_ok = m < p.M;
      // this warp's chunks: c0 = half*32 + 64*i with n0 + c0 < N; the next
      // chunk's TMEM load is in flight while the current one is finished,
      // and the accumulator is released as soon as its last chunk is read
      const int64_t ncols = min((int64_t)BN, p.N - n0);
      if (p.epi.dtype_c == EVO_BF16 && p.store_mode != 0 && p.split == 1) {
        // 64-column units (two TMEM loads, both halves finished together for
        // ILP): one 32 x 64 SW128 box (box_w 64) or two 32 x 32 boxes (SW64
        // for the tensor maps, plain rows for the mode-4 block store)
        const int nun = ncols > half * 64 ? (int)((ncols - half * 64 + 127) / 128) : 0;
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
        if (nun == 0) {
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
#pragma unroll 1
        for (int ui = 0; ui < nun; ++ui) {
          const int c0 = half * 64 + 128 * ui;
          uint32_t va[32], vb[32];
          tmem_ld32_nw(tb + c0, va);
          tmem_ld32_nw(tb + c0 + 32, vb);
          tmem_wait_ld();
          if (ui + 1 == nun) {
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
          }
          const int64_t nb = n0 + c0;
          if ((mt * BM + q * 32) >= p.M) continue;
          uint8_t *box = wreg + (chunk_ctr & 1) * 4096;
          ++chunk_ctr;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          const bool second = nb + 32 < p.N;  // warp-uniform
          // byte offset of 16-byte chunk c (0..7) of this lane's row
          auto off = [&](int c) -> int {
            if (p.box_w == 64) return lane * 128 + ((c ^ (lane & 7)) << 4);
            if (p.box_w == 65)  // rows 2*lane + j of 64 B, SW64: chunk ^ ((row >> 1) & 3)
              return (2 * lane + (c >> 2)) * 64 + (((c & 3) ^ (lane & 3)) << 4);
            const int hh = c >> 2, cc = c & 3;
            const int sw = p.store_mode == 4 ? 0 : ((lane >> 1) & 3);
            return hh * 2048 + lane * 64 + ((cc ^ sw) << 4);
          };
          // finish and stage one 32-column half at a time (register budget:
          // 10 warps cap the kernel at 168 registers per thread)
          auto half_out = [&](const uint32_t(&v)[32], int64_t nbh, int cbase) {
            float x[32];
            epi_math<EPI>(p, e, v, nbh, x, bias);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t w[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(x[8 * c + 2 * u], x[8 * c + 2 * u + 1]);
                w[u] = *reinterpret_cast<uint32_t *>(&h2);
              }
              *reinterpret_cast<uint4 *>(box + off(cbase + c)) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          };
          half_out(va, nb, 0);
          if (second) half_out(vb, nb + 32, 4);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int mrow = (int)(mt * BM + q * 32);
            const int nsub = p.box_w >= 64 ? 1 : (second ? 2 : 1);
            for (int sb = 0; sb < nsub; ++sb) {
              const int64_t nbs = nb + 32 * sb;
              const uint8_t *bx = box + sb * 2048;
              if (p.store_mode == 4) {
                bf16 *dst = reinterpret_cast<bf16 *>(e.C) + e.cmap.row(mrow) + e.cmap.col(nbs);
                bulk_store(dst, bx, 2048);
              } else if (p.store_mode == 1) {
                tma_store_2d(&tmC, bx, (int)nbs, mrow);
              } else if (p.store_mode == 2) {
                tma_store_3d(&tmC, bx, (int)(nbs % p.cdiv), (int)(nbs / p.cdiv), mrow);
              } else {
                tma_store_4d(&tmC, bx, (int)(nbs % p.cdiv), (int)(nbs / p.cdiv),
                             (int)(mrow % p.rdiv), (int)(mrow / p.rdiv));
              }
            }
            bulk_commit();
          }
        }
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
        continue;
      }
      // destination row base: only the thread-store / plain-residual paths
      // need it (64-bit divisions kept off the bf16 TMA-store path)
      int64_t rbase = 0;
      if (row_ok && p.split == 1) {
        const int64_t b1 = bidx / p.B2, b2 = bidx % p.B2;
        rbase = b1 * e.c_b1 + b2 * e.c_b2 + e.cmap.row(m);
      }
      const int nch = ncols > half * 32 ? (int)((ncols - half * 32 + 63) / 64) : 0;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + half * 32;
      uint32_t vn[32];
      if (nch > 0) tmem_ld32_nw(tbase, vn);
      if (nch == 0) {
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
#pragma unroll 1
      for (int ci = 0; ci < nch; ++ci) {
        const int c0 = half * 32 + 64 * ci;
        uint32_t v[32];
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = vn[j];
        if (ci + 1 < nch) {
          tmem_ld32_nw(tbase + 64 * (ci + 1), vn);
        } else {
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const int64_t nb = n0 + c0;
        if (p.split > 1) {
          if (!row_ok) continue;
          float *dst = p.partial + (((int64_t)sp * p.nbatch + bidx) * p.M + m) * p.N + nb;
          if (nb + 32 <= p.N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4 *>(dst)[j] =
                  make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                              __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nb + j < p.N) dst[j] = __uint_as_float(v[j]);
          }
          continue;
        }
        if (p.store_mode != 0 && (mt * BM + q * 32) < p.M) {
          // TMA bulk store (or reduce-add, for accumulate) of this warp's
          // 32 x 32 chunk; rows/cols beyond M/N are clipped by the map
          float x[32];
          epi_math<EPI>(p, e, v, nb, x, bias);
          if (p.res_tma) {
            // residual chunk arrives in this chunk's box (TMA, SW128 like the
            // store); issued one chunk ahead (or now, at a tile's first chunk)
            const int bx = (int)(chunk_ctr & 1);
            uint8_t *rbox = wreg + bx * 4096;
            uint64_t *rb = &rbar[ew * 2 + bx];
            if (ci == 0) {
              if (lane == 0) {
                bulk_wait_read<1>();
                mbar_expect_tx(rb, 4096);
                tma_load_2d(rbox, &tmR, rb, (int)nb, (int)(mt * BM + q * 32));
              }
              __syncwarp();
            }
            mbar_wait(rb, (rph >> bx) & 1u);
            rph ^= 1u << bx;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float4 r4 = *reinterpret_cast<const float4 *>(rbox + lane * 128 + ((c ^ (lane & 7)) << 4));
              x[4 * c] += r4.x; x[4 * c + 1] += r4.y; x[4 * c + 2] += r4.z; x[4 * c + 3] += r4.w;
            }
          } else if (e.residual) {  // fp32, plain 2-D layout (same map as C)
            if (row_ok) {
              const float4 *rp = reinterpret_cast<const float4 *>(e.residual + rbase + nb);
              if (nb + 32 <= p.N) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float4 r4 = __ldg(rp + j);
                  x[4 * j] += r4.x; x[4 * j + 1] += r4.y; x[4 * j + 2] += r4.z; x[4 * j + 3] += r4.w;
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (nb + j < p.N) x[j] += e.residual[rbase + nb + j];
              }
            }
          }
          uint8_t *box = wreg + (chunk_ctr & 1) * 4096;
          ++chunk_ctr;
          if (lane == 0) bulk_wait_read<1>();  // box's previous store has read it
          __syncwarp();
          if (e.dtype_c == EVO_BF16) {
            // SW64 box for the tensor map; plain 64-byte rows for mode 4
            const int sw = p.store_mode == 4 ? 0 : ((lane >> 1) & 3);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t w[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(x[8 * c + 2 * u], x[8 * c + 2 * u + 1]);
                w[u] = *reinterpret_cast<uint32_t *>(&h2);
              }
              *reinterpret_cast<uint4 *>(box + lane * 64 + ((c ^ sw) << 4)) =
                  make_uint4(w[0], w[1], w[2], w[3]);
            }
          } else {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<float4 *>(box + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                  make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && p.store_mode == 4) {
            const int64_t mrow = mt * BM + q * 32;
            bf16 *dst = reinterpret_cast<bf16 *>(e.C) + e.cmap.row(mrow) + e.cmap.col(nb);
            bulk_store(dst, box, 2048);
            bulk_commit();
          } else if (lane == 0) {
            const int mrow = (int)(mt * BM + q * 32);
            if (e.accumulate) {
              if (p.store_mode == 1)
                tma_radd_2d(&tmC, box, (int)nb, mrow);
              else if (p.store_mode == 2)
                tma_radd_3d(&tmC, box, (int)(nb % p.cdiv), (int)(nb / p.cdiv), mrow);
              else
                tma_radd_4d(&tmC, box, (int)(nb % p.cdiv), (int)(nb / p.cdiv),
                            (int)(mrow % p.rdiv), (int)(mrow / p.rdiv));
            } else if (p.store_mode == 1) {
              tma_store_2d(&tmC, box, (int)nb, mrow);
            } else if (p.store_mode == 2) {
              tma_store_3d(&tmC, box, (int)(nb % p.cdiv), (int)(nb / p.cdiv), mrow);
            } else {
              tma_store_4d(&tmC, box, (int)(nb % p.cdiv), (int)(nb / p.cdiv),
                           (int)(mrow % p.rdiv), (int)(mrow / p.rdiv));
            }
            bulk_commit();
            if (p.res_tma && ci + 1 < nch) {  // next chunk's residual into the other box
              const int bx = (int)(chunk_ctr & 1);
              bulk_wait_read<1>();  // that box's previous store has read it
              mbar_expect_tx(&rbar[ew * 2 + bx], 4096);
              tma_load_2d(wreg + bx * 4096, &tmR, &rbar[ew * 2 + bx], (int)(nb + 64), mrow);
            }
          }
          continue;
        }
        epi_chunk<EPI>(p, e, v, rbase, nb, row_ok, stage);
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (lane == 0) bulk_wait_all();
  }

  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host
struct OperandPlan {
  bool kmajor;
  bool bat1, bat2;
};

// Which layout does a (rows x K) operand view have?  rows = M or N.
bool plan_operand(const evo_mat &x, int64_t rows, int64_t K, OperandPlan &pl) {
  if ((reinterpret_cast<uintptr_t>(x.ptr) & 15) != 0) return false;
  auto ok_batch = [](int64_t s) { return s == 0 || (s % 8 == 0 && s > 0); };
  if (!ok_batch(x.bs1) || !ok_batch(x.bs2)) return false;
  if (x.cs == 1 && (x.rs % 8 == 0) && x.rs > 0 && (rows > 1 || true)) {
    pl.kmajor = true;
  } else if (x.rs == 1 && (x.cs % 8 == 0) && x.cs > 0) {
    pl.kmajor = false;
  } else {
    return false;
  }
  pl.bat1 = x.bs1 != 0;
  pl.bat2 = x.bs2 != 0;
  (void)K;
  return true;
}

bool make_map(CUtensorMap *map, const evo_mat &x, const OperandPlan &pl, int64_t rows,
              int64_t K, int64_t B1, int64_t B2, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
  if (pl.kmajor) {
    dims[0] = (cuuint64_t)K;
    dims[1] = (cuuint64_t)rows;
    strides[0] = (cuuint64_t)x.rs * 2;
    box[0] = BK;
    box[1] = (cuuint32_t)box_rows;
  } else {
    dims[0] = (cuuint64_t)rows;
    dims[1] = (cuuint64_t)K;
    strides[0] = (cuuint64_t)x.cs * 2;
    box[0] = 64;
    box[1] = BK;
  }
  const cuuint64_t span = strides[0] * dims[1];
  const cuuint64_t dummy = ((span + 15) / 16) * 16;
  dims[2] = pl.bat1 ? (cuuint64_t)B1 : 1;
  dims[3] = pl.bat2 ? (cuuint64_t)B2 : 1;
  strides[1] = pl.bat1 ? (cuuint64_t)x.bs1 * 2 : dummy;
  strides[2] = pl.bat2 ? (cuuint64_t)x.bs2 * 2 : strides[1] * dims[2];
  if (strides[2] == 0) strides[2] = 16;
  box[2] = 1;
  box[3] = 1;
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x.ptr, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int choose_bn(const evo_gemm_desc *d) {
  if (d->N <= 128) return 128;
  // split-K (weight gradients): 128 x 256 tiles, the split doubled to fill
  // the SMs (kernels.pick_split) -- fewer operand bytes per FLOP per SM,
  // 5-7 % faster than 128 x 128 at [256|1024] x [1024|256] x 32768
  if (d->split_k > 1) return 256;
  const int64_t tiles256 = ((d->M + BM - 1) / BM) * ((d->N + 255) / 256) * d->B1 * d->B2 *
                           std::max(1, d->split_k);
  return tiles256 < (int64_t)num_sms() ? 128 : 256;
}

int choose_split(const evo_gemm_desc *d, int BN, int64_t &k_chunk) {
  int split = d->split_k < 1 ? 1 : d->split_k;
  k_chunk = (d->K + split - 1) / split;
  k_chunk = ((k_chunk + BK - 1) / BK) * BK;
  if (k_chunk < BK) k_chunk = BK;
  split = (int)((d->K + k_chunk - 1) / k_chunk);
  (void)BN;
  return split < 1 ? 1 : split;
}

// Bulk-copy fallback for the outer-product-mean layouts o[i,j,p,q] and
// do'[i,p,j,q] when their 4-D tensor map cannot be built (mode 4): every
// warp chunk (32 rows x 32 columns) is one contiguous 2 KiB bf16 block --
// rows 32 elements apart inside a 32-aligned row group, columns unit-stride
// inside a 32-aligned column group.  (The 4-D map with two 32-column SW64
// boxes per 64-column unit measured 47 us against 54 us for this at the C2
// OPM GEMM; a single {32 q, 2 j, 32 p, 1 i} box with 128-byte swizzle -- a
// 64-byte inner box -- does NOT match the SW128 staging image and was
// removed.)
static int bulk_block_mode(const evo_gemm_desc *d) {
  const evo_mat &c = d->C;
  if (d->dtype_c == EVO_BF16 && !d->residual && !d->accumulate && c.rdiv > 0 &&
      c.rdiv % 32 == 0 && c.rs0 == 32 && c.cdiv > 0 && c.cdiv % 32 == 0 && c.cs0 == 1 &&
      d->M % 32 == 0 && d->N % 32 == 0 && (reinterpret_cast<uintptr_t>(c.ptr) & 15) == 0 &&
      (c.rs % 8) == 0 && (c.cs % 8) == 0)
    return 4;
  return 0;
}

// EVO_GEMM_OPM_BOX=0: the OPM layouts as two 32-column boxes per unit
static const bool g_opm_box = [] {
  const char *e = getenv("EVO_GEMM_OPM_BOX");
  return !(e && e[0] == '0');
}();

// TMA store map for C when its index map is expressible (no batching; a
// residual only for fp32 plain 2-D outputs, accumulate only for fp32, done
// as a bulk reduce-add): returns the store mode (0 = not expressible).
int make_store_map(CUtensorMap *map, const evo_gemm_desc *d, int *box_w) {
  if (d->B1 * d->B2 != 1) return 0;
  {
    // 32-column groups (the outer-product-mean layouts, c = 32): one 4-D box
    // {32 q, 2 j, 32 p, 1 i} per 64-column unit.  Its inner dimension is 64
    // bytes, so the swizzle must be the 64-byte one (a 64-byte box row under
    // SW128 is not the SW128 image of a 128-byte row); the staging writes
    // each output row p as box rows 2p, 2p+1 (box_w code 65)
    const evo_mat &c = d->C;
    const int64_t es = 2;
    auto ok16 = [&](int64_t st) { return st > 0 && (st * es) % 16 == 0; };
    if (g_opm_box && d->dtype_c == EVO_BF16 && !d->residual && !d->accumulate &&
        c.cdiv == 32 && c.cs0 == 1 && c.rdiv > 0 && c.rdiv % 32 == 0 && d->M % c.rdiv == 0 &&
        d->N % 64 == 0 && ok16(c.cs) && ok16(c.rs0) && ok16(c.rs) &&
        (reinterpret_cast<uintptr_t>(c.ptr) & 15) == 0) {
      cuuint64_t dims[4] = {32, (cuuint64_t)(d->N / 32), (cuuint64_t)c.rdiv,
                            (cuuint64_t)(d->M / c.rdiv)};
      cuuint64_t strides[3] = {(cuuint64_t)(c.cs * es), (cuuint64_t)(c.rs0 * es),
                               (cuuint64_t)(c.rs * es)};
      cuuint32_t box[4] = {32, 2, 32, 1}, estr[4] = {1, 1, 1, 1};
      EncodeTiledFn fn = encode_fn();
      if (fn && fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, c.ptr, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
        *box_w = 65;
        return 3;
      }
    }
  }
  if ((d->residual || d->accumulate) && d->dtype_c != EVO_F32) return 0;
  if (d->residual && (d->accumulate || d->C.cdiv || d->C.rdiv ||
                      (reinterpret_cast<uintptr_t>(d->residual) & 15) != 0))
    return 0;
  const evo_mat &c = d->C;
  const int64_t es = d->dtype_c == EVO_BF16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(c.ptr) & 15) != 0) return 0;
  auto ok16 = [&](int64_t st) { return st > 0 && (st * es) % 16 == 0; };
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
  int rank, mode;
  // bf16 rows of 64 columns (128 B) halve the number of store requests;
  // needs 64-aligned column blocks
  const bool wide = d->dtype_c == EVO_BF16 && !d->residual && !d->accumulate &&
                    (c.cdiv == 0 ? true : c.cdiv % 64 == 0);
  const cuuint32_t bw = wide ? 64 : 32;
  if (c.cdiv == 0 && c.rdiv == 0) {
    if (c.cs != 1 || !ok16(c.rs)) return 0;
    dims[0] = d->N; dims[1] = d->M;
    strides[0] = c.rs * es;
    box[0] = bw; box[1] = 32;
    rank = 2; mode = 1;
  } else if (c.cdiv > 0 && c.rdiv == 0) {
    if (c.cs0 != 1 || c.cdiv % 32 || d->N % c.cdiv || !ok16(c.cs) || !ok16(c.rs)) return 0;
    dims[0] = c.cdiv; dims[1] = d->N / c.cdiv; dims[2] = d->M;
    strides[0] = c.cs * es; strides[1] = c.rs * es;
    box[0] = bw; box[1] = 1; box[2] = 32;
    rank = 3; mode = 2;
  } else if (c.cdiv > 0 && c.rdiv > 0) {
    if (c.cs0 != 1 || c.cdiv % 32 || d->N % c.cdiv || c.rdiv % 32 || d->M % c.rdiv ||
        !ok16(c.cs) || !ok16(c.rs0) || !ok16(c.rs))
      return bulk_block_mode(d);
    dims[0] = c.cdiv; dims[1] = d->N / c.cdiv; dims[2] = c.rdiv; dims[3] = d->M / c.rdiv;
    strides[0] = c.cs * es; strides[1] = c.rs0 * es; strides[2] = c.rs * es;
    box[0] = bw; box[1] = 1; box[2] = 32; box[3] = 1;
    rank = 4; mode = 3;
  } else {
    return 0;
  }
  *box_w = (int)bw;
  EncodeTiledFn fn = encode_fn();
  if (!fn) return mode == 3 ? bulk_block_mode(d) : 0;
  CUresult r = fn(map, d->dtype_c == EVO_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                  rank, c.ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  (d->dtype_c == EVO_BF16 && bw == 32) ? CU_TENSOR_MAP_SWIZZLE_64B
                                                       : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return mode == 3 ? bulk_block_mode(d) : 0;
  return mode;
}

template <int BN, int STAGES, int EPI>
int launch(const evo_gemm_desc *d, cudaStream_t st) {
  OperandPlan pa, pb;
  plan_operand(d->A, d->M, d->K, pa);
  plan_operand(d->B, d->N, d->K, pb);
  CUtensorMap ma, mb;
  if (!make_map(&ma, d->A, pa, d->M, d->K, d->B1, d->B2, BM) ||
      !make_map(&mb, d->B, pb, d->N, d->K, d->B1, d->B2, BN))
    return EVO_EUNSUP;
  TcParams p;
  p.M = d->M; p.N = d->N; p.K = d->K; p.B2 = d->B2; p.nbatch = d->B1 * d->B2;
  p.c_aligned = (reinterpret_cast<uintptr_t>(d->C.ptr) & 15) == 0 &&
                (!d->residual || (reinterpret_cast<uintptr_t>(d->residual) & 15) == 0);
  p.tiles_m = (d->M + BM - 1) / BM;
  p.tiles_n = (d->N + BN - 1) / BN;
  p.split = choose_split(d, BN, p.k_chunk);
  p.num_tiles = p.tiles_m * p.tiles_n * p.split * d->B1 * d->B2;
  if (p.num_tiles >= (1ll << 31)) return EVO_EUNSUP;
  p.a_kmajor = pa.kmajor; p.b_kmajor = pb.kmajor;
  p.a_bat1 = pa.bat1; p.a_bat2 = pa.bat2; p.b_bat1 = pb.bat1; p.b_bat2 = pb.bat2;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((pa.kmajor ? 0u : 1u) << 15) |
            ((pb.kmajor ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
            ((uint32_t)(BM >> 4) << 24);
  p.epi = epi_args_of(d);
  p.partial = reinterpret_cast<float *>(d->workspace);
  CUtensorMap mc;
  p.box_w = 32;
  p.store_mode = p.split > 1 ? 0 : make_store_map(&mc, d, &p.box_w);
  // fp32 residual through TMA (same geometry as C's 2-D map, its own pointer)
  CUtensorMap mr = mc;
  p.res_tma = 0;
  if (p.store_mode == 1 && d->residual && d->dtype_c == EVO_F32) {
    evo_gemm_desc dr = *d;
    dr.C.ptr = const_cast<float *>(d->residual);
    dr.residual = nullptr;
    int bw = 32;
    if (make_store_map(&mr, &dr, &bw) == 1) p.res_tma = 1;
  }
  p.cdiv = d->C.cdiv > 0 ? d->C.cdiv : 1;
  p.rdiv = d->C.rdiv > 0 ? d->C.rdiv : 1;
  if (p.store_mode == 0 || p.store_mode == 4) mc = ma;  // unused
  if (p.split > 1) {
    size_t need = (size_t)p.split * d->B1 * d->B2 * d->M * d->N * sizeof(float);
    EVO_REQUIRE(d->workspace && d->workspace_bytes >= need, EVO_EARG,
                "evo_gemm(tc): split=%d needs %zu workspace bytes", p.split, need);
  }
  p.bias_smem = (d->bias && d->N <= BIAS_SMEM_MAX && p.split == 1) ? 1 : 0;
  const size_t smem = 1024 + (size_t)STAGES * (SMEM_A + BN * BK * 2) +
                      (EPI == EK_SPLIT ? (size_t)0 : (size_t)EPI_WARPS * 8192) + 512 +
                      (size_t)BIAS_SMEM_MAX * 4;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, EPI>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  int64_t grid = std::min<int64_t>(p.num_tiles, (int64_t)num_sms());
  if (!p.res_tma) mr = mc;  // unused
  launch_k(gemm_tc_kernel<BN, STAGES, EPI>, (unsigned)grid, NTHREADS, smem, st, ma, mb, mc, mr, p);
  EVO_LAUNCHED("gemm_tc_kernel");
  if (p.split > 1) return gemm_splitk_reduce(d, p.split, p.partial, st);
  return EVO_OK;
}

}  // namespace

bool gemm_tc_accepts(const evo_gemm_desc *d) {
  if (d->dtype_ab != EVO_BF16 || d->K < 1 || d->M < 1 || d->N < 1) return false;
  if (d->B1 * d->B2 > 65535 || d->K > (1ll << 31) || d->M > (1ll << 31) || d->N > (1ll << 31))
    return false;
  if (!encode_fn()) return false;
  OperandPlan pa, pb;
  return plan_operand(d->A, d->M, d->K, pa) && plan_operand(d->B, d->N, d->K, pb);
}

size_t gemm_tc_workspace(const evo_gemm_desc *d) {
  int64_t kc;
  int split = choose_split(d, choose_bn(d), kc);
  if (split <= 1) return 0;
  return (size_t)split * d->B1 * d->B2 * d->M * d->N * sizeof(float);
}

template <int EPI>
int launch_bn(const evo_gemm_desc *d, cudaStream_t st) {
  if (choose_bn(d) == 256) return launch<256, 3, EPI>(d, st);
  return launch<128, 4, EPI>(d, st);
}

int gemm_tc(const evo_gemm_desc *d, cudaStream_t st) {
  if (!gemm_tc_accepts(d)) return EVO_EUNSUP;
  // split-K partials carry no epilogue (applied by the reducer)
  int64_t kc;
  const bool split = choose_split(d, choose_bn(d), kc) > 1;
  if (split) {
    if (choose_bn(d) == 256) return launch<256, 4, EK_SPLIT>(d, st);
    return launch<128, 6, EK_SPLIT>(d, st);
  }
  if (!d->bias && d->epilogue == EVO_EPI_NONE) return launch_bn<EK_NONE>(d, st);
  if (!d->bias) return EVO_EUNSUP;  // activation without bias: SIMT handles it
  if (d->epilogue == EVO_EPI_RELU) return launch_bn<EK_BIAS_RELU>(d, st);
  if (d->epilogue == EVO_EPI_SIGMOID_FROM) return launch_bn<EK_BIAS_SIGMOID>(d, st);
  return launch_bn<EK_BIAS>(d, st);
}

}  // namespace evo
