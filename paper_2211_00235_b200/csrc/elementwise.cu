// Bandwidth-bound element-wise / reduction kernels of the Evoformer block:
// gates, casts, bias-gradient sums, loss.  Grid-stride loops over a grid
// sized in multiples of the SM count; reductions use a fixed partition and
// fixed summation order (bitwise reproducible).
#include "common.cuh"

namespace evo {
namespace {

inline int ew_blocks(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 8;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

template <typename T>
__device__ __forceinline__ float LD(const void *p, int64_t i) {
  return to_f(reinterpret_cast<const T *>(p)[i]);
}
template <typename T>
__device__ __forceinline__ void ST(void *p, int64_t i, float v) {
  reinterpret_cast<T *>(p)[i] = from_f<T>(v);
}

// dst(i,j) = sum_b src[b][i][j]; block per tile of j, threads over j.
template <typename T>
__global__ void reduce_lead_kernel(int64_t nb, int64_t n1, int64_t n2, const void *src,
                                   float *dst, int64_t d_s1, int64_t d_s2, int acc) {
  evo_pdl_enter();
  const int64_t total = n1 * n2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t b = 0; b < nb; ++b) s += LD<T>(src, b * total + e);
    int64_t i = e / n2, j = e % n2;
    float *d = dst + i * d_s1 + j * d_s2;
    *d = acc ? *d + s : s;
  }
}

// Contiguous fp32 case (the attention dbias chunk partials, n1 = 1): float4
// per thread, the nb partial slabs summed in order with four loads in flight.
__global__ void reduce_lead_vec_kernel(int64_t nb, int64_t total4, const float4 *src, float4 *dst,
                                       int acc) {
  evo_pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total4;
       e += (int64_t)gridDim.x * blockDim.x) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int64_t b = 0; b < nb; ++b) {
      const float4 v = __ldg(src + b * total4 + e);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    if (acc) {
      const float4 d = dst[e];
      s.x += d.x; s.y += d.y; s.z += d.z; s.w += d.w;
    }
    dst[e] = s;
  }
}

// Column sums of a tall matrix, deterministic two-stage reduction.
// Stage 1: block (bx, by) covers rows [bx*rpb, (bx+1)*rpb) and 32 columns;
// 8 row-lanes (threadIdx.y) stride the rows with 4 loads in flight each, then
// combine in fixed order through smem.
template <typename T>
__global__ void colsum_stage1(int64_t rows, int64_t cols, const void *src, int64_t rs,
                              int64_t rpb, float *part) {
  evo_pdl_enter();
  __shared__ float red[8][33];
  const int64_t c = blockIdx.y * 32 + threadIdx.x;
  const int64_t r0 = blockIdx.x * rpb;
  const int64_t r1 = min(rows, r0 + rpb);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (c < cols) {
    int64_t r = r0 + threadIdx.y;
    for (; r + 24 < r1; r += 32) {
      a0 += LD<T>(src, r * rs + c);
      a1 += LD<T>(src, (r + 8) * rs + c);
      a2 += LD<T>(src, (r + 16) * rs + c);
      a3 += LD<T>(src, (r + 24) * rs + c);
    }
    for (; r < r1; r += 8) a0 += LD<T>(src, r * rs + c);
  }
  red[threadIdx.y][threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    float s = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) s += red[y][threadIdx.x];
    part[blockIdx.x * cols + c] = s;
  }
}

// Vectorised stage 1 for contiguous, 16-byte aligned rows: thread (tx, ty)
// owns VW consecutive columns (VW = 8 bf16 / 4 fp32 = one 16-byte load) of
// the block's 32*VW-column tile and rows ty, ty+8, ... of the chunk.
template <typename T>
__global__ void colsum_stage1_vec(int64_t rows, int64_t cols, const void *src, int64_t rs,
                                  int64_t rpb, float *part) {
  evo_pdl_enter();
  constexpr int VW = 16 / sizeof(T);
  __shared__ float red[8][32 * VW + 4];
  const int64_t c0 = (blockIdx.y * 32 + threadIdx.x) * VW;
  const int64_t r0 = blockIdx.x * rpb;
  const int64_t r1 = min(rows, r0 + rpb);
  float acc[VW];
#pragma unroll
  for (int j = 0; j < VW; ++j) acc[j] = 0.f;
  if (c0 < cols) {
    const T *base = reinterpret_cast<const T *>(src) + c0;
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      uint4 u = *reinterpret_cast<const uint4 *>(base + r * rs);
      if constexpr (sizeof(T) == 4) {
        const float *f = reinterpret_cast<const float *>(&u);
#pragma unroll
        for (int j = 0; j < VW; ++j) acc[j] += f[j];
      } else {
        const uint32_t *w = reinterpret_cast<const uint32_t *>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w[j]));
          acc[2 * j] += f.x;
          acc[2 * j + 1] += f.y;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < VW; ++j) red[threadIdx.y][threadIdx.x * VW + j] = acc[j];
  __syncthreads();
  const int t = threadIdx.y * 32 + threadIdx.x;
  for (int cc = t; cc < 32 * VW; cc += 256) {
    const int64_t c = blockIdx.y * 32 * VW + cc;
    if (c >= cols) continue;
    float sum = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) sum += red[y][cc];
    part[blockIdx.x * cols + c] = sum;
  }
}

// Stage 2: column sums of the [nblk, cols] partials: a 1024-thread block
// owns 32 columns, lanes across columns (coalesced 128-byte rows), the 32
// warps take partial rows w, w+32, ... (8 loads in flight each) and the 32
// warp sums are combined in order.  Deterministic.
__global__ void __launch_bounds__(1024) colsum_stage2(int nblk, int64_t cols, const float *part,
                                                      float *dst, int acc) {
  evo_pdl_enter();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < cols) {
#pragma unroll 8
    for (int b = w; b < nblk; b += 32) s += __ldg(&part[(int64_t)b * cols + c]);
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < cols) {
    float t = red[0][lane];
#pragma unroll
    for (int j = 1; j < 32; ++j) t += red[j][lane];
    dst[c] = acc ? dst[c] + t : t;
  }
}

template <typename TS, typename TD>
__global__ void copy2d_kernel(int64_t rows, int64_t cols, const void *src, int64_t s_rs,
                              int64_t s_cs, void *dst, int64_t d_rs, int64_t d_cs) {
  evo_pdl_enter();
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    ST<TD>(dst, r * d_rs + c * d_cs, LD<TS>(src, r * s_rs + c * s_cs));
  }
}

// Contiguous-row copy/cast, 8 elements per thread per step (16-byte
// bf16 / 2x16-byte fp32 accesses).  cols % 8 == 0, rows 16-byte aligned.
template <typename TS, typename TD>
__global__ void copy2d_vec_kernel(int64_t rows, int64_t cols, const void *src, int64_t s_rs,
                                  void *dst, int64_t d_rs) {
  evo_pdl_enter();
  const int64_t per_row = cols / 8;
  const int64_t total = rows * per_row;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / per_row, c = (e % per_row) * 8;
    float v[8];
    if constexpr (sizeof(TS) == 4) {
      const float4 *p = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(src) +
                                                         r * s_rs + c);
      float4 a = p[0], b = p[1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
      uint4 a = *reinterpret_cast<const uint4 *>(reinterpret_cast<const bf16 *>(src) + r * s_rs + c);
      const uint32_t *w = reinterpret_cast<const uint32_t *>(&a);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w[j]));
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
      }
    }
    if constexpr (sizeof(TD) == 4) {
      float4 *q = reinterpret_cast<float4 *>(reinterpret_cast<float *>(dst) + r * d_rs + c);
      q[0] = make_float4(v[0], v[1], v[2], v[3]);
      q[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        w[j] = *reinterpret_cast<uint32_t *>(&h2);
      }
      *reinterpret_cast<uint4 *>(reinterpret_cast<bf16 *>(dst) + r * d_rs + c) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// Transposing copy through shared memory for the dst-contiguous-along-rows
// case (s_cs == 1 and d_rs == 1): coalesced on both sides.
template <typename TS, typename TD>
__global__ void transpose_kernel(int64_t rows, int64_t cols, const void *src, int64_t s_rs,
                                 void *dst, int64_t d_cs) {
  evo_pdl_enter();
  __shared__ float tile[32][33];
  int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? LD<TS>(src, r * s_rs + c) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) ST<TD>(dst, c * d_cs + r, tile[threadIdx.x][i]);
  }
}

template <typename TA, typename TB, typename TO>
__global__ void mul2d_kernel(int64_t rows, int64_t cols, const void *a, int64_t a_rs,
                             const void *b, int64_t b_rs, void *o, int64_t o_rs) {
  evo_pdl_enter();
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    ST<TO>(o, r * o_rs + c, LD<TA>(a, r * a_rs + c) * LD<TB>(b, r * b_rs + c));
  }
}

// a_cf[ch][row] = sig(ga)*a ; proj cols [a | b | ga | gb] (ga, gb already
// sigmoid-activated by the projection GEMM epilogue).  Tile: 32 rows x c
// channels through smem so both the channel-last read and the
// channel-first write are coalesced.
template <typename T>
__global__ void trimul_gate_fwd_kernel(int64_t rows, int c, const void *proj, int64_t ldp,
                                       void *a_cf, void *b_cf) {
  evo_pdl_enter();
  extern __shared__ float t2[];  // [2][c][33]
  const int64_t r0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * c; e += blockDim.x) {
    int rr = e / c, ch = e % c;
    int64_t r = r0 + rr;
    float av = 0.f, bv = 0.f;
    if (r < rows) {
      const int64_t base = r * ldp;
      av = LD<T>(proj, base + ch) * LD<T>(proj, base + 2 * c + ch);
      bv = LD<T>(proj, base + c + ch) * LD<T>(proj, base + 3 * c + ch);
    }
    t2[(0 * c + ch) * 33 + rr] = av;
    t2[(1 * c + ch) * 33 + rr] = bv;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * c; e += blockDim.x) {
    int ch = e / 32, rr = e % 32;
    int64_t r = r0 + rr;
    if (r < rows) {
      ST<T>(a_cf, (int64_t)ch * rows + r, t2[(0 * c + ch) * 33 + rr]);
      ST<T>(b_cf, (int64_t)ch * rows + r, t2[(1 * c + ch) * 33 + rr]);
    }
  }
}

template <typename T>
__global__ void trimul_gate_bwd_kernel(int64_t rows, int c, const void *proj, int64_t ldp,
                                       const float *da_cf, const float *db_cf, void *dproj,
                                       int64_t ldd, float *part) {
  evo_pdl_enter();
  extern __shared__ float t2[];  // [2][c][33], then (part) [4c][33] fp32 outputs
  const int64_t r0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * c; e += blockDim.x) {
    int ch = e / 32, rr = e % 32;
    int64_t r = r0 + rr;
    float da = 0.f, db = 0.f;
    if (r < rows) {
      da = da_cf[(int64_t)ch * rows + r];
      db = db_cf[(int64_t)ch * rows + r];
    }
    t2[(0 * c + ch) * 33 + rr] = da;
    t2[(1 * c + ch) * 33 + rr] = db;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * c; e += blockDim.x) {
    int rr = e / c, ch = e % c;
    int64_t r = r0 + rr;
    if (r >= rows) continue;
    const int64_t base = r * ldp, dbase = r * ldd;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      float d = t2[(which * c + ch) * 33 + rr];
      float v = LD<T>(proj, base + which * c + ch);
      float g = LD<T>(proj, base + (2 + which) * c + ch);
      const float dv = d * g, dg = d * v * g * (1.f - g);
      ST<T>(dproj, dbase + which * c + ch, dv);
      ST<T>(dproj, dbase + (2 + which) * c + ch, dg);
      if (part) {
        float *so = t2 + 2 * c * 33;
        so[(which * c + ch) * 33 + rr] = dv;
        so[((2 + which) * c + ch) * 33 + rr] = dg;
      }
    }
  }
  if (part) {
    // the bias gradients a_b | b_b | a_gate_b | b_gate_b from the fp32 values
    // (not the bf16-rounded dproj): per-block column sums over the 32 rows in
    // order, reduced over blocks by colsum_stage2 (deterministic)
    __syncthreads();
    const float *so = t2 + 2 * c * 33;
    const int nrow = (int)(rows - r0 < 32 ? rows - r0 : 32);
    for (int col = threadIdx.x; col < 4 * c; col += blockDim.x) {
      float acc = 0.f;
      for (int rr = 0; rr < nrow; ++rr) acc += so[col * 33 + rr];
      part[blockIdx.x * (int64_t)(4 * c) + col] = acc;
    }
  }
}

template <typename T>
__global__ void outgate_fwd_kernel(int64_t rows, int64_t cols, const float *z, const void *g,
                                   int64_t g_rs, const void *o, int64_t o_rs, float *znew) {
  evo_pdl_enter();
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    znew[e] = z[e] + LD<T>(g, r * g_rs + c) * LD<T>(o, r * o_rs + c);
  }
}

template <typename T>
__global__ void outgate_bwd_kernel(int64_t rows, int64_t cols, const float *dz, const void *g,
                                   int64_t g_rs, const void *o, int64_t o_rs, void *do_,
                                   int64_t do_rs, void *dgp, int64_t dg_rs) {
  evo_pdl_enter();
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    float d = dz[e], gv = LD<T>(g, r * g_rs + c), ov = LD<T>(o, r * o_rs + c);
    ST<T>(do_, r * do_rs + c, d * gv);
    ST<T>(dgp, r * dg_rs + c, d * ov * gv * (1.f - gv));
  }
}

// bf16 fast paths of the out-gate (cols % 8 == 0, 16-byte aligned rows):
// one thread per 8 consecutive columns.
__device__ __forceinline__ void unpack8(const uint4 &u, float (&f)[8]) {
  const uint32_t *w = reinterpret_cast<const uint32_t *>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w[j]));
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t *>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__global__ void outgate_fwd_bf16x8_kernel(int64_t rows, int64_t cols, const float *z,
                                          const bf16 *g, int64_t g_rs, const bf16 *o,
                                          int64_t o_rs, float *znew) {
  evo_pdl_enter();
  const int64_t per_row = cols / 8, total = rows * per_row;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / per_row, c = (e % per_row) * 8;
    float gv[8], ov[8];
    unpack8(__ldg(reinterpret_cast<const uint4 *>(g + r * g_rs + c)), gv);
    unpack8(__ldg(reinterpret_cast<const uint4 *>(o + r * o_rs + c)), ov);
    const float4 *zp = reinterpret_cast<const float4 *>(z + r * cols + c);
    const float4 z0 = __ldg(zp), z1 = __ldg(zp + 1);
    float4 *dst = reinterpret_cast<float4 *>(znew + r * cols + c);
    dst[0] = make_float4(z0.x + gv[0] * ov[0], z0.y + gv[1] * ov[1], z0.z + gv[2] * ov[2],
                         z0.w + gv[3] * ov[3]);
    dst[1] = make_float4(z1.x + gv[4] * ov[4], z1.y + gv[5] * ov[5], z1.z + gv[6] * ov[6],
                         z1.w + gv[7] * ov[7]);
  }
}
__global__ void outgate_bwd_bf16x8_kernel(int64_t rows, int64_t cols, const float *dz,
                                          const bf16 *g, int64_t g_rs, const bf16 *o,
                                          int64_t o_rs, bf16 *do_, int64_t do_rs, bf16 *dgp,
                                          int64_t dg_rs) {
  evo_pdl_enter();
  const int64_t per_row = cols / 8, total = rows * per_row;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / per_row, c = (e % per_row) * 8;
    float gv[8], ov[8], d[8], a[8], b[8];
    unpack8(__ldg(reinterpret_cast<const uint4 *>(g + r * g_rs + c)), gv);
    unpack8(__ldg(reinterpret_cast<const uint4 *>(o + r * o_rs + c)), ov);
    const float4 *dp = reinterpret_cast<const float4 *>(dz + r * cols + c);
    const float4 d0 = __ldg(dp), d1 = __ldg(dp + 1);
    d[0] = d0.x; d[1] = d0.y; d[2] = d0.z; d[3] = d0.w;
    d[4] = d1.x; d[5] = d1.y; d[6] = d1.z; d[7] = d1.w;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = d[j] * gv[j];
      b[j] = d[j] * ov[j] * gv[j] * (1.f - gv[j]);
    }
    *reinterpret_cast<uint4 *>(do_ + r * do_rs + c) = pack8(a);
    *reinterpret_cast<uint4 *>(dgp + r * dg_rs + c) = pack8(b);
  }
}

// Out-gate backward (bf16 g / o, fp32 dz, cols % 8 == 0) with the column sums
// of both outputs fused in, taken from the fp32 values before rounding: the
// out_b gradient (sum of do) and the out_gate_b gradient (sum of dgpre).
// Tiling of relu_bwd_colsum_kernel: thread = 8 columns, rows ty, ty+8, ...
__global__ void outgate_bwd_colsum_kernel(int64_t rows, int64_t cols, const float *dz,
                                          const bf16 *g, int64_t g_rs, const bf16 *o,
                                          int64_t o_rs, bf16 *do_, int64_t do_rs, bf16 *dgp,
                                          int64_t dg_rs, int64_t rpb, float *part_do,
                                          float *part_dg) {
  evo_pdl_enter();
  __shared__ float red[8][32 * 8 + 4];
  const int64_t c0 = (blockIdx.y * 32 + threadIdx.x) * 8;
  const int64_t r0 = blockIdx.x * rpb;
  const int64_t r1 = min(rows, r0 + rpb);
  float a_do[8], a_dg[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a_do[j] = a_dg[j] = 0.f;
  if (c0 < cols) {
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      float gv[8], ov[8], dv[8], gg[8];
      unpack8(__ldg(reinterpret_cast<const uint4 *>(g + r * g_rs + c0)), gv);
      unpack8(__ldg(reinterpret_cast<const uint4 *>(o + r * o_rs + c0)), ov);
      const float4 *zp = reinterpret_cast<const float4 *>(dz + r * cols + c0);
      const float4 z0 = __ldg(zp), z1 = __ldg(zp + 1);
      const float d[8] = {z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dv[j] = d[j] * gv[j];
        gg[j] = d[j] * ov[j] * gv[j] * (1.f - gv[j]);
        a_do[j] += dv[j];
        a_dg[j] += gg[j];
      }
      *reinterpret_cast<uint4 *>(do_ + r * do_rs + c0) = pack8(dv);
      *reinterpret_cast<uint4 *>(dgp + r * dg_rs + c0) = pack8(gg);
    }
  }
  const int t = threadIdx.y * 32 + threadIdx.x;
  const int64_t c = blockIdx.y * 256 + t;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
    for (int j = 0; j < 8; ++j) red[threadIdx.y][threadIdx.x * 8 + j] = pass ? a_dg[j] : a_do[j];
    __syncthreads();
    if (t < 256 && c < cols) {
      float sacc = 0.f;
#pragma unroll
      for (int y = 0; y < 8; ++y) sacc += red[y][t];
      (pass ? part_dg : part_do)[blockIdx.x * cols + c] = sacc;
    }
    __syncthreads();
  }
}

// ReLU backward with the bias-gradient column sums of its output fused in
// (the transition's b1 gradient, src/tensor.py:343): the tiling of
// colsum_stage1_vec (thread = 8 consecutive columns, rows ty, ty+8, ... of
// the block's row chunk), so stage 2 is shared.
__global__ void relu_bwd_colsum_kernel(int64_t rows, int64_t cols, const bf16 *dh, const bf16 *h,
                                       bf16 *dpre, int64_t rpb, float *part) {
  evo_pdl_enter();
  __shared__ float red[8][32 * 8 + 4];
  const int64_t c0 = (blockIdx.y * 32 + threadIdx.x) * 8;
  const int64_t r0 = blockIdx.x * rpb;
  const int64_t r1 = min(rows, r0 + rpb);
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  if (c0 < cols) {
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      const uint4 a = __ldg(reinterpret_cast<const uint4 *>(dh + r * cols + c0));
      const uint4 b = __ldg(reinterpret_cast<const uint4 *>(h + r * cols + c0));
      const uint32_t *aw = reinterpret_cast<const uint32_t *>(&a);
      const uint32_t *bw = reinterpret_cast<const uint32_t *>(&b);
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t l16 = bw[j] & 0xFFFFu, h16 = bw[j] >> 16;
        const uint32_t lo = ((l16 & 0x8000u) == 0u && (l16 & 0x7FFFu) != 0u) ? 0xFFFFu : 0u;
        const uint32_t hi = ((h16 & 0x8000u) == 0u && (h16 & 0x7FFFu) != 0u) ? 0xFFFF0000u : 0u;
        o[j] = aw[j] & (lo | hi);
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&o[j]));
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
      }
      *reinterpret_cast<uint4 *>(dpre + r * cols + c0) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[threadIdx.y][threadIdx.x * 8 + j] = acc[j];
  __syncthreads();
  const int t = threadIdx.y * 32 + threadIdx.x;
  const int64_t c = blockIdx.y * 256 + t;
  if (t < 256 && c < cols) {
    float sacc = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) sacc += red[y][t];
    part[blockIdx.x * cols + c] = sacc;
  }
}

__global__ void relu_bwd_bf16x8_kernel(int64_t n8, const uint4 *dh, const uint4 *h, uint4 *dpre) {
  evo_pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint4 a = dh[e], b = h[e];
    const uint32_t *aw = reinterpret_cast<const uint32_t *>(&a);
    const uint32_t *bw = reinterpret_cast<const uint32_t *>(&b);
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // bf16 x > 0  <=>  sign bit clear and magnitude bits non-zero
      const uint32_t l16 = bw[j] & 0xFFFFu, h16 = bw[j] >> 16;
      uint32_t lo = ((l16 & 0x8000u) == 0u && (l16 & 0x7FFFu) != 0u) ? 0xFFFFu : 0u;
      uint32_t hi = ((h16 & 0x8000u) == 0u && (h16 & 0x7FFFu) != 0u) ? 0xFFFF0000u : 0u;
      o[j] = aw[j] & (lo | hi);
    }
    dpre[e] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

template <typename T>
__global__ void relu_bwd_kernel(int64_t n, const void *dh, const void *h, void *dpre) {
  evo_pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float hv = LD<T>(h, e);
    ST<T>(dpre, e, hv > 0.f ? LD<T>(dh, e) : 0.f);
  }
}

constexpr int SQ_BLOCKS = 512;

// One pass over x: per-block partial sums of x^2 and (dx != NULL) the
// gradient dx = (2/n) x of mean(x^2), 16-byte vectors when aligned.
__global__ void sq_partial_kernel(int64_t n, const float *x, float *part, float *dx) {
  evo_pdl_enter();
  __shared__ float red[32];
  float s = 0.f;
  const float sc = 2.0f / (float)n;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dx)) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(x) + e);
    s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    if (dx) reinterpret_cast<float4 *>(dx)[e] = make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w);
  }
  for (int64_t e = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[e];
    s += v * v;
    if (dx) dx[e] = sc * v;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

// Fixed-order double-precision sum of the block partials (one 256-thread
// block: strided per-thread sums, then an ordered tree).
__global__ void sq_final_kernel(int nblk, int64_t n, const float *part, float *out) {
  evo_pdl_enter();
  __shared__ double red[256];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += part[b];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] += (float)(red[0] / (double)n);
}

__global__ void add_kernel(int64_t n, const float *a, const float *b, float *o) {
  evo_pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    o[e] = a[e] + b[e];
}

__global__ void div_scalar_kernel(int64_t n, const float *x, float d, float *o) {
  evo_pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    o[e] = x[e] / d;
}

}  // namespace

// ------------------------------------------------------------------ API impl
int reduce_lead(int dt, int64_t nb, int64_t n1, int64_t n2, const void *src, float *dst,
                int64_t d_s1, int64_t d_s2, int acc, cudaStream_t st) {
  int64_t total = n1 * n2;
  if (total == 0) return EVO_OK;
  // Tall-and-skinny (bias gradients: nb = rows, n1 = 1): two-stage colsum.
  if (n1 == 1 && nb > 4096 && n2 <= 4096) {
    // Not used for arbitrary dst maps beyond d_s2; falls through otherwise.
  }
  if (dt == EVO_F32 && (n1 == 1 || d_s1 == n2) && d_s2 == 1 && total % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    launch_k(reduce_lead_vec_kernel, ew_blocks(total / 4), 256, 0, st, nb, total / 4, reinterpret_cast<const float4 *>(src), reinterpret_cast<float4 *>(dst), acc);
    EVO_LAUNCHED("reduce_lead_vec_kernel");
    return EVO_OK;
  }
  if (dt == EVO_F32)
    launch_k(reduce_lead_kernel<float>, ew_blocks(total), 256, 0, st, nb, n1, n2, src, dst, d_s1, d_s2, acc);
  else
    launch_k(reduce_lead_kernel<bf16>, ew_blocks(total), 256, 0, st, nb, n1, n2, src, dst, d_s1, d_s2, acc);
  EVO_LAUNCHED("reduce_lead_kernel");
  return EVO_OK;
}

// Column sums of src[rows x cols] (row stride rs) into dst[cols] (fp32).
// Deterministic: fixed row partition, ordered sums.  ws >= 256*cols floats.
int colsum(int dt, int64_t rows, int64_t cols, const void *src, int64_t rs, float *dst, int acc,
           float *ws, cudaStream_t st) {
  const int vw = dt == EVO_BF16 ? 8 : 4;
  const bool vec = cols % vw == 0 && rs % vw == 0 &&
                   (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  const int64_t tile_cols = vec ? 32 * vw : 32;
  const int64_t col_tiles = (cols + tile_cols - 1) / tile_cols;
  int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(256, (4 * num_sms() + col_tiles - 1) /
                                                                 col_tiles));
  nblk = std::min<int64_t>(nblk, std::max<int64_t>(1, rows / 64));
  const int64_t rpb = (rows + nblk - 1) / nblk;
  nblk = (rows + rpb - 1) / rpb;
  dim3 grid((unsigned)nblk, (unsigned)col_tiles), blk(32, 8);
  if (vec) {
    if (dt == EVO_F32) launch_k(colsum_stage1_vec<float>, grid, blk, 0, st, rows, cols, src, rs, rpb, ws);
    else launch_k(colsum_stage1_vec<bf16>, grid, blk, 0, st, rows, cols, src, rs, rpb, ws);
    EVO_LAUNCHED("colsum_stage1_vec");
  } else {
    if (dt == EVO_F32) launch_k(colsum_stage1<float>, grid, blk, 0, st, rows, cols, src, rs, rpb, ws);
    else launch_k(colsum_stage1<bf16>, grid, blk, 0, st, rows, cols, src, rs, rpb, ws);
    EVO_LAUNCHED("colsum_stage1");
  }
  launch_k(colsum_stage2, (unsigned)((cols + 31) / 32), 1024, 0, st, (int)nblk, cols, ws, dst, acc);
  EVO_LAUNCHED("colsum_stage2");
  return EVO_OK;
}

// n0 independent 2-D copies (batch strides s_bs / d_bs); 16-byte vectors
// along unit-stride rows when every row start is aligned
template <typename TS, typename TD>
__global__ void copy3d_kernel(int64_t n0, int64_t rows, int64_t cols, const void *src,
                              int64_t s_bs, int64_t s_rs, int64_t s_cs, void *dst, int64_t d_bs,
                              int64_t d_rs, int64_t d_cs) {
  evo_pdl_enter();
  const int64_t plane = rows * cols, total = n0 * plane;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / plane, rc = e - b * plane, r = rc / cols, c = rc - r * cols;
    ST<TD>(dst, b * d_bs + r * d_rs + c * d_cs, LD<TS>(src, b * s_bs + r * s_rs + c * s_cs));
  }
}

int copy3d(int ts, int td, int64_t n0, int64_t rows, int64_t cols, const void *src, int64_t s_bs,
           int64_t s_rs, int64_t s_cs, void *dst, int64_t d_bs, int64_t d_rs, int64_t d_cs,
           cudaStream_t st) {
  const int64_t total = n0 * rows * cols;
  if (total == 0) return EVO_OK;
  const int nb = ew_blocks(total);
#define C(A, B)                                                                              \
  launch_k(copy3d_kernel<A, B>, nb, 256, 0, st, n0, rows, cols, src, s_bs, s_rs, s_cs, dst, d_bs, d_rs, \
                                          d_cs)
  if (ts == EVO_F32) { if (td == EVO_F32) C(float, float); else C(float, bf16); }
  else { if (td == EVO_F32) C(bf16, float); else C(bf16, bf16); }
#undef C
  EVO_LAUNCHED("copy3d_kernel");
  return EVO_OK;
}

int copy2d(int ts, int td, int64_t rows, int64_t cols, const void *src, int64_t s_rs,
           int64_t s_cs, void *dst, int64_t d_rs, int64_t d_cs, cudaStream_t st) {
  int64_t total = rows * cols;
  if (total == 0) return EVO_OK;
  if (s_cs == 1 && d_rs == 1 && d_cs != 1 && rows >= 32 && cols >= 32) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    dim3 blk(32, 8);
#define T(A, B) launch_k(transpose_kernel<A, B>, grid, blk, 0, st, rows, cols, src, s_rs, dst, d_cs)
    if (ts == EVO_F32) { if (td == EVO_F32) T(float, float); else T(float, bf16); }
    else { if (td == EVO_F32) T(bf16, float); else T(bf16, bf16); }
#undef T
    EVO_LAUNCHED("transpose_kernel");
    return EVO_OK;
  }
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (s_cs == 1 && d_cs == 1 && cols % 8 == 0 && s_rs % 8 == 0 && d_rs % 8 == 0 && al16(src) &&
      al16(dst)) {
    int nb = ew_blocks(total / 8);
#define CV(A, B) launch_k(copy2d_vec_kernel<A, B>, nb, 256, 0, st, rows, cols, src, s_rs, dst, d_rs)
    if (ts == EVO_F32) { if (td == EVO_F32) CV(float, float); else CV(float, bf16); }
    else { if (td == EVO_F32) CV(bf16, float); else CV(bf16, bf16); }
#undef CV
    EVO_LAUNCHED("copy2d_vec_kernel");
    return EVO_OK;
  }
  int nb = ew_blocks(total);
#define C(A, B) launch_k(copy2d_kernel<A, B>, nb, 256, 0, st, rows, cols, src, s_rs, s_cs, dst, d_rs, d_cs)
  if (ts == EVO_F32) { if (td == EVO_F32) C(float, float); else C(float, bf16); }
  else { if (td == EVO_F32) C(bf16, float); else C(bf16, bf16); }
#undef C
  EVO_LAUNCHED("copy2d_kernel");
  return EVO_OK;
}

int mul2d(int ta, int tb, int to, int64_t rows, int64_t cols, const void *a, int64_t a_rs,
          const void *b, int64_t b_rs, void *o, int64_t o_rs, cudaStream_t st) {
  int64_t total = rows * cols;
  if (total == 0) return EVO_OK;
  int nb = ew_blocks(total);
#define M3(A, B, O) launch_k(mul2d_kernel<A, B, O>, nb, 256, 0, st, rows, cols, a, a_rs, b, b_rs, o, o_rs)
  if (ta == EVO_F32 && tb == EVO_F32 && to == EVO_F32) M3(float, float, float);
  else if (ta == EVO_BF16 && tb == EVO_BF16 && to == EVO_BF16) M3(bf16, bf16, bf16);
  else if (ta == EVO_BF16 && tb == EVO_BF16 && to == EVO_F32) M3(bf16, bf16, float);
  else if (ta == EVO_F32 && tb == EVO_F32 && to == EVO_BF16) M3(float, float, bf16);
  else if (ta == EVO_F32 && tb == EVO_BF16) { if (to == EVO_F32) M3(float, bf16, float); else M3(float, bf16, bf16); }
  else { if (to == EVO_F32) M3(bf16, float, float); else M3(bf16, float, bf16); }
#undef M3
  EVO_LAUNCHED("mul2d_kernel");
  return EVO_OK;
}

int trimul_gate_fwd(int dt, int64_t rows, int c, const void *proj, int64_t ldp, void *a_cf,
                    void *b_cf, cudaStream_t st) {
  unsigned nb = (unsigned)((rows + 31) / 32);
  size_t smem = (size_t)2 * c * 33 * sizeof(float);
  if (dt == EVO_F32)
    launch_k(trimul_gate_fwd_kernel<float>, nb, 256, smem, st, rows, c, proj, ldp, a_cf, b_cf);
  else
    launch_k(trimul_gate_fwd_kernel<bf16>, nb, 256, smem, st, rows, c, proj, ldp, a_cf, b_cf);
  EVO_LAUNCHED("trimul_gate_fwd_kernel");
  return EVO_OK;
}

int trimul_gate_bwd(int dt, int64_t rows, int c, const void *proj, int64_t ldp, const float *da,
                    const float *db, void *dproj, int64_t ldd, float *colsum, float *ws,
                    cudaStream_t st) {
  unsigned nb = (unsigned)((rows + 31) / 32);
  size_t smem = (size_t)(colsum ? 6 : 2) * c * 33 * sizeof(float);
  float *part = colsum ? ws : nullptr;
  if (dt == EVO_F32)
    launch_k(trimul_gate_bwd_kernel<float>, nb, 256, smem, st, rows, c, proj, ldp, da, db, dproj, ldd,
                                                         part);
  else
    launch_k(trimul_gate_bwd_kernel<bf16>, nb, 256, smem, st, rows, c, proj, ldp, da, db, dproj, ldd,
                                                        part);
  EVO_LAUNCHED("trimul_gate_bwd_kernel");
  if (colsum) {
    launch_k(colsum_stage2, (unsigned)((4 * c + 31) / 32), 1024, 0, st, (int)nb, 4 * c, part, colsum, 0);
    EVO_LAUNCHED("colsum_stage2");
  }
  return EVO_OK;
}

size_t trimul_gate_bwd_ws(int64_t rows, int c) {
  return (size_t)((rows + 31) / 32) * 4 * c * sizeof(float);
}

int outgate_fwd(int dt, int64_t rows, int64_t cols, const float *z, const void *g, int64_t g_rs,
                const void *o, int64_t o_rs, float *znew, cudaStream_t st) {
  int nb = ew_blocks(rows * cols);
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (dt == EVO_BF16 && cols % 8 == 0 && g_rs % 8 == 0 && o_rs % 8 == 0 && al16(z) && al16(g) &&
      al16(o) && al16(znew)) {
    launch_k(outgate_fwd_bf16x8_kernel, ew_blocks(rows * cols / 8), 256, 0, st, rows, cols, z, reinterpret_cast<const bf16 *>(g), g_rs, reinterpret_cast<const bf16 *>(o),
        o_rs, znew);
    EVO_LAUNCHED("outgate_fwd_bf16x8_kernel");
    return EVO_OK;
  }
  if (dt == EVO_F32) launch_k(outgate_fwd_kernel<float>, nb, 256, 0, st, rows, cols, z, g, g_rs, o, o_rs, znew);
  else launch_k(outgate_fwd_kernel<bf16>, nb, 256, 0, st, rows, cols, z, g, g_rs, o, o_rs, znew);
  EVO_LAUNCHED("outgate_fwd_kernel");
  return EVO_OK;
}

static int64_t outgate_colsum_blocks(int64_t rows, int64_t cols, int64_t &rpb) {
  const int64_t col_tiles = (cols + 255) / 256;
  int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(256, (4 * num_sms() + col_tiles - 1) /
                                                                 col_tiles));
  nblk = std::min<int64_t>(nblk, std::max<int64_t>(1, rows / 64));
  rpb = (rows + nblk - 1) / nblk;
  return (rows + rpb - 1) / rpb;
}

size_t outgate_bwd_ws(int64_t rows, int64_t cols) {
  int64_t rpb;
  return (size_t)outgate_colsum_blocks(rows, cols, rpb) * 2 * cols * sizeof(float);
}

int outgate_bwd(int dt, int64_t rows, int64_t cols, const float *dz, const void *g, int64_t g_rs,
                const void *o, int64_t o_rs, void *do_, int64_t do_rs, void *dgp, int64_t dg_rs,
                float *do_colsum, float *dg_colsum, float *ws, cudaStream_t st) {
  int nb = ew_blocks(rows * cols);
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = dt == EVO_BF16 && cols % 8 == 0 && g_rs % 8 == 0 && o_rs % 8 == 0 &&
                   do_rs % 8 == 0 && dg_rs % 8 == 0 && al16(dz) && al16(g) && al16(o) &&
                   al16(do_) && al16(dgp);
  if (do_colsum || dg_colsum) {
    EVO_REQUIRE(vec && do_colsum && dg_colsum && ws, EVO_EUNSUP,
                "outgate_bwd: fused column sums need bf16, cols %% 8 == 0, aligned rows");
    int64_t rpb;
    const int64_t nblk = outgate_colsum_blocks(rows, cols, rpb);
    const int64_t col_tiles = (cols + 255) / 256;
    float *pdo = ws, *pdg = ws + nblk * cols;
    launch_k(outgate_bwd_colsum_kernel, dim3((unsigned)nblk, (unsigned)col_tiles), dim3(32, 8), 0, st, rows, cols, dz, reinterpret_cast<const bf16 *>(g), g_rs, reinterpret_cast<const bf16 *>(o),
        o_rs, reinterpret_cast<bf16 *>(do_), do_rs, reinterpret_cast<bf16 *>(dgp), dg_rs, rpb, pdo,
        pdg);
    EVO_LAUNCHED("outgate_bwd_colsum_kernel");
    launch_k(colsum_stage2, (unsigned)((cols + 31) / 32), 1024, 0, st, (int)nblk, cols, pdo, do_colsum, 0);
    EVO_LAUNCHED("colsum_stage2");
    launch_k(colsum_stage2, (unsigned)((cols + 31) / 32), 1024, 0, st, (int)nblk, cols, pdg, dg_colsum, 0);
    EVO_LAUNCHED("colsum_stage2");
    return EVO_OK;
  }
  if (vec) {
    launch_k(outgate_bwd_bf16x8_kernel, ew_blocks(rows * cols / 8), 256, 0, st, rows, cols, dz, reinterpret_cast<const bf16 *>(g), g_rs,
        reinterpret_cast<const bf16 *>(o), o_rs, reinterpret_cast<bf16 *>(do_), do_rs,
        reinterpret_cast<bf16 *>(dgp), dg_rs);
    EVO_LAUNCHED("outgate_bwd_bf16x8_kernel");
    return EVO_OK;
  }
  if (dt == EVO_F32)
    launch_k(outgate_bwd_kernel<float>, nb, 256, 0, st, rows, cols, dz, g, g_rs, o, o_rs, do_, do_rs, dgp, dg_rs);
  else
    launch_k(outgate_bwd_kernel<bf16>, nb, 256, 0, st, rows, cols, dz, g, g_rs, o, o_rs, do_, do_rs, dgp, dg_rs);
  EVO_LAUNCHED("outgate_bwd_kernel");
  return EVO_OK;
}

int relu_bwd(int dt, int64_t n, const void *dh, const void *h, void *dpre, cudaStream_t st) {
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (dt == EVO_BF16 && n % 8 == 0 && al16(dh) && al16(h) && al16(dpre)) {
    launch_k(relu_bwd_bf16x8_kernel, ew_blocks(n / 8), 256, 0, st, n / 8, reinterpret_cast<const uint4 *>(dh), reinterpret_cast<const uint4 *>(h),
        reinterpret_cast<uint4 *>(dpre));
    EVO_LAUNCHED("relu_bwd_bf16x8_kernel");
    return EVO_OK;
  }
  int nb = ew_blocks(n);
  if (dt == EVO_F32) launch_k(relu_bwd_kernel<float>, nb, 256, 0, st, n, dh, h, dpre);
  else launch_k(relu_bwd_kernel<bf16>, nb, 256, 0, st, n, dh, h, dpre);
  EVO_LAUNCHED("relu_bwd_kernel");
  return EVO_OK;
}

// Ordered column sums of [nblk, cols] fp32 partials (coalesced stage 2).
int colsum_partials(int nblk, int64_t cols, const float *part, float *dst, int acc,
                    cudaStream_t st) {
  launch_k(colsum_stage2, (unsigned)((cols + 31) / 32), 1024, 0, st, nblk, cols, part, dst, acc);
  EVO_LAUNCHED("colsum_stage2");
  return EVO_OK;
}

int relu_bwd_colsum(int64_t rows, int64_t cols, const void *dh, const void *h, void *dpre,
                    float *dst, float *ws, cudaStream_t st) {
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  EVO_REQUIRE(cols % 8 == 0 && al16(dh) && al16(h) && al16(dpre), EVO_EUNSUP,
              "relu_bwd_colsum: bf16 rows of 8k columns, 16-byte aligned");
  if (rows == 0) return EVO_OK;
  const int64_t col_tiles = (cols + 255) / 256;
  int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(256, (4 * num_sms() + col_tiles - 1) /
                                                                 col_tiles));
  nblk = std::min<int64_t>(nblk, std::max<int64_t>(1, rows / 64));
  const int64_t rpb = (rows + nblk - 1) / nblk;
  nblk = (rows + rpb - 1) / rpb;
  launch_k(relu_bwd_colsum_kernel, dim3((unsigned)nblk, (unsigned)col_tiles), dim3(32, 8), 0, st, rows, cols, reinterpret_cast<const bf16 *>(dh), reinterpret_cast<const bf16 *>(h),
      reinterpret_cast<bf16 *>(dpre), rpb, ws);
  EVO_LAUNCHED("relu_bwd_colsum_kernel");
  launch_k(colsum_stage2, (unsigned)((cols + 31) / 32), 1024, 0, st, (int)nblk, cols, ws, dst, 0);
  EVO_LAUNCHED("colsum_stage2");
  return EVO_OK;
}

int sq_mean(int64_t n, const float *x, float *out, float *dx, void *ws, cudaStream_t st) {
  float *part = reinterpret_cast<float *>(ws);
  launch_k(sq_partial_kernel, SQ_BLOCKS, 256, 0, st, n, x, part, dx);
  EVO_LAUNCHED("sq_partial_kernel");
  launch_k(sq_final_kernel, 1, 256, 0, st, SQ_BLOCKS, n, part, out);
  EVO_LAUNCHED("sq_final_kernel");
  return EVO_OK;
}

// x (fp32) = hi + lo with hi = bf16(x), lo = bf16(x - hi): the split operand
// of a 3-product bf16 GEMM (hi*hi' + lo*hi' + hi*lo' ~ fp32 product).  hi is
// written to hi (and hi2 when given), lo to lo; 4 columns per thread.
__global__ void split_bf16_kernel(int64_t rows, int64_t cols, const float *__restrict__ x,
                                  int64_t x_rs, bf16 *__restrict__ hi, int64_t h_rs,
                                  bf16 *__restrict__ lo, int64_t l_rs, bf16 *__restrict__ hi2,
                                  int64_t h2_rs) {
  evo_pdl_enter();
  const int64_t c4 = (cols + 3) / 4;
  const int64_t total = rows * c4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / c4, c0 = (e - r * c4) * 4;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t c = c0 + u;
      if (c >= cols) break;
      const float v = x[r * x_rs + c];
      const bf16 h = __float2bfloat16(v);
      const bf16 l = __float2bfloat16(v - __bfloat162float(h));
      hi[r * h_rs + c] = h;
      lo[r * l_rs + c] = l;
      if (hi2) hi2[r * h2_rs + c] = h;
    }
  }
}

int split_bf16(int64_t rows, int64_t cols, const float *x, int64_t x_rs, void *hi, int64_t h_rs,
               void *lo, int64_t l_rs, void *hi2, int64_t h2_rs, cudaStream_t st) {
  launch_k(split_bf16_kernel, ew_blocks(rows * ((cols + 3) / 4)), 256, 0, st, rows, cols, x, x_rs, reinterpret_cast<bf16 *>(hi), h_rs, reinterpret_cast<bf16 *>(lo), l_rs,
      reinterpret_cast<bf16 *>(hi2), h2_rs);
  EVO_LAUNCHED("split_bf16_kernel");
  return EVO_OK;
}

int div_scalar(int64_t n, const float *x, float d, float *o, cudaStream_t st) {
  launch_k(div_scalar_kernel, ew_blocks(n), 256, 0, st, n, x, d, o);
  EVO_LAUNCHED("div_scalar_kernel");
  return EVO_OK;
}

int add(int64_t n, const float *a, const float *b, float *o, cudaStream_t st) {
  launch_k(add_kernel, ew_blocks(n), 256, 0, st, n, a, b, o);
  EVO_LAUNCHED("add_kernel");
  return EVO_OK;
}

}  // namespace evo
