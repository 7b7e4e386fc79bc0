// LayerNorm forward/backward over the last axis (src/tensor.py:366-392).
// Warp per row with the row in registers; two-pass population variance as
// in the reference.  Contiguous rows with cols % 128 == 0 (c_m = 256,
// c_z = 128) take a vectorised fast path (16-byte loads/stores, ~8 rows in
// flight per SM scheduler); other shapes (channel-first p of the triangle
// multiplication, tiny test dims) a generic strided path.  gamma/beta
// gradients: per-warp register partials -> per-block partials -> an ordered
// warp-per-column reduction (fixed grid, bitwise reproducible).
#include "tc_common.cuh"

namespace evo {
namespace {

constexpr int LN_WARPS = 8;
constexpr int LN_BWD_BLOCKS = 592;  // 4 x 148; fixed => reproducible sums
constexpr int MAXV = 16;            // generic path: cols <= 32*MAXV

// ----------------------------------------------------------- vector helpers
template <typename T, int N> struct Vec;
template <> struct Vec<float, 4> {
  static __device__ __forceinline__ void load(const float *p, float (&v)[4]) {
    float4 a = *reinterpret_cast<const float4 *>(p);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
  static __device__ __forceinline__ void store(float *p, const float (&v)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct Vec<bf16, 4> {
  static __device__ __forceinline__ void load(const bf16 *p, float (&v)[4]) {
    uint2 a = *reinterpret_cast<const uint2 *>(p);
    float2 lo = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162 *>(&a.x));
    float2 hi = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162 *>(&a.y));
    v[0] = lo.x; v[1] = lo.y; v[2] = hi.x; v[3] = hi.y;
  }
  static __device__ __forceinline__ void store(bf16 *p, const float (&v)[4]) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 hi = __floats2bfloat162_rn(v[2], v[3]);
    uint2 a;
    a.x = *reinterpret_cast<uint32_t *>(&lo);
    a.y = *reinterpret_cast<uint32_t *>(&hi);
    *reinterpret_cast<uint2 *>(p) = a;
  }
};

// ------------------------------------------------------------ fast forward
// NV = cols / 128 float4-groups per lane; lane owns columns 4*lane + 128*i.
template <typename TX, typename TY, int NV>
__global__ void __launch_bounds__(LN_WARPS * 32)
ln_fwd_vec_kernel(int64_t rows, const TX *__restrict__ x, int64_t x_rs,
                  const float *__restrict__ gamma, const float *__restrict__ beta,
                  TY *__restrict__ y, int64_t y_rs, float *__restrict__ mean_out,
                  float *__restrict__ rstd_out, float eps) {
  evo_pdl_enter();
  // RPW rows per warp, all loads issued before the first reduction
  constexpr int cols = NV * 128, RPW = 4;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = ((int64_t)blockIdx.x * LN_WARPS + (threadIdx.x >> 5)) * RPW;
  if (row0 >= rows) return;
  float v[RPW][NV][4];
#pragma unroll
  for (int r = 0; r < RPW; ++r)
    if (row0 + r < rows) {
#pragma unroll
      for (int i = 0; i < NV; ++i)
        Vec<TX, 4>::load(x + (row0 + r) * x_rs + 4 * lane + 128 * i, v[r][i]);
    }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int64_t row = row0 + r;
    if (row >= rows) break;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s += v[r][i][j];
    const float mu = warp_sum(s) * (1.f / cols);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float d = v[r][i][j] - mu;
        q += d * d;
      }
    const float rs = 1.f / sqrtf(warp_sum(q) * (1.f / cols) + eps);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = 4 * lane + 128 * i;
      float4 g4 = *reinterpret_cast<const float4 *>(gamma + c);
      float4 b4 = *reinterpret_cast<const float4 *>(beta + c);
      float o[4] = {(v[r][i][0] - mu) * rs * g4.x + b4.x, (v[r][i][1] - mu) * rs * g4.y + b4.y,
                    (v[r][i][2] - mu) * rs * g4.z + b4.z, (v[r][i][3] - mu) * rs * g4.w + b4.w};
      Vec<TY, 4>::store(y + row * y_rs + c, o);
    }
    if (lane == 0) {
      mean_out[row] = mu;
      rstd_out[row] = rs;
    }
  }
}

// Sum 8 per-lane values over the warp with a transposing butterfly (9
// shuffles instead of 8 x 5): returns, in every lane, the total of value
// h8(lane) = 4*bit4 + 2*bit3 + bit2 of the lane id (fixed order: bitwise
// reproducible).
__device__ __forceinline__ float warp_sum8_scatter(const float (&v)[8], int lane) {
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
  float w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float send = u16 ? v[k] : v[k + 4];
    const float keep = u16 ? v[k + 4] : v[k];
    w[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float x2[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float send = u8 ? w[k] : w[k + 2];
    const float keep = u8 ? w[k + 2] : w[k];
    x2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const float send = u4 ? x2[0] : x2[1];
  float y = (u4 ? x2[1] : x2[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
  y += __shfl_xor_sync(0xffffffffu, y, 2);
  y += __shfl_xor_sync(0xffffffffu, y, 1);
  return y;
}

// --------------------------------------------------------- generic forward
template <typename TX, typename TY, int V>
__global__ void __launch_bounds__(LN_WARPS * 32)
ln_fwd_kernel(int64_t rows, int cols, const TX *__restrict__ x, int64_t x_rs, int64_t x_cs,
              const float *__restrict__ gamma, const float *__restrict__ beta, TY *__restrict__ y,
              int64_t y_rs, float *__restrict__ mean_out, float *__restrict__ rstd_out, float eps) {
  evo_pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * LN_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  float v[V];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    int c = lane + 32 * j;
    v[j] = (c < cols) ? to_f(x[row * x_rs + (int64_t)c * x_cs]) : 0.f;
    s += v[j];
  }
  const float inv_n = 1.f / (float)cols;
  const float mu = warp_sum(s) * inv_n;
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    int c = lane + 32 * j;
    float d = (c < cols) ? v[j] - mu : 0.f;
    q += d * d;
  }
  const float rs = 1.f / sqrtf(warp_sum(q) * inv_n + eps);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    int c = lane + 32 * j;
    if (c < cols) y[row * y_rs + c] = from_f<TY>((v[j] - mu) * rs * gamma[c] + beta[c]);
  }
  if (lane == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
}

// ----------------------------------------------------------- fast backward
template <typename TDY, typename TX, typename TDX, int NV>
__global__ void __launch_bounds__(LN_WARPS * 32)
ln_bwd_vec_kernel(int64_t rows, const TDY *__restrict__ dy, int64_t dy_rs,
                  const TX *__restrict__ x, int64_t x_rs, const float *__restrict__ mean,
                  const float *__restrict__ rstd, const float *__restrict__ gamma,
                  const float *__restrict__ dres, TDX *__restrict__ dx, int64_t dx_rs,
                  bf16 *__restrict__ dxa, int64_t dxa_rs, float *__restrict__ partial,
                  int nparts) {
  evo_pdl_enter();
  // partial[block][0..nparts)[cols]: dgamma, dbeta, and (nparts == 3) the
  // column sums of dx itself (the next consumer's bias gradient)
  constexpr int cols = NV * 128;
  __shared__ float red[LN_WARPS][3][cols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float pg[NV][4], pb[NV][4], pc[NV][4], g[NV][4];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float4 g4 = *reinterpret_cast<const float4 *>(gamma + 4 * lane + 128 * i);
    g[i][0] = g4.x; g[i][1] = g4.y; g[i][2] = g4.z; g[i][3] = g4.w;
#pragma unroll
    for (int j = 0; j < 4; ++j) pg[i][j] = pb[i][j] = pc[i][j] = 0.f;
  }
  constexpr float inv_n = 1.f / cols;
  // A warp walks rows with a stride; the loads of its next row are issued
  // before the current row's reductions (two row buffers, swapped by
  // unrolling the loop by two), so each warp keeps two rows in flight.
  struct RowIn {
    float dv[NV][4], xv[NV][4], dr[NV][4];
    float mu, rs;
  };
  auto load = [&](int64_t row, RowIn &in) {
    in.mu = mean[row];
    in.rs = rstd[row];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = 4 * lane + 128 * i;
      Vec<TDY, 4>::load(dy + row * dy_rs + c, in.dv[i]);
      Vec<TX, 4>::load(x + row * x_rs + c, in.xv[i]);
      if (dres) {
        const float4 d4 = *reinterpret_cast<const float4 *>(dres + row * dx_rs + c);
        in.dr[i][0] = d4.x; in.dr[i][1] = d4.y; in.dr[i][2] = d4.z; in.dr[i][3] = d4.w;
      }
    }
  };
  auto process = [&](int64_t row, const RowIn &in) {
    const float mu = in.mu, rs = in.rs;
    float xh[NV][4], dxh[NV][4];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float dv = in.dv[i][j];
        xh[i][j] = (in.xv[i][j] - mu) * rs;
        dxh[i][j] = dv * g[i][j];
        s1 += dxh[i][j];
        s2 += dxh[i][j] * xh[i][j];
        pg[i][j] += dv * xh[i][j];
        pb[i][j] += dv;
      }
    }
    const float m1 = warp_sum(s1) * inv_n;
    const float m2 = warp_sum(s2) * inv_n;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = 4 * lane + 128 * i;
      float r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = rs * (dxh[i][j] - m1 - xh[i][j] * m2);
      if (dres) {
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] += in.dr[i][j];
      }
      Vec<TDX, 4>::store(dx + row * dx_rs + c, r);
      if (dxa) Vec<bf16, 4>::store(dxa + row * dxa_rs + c, r);
#pragma unroll
      for (int j = 0; j < 4; ++j) pc[i][j] += r[j];
    }
  };
  const int64_t stride = (int64_t)gridDim.x * LN_WARPS;
  int64_t row = (int64_t)blockIdx.x * LN_WARPS + warp;
  RowIn ra, rb;
  if (row < rows) load(row, ra);
  for (; row < rows; row += 2 * stride) {
    if (row + stride < rows) load(row + stride, rb);
    process(row, ra);
    if (row + stride >= rows) break;
    if (row + 2 * stride < rows) load(row + 2 * stride, ra);
    process(row + stride, rb);
  }
  if (!nparts) return;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      red[warp][0][4 * lane + 128 * i + j] = pg[i][j];
      red[warp][1][4 * lane + 128 * i + j] = pb[i][j];
      red[warp][2][4 * lane + 128 * i + j] = pc[i][j];
    }
  __syncthreads();
  for (int c = threadIdx.x; c < nparts * cols; c += blockDim.x) {
    const int which = c / cols, cc = c % cols;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < LN_WARPS; ++w) s += red[w][which][cc];
    partial[((int64_t)blockIdx.x * nparts + which) * cols + cc] = s;
  }
}

// ------------------------------------- backward + pair-bias projection
// c_z = 128 rows.  dy_tot = dy (may be NULL) + dproj^T Wp^T with dproj fp32
// [NH, p_rs] (the pair-bias gradient summed over heads' batch rows);
// dx = LN_bwd(dy_tot) (+ dres), optional bf16 copy and column sums of dx as
// in ln_bwd_vec_kernel; partials [block][3 + NH][128]: dgamma, dbeta, colsum,
// and dWp^T[hh][c] = sum_rows bf16(y[row,c]) * dproj[hh,row] with y = LN(x)
// recomputed exactly as the forward rounded it.
template <int NH>
__global__ void __launch_bounds__(LN_WARPS * 32)
ln_bwd_proj_kernel(int64_t rows, const float *__restrict__ dy, const float *__restrict__ x,
                   const float *__restrict__ mean, const float *__restrict__ rstd,
                   const float *__restrict__ gamma, const float *__restrict__ beta,
                   const float *__restrict__ dres, const float *__restrict__ dproj, int64_t p_rs,
                   const bf16 *__restrict__ Wp, int nh, float *__restrict__ dx,
                   bf16 *__restrict__ dxa, float *__restrict__ partial) {
  evo_pdl_enter();
  constexpr int cols = 128, NP = 3 + NH;
  __shared__ float red[LN_WARPS][NP][cols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float W[4][NH], pw[4][NH], pg[4], pb[4], pc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    pg[j] = pb[j] = pc[j] = 0.f;
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) {
      W[j][hh] = hh < nh ? __bfloat162float(Wp[(4 * lane + j) * nh + hh]) : 0.f;
      pw[j][hh] = 0.f;
    }
  }
  const float4 g4 = *reinterpret_cast<const float4 *>(gamma + 4 * lane);
  const float4 b4 = *reinterpret_cast<const float4 *>(beta + 4 * lane);
  const float g[4] = {g4.x, g4.y, g4.z, g4.w}, bt[4] = {b4.x, b4.y, b4.z, b4.w};
  constexpr float inv_n = 1.f / cols;
  for (int64_t row = (int64_t)blockIdx.x * LN_WARPS + warp; row < rows;
       row += (int64_t)gridDim.x * LN_WARPS) {
    const float mu = mean[row], rs = rstd[row];
    // this row's NH projection gradients: lane hh loads, shuffles broadcast
    const float mine = lane < nh ? __ldg(&dproj[(int64_t)lane * p_rs + row]) : 0.f;
    float dp[NH];
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) dp[hh] = __shfl_sync(0xffffffffu, mine, hh);
    float dv[4] = {0.f, 0.f, 0.f, 0.f}, xv[4];
    if (dy) Vec<float, 4>::load(dy + row * cols + 4 * lane, dv);
    Vec<float, 4>::load(x + row * cols + 4 * lane, xv);
    float xh[4], dxh[4], s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float d = dv[j];
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) d = fmaf(dp[hh], W[j][hh], d);
      xh[j] = (xv[j] - mu) * rs;
      // y exactly as the forward produced it (bf16), for dWp
      const float yv = __bfloat162float(__float2bfloat16_rn((xv[j] - mu) * rs * g[j] + bt[j]));
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) pw[j][hh] = fmaf(yv, dp[hh], pw[j][hh]);
      dxh[j] = d * g[j];
      s1 += dxh[j];
      s2 += dxh[j] * xh[j];
      pg[j] += d * xh[j];
      pb[j] += d;
    }
    const float m1 = warp_sum(s1) * inv_n;
    const float m2 = warp_sum(s2) * inv_n;
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = rs * (dxh[j] - m1 - xh[j] * m2);
    if (dres) {
      float4 d4 = *reinterpret_cast<const float4 *>(dres + row * cols + 4 * lane);
      r[0] += d4.x; r[1] += d4.y; r[2] += d4.z; r[3] += d4.w;
    }
    Vec<float, 4>::store(dx + row * cols + 4 * lane, r);
    if (dxa) Vec<bf16, 4>::store(dxa + row * cols + 4 * lane, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) pc[j] += r[j];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = 4 * lane + j;
    red[warp][0][c] = pg[j];
    red[warp][1][c] = pb[j];
    red[warp][2][c] = pc[j];
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) red[warp][3 + hh][c] = pw[j][hh];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < NP * cols; c += blockDim.x) {
    const int which = c / cols, cc = c % cols;
    float sacc = 0.f;
#pragma unroll
    for (int w = 0; w < LN_WARPS; ++w) sacc += red[w][which][cc];
    partial[((int64_t)blockIdx.x * NP + which) * cols + cc] = sacc;
  }
}

// ------------------------------------------- TMA-staged backward (fp32)
// The register-staged kernels above keep ~1.5 rows in flight per warp and
// stall at ~4 TB/s (the proj variant, 128 registers for W / dW, at ~2).
// Here one persistent CTA per SM splits producer and consumers: a producer
// lane streams chunks of RCH contiguous rows -- x, dy, dres, mean, rstd and
// the NH projection-gradient rows -- into an LNT_NS-deep smem ring with
// bulk async copies (cp.async.bulk, mbarrier completion), so ~3 chunks
// (~150 KB) per SM are in flight regardless of the consumers' reduction
// latency; 12 consumer warps finish two rows per pass from smem with
// exactly the per-row arithmetic of ln_bwd_vec_kernel / ln_bwd_proj_kernel.
// Partials: [block][nparts][cols], reduced by ln_param_reduce_kernel.

// consumer warps: 12 (registers cap 128) / 8 with the projection's W, dW
template <int NV, int NH> constexpr int lnt_cw() { return NH > 0 ? 8 : 12; }

template <int NV, int NH>
struct LntLayout {
  static constexpr int CW = lnt_cw<NV, NH>();
  static constexpr int cols = NV * 128, RCH = (NH > 0 ? 4 : 2) * CW / NV;
  static constexpr uint32_t RB = RCH * cols * 4;  // 12 KB per row tensor
  static constexpr uint32_t OFF_DY = RB, OFF_DR = 2 * RB, OFF_MU = 3 * RB;
  static constexpr uint32_t OFF_RS = OFF_MU + 128, OFF_DP = OFF_RS + 128;
  static constexpr uint32_t STAGE = OFF_DP + (NH > 0 ? NH : 1) * 128;
  static constexpr int NS = 5 * STAGE <= 200 * 1024 ? 5 : 4;  // ring depth
  static constexpr uint32_t SMEM = NS * STAGE + 2 * NS * 8;
  static_assert(RCH * 4 <= 128 && NS * STAGE <= 200 * 1024, "ring layout");
};

template <int NV, int NH>
__global__ void __launch_bounds__((lnt_cw<NV, NH>() + 1) * 32, 1)
ln_bwd_tma_kernel(int64_t rows, const float *__restrict__ dy, const float *__restrict__ x,
                  const float *__restrict__ mean, const float *__restrict__ rstd,
                  const float *__restrict__ gamma, const float *__restrict__ beta,
                  const float *__restrict__ dres, const float *__restrict__ dproj, int64_t p_rs,
                  const bf16 *__restrict__ Wp, int nh, float *__restrict__ dx,
                  bf16 *__restrict__ dxa, float *__restrict__ partial, int nparts) {
  evo_pdl_enter();
  using Lay = LntLayout<NV, NH>;
  constexpr int LNT_CW = Lay::CW, LNT_NS = Lay::NS;
  constexpr int cols = Lay::cols, RCH = Lay::RCH;
  constexpr int NHR = NH > 0 ? NH : 1;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + LNT_NS * Lay::STAGE);
  uint64_t *empty = full + LNT_NS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (rows + RCH - 1) / RCH;
  if (threadIdx.x == 0) {
    for (int s = 0; s < LNT_NS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], LNT_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float pg[NV][4], pb[NV][4], pc[NV][4], g[NV][4], bt[NV][4];
  float W[4][NHR], pw[4][NHR];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float4 g4 = *reinterpret_cast<const float4 *>(gamma + 4 * lane + 128 * i);
    g[i][0] = g4.x; g[i][1] = g4.y; g[i][2] = g4.z; g[i][3] = g4.w;
    if constexpr (NH > 0) {
      const float4 b4 = *reinterpret_cast<const float4 *>(beta + 4 * lane + 128 * i);
      bt[i][0] = b4.x; bt[i][1] = b4.y; bt[i][2] = b4.z; bt[i][3] = b4.w;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) pg[i][j] = pb[i][j] = pc[i][j] = 0.f;
  }
  if constexpr (NH > 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        W[j][hh] = hh < nh ? __bfloat162float(Wp[(4 * lane + j) * nh + hh]) : 0.f;
        pw[j][hh] = 0.f;
      }
  }
  if (warp == LNT_CW) {
    if (lane == 0) {
      int it = 0;
      for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % LNT_NS;
        if (it >= LNT_NS) tc::mbar_wait(&empty[s], ((it / LNT_NS) - 1) & 1);
        const int64_t r0 = c * RCH;
        const uint32_t nr = (uint32_t)(rows - r0 < RCH ? rows - r0 : RCH);
        const uint32_t rb = nr * cols * 4, sb = nr * 4;
        uint8_t *st = sm + s * Lay::STAGE;
        uint32_t tx = rb + 2 * sb + (dy ? rb : 0) + (dres ? rb : 0);
        if constexpr (NH > 0) tx += (uint32_t)nh * sb;
        tc::mbar_expect_tx(&full[s], tx);
        tc::bulk_load(st, x + r0 * cols, rb, &full[s]);
        if (dy) tc::bulk_load(st + Lay::OFF_DY, dy + r0 * cols, rb, &full[s]);
        if (dres) tc::bulk_load(st + Lay::OFF_DR, dres + r0 * cols, rb, &full[s]);
        tc::bulk_load(st + Lay::OFF_MU, mean + r0, sb, &full[s]);
        tc::bulk_load(st + Lay::OFF_RS, rstd + r0, sb, &full[s]);
        if constexpr (NH > 0) {
          for (int hh = 0; hh < nh; ++hh)
            tc::bulk_load(st + Lay::OFF_DP + hh * 128, dproj + hh * p_rs + r0, sb, &full[s]);
        }
      }
    }
  } else {
    constexpr float inv_n = 1.f / cols;
    int it = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
      const int s = it % LNT_NS;
      tc::mbar_wait(&full[s], (it / LNT_NS) & 1);
      const int64_t r0 = c * RCH;
      const int nr = (int)(rows - r0 < RCH ? rows - r0 : RCH);
      const uint8_t *st = sm + s * Lay::STAGE;
      // two rows per pass (r, r + LNT_CW): their shuffle reductions interleave
      for (int rp = warp; rp < nr; rp += 2 * LNT_CW) {
        float xh[2][NV][4], dxh[2][NV][4], rsv[2], m1[2], m2[2];
        bool ok[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = rp + q * LNT_CW;
          ok[q] = r < nr;  // warp-uniform
          if (!ok[q]) continue;
          const float mu = reinterpret_cast<const float *>(st + Lay::OFF_MU)[r];
          const float rs = reinterpret_cast<const float *>(st + Lay::OFF_RS)[r];
          rsv[q] = rs;
          float dp[NHR];
          if constexpr (NH > 0) {
#pragma unroll
            for (int hh = 0; hh < NH; ++hh)
              dp[hh] = hh < nh ? reinterpret_cast<const float *>(st + Lay::OFF_DP + hh * 128)[r] : 0.f;
          }
          float s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            const uint32_t o = (uint32_t)(r * cols + 4 * lane + 128 * i) * 4;
            float xv[4], dv[4] = {0.f, 0.f, 0.f, 0.f};
            Vec<float, 4>::load(reinterpret_cast<const float *>(st + o), xv);
            if (dy) Vec<float, 4>::load(reinterpret_cast<const float *>(st + Lay::OFF_DY + o), dv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float d = dv[j];
              xh[q][i][j] = (xv[j] - mu) * rs;
              if constexpr (NH > 0) {
#pragma unroll
                for (int hh = 0; hh < NH; ++hh) d = fmaf(dp[hh], W[j][hh], d);
                const float yv =
                    __bfloat162float(__float2bfloat16_rn((xv[j] - mu) * rs * g[i][j] + bt[i][j]));
#pragma unroll
                for (int hh = 0; hh < NH; ++hh) pw[j][hh] = fmaf(yv, dp[hh], pw[j][hh]);
              }
              dxh[q][i][j] = d * g[i][j];
              s1 += dxh[q][i][j];
              s2 += dxh[q][i][j] * xh[q][i][j];
              pg[i][j] += d * xh[q][i][j];
              pb[i][j] += d;
            }
          }
          m1[q] = s1;
          m2[q] = s2;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (!ok[q]) continue;
          m1[q] = warp_sum(m1[q]) * inv_n;
          m2[q] = warp_sum(m2[q]) * inv_n;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (!ok[q]) continue;
          const int r = rp + q * LNT_CW;
          const int64_t row = r0 + r;
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            const int cc = 4 * lane + 128 * i;
            float rr[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) rr[j] = rsv[q] * (dxh[q][i][j] - m1[q] - xh[q][i][j] * m2[q]);
            if (dres) {
              float d4[4];
              Vec<float, 4>::load(
                  reinterpret_cast<const float *>(st + Lay::OFF_DR + (uint32_t)(r * cols + cc) * 4), d4);
#pragma unroll
              for (int j = 0; j < 4; ++j) rr[j] += d4[j];
            }
            Vec<float, 4>::store(dx + row * cols + cc, rr);
            if (dxa) Vec<bf16, 4>::store(dxa + row * cols + cc, rr);
#pragma unroll
            for (int j = 0; j < 4; ++j) pc[i][j] += rr[j];
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[s]);
    }
  }
  // every chunk consumed => every bulk copy landed; the ring becomes the
  // partials buffer [LNT_CW][nparts][cols]
  __syncthreads();
  if (!nparts) return;
  if (warp < LNT_CW) {
    float *red = reinterpret_cast<float *>(sm);
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cc = 4 * lane + 128 * i + j;
        red[(warp * nparts + 0) * cols + cc] = pg[i][j];
        red[(warp * nparts + 1) * cols + cc] = pb[i][j];
        if (nparts > 2) red[(warp * nparts + 2) * cols + cc] = pc[i][j];
        if constexpr (NH > 0) {
#pragma unroll
          for (int hh = 0; hh < NH; ++hh) red[(warp * nparts + 3 + hh) * cols + cc] = pw[j][hh];
        }
      }
  }
  __syncthreads();
  const float *red = reinterpret_cast<const float *>(sm);
  for (int c = threadIdx.x; c < nparts * cols; c += blockDim.x) {
    float sacc = 0.f;
#pragma unroll
    for (int w = 0; w < LNT_CW; ++w) sacc += red[w * nparts * cols + c];
    partial[(int64_t)blockIdx.x * nparts * cols + c] = sacc;
  }
}

// --------------------------------------------- TMA-staged forward (fp32 x)
// Same producer / consumer split as the backward: the producer lane streams
// RCH-row chunks of x into an LNF_NS-deep ring.  The forward has no
// per-column accumulators, so a consumer warp normalises FOUR rows at once,
// eight lanes per row (lane l8 owns columns 4*l8 + 32*i): the two dependent
// row reductions are 3-level 8-lane butterflies shared by the four rows
// instead of 5-level full-warp ones per row (the 32-lane mapping measured
// shuffle-latency bound at ~2.7 TB/s).  gamma / beta (and the projection
// weights) sit in smem.  NH > 0 fuses the pair-bias projection of the bf16 y
// (staged per warp in smem, then a 32-lane pass with W in registers):
// proj[hh * p_rs + row] = sum_c y[row, c] * Wp[c, hh]  (src/evoformer.py:279).
constexpr int LNF_CW = 16, LNF_NS = 6;

template <int NV>
struct LnfLayout {
  static constexpr int cols = NV * 128, RCH = 4 * LNF_CW / NV;
  static constexpr uint32_t STAGE = RCH * cols * 4;
  static constexpr uint32_t OFF_P = LNF_NS * STAGE;  // gamma, beta
  static constexpr uint32_t OFF_BAR = OFF_P + 2 * cols * 4;
  static constexpr uint32_t SMEM = OFF_BAR + 2 * LNF_NS * 8;
};

// Sum 8 per-lane values over the 8 lanes of a row group (xor 4, 2, 1) with a
// transposing butterfly: lane l8 ends with the total of value l8.
__device__ __forceinline__ float group8_sum8_scatter(const float (&v)[8], int l8) {
  const bool u4 = l8 & 4, u2 = l8 & 2, u1 = l8 & 1;
  float w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float send = u4 ? v[k] : v[k + 4];
    const float keep = u4 ? v[k + 4] : v[k];
    w[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  float x2[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float send = u2 ? w[k] : w[k + 2];
    const float keep = u2 ? w[k + 2] : w[k];
    x2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  const float send = u1 ? x2[0] : x2[1];
  return (u1 ? x2[1] : x2[0]) + __shfl_xor_sync(0xffffffffu, send, 1);
}

__device__ __forceinline__ float group8_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

// SPLIT: y is bf16 [rows, 3*cols] = hi | lo | hi with hi = bf16(LN(x)),
// lo = bf16(LN(x) - hi): the A operand of the transitions' 3-product bf16
// first projection (engine.transition_fwd)
template <int NV, int SPLIT, typename TY>
__global__ void __launch_bounds__((LNF_CW + 1) * 32, 1)
ln_fwd_tma_kernel(int64_t rows, const float *__restrict__ x, const float *__restrict__ gamma,
                  const float *__restrict__ beta, TY *__restrict__ y, float *__restrict__ mean_out,
                  float *__restrict__ rstd_out, float eps) {
  evo_pdl_enter();
  using Lay = LnfLayout<NV>;
  constexpr int cols = Lay::cols, RCH = Lay::RCH, NI = 4 * NV;
  static_assert(!SPLIT || std::is_same<TY, bf16>::value, "split output is bf16");
  extern __shared__ __align__(128) uint8_t sm[];
  float *sg = reinterpret_cast<float *>(sm + Lay::OFF_P), *sbt = sg + cols;
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + Lay::OFF_BAR);
  uint64_t *empty = full + LNF_NS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (rows + RCH - 1) / RCH;
  if (threadIdx.x == 0) {
    for (int s = 0; s < LNF_NS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], LNF_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < cols; i += blockDim.x) {
    sg[i] = gamma[i];
    sbt[i] = beta[i];
  }
  __syncthreads();
  if (warp == LNF_CW) {
    if (lane == 0) {
      int it = 0;
      for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % LNF_NS;
        if (it >= LNF_NS) tc::mbar_wait(&empty[s], ((it / LNF_NS) - 1) & 1);
        const int64_t r0 = c * RCH;
        const uint32_t nr = (uint32_t)(rows - r0 < RCH ? rows - r0 : RCH);
        tc::mbar_expect_tx(&full[s], nr * cols * 4);
        tc::bulk_load(sm + s * Lay::STAGE, x + r0 * cols, nr * cols * 4, &full[s]);
      }
    }
    return;
  }
  const int l8 = lane & 7, rg = lane >> 3;
  constexpr float inv_n = 1.f / cols;
  int it = 0;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int s = it % LNF_NS;
    tc::mbar_wait(&full[s], (it / LNF_NS) & 1);
    const int64_t r0 = c * RCH;
    const int nr = (int)(rows - r0 < RCH ? rows - r0 : RCH);
    const float *st = reinterpret_cast<const float *>(sm + s * Lay::STAGE);
    for (int q4 = warp; 4 * q4 < nr; q4 += LNF_CW) {
      const int r = 4 * q4 + rg;
      const bool ok = r < nr;  // per row group; the shuffles stay in-group
      float v[NI][4];
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        if (ok) Vec<float, 4>::load(st + r * cols + 4 * l8 + 32 * i, v[i]);
        else v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) sum += v[i][j];
      }
      const float mu = group8_sum(sum) * inv_n;
      float qq = 0.f;
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float d = v[i][j] - mu;
          qq += d * d;
        }
      const float rs = 1.f / sqrtf(group8_sum(qq) * inv_n + eps);
      const int64_t row = r0 + r;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int cc = 4 * l8 + 32 * i;
        const float4 g4 = *reinterpret_cast<const float4 *>(sg + cc);
        const float4 b4 = *reinterpret_cast<const float4 *>(sbt + cc);
        float o[4] = {(v[i][0] - mu) * rs * g4.x + b4.x, (v[i][1] - mu) * rs * g4.y + b4.y,
                      (v[i][2] - mu) * rs * g4.z + b4.z, (v[i][3] - mu) * rs * g4.w + b4.w};
        if (!ok) continue;
        if constexpr (SPLIT) {
          float hi[4], lo[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            hi[j] = __bfloat162float(__float2bfloat16(o[j]));
            lo[j] = o[j] - hi[j];
          }
          TY *yr = y + row * (3 * cols) + cc;
          Vec<TY, 4>::store(yr, hi);
          Vec<TY, 4>::store(yr + cols, lo);
          Vec<TY, 4>::store(yr + 2 * cols, hi);
        } else {
          Vec<TY, 4>::store(y + row * cols + cc, o);
        }
      }
      if (ok && l8 == 0) {
        mean_out[row] = mu;
        rstd_out[row] = rs;
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[s]);
  }
}

template <int NV, int SPLIT, typename TY>
int ln_fwd_tma_launch(int64_t rows, const float *x, const float *gamma, const float *beta, TY *y,
                      float *mean, float *rstd, float eps, cudaStream_t st) {
  using Lay = LnfLayout<NV>;
  const int64_t nchunks = (rows + Lay::RCH - 1) / Lay::RCH;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms(), nchunks));
  auto kfn = ln_fwd_tma_kernel<NV, SPLIT, TY>;
  EVO_MAX_SMEM_ONCE(kfn);
  launch_k(kfn, nb, (LNF_CW + 1) * 32, Lay::SMEM, st, rows, x, gamma, beta, y, mean, rstd, eps);
  EVO_LAUNCHED("ln_fwd_tma_kernel");
  return EVO_OK;
}

// ---------------------------------------------- channel-first (c <= 32)
// The triangle multiplication normalises p[c, i, j] over c with the data
// channel-first (x[c*rows + row]): one thread per row, the C channel values
// in registers, loads coalesced across threads for each channel.
template <int C, typename TY>
__global__ void __launch_bounds__(128)
ln_fwd_cf_kernel(int64_t rows, int cols, const float *__restrict__ x,
                 const float *__restrict__ gamma, const float *__restrict__ beta,
                 TY *__restrict__ y, int64_t y_rs, float *__restrict__ mean_out,
                 float *__restrict__ rstd_out, float eps) {
  evo_pdl_enter();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
  float v[C];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    v[c] = c < cols ? __ldg(&x[(int64_t)c * rows + row]) : 0.f;
    s += v[c];
  }
  const float inv_n = 1.f / (float)cols;
  const float mu = s * inv_n;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const float d = c < cols ? v[c] - mu : 0.f;
    q += d * d;
  }
  const float rs = 1.f / sqrtf(q * inv_n + eps);
  if constexpr (std::is_same<TY, bf16>::value && C % 8 == 0) {
    if (cols == C && (y_rs % 8) == 0 && ((reinterpret_cast<uintptr_t>(y) & 15) == 0)) {
#pragma unroll
      for (int c8 = 0; c8 < C; c8 += 8) {  // 16-byte stores of the row
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (v[c8 + j] - mu) * rs * gamma[c8 + j] + beta[c8 + j];
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __nv_bfloat162 h2 = __floats2bfloat162_rn(o[2 * j], o[2 * j + 1]);
          w[j] = *reinterpret_cast<uint32_t *>(&h2);
        }
        *reinterpret_cast<uint4 *>(y + row * y_rs + c8) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      mean_out[row] = mu;
      rstd_out[row] = rs;
      return;
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (c < cols) y[row * y_rs + c] = from_f<TY>((v[c] - mu) * rs * gamma[c] + beta[c]);
  mean_out[row] = mu;
  rstd_out[row] = rs;
}

// partial[block][2][C]: dgamma, dbeta of the block's 128 rows (fixed order)
template <int C, typename TDX>
__global__ void __launch_bounds__(128)
ln_bwd_cf_kernel(int64_t rows, int cols, const float *__restrict__ dy, int64_t dy_rs,
                 const float *__restrict__ x, const float *__restrict__ mean,
                 const float *__restrict__ rstd, const float *__restrict__ gamma,
                 TDX *__restrict__ dx, float *__restrict__ partial) {
  evo_pdl_enter();
  __shared__ float wred[4][2 * C];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool ok = row < rows;
  const float mu = ok ? mean[row] : 0.f, rs = ok ? rstd[row] : 0.f;
  float xh[C], dv[C];
  float s1 = 0.f, s2 = 0.f;
  const bool dvec = ok && cols == C && (dy_rs % 4) == 0 &&
                    ((reinterpret_cast<uintptr_t>(dy) & 15) == 0);
  if (dvec) {  // the row's gradients as 16-byte loads
#pragma unroll
    for (int c4 = 0; c4 < C; c4 += 4) {
      const float4 t = __ldg(reinterpret_cast<const float4 *>(dy + row * dy_rs + c4));
      dv[c4] = t.x; dv[c4 + 1] = t.y; dv[c4 + 2] = t.z; dv[c4 + 3] = t.w;
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const bool in = ok && c < cols;
    const float xv = in ? __ldg(&x[(int64_t)c * rows + row]) : 0.f;
    if (!dvec) dv[c] = in ? __ldg(&dy[row * dy_rs + c]) : 0.f;
    xh[c] = (xv - mu) * rs;
    const float d = dv[c] * (in ? gamma[c] : 0.f);
    s1 += d;
    s2 += d * xh[c];
  }
  const float inv_n = 1.f / (float)cols;
  const float m1 = s1 * inv_n, m2 = s2 * inv_n;
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (ok && c < cols)
      dx[(int64_t)c * rows + row] = from_f<TDX>(rs * (dv[c] * gamma[c] - m1 - xh[c] * m2));
  if constexpr (C == 32) {
    // transposing butterfly: after it lane c holds the warp's sum of column
    // c (31 shuffles per quantity instead of 32 x 5)
    float vg[32], vb[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      vg[c] = dv[c] * xh[c];
      vb[c] = dv[c];
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool up = lane & o;
#pragma unroll
      for (int k = 0; k < o; ++k) {
        const float sg = up ? vg[k] : vg[k + o], kg = up ? vg[k + o] : vg[k];
        const float sb = up ? vb[k] : vb[k + o], kb = up ? vb[k + o] : vb[k];
        vg[k] = kg + __shfl_xor_sync(0xffffffffu, sg, o);
        vb[k] = kb + __shfl_xor_sync(0xffffffffu, sb, o);
      }
    }
    wred[warp][lane] = vg[0];
    wred[warp][C + lane] = vb[0];
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const float pg = warp_sum(dv[c] * xh[c]);
      const float pb = warp_sum(dv[c]);
      if (lane == 0) {
        wred[warp][c] = pg;
        wred[warp][C + c] = pb;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * C) {
    const int which = threadIdx.x / C, c = threadIdx.x % C;
    const float t = (wred[0][threadIdx.x] + wred[1][threadIdx.x]) +
                    (wred[2][threadIdx.x] + wred[3][threadIdx.x]);
    if (c < cols) partial[((int64_t)blockIdx.x * 2 + which) * cols + c] = t;
  }
}

// -------------------------------------------------------- generic backward
template <typename TDY, typename TX, typename TDX, int V>
__global__ void __launch_bounds__(LN_WARPS * 32)
ln_bwd_kernel(int64_t rows, int cols, const TDY *__restrict__ dy, int64_t dy_rs,
              const TX *__restrict__ x, int64_t x_rs, int64_t x_cs, const float *__restrict__ mean,
              const float *__restrict__ rstd, const float *__restrict__ gamma,
              const float *__restrict__ dres, TDX *__restrict__ dx, int64_t dx_rs, int64_t dx_cs,
              float *__restrict__ partial /* [gridDim.x][2][cols] */, int want_params) {
  evo_pdl_enter();
  extern __shared__ float red[];  // [LN_WARPS][2][cols]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float pg[V], pb[V], g[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    pg[j] = 0.f;
    pb[j] = 0.f;
    int c = lane + 32 * j;
    g[j] = (c < cols) ? gamma[c] : 0.f;
  }
  const float inv_n = 1.f / (float)cols;
  for (int64_t row = (int64_t)blockIdx.x * LN_WARPS + warp; row < rows;
       row += (int64_t)gridDim.x * LN_WARPS) {
    const float mu = mean[row], rs = rstd[row];
    float xh[V], dxh[V];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      int c = lane + 32 * j;
      float dyv = 0.f, xv = 0.f;
      if (c < cols) {
        dyv = to_f(dy[row * dy_rs + c]);
        xv = (to_f(x[row * x_rs + (int64_t)c * x_cs]) - mu) * rs;
      }
      xh[j] = xv;
      dxh[j] = dyv * g[j];
      s1 += dxh[j];
      s2 += dxh[j] * xv;
      pg[j] += dyv * xv;
      pb[j] += dyv;
    }
    const float m1 = warp_sum(s1) * inv_n;
    const float m2 = warp_sum(s2) * inv_n;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      int c = lane + 32 * j;
      if (c < cols) {
        int64_t off = row * dx_rs + (int64_t)c * dx_cs;
        float r = rs * (dxh[j] - m1 - xh[j] * m2);
        if (dres) r += dres[off];
        dx[off] = from_f<TDX>(r);
      }
    }
  }
  if (!want_params) return;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    int c = lane + 32 * j;
    if (c < cols) {
      red[(warp * 2 + 0) * cols + c] = pg[j];
      red[(warp * 2 + 1) * cols + c] = pb[j];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * cols; c += blockDim.x) {
    float s = 0.f;
    int which = c / cols, cc = c % cols;
    for (int w = 0; w < LN_WARPS; ++w) s += red[(w * 2 + which) * cols + cc];
    partial[((int64_t)blockIdx.x * 2 + which) * cols + cc] = s;
  }
}

// Ordered reduction of the per-block partials: one warp per output value;
// lane l sums partials l, l+32, ... then a fixed shuffle tree.
// Column sums of the [nblk, nparts*cols] partials (see colsum_stage2): a
// 1024-thread block owns 32 output columns with lanes across columns
// (coalesced), the 32 warps take partial rows w, w+32, ..., combined in order.
__global__ void __launch_bounds__(1024) ln_param_reduce_kernel(int nblk, int cols, int nparts,
                                                              const float *__restrict__ partial,
                                                              float *__restrict__ dgamma,
                                                              float *__restrict__ dbeta,
                                                              float *__restrict__ dcol,
                                                              int accumulate,
                                                              float *__restrict__ dWp = nullptr,
                                                              int nh = 0) {
  evo_pdl_enter();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int width = nparts * cols;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < width) {
#pragma unroll 8
    for (int b = w; b < nblk; b += 32) s += __ldg(&partial[(int64_t)b * width + c]);
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < width) {
    float t = red[0][lane];
#pragma unroll
    for (int j = 1; j < 32; ++j) t += red[j][lane];
    const int which = c / cols, cc = c % cols;
    if (which >= 3) {
      if (which - 3 < nh) dWp[cc * nh + (which - 3)] = t;
    } else {
      float *dst = which == 0 ? dgamma : (which == 1 ? dbeta : dcol);
      if (dst) dst[cc] = (accumulate && which < 2) ? dst[cc] + t : t;
    }
  }
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename TX, typename TY>
int ln_fwd_launch(int64_t rows, int cols, const void *x, int64_t x_rs, int64_t x_cs,
                  const float *gamma, const float *beta, void *y, int64_t y_rs, float *mean,
                  float *rstd, float eps, cudaStream_t st) {
  dim3 grid((unsigned)((rows + LN_WARPS - 1) / LN_WARPS));
  const TX *xp = reinterpret_cast<const TX *>(x);
  TY *yp = reinterpret_cast<TY *>(y);
  if constexpr (std::is_same<TX, float>::value) {
    if (x_rs == 1 && x_cs == rows && cols <= 32) {  // channel-first
      launch_k(ln_fwd_cf_kernel<32, TY>, (unsigned)((rows + 127) / 128), 128, 0, st, rows, cols, xp, gamma, beta, yp, y_rs, mean, rstd, eps);
      EVO_LAUNCHED("ln_fwd_cf_kernel");
      return EVO_OK;
    }
  }
  const bool vec = x_cs == 1 && (cols == 128 || cols == 256) && x_rs % 4 == 0 && y_rs % 4 == 0 &&
                   aligned16(x) && aligned16(y) && aligned16(gamma) && aligned16(beta);
  if constexpr (std::is_same<TX, float>::value) {
    if (vec && x_rs == cols && y_rs == cols) {
      if (cols == 128)
        return ln_fwd_tma_launch<1, 0, TY>(rows, xp, gamma, beta, yp, mean, rstd, eps, st);
      return ln_fwd_tma_launch<2, 0, TY>(rows, xp, gamma, beta, yp, mean, rstd, eps, st);
    }
  }
  if (vec) {
    dim3 vgrid((unsigned)((rows + 4 * LN_WARPS - 1) / (4 * LN_WARPS)));  // 4 rows per warp
    if (cols == 128)
      launch_k(ln_fwd_vec_kernel<TX, TY, 1>, vgrid, LN_WARPS * 32, 0, st, rows, xp, x_rs, gamma, beta, yp,
                                                                   y_rs, mean, rstd, eps);
    else
      launch_k(ln_fwd_vec_kernel<TX, TY, 2>, vgrid, LN_WARPS * 32, 0, st, rows, xp, x_rs, gamma, beta, yp,
                                                                   y_rs, mean, rstd, eps);
    EVO_LAUNCHED("ln_fwd_vec_kernel");
    return EVO_OK;
  }
#define L(Vn)                                                                                \
  launch_k(ln_fwd_kernel<TX, TY, Vn>, grid, LN_WARPS * 32, 0, st, rows, cols, xp, x_rs, x_cs, gamma, \
                                                            beta, yp, y_rs, mean, rstd, eps)
  if (cols <= 32) L(1);
  else if (cols <= 64) L(2);
  else if (cols <= 128) L(4);
  else if (cols <= 256) L(8);
  else L(16);
#undef L
  EVO_LAUNCHED("ln_fwd_kernel");
  return EVO_OK;
}

// *nb_out = the grid size (= number of partial blocks)
int ln_bwd_tma_launch(int64_t rows, int cols, const float *dy, const float *x, const float *mean,
                      const float *rstd, const float *gamma, const float *beta,
                      const float *dres, const float *dproj, int64_t p_rs, const bf16 *Wp,
                      int nh, float *dx, bf16 *dxa, float *ws, int nparts, cudaStream_t st,
                      int *nb_out) {
  const int rch = dproj ? LntLayout<1, 8>::RCH : (cols == 128 ? LntLayout<1, 0>::RCH : LntLayout<2, 0>::RCH);
  const int64_t nchunks = (rows + rch - 1) / rch;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms(), nchunks));
#define LT(NV_, NH_)                                                                        \
  do {                                                                                      \
    auto kfn = ln_bwd_tma_kernel<NV_, NH_>;                                                 \
    EVO_MAX_SMEM_ONCE(kfn);                                                                 \
    launch_k(kfn, nb, (LntLayout<NV_, NH_>::CW + 1) * 32, LntLayout<NV_, NH_>::SMEM, st, \
        rows, dy, x, mean, rstd, gamma, beta, dres, dproj, p_rs, Wp, nh, dx, dxa, ws, nparts); \
  } while (0)
  if (dproj) LT(1, 8);
  else if (cols == 128) LT(1, 0);
  else LT(2, 0);
#undef LT
  EVO_LAUNCHED("ln_bwd_tma_kernel");
  *nb_out = nb;
  return EVO_OK;
}

template <typename TDY, typename TX, typename TDX>
int ln_bwd_launch(int64_t rows, int cols, const void *dy, int64_t dy_rs, const void *x,
                  int64_t x_rs, int64_t x_cs, const float *mean, const float *rstd,
                  const float *gamma, const float *dres, void *dx, int64_t dx_rs, int64_t dx_cs,
                  float *dgamma, float *dbeta, int acc, float *ws, cudaStream_t st,
                  void *dx_act = nullptr, int64_t dxa_rs = 0, float *dx_colsum = nullptr) {
  int want = (dgamma || dbeta || dx_colsum) ? 1 : 0;
  int64_t need_blocks = (rows + LN_WARPS - 1) / LN_WARPS;
  int nblk = (int)std::min<int64_t>(LN_BWD_BLOCKS, std::max<int64_t>(need_blocks, 1));
  const TDY *dyp = reinterpret_cast<const TDY *>(dy);
  const TX *xp = reinterpret_cast<const TX *>(x);
  TDX *dxp = reinterpret_cast<TDX *>(dx);
  const bool vec = x_cs == 1 && dx_cs == 1 && (cols == 128 || cols == 256) && dy_rs % 4 == 0 &&
                   x_rs % 4 == 0 && dx_rs % 4 == 0 && aligned16(dy) && aligned16(x) &&
                   aligned16(dx) && aligned16(gamma) && (!dres || aligned16(dres)) &&
                   (!dx_act || (aligned16(dx_act) && dxa_rs % 4 == 0));
  int nparts = 2;
  if constexpr (std::is_same<TDY, float>::value && std::is_same<TX, float>::value) {
    if (x_rs == 1 && x_cs == rows && dx_rs == 1 && dx_cs == rows && cols <= 32 && !dres &&
        !dx_act && !dx_colsum) {  // channel-first (triangle multiplication p)
      const int nb = (int)((rows + 127) / 128);
      EVO_REQUIRE(!want || nb * 2 <= LN_BWD_BLOCKS * 11, EVO_EUNSUP,
                  "layernorm_bwd: channel-first rows=%lld exceed the workspace", (long long)rows);
      launch_k(ln_bwd_cf_kernel<32, TDX>, nb, 128, 0, st, rows, cols, dyp, dy_rs, xp, mean, rstd, gamma,
                                                  dxp, ws);
      EVO_LAUNCHED("ln_bwd_cf_kernel");
      if (want) {
        launch_k(ln_param_reduce_kernel, (2 * cols + 31) / 32, 1024, 0, st, nb, cols, 2, ws, dgamma,
                                                                     dbeta, nullptr, acc,
                                                                     nullptr, 0);
        EVO_LAUNCHED("ln_param_reduce_kernel");
      }
      return EVO_OK;
    }
  }
  if constexpr (std::is_same<TDY, float>::value && std::is_same<TX, float>::value &&
                std::is_same<TDX, float>::value) {
    if (vec && dy_rs == cols && x_rs == cols && dx_rs == cols && (!dx_act || dxa_rs == cols) &&
        rows % 4 == 0 && aligned16(mean) && aligned16(rstd)) {
      nparts = want ? (dx_colsum ? 3 : 2) : 0;
      int nb = 0;
      const int rc = ln_bwd_tma_launch(rows, cols, dyp, xp, mean, rstd, gamma, nullptr, dres,
                                       nullptr, 0, nullptr, 0, dxp,
                                       reinterpret_cast<bf16 *>(dx_act), ws, nparts, st, &nb);
      if (rc != EVO_OK) return rc;
      if (want) {
        launch_k(ln_param_reduce_kernel, (nparts * cols + 31) / 32, 1024, 0, st, nb, cols, nparts, ws,
                                                                          dgamma, dbeta,
                                                                          dx_colsum, acc, nullptr, 0);
        EVO_LAUNCHED("ln_param_reduce_kernel");
      }
      return EVO_OK;
    }
  }
  if (vec) {
    bf16 *dxa = reinterpret_cast<bf16 *>(dx_act);
    nparts = want ? (dx_colsum ? 3 : 2) : 0;
    if (cols == 128)
      launch_k(ln_bwd_vec_kernel<TDY, TX, TDX, 1>, nblk, LN_WARPS * 32, 0, st, rows, dyp, dy_rs, xp, x_rs, mean, rstd, gamma, dres, dxp, dx_rs, dxa, dxa_rs, ws, nparts);
    else
      launch_k(ln_bwd_vec_kernel<TDY, TX, TDX, 2>, nblk, LN_WARPS * 32, 0, st, rows, dyp, dy_rs, xp, x_rs, mean, rstd, gamma, dres, dxp, dx_rs, dxa, dxa_rs, ws, nparts);
    EVO_LAUNCHED("ln_bwd_vec_kernel");
  } else {
    EVO_REQUIRE(!dx_act && !dx_colsum, EVO_EUNSUP,
                "layernorm_bwd: fused dx copy / column sums need the vectorised layout");
    size_t smem = (size_t)LN_WARPS * 2 * cols * sizeof(float);
#define L(Vn)                                                                                 \
  launch_k(ln_bwd_kernel<TDY, TX, TDX, Vn>, nblk, LN_WARPS * 32, smem, st, \
      rows, cols, dyp, dy_rs, xp, x_rs, x_cs, mean, rstd, gamma, dres, dxp, dx_rs, dx_cs, ws, want)
    if (cols <= 32) L(1);
    else if (cols <= 64) L(2);
    else if (cols <= 128) L(4);
    else if (cols <= 256) L(8);
    else L(16);
#undef L
    EVO_LAUNCHED("ln_bwd_kernel");
  }
  if (want) {
    const int outs = nparts * cols;
    launch_k(ln_param_reduce_kernel, (outs + 31) / 32, 1024, 0, st, nblk, cols, nparts, ws, dgamma,
                                                             dbeta, dx_colsum, acc, nullptr, 0);
    EVO_LAUNCHED("ln_param_reduce_kernel");
  }
  return EVO_OK;
}

}  // namespace

size_t layernorm_bwd_ws(int64_t rows, int cols) {
  (void)rows;
  // dgamma, dbeta, column sums, and up to 8 projection-weight gradients
  return (size_t)LN_BWD_BLOCKS * 11 * cols * sizeof(float);
}

int layernorm_fwd(int tx, int ty, int64_t rows, int cols, const void *x, int64_t x_rs,
                  int64_t x_cs, const float *gamma, const float *beta, void *y, int64_t y_rs,
                  float *mean, float *rstd, float eps, cudaStream_t st) {
  EVO_REQUIRE(cols >= 1 && cols <= 32 * MAXV, EVO_EUNSUP, "layernorm: cols=%d unsupported", cols);
  if (rows == 0) return EVO_OK;
  if (tx == EVO_F32 && ty == EVO_F32)
    return ln_fwd_launch<float, float>(rows, cols, x, x_rs, x_cs, gamma, beta, y, y_rs, mean, rstd, eps, st);
  if (tx == EVO_F32 && ty == EVO_BF16)
    return ln_fwd_launch<float, bf16>(rows, cols, x, x_rs, x_cs, gamma, beta, y, y_rs, mean, rstd, eps, st);
  if (tx == EVO_BF16 && ty == EVO_BF16)
    return ln_fwd_launch<bf16, bf16>(rows, cols, x, x_rs, x_cs, gamma, beta, y, y_rs, mean, rstd, eps, st);
  return ln_fwd_launch<bf16, float>(rows, cols, x, x_rs, x_cs, gamma, beta, y, y_rs, mean, rstd, eps, st);
}

int layernorm_fwd_split(int64_t rows, int cols, const float *x, const float *gamma,
                        const float *beta, void *y3, float *mean, float *rstd, float eps,
                        cudaStream_t st) {
  EVO_REQUIRE((cols == 128 || cols == 256) && aligned16(x) && aligned16(y3) && aligned16(gamma) &&
                  aligned16(beta),
              EVO_EUNSUP, "layernorm_fwd_split: contiguous fp32 rows of 128 / 256, aligned");
  if (rows == 0) return EVO_OK;
  bf16 *y = reinterpret_cast<bf16 *>(y3);
  if (cols == 128) return ln_fwd_tma_launch<1, 1, bf16>(rows, x, gamma, beta, y, mean, rstd, eps, st);
  return ln_fwd_tma_launch<2, 1, bf16>(rows, x, gamma, beta, y, mean, rstd, eps, st);
}

int layernorm_bwd_ex(int64_t rows, int cols, const float *dy, const void *x, int tx,
                     const float *mean, const float *rstd, const float *gamma, const float *dres,
                     float *dx, void *dx_act, float *dgamma, float *dbeta, float *dx_colsum,
                     void *ws, size_t ws_bytes, cudaStream_t st) {
  EVO_REQUIRE(cols == 128 || cols == 256, EVO_EUNSUP,
              "layernorm_bwd_ex: cols=%d (fused path: 128 or 256)", cols);
  EVO_REQUIRE(ws && ws_bytes >= layernorm_bwd_ws(rows, cols), EVO_EARG,
              "layernorm_bwd_ex: workspace too small");
  if (rows == 0) return EVO_OK;
  float *w = reinterpret_cast<float *>(ws);
  if (tx == EVO_F32)
    return ln_bwd_launch<float, float, float>(rows, cols, dy, cols, x, cols, 1, mean, rstd, gamma,
                                              dres, dx, cols, 1, dgamma, dbeta, 0, w, st, dx_act,
                                              cols, dx_colsum);
  return ln_bwd_launch<float, bf16, float>(rows, cols, dy, cols, x, cols, 1, mean, rstd, gamma,
                                           dres, dx, cols, 1, dgamma, dbeta, 0, w, st, dx_act, cols,
                                           dx_colsum);
}

int layernorm_bwd_proj(int64_t rows, int cols, const float *dy, const float *x, const float *mean,
                       const float *rstd, const float *gamma, const float *beta,
                       const float *dres, const float *dproj, int64_t p_rs, const void *Wp, int nh,
                       float *dx, void *dx_act, float *dgamma, float *dbeta, float *dx_colsum,
                       float *dWp, void *ws, size_t ws_bytes, cudaStream_t st) {
  EVO_REQUIRE(cols == 128 && nh >= 1 && nh <= 8, EVO_EUNSUP,
              "layernorm_bwd_proj: cols=%d nh=%d (fused path: cols 128, nh <= 8)", cols, nh);
  EVO_REQUIRE(ws && ws_bytes >= layernorm_bwd_ws(rows, cols), EVO_EARG,
              "layernorm_bwd_proj: workspace too small");
  EVO_REQUIRE(aligned16(x) && aligned16(dx) && (!dy || aligned16(dy)) && (!dres || aligned16(dres)) &&
                  (!dx_act || aligned16(dx_act)),
              EVO_EARG, "layernorm_bwd_proj: operands must be 16-byte aligned");
  if (rows == 0) return EVO_OK;
  float *w = reinterpret_cast<float *>(ws);
  const int nparts = 3 + 8;
  if (rows % 4 == 0 && p_rs % 4 == 0 && aligned16(dproj) && aligned16(mean) && aligned16(rstd)) {
    int nb = 0;
    const int rc = ln_bwd_tma_launch(rows, cols, dy, x, mean, rstd, gamma, beta, dres, dproj, p_rs,
                                     reinterpret_cast<const bf16 *>(Wp), nh, dx,
                                     reinterpret_cast<bf16 *>(dx_act), w, nparts, st, &nb);
    if (rc != EVO_OK) return rc;
    launch_k(ln_param_reduce_kernel, (nparts * cols + 31) / 32, 1024, 0, st, nb, cols, nparts, w, dgamma, dbeta, dx_colsum, 0, dWp, nh);
    EVO_LAUNCHED("ln_param_reduce_kernel");
    return EVO_OK;
  }
  const int64_t need_blocks = (rows + LN_WARPS - 1) / LN_WARPS;
  const int nblk = (int)std::min<int64_t>(LN_BWD_BLOCKS, std::max<int64_t>(need_blocks, 1));
  launch_k(ln_bwd_proj_kernel<8>, nblk, LN_WARPS * 32, 0, st, rows, dy, x, mean, rstd, gamma, beta, dres, dproj, p_rs,
      reinterpret_cast<const bf16 *>(Wp), nh, dx, reinterpret_cast<bf16 *>(dx_act), w);
  EVO_LAUNCHED("ln_bwd_proj_kernel");
  launch_k(ln_param_reduce_kernel, (nparts * cols + 31) / 32, 1024, 0, st, nblk, cols, nparts, w, dgamma, dbeta, dx_colsum, 0, dWp, nh);
  EVO_LAUNCHED("ln_param_reduce_kernel");
  return EVO_OK;
}

int layernorm_bwd(int tdy, int tx, int tdx, int64_t rows, int cols, const void *dy, int64_t dy_rs,
                  const void *x, int64_t x_rs, int64_t x_cs, const float *mean, const float *rstd,
                  const float *gamma, const float *dres, void *dx, int64_t dx_rs, int64_t dx_cs,
                  float *dgamma, float *dbeta, int acc, void *ws, size_t ws_bytes,
                  cudaStream_t st) {
  EVO_REQUIRE(cols >= 1 && cols <= 32 * MAXV, EVO_EUNSUP, "layernorm_bwd: cols=%d unsupported",
              cols);
  if ((dgamma || dbeta))
    EVO_REQUIRE(ws && ws_bytes >= layernorm_bwd_ws(rows, cols), EVO_EARG,
                "layernorm_bwd: workspace too small");
  if (rows == 0) return EVO_OK;
  float *w = reinterpret_cast<float *>(ws);
#define D(A, B, C)                                                                              \
  return ln_bwd_launch<A, B, C>(rows, cols, dy, dy_rs, x, x_rs, x_cs, mean, rstd, gamma, dres, \
                                dx, dx_rs, dx_cs, dgamma, dbeta, acc, w, st)
  if (tdy == EVO_F32) {
    if (tx == EVO_F32) { if (tdx == EVO_F32) D(float, float, float); else D(float, float, bf16); }
    else { if (tdx == EVO_F32) D(float, bf16, float); else D(float, bf16, bf16); }
  } else {
    if (tx == EVO_F32) { if (tdx == EVO_F32) D(bf16, float, float); else D(bf16, float, bf16); }
    else { if (tdx == EVO_F32) D(bf16, bf16, float); else D(bf16, bf16, bf16); }
  }
#undef D
}

}  // namespace evo
