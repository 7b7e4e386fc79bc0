// LayerNorm forward/backward over the last axis (src/tensor.py:366-392).
// Warp per row, the row held in registers (cols <= 512), two-pass
// population variance like the reference; gamma/beta gradients reduced
// deterministically (fixed grid, per-block partials, ordered final sum).
#include "common.cuh"

namespace evo {
namespace {

constexpr int LN_WARPS = 8;
constexpr int LN_BWD_BLOCKS = 512;  // fixed => bitwise-reproducible sums
constexpr int MAXV = 16;            // cols <= 32*MAXV

template <typename TX, typename TY, int V>
__global__ void __launch_bounds__(LN_WARPS * 32)
ln_fwd_kernel(int64_t rows, int cols, const TX *__restrict__ x, int64_t x_rs, int64_t x_cs,
              const float *__restrict__ gamma, const float *__restrict__ beta, TY *__restrict__ y,
              int64_t y_rs, float *__restrict__ mean_out, float *__restrict__ rstd_out, float eps) {
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
  const float var = warp_sum(q) * inv_n;
  const float rs = 1.f / sqrtf(var + eps);
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

template <typename TDY, typename TX, typename TDX, int V>
__global__ void __launch_bounds__(LN_WARPS * 32)
ln_bwd_kernel(int64_t rows, int cols, const TDY *__restrict__ dy, int64_t dy_rs,
              const TX *__restrict__ x, int64_t x_rs, int64_t x_cs, const float *__restrict__ mean,
              const float *__restrict__ rstd, const float *__restrict__ gamma,
              const float *__restrict__ dres, TDX *__restrict__ dx, int64_t dx_rs, int64_t dx_cs,
              float *__restrict__ partial /* [gridDim.x][2][cols] */, int want_params) {
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

__global__ void ln_param_reduce_kernel(int nblk, int cols, const float *__restrict__ partial,
                                       float *__restrict__ dgamma, float *__restrict__ dbeta,
                                       int accumulate) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < 2 * cols; c += gridDim.x * blockDim.x) {
    int which = c / cols, cc = c % cols;
    float s = 0.f;
    for (int b = 0; b < nblk; ++b) s += partial[((int64_t)b * 2 + which) * cols + cc];
    float *dst = which == 0 ? dgamma : dbeta;
    if (dst) dst[cc] = accumulate ? dst[cc] + s : s;
  }
}

template <typename TX, typename TY>
int ln_fwd_launch(int64_t rows, int cols, const void *x, int64_t x_rs, int64_t x_cs,
                  const float *gamma, const float *beta, void *y, int64_t y_rs, float *mean,
                  float *rstd, float eps, cudaStream_t st) {
  dim3 grid((unsigned)((rows + LN_WARPS - 1) / LN_WARPS));
  const TX *xp = reinterpret_cast<const TX *>(x);
  TY *yp = reinterpret_cast<TY *>(y);
#define L(Vn)                                                                                \
  ln_fwd_kernel<TX, TY, Vn><<<grid, LN_WARPS * 32, 0, st>>>(rows, cols, xp, x_rs, x_cs, gamma, \
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

template <typename TDY, typename TX, typename TDX>
int ln_bwd_launch(int64_t rows, int cols, const void *dy, int64_t dy_rs, const void *x,
                  int64_t x_rs, int64_t x_cs, const float *mean, const float *rstd,
                  const float *gamma, const float *dres, void *dx, int64_t dx_rs, int64_t dx_cs,
                  float *dgamma, float *dbeta, int acc, float *ws, cudaStream_t st) {
  int want = (dgamma || dbeta) ? 1 : 0;
  int64_t need_blocks = (rows + LN_WARPS - 1) / LN_WARPS;
  int nblk = (int)std::min<int64_t>(LN_BWD_BLOCKS, std::max<int64_t>(need_blocks, 1));
  size_t smem = (size_t)LN_WARPS * 2 * cols * sizeof(float);
  const TDY *dyp = reinterpret_cast<const TDY *>(dy);
  const TX *xp = reinterpret_cast<const TX *>(x);
  TDX *dxp = reinterpret_cast<TDX *>(dx);
#define L(Vn)                                                                                 \
  ln_bwd_kernel<TDY, TX, TDX, Vn><<<nblk, LN_WARPS * 32, smem, st>>>(                          \
      rows, cols, dyp, dy_rs, xp, x_rs, x_cs, mean, rstd, gamma, dres, dxp, dx_rs, dx_cs, ws, want)
  if (cols <= 32) L(1);
  else if (cols <= 64) L(2);
  else if (cols <= 128) L(4);
  else if (cols <= 256) L(8);
  else L(16);
#undef L
  EVO_LAUNCHED("ln_bwd_kernel");
  if (want) {
    ln_param_reduce_kernel<<<(2 * cols + 255) / 256, 256, 0, st>>>(nblk, cols, ws, dgamma, dbeta,
                                                                   acc);
    EVO_LAUNCHED("ln_param_reduce_kernel");
  }
  return EVO_OK;
}

}  // namespace

size_t layernorm_bwd_ws(int64_t rows, int cols) {
  (void)rows;
  return (size_t)LN_BWD_BLOCKS * 2 * cols * sizeof(float);
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
