// Fused gated attention with pair bias, SIMT (FFMA) form: the fp32 parity
// path and the fallback for head dims the tensor-core kernel does not take.
//
// Forward (src/evoformer.py:274-286, softmax src/tensor.py:352-357):
//   O[b,q,h,:] = sum_k softmax_k(scale*q.k + bias[h,q,k]) v[b,k,h,:]
//   GM = G * O  (sigmoid gate applied before the out-projection)
// Backward (src/tensor.py:305-309 matmul, 359-361 softmax):
//   dO = dGM*G,  dGpre = dGM*O*G*(1-G),  Dq = sum_d dO*O
//   dS = P*(dO.v - Dq),  dq = scale*dS k,  dk = scale*dS^T q,  dv = P^T dO
//   dbias[h,q,k] = sum_b dS  (chunk partials + ordered reduce: deterministic)
// All keys of one (b,h) are resident in shared memory (L <= 1024, the
// register row of logits sized per instantiation: 256 / 512 / 1024), so the
// softmax is exact single-pass; no logits ever reach HBM.
#include "common.cuh"

namespace evo {

int reduce_lead(int dt, int64_t nb, int64_t n1, int64_t n2, const void *src, float *dst,
                int64_t d_s1, int64_t d_s2, int acc, cudaStream_t st);
int colsum_partials(int nblk, int64_t cols, const float *part, float *dst, int acc,
                    cudaStream_t st);

namespace {

constexpr int AW = 8;      // warps per block
constexpr int QT = 32;     // queries (or keys) per block
constexpr int MAXL = 1024; // resident keys (kernels instantiated for 256 / 512 / 1024)
constexpr int MAXD = 64;

template <typename T>
__device__ __forceinline__ float ld(const void *p, int64_t off) {
  return to_f(reinterpret_cast<const T *>(p)[off]);
}
template <typename T>
__device__ __forceinline__ void st(void *p, int64_t off, float v) {
  reinterpret_cast<T *>(p)[off] = from_f<T>(v);
}

// Load rows [0, L) of head h, batch b of a (b,l,h,d) strided tensor into
// smem laid out [L][D+1] fp32.
template <typename T>
__device__ void load_rows(float *dst, const void *src, int64_t base, int64_t sl, int L, int D) {
  const int Dp = D + 1;
  for (int e = threadIdx.x; e < L * D; e += blockDim.x) {
    int l = e / D, d = e % D;
    dst[l * Dp + d] = ld<T>(src, base + l * sl + d);
  }
}

template <typename T, int ML>
__global__ void __launch_bounds__(AW * 32) attn_fwd_kernel(evo_attn_desc a) {
  evo_pdl_enter();
  extern __shared__ float sm[];
  const int L = a.L, D = a.D, Dp = D + 1;
  float *Ks = sm;
  float *Vs = Ks + L * Dp;
  float *Pw = Vs + L * Dp;          // [AW][L]
  float *Qw = Pw + AW * L;          // [AW][D]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int64_t base = b * a.sb + (int64_t)h * D;
  load_rows<T>(Ks, a.k, base, a.sl, L, D);
  load_rows<T>(Vs, a.v, base, a.sl, L, D);
  __syncthreads();
  float *P = Pw + warp * L;
  float *Qv = Qw + warp * D;
  const int nk = (L + 31) / 32;
  for (int qi = warp; qi < QT; qi += AW) {
    const int q = blockIdx.x * QT + qi;
    if (q >= L) break;
    const int64_t qoff = base + (int64_t)q * a.sl;
    for (int d = lane; d < D; d += 32) Qv[d] = ld<T>(a.q, qoff + d);
    __syncwarp();
    float s[ML / 32];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < ML / 32; ++j) {
      int k = lane + 32 * j;
      s[j] = -INFINITY;
      if (j < nk && k < L) {
        float acc = 0.f;
        for (int d = 0; d < D; ++d) acc = fmaf(Qv[d], Ks[k * Dp + d], acc);
        acc *= a.scale;
        if (a.bias) acc += a.bias[(int64_t)h * a.bh + (int64_t)q * a.bq + (int64_t)k * a.bk];
        s[j] = acc;
        mx = fmaxf(mx, acc);
      }
    }
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < ML / 32; ++j) {
      int k = lane + 32 * j;
      float p = (j < nk && k < L) ? expf(s[j] - mx) : 0.f;
      s[j] = p;
      sum += p;
    }
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
#pragma unroll
    for (int j = 0; j < ML / 32; ++j) {
      int k = lane + 32 * j;
      if (j < nk && k < L) P[k] = s[j] * inv;
    }
    __syncwarp();
    const int64_t ooff = b * a.o_sb + (int64_t)q * a.o_sl + (int64_t)h * D;
    for (int d = lane; d < D; d += 32) {
      float o = 0.f;
      for (int k = 0; k < L; ++k) o = fmaf(P[k], Vs[k * Dp + d], o);
      float g = ld<T>(a.g, qoff + d);
      st<T>(a.o, ooff + d, o);
      st<T>(a.gm, ooff + d, g * o);
    }
    if (lane == 0) a.lse[(b * a.H + h) * (int64_t)L + q] = mx + logf(sum);
    __syncwarp();
  }
}

// dq, dgpre and per-chunk dbias partials.  grid (ceil(L/QT), H, nchunk).
template <typename T, int ML>
__global__ void __launch_bounds__(AW * 32)
attn_bwd_dq_kernel(evo_attn_desc a, int64_t chunk, float *dbias_part) {
  evo_pdl_enter();
  extern __shared__ float sm[];
  const int L = a.L, D = a.D, Dp = D + 1;
  float *Ks = sm;
  float *Vs = Ks + L * Dp;
  float *Pw = Vs + L * Dp;              // [AW][L]  dS row
  float *Ow = Pw + AW * L;              // [AW][D]  dO row
  float *Qw = Ow + AW * D;              // [AW][D]  q row
  float *Bt = Qw + AW * D;              // [QT][L]  dbias tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * QT;
  const bool want_bias = (dbias_part != nullptr);
  if (want_bias)
    for (int e = threadIdx.x; e < QT * L; e += blockDim.x) Bt[e] = 0.f;
  const int64_t b_lo = blockIdx.z * chunk;
  const int64_t b_hi = min(a.nb, b_lo + chunk);
  const int nk = (L + 31) / 32;
  for (int64_t b = b_lo; b < b_hi; ++b) {
    const int64_t base = b * a.sb + (int64_t)h * D;
    __syncthreads();
    load_rows<T>(Ks, a.k, base, a.sl, L, D);
    load_rows<T>(Vs, a.v, base, a.sl, L, D);
    __syncthreads();
    float *dS = Pw + warp * L;
    float *dOv = Ow + warp * D;
    float *Qv = Qw + warp * D;
    for (int qi = warp; qi < QT; qi += AW) {
      const int q = q0 + qi;
      if (q >= L) break;
      const int64_t qoff = base + (int64_t)q * a.sl;
      const int64_t ooff = b * a.o_sb + (int64_t)q * a.o_sl + (int64_t)h * D;
      float Dq = 0.f;
      for (int d = lane; d < D; d += 32) {
        float g = ld<T>(a.g, qoff + d);
        float o = ld<T>(a.o, ooff + d);
        float dgm = ld<T>(a.dgm, ooff + d);
        float dov = dgm * g;
        dOv[d] = dov;
        Qv[d] = ld<T>(a.q, qoff + d);
        st<T>(a.dgpre, qoff + d, dgm * o * g * (1.f - g));
        Dq += dov * o;
      }
      Dq = warp_sum(Dq);
      __syncwarp();
      const float lse = a.lse[(b * a.H + h) * (int64_t)L + q];
#pragma unroll
      for (int j = 0; j < ML / 32; ++j) {
        int k = lane + 32 * j;
        if (j < nk && k < L) {
          float sc = 0.f, dp = 0.f;
          for (int d = 0; d < D; ++d) {
            sc = fmaf(Qv[d], Ks[k * Dp + d], sc);
            dp = fmaf(dOv[d], Vs[k * Dp + d], dp);
          }
          sc *= a.scale;
          if (a.bias) sc += a.bias[(int64_t)h * a.bh + (int64_t)q * a.bq + (int64_t)k * a.bk];
          float p = expf(sc - lse);
          float ds = p * (dp - Dq);
          dS[k] = ds;
          if (want_bias) Bt[qi * L + k] += ds;
        }
      }
      __syncwarp();
      for (int d = lane; d < D; d += 32) {
        float acc = 0.f;
        for (int k = 0; k < L; ++k) acc = fmaf(dS[k], Ks[k * Dp + d], acc);
        st<T>(a.dq, qoff + d, acc * a.scale);
      }
      __syncwarp();
    }
  }
  if (!want_bias) return;
  __syncthreads();
  // partial slab uses dbias's own (dense) [H, L, L] index map
  float *dst = dbias_part + (int64_t)blockIdx.z * a.H * (int64_t)L * L;
  for (int e = threadIdx.x; e < QT * L; e += blockDim.x) {
    int qi = e / L, k = e % L;
    if (q0 + qi < L)
      dst[(int64_t)h * a.bh + (int64_t)(q0 + qi) * a.bq + (int64_t)k * a.bk] = Bt[e];
  }
}

// dk, dv.  grid (ceil(L/QT) key tiles, H, nb).
template <typename T, int ML>
__global__ void __launch_bounds__(AW * 32) attn_bwd_dkv_kernel(evo_attn_desc a) {
  evo_pdl_enter();
  extern __shared__ float sm[];
  const int L = a.L, D = a.D, Dp = D + 1;
  float *Qs = sm;                  // [L][Dp]
  float *dOs = Qs + L * Dp;        // [L][Dp]
  float *lse = dOs + L * Dp;       // [L]
  float *Dqs = lse + L;            // [L]
  float *Pw = Dqs + L;             // [AW][2][L]
  float *Kw = Pw + AW * 2 * L;     // [AW][2][D]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int64_t base = b * a.sb + (int64_t)h * D;
  const int64_t obase = b * a.o_sb + (int64_t)h * D;
  load_rows<T>(Qs, a.q, base, a.sl, L, D);
  for (int e = threadIdx.x; e < L * D; e += blockDim.x) {
    int l = e / D, d = e % D;
    int64_t ooff = obase + (int64_t)l * a.o_sl + d;
    dOs[l * Dp + d] = ld<T>(a.dgm, ooff) * ld<T>(a.g, base + (int64_t)l * a.sl + d);
  }
  __syncthreads();
  // Dq = sum_d dO*O per query; lse
  for (int q = warp; q < L; q += AW) {
    float acc = 0.f;
    for (int d = lane; d < D; d += 32)
      acc += dOs[q * Dp + d] * ld<T>(a.o, obase + (int64_t)q * a.o_sl + d);
    acc = warp_sum(acc);
    if (lane == 0) {
      Dqs[q] = acc;
      lse[q] = a.lse[(b * a.H + h) * (int64_t)L + q];
    }
  }
  __syncthreads();
  float *Pk = Pw + warp * 2 * L;
  float *dSk = Pk + L;
  float *Kv = Kw + warp * 2 * D;
  float *Vv = Kv + D;
  const int nq = (L + 31) / 32;
  for (int ki = warp; ki < QT; ki += AW) {
    const int k = blockIdx.x * QT + ki;
    if (k >= L) break;
    const int64_t koff = base + (int64_t)k * a.sl;
    for (int d = lane; d < D; d += 32) {
      Kv[d] = ld<T>(a.k, koff + d);
      Vv[d] = ld<T>(a.v, koff + d);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < ML / 32; ++j) {
      int q = lane + 32 * j;
      if (j < nq && q < L) {
        float sc = 0.f, dp = 0.f;
        for (int d = 0; d < D; ++d) {
          sc = fmaf(Qs[q * Dp + d], Kv[d], sc);
          dp = fmaf(dOs[q * Dp + d], Vv[d], dp);
        }
        sc *= a.scale;
        if (a.bias) sc += a.bias[(int64_t)h * a.bh + (int64_t)q * a.bq + (int64_t)k * a.bk];
        float p = expf(sc - lse[q]);
        Pk[q] = p;
        dSk[q] = p * (dp - Dqs[q]);
      }
    }
    __syncwarp();
    for (int d = lane; d < D; d += 32) {
      float dv = 0.f, dk = 0.f;
      for (int q = 0; q < L; ++q) {
        dv = fmaf(Pk[q], dOs[q * Dp + d], dv);
        dk = fmaf(dSk[q], Qs[q * Dp + d], dk);
      }
      st<T>(a.dv, koff + d, dv);
      st<T>(a.dk, koff + d, dk * a.scale);
    }
    __syncwarp();
  }
}

int64_t dbias_chunks(const evo_attn_desc *a) {
  int64_t tiles = (int64_t)a->H * ((a->L + QT - 1) / QT);
  int64_t want = (4 * 148 + tiles - 1) / tiles;
  return std::max<int64_t>(1, std::min<int64_t>(a->nb, want));
}

}  // namespace

// gate-bias column sums: GB_PARTS ordered row ranges, then colsum_partials
constexpr int GB_PARTS = 4 * 148;

size_t dbias_ws_bytes(const evo_attn_desc *a) {
  if (!a->dbias) return 0;
  return ((size_t)dbias_chunks(a) * a->H * a->L * a->L * sizeof(float) + 255) & ~(size_t)255;
}

size_t attention_simt_bwd_ws(const evo_attn_desc *a) {
  return dbias_ws_bytes(a) +
         (a->dgate_bias ? (size_t)GB_PARTS * a->H * a->D * sizeof(float) : 0);
}

int attention_simt_fwd(const evo_attn_desc *a, cudaStream_t st) {
  EVO_REQUIRE(a->L >= 1 && a->L <= MAXL && a->D >= 1 && a->D <= MAXD, EVO_EUNSUP,
              "attention: L=%d D=%d unsupported (L<=1024, D<=64)", a->L, a->D);
  dim3 grid((a->L + QT - 1) / QT, a->H, (unsigned)a->nb);
  size_t smem = (size_t)(2 * a->L * (a->D + 1) + AW * a->L + AW * a->D) * sizeof(float);
  EVO_REQUIRE(smem <= 227 * 1024, EVO_EUNSUP, "attention: L=%d D=%d exceeds shared memory",
              a->L, a->D);
#define EVO_SIMT_FWD(T, ML)                                             \
  {                                                                    \
    EVO_MAX_SMEM_ONCE((attn_fwd_kernel<T, ML>));                       \
    launch_k(attn_fwd_kernel<T, ML>, grid, AW * 32, smem, st, *a);           \
  }
  const bool f32 = a->dtype == EVO_F32;
  if (a->L <= 256) { if (f32) EVO_SIMT_FWD(float, 256) else EVO_SIMT_FWD(bf16, 256) }
  else if (a->L <= 512) { if (f32) EVO_SIMT_FWD(float, 512) else EVO_SIMT_FWD(bf16, 512) }
  else { if (f32) EVO_SIMT_FWD(float, 1024) else EVO_SIMT_FWD(bf16, 1024) }
#undef EVO_SIMT_FWD
  EVO_LAUNCHED("attn_fwd_kernel");
  return EVO_OK;
}

// dgate_bias[h*D + d] = sum over (b, l) of dGpre, deterministic two-stage:
// block p sums the (b, l) rows [p*rpp, (p+1)*rpp) in order (threads across
// columns), then colsum_partials adds the GB_PARTS partials in order.
template <typename T>
__global__ void gate_bias_part_kernel(const evo_attn_desc a, int64_t rpp, float *part) {
  evo_pdl_enter();
  const int cols = a.H * a.D;
  const int64_t n = a.nb * (int64_t)a.L;
  const int64_t r0 = blockIdx.x * rpp, r1 = min(n, r0 + rpp);
  const T *g = reinterpret_cast<const T *>(a.dgpre);
  for (int col = threadIdx.x; col < cols; col += blockDim.x) {
    float s = 0.f;
#pragma unroll 8
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t b = r / a.L;
      const int l = (int)(r - b * a.L);
      s += to_f(g[b * a.sb + (int64_t)l * a.sl + col]);
    }
    part[(int64_t)blockIdx.x * cols + col] = s;
  }
}

int attention_simt_bwd(const evo_attn_desc *a, cudaStream_t st) {
  EVO_REQUIRE(a->L >= 1 && a->L <= MAXL && a->D >= 1 && a->D <= MAXD, EVO_EUNSUP,
              "attention bwd: L=%d D=%d unsupported", a->L, a->D);
  const int L = a->L, D = a->D;
  int64_t nch = a->dbias ? dbias_chunks(a) : a->nb;
  int64_t chunk = (a->nb + nch - 1) / nch;
  nch = (a->nb + chunk - 1) / chunk;
  float *part = nullptr;
  if (a->dbias) {
    EVO_REQUIRE(a->workspace && a->workspace_bytes >= attention_simt_bwd_ws(a), EVO_EARG,
                "attention bwd: workspace too small");
    part = reinterpret_cast<float *>(a->workspace);
  }
  {
    dim3 grid((L + QT - 1) / QT, a->H, (unsigned)nch);
    size_t smem = (size_t)(2 * L * (D + 1) + AW * L + 2 * AW * D + (a->dbias ? QT * L : 0)) *
                  sizeof(float);
    EVO_REQUIRE(smem <= 227 * 1024, EVO_EUNSUP,
                "attention bwd: L=%d D=%d exceeds shared memory", L, D);
#define EVO_SIMT_DQ(T, ML)                                                   \
  {                                                                         \
    EVO_MAX_SMEM_ONCE((attn_bwd_dq_kernel<T, ML>));                         \
    launch_k(attn_bwd_dq_kernel<T, ML>, grid, AW * 32, smem, st, *a, chunk, part); \
  }
    const bool f32 = a->dtype == EVO_F32;
    if (L <= 256) { if (f32) EVO_SIMT_DQ(float, 256) else EVO_SIMT_DQ(bf16, 256) }
    else if (L <= 512) { if (f32) EVO_SIMT_DQ(float, 512) else EVO_SIMT_DQ(bf16, 512) }
    else { if (f32) EVO_SIMT_DQ(float, 1024) else EVO_SIMT_DQ(bf16, 1024) }
#undef EVO_SIMT_DQ
    EVO_LAUNCHED("attn_bwd_dq_kernel");
  }
  {
    dim3 grid((L + QT - 1) / QT, a->H, (unsigned)a->nb);
    size_t smem = (size_t)(2 * L * (D + 1) + 2 * L + AW * 2 * L + AW * 2 * D) * sizeof(float);
    EVO_REQUIRE(smem <= 227 * 1024, EVO_EUNSUP,
                "attention bwd: L=%d D=%d exceeds shared memory", L, D);
#define EVO_SIMT_DKV(T, ML)                                      \
  {                                                             \
    EVO_MAX_SMEM_ONCE((attn_bwd_dkv_kernel<T, ML>));            \
    launch_k(attn_bwd_dkv_kernel<T, ML>, grid, AW * 32, smem, st, *a); \
  }
    const bool f32 = a->dtype == EVO_F32;
    if (L <= 256) { if (f32) EVO_SIMT_DKV(float, 256) else EVO_SIMT_DKV(bf16, 256) }
    else if (L <= 512) { if (f32) EVO_SIMT_DKV(float, 512) else EVO_SIMT_DKV(bf16, 512) }
    else { if (f32) EVO_SIMT_DKV(float, 1024) else EVO_SIMT_DKV(bf16, 1024) }
#undef EVO_SIMT_DKV
    EVO_LAUNCHED("attn_bwd_dkv_kernel");
  }
  if (a->dbias) {
    // dbias = ordered sum of the chunk slabs (same dense index map)
    int rc = reduce_lead(EVO_F32, nch, 1, (int64_t)a->H * L * L, part, a->dbias, 0, 1, 0, st);
    if (rc != EVO_OK) return rc;
  }
  if (a->dgate_bias) {
    EVO_REQUIRE(a->workspace && a->workspace_bytes >= attention_simt_bwd_ws(a), EVO_EARG,
                "attention bwd: workspace too small");
    const int cols = a->H * a->D;
    float *gpart = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(a->workspace) +
                                             dbias_ws_bytes(a));
    const int64_t n = a->nb * (int64_t)L;
    const int64_t rpp = (n + GB_PARTS - 1) / GB_PARTS;
    const int parts = (int)((n + rpp - 1) / rpp);
    const int thr = std::min(256, ((cols + 31) / 32) * 32);
    if (a->dtype == EVO_F32)
      launch_k(gate_bias_part_kernel<float>, parts, thr, 0, st, *a, rpp, gpart);
    else
      launch_k(gate_bias_part_kernel<bf16>, parts, thr, 0, st, *a, rpp, gpart);
    EVO_LAUNCHED("gate_bias_part_kernel");
    int rc = colsum_partials(parts, cols, gpart, a->dgate_bias, 0, st);
    if (rc != EVO_OK) return rc;
  }
  return EVO_OK;
}

}  // namespace evo
