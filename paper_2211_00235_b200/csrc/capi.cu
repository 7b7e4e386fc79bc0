// extern "C" boundary (include/evo_b200.h): argument validation, status
// codes, thread-local error strings and kernel dispatch.
#include <stdarg.h>
#include <algorithm>

#include "common.cuh"
#include "gemm.cuh"
#include "tc_common.cuh"

namespace evo {

std::atomic<int64_t> g_launches{0};
static thread_local char g_err[512] = "";
static std::atomic<int> g_strict_tc{1};
static std::atomic<int64_t> g_backend[EVO_BK_COUNT];
static thread_local int g_last_backend = -1;

void note_backend(int b) {
  g_backend[b].fetch_add(1, std::memory_order_relaxed);
  g_last_backend = b;
}

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// implemented in the other translation units
size_t layernorm_bwd_ws(int64_t rows, int cols);
int layernorm_fwd(int, int, int64_t, int, const void *, int64_t, int64_t, const float *,
                  const float *, void *, int64_t, float *, float *, float, cudaStream_t);
int layernorm_bwd(int, int, int, int64_t, int, const void *, int64_t, const void *, int64_t,
                  int64_t, const float *, const float *, const float *, const float *, void *,
                  int64_t, int64_t, float *, float *, int, void *, size_t, cudaStream_t);
int layernorm_fwd_split(int64_t, int, const float *, const float *, const float *, void *, float *,
                        float *, float, cudaStream_t);
int layernorm_bwd_ex(int64_t, int, const float *, const void *, int, const float *, const float *,
                     const float *, const float *, float *, void *, float *, float *, float *,
                     void *, size_t, cudaStream_t);
int layernorm_bwd_proj(int64_t, int, const float *, const float *, const float *, const float *,
                       const float *, const float *, const float *, const float *, int64_t,
                       const void *, int, float *, void *, float *, float *, float *, float *,
                       void *, size_t, cudaStream_t);
int attention_simt_fwd(const evo_attn_desc *, cudaStream_t);
int attention_simt_bwd(const evo_attn_desc *, cudaStream_t);
size_t attention_simt_bwd_ws(const evo_attn_desc *);
int attention_tc_fwd(const evo_attn_desc *, cudaStream_t);
int attention_tc_bwd(const evo_attn_desc *, cudaStream_t);
bool attention_tc_accepts(const evo_attn_desc *);
size_t attention_tc_bwd_ws(const evo_attn_desc *);
int reduce_lead(int, int64_t, int64_t, int64_t, const void *, float *, int64_t, int64_t, int,
                cudaStream_t);
int colsum(int, int64_t, int64_t, const void *, int64_t, float *, int, float *, cudaStream_t);
int copy3d(int, int, int64_t, int64_t, int64_t, const void *, int64_t, int64_t, int64_t, void *,
           int64_t, int64_t, int64_t, cudaStream_t);
int copy2d(int, int, int64_t, int64_t, const void *, int64_t, int64_t, void *, int64_t, int64_t,
           cudaStream_t);
int mul2d(int, int, int, int64_t, int64_t, const void *, int64_t, const void *, int64_t, void *,
          int64_t, cudaStream_t);
int trimul_gate_fwd(int, int64_t, int, const void *, int64_t, void *, void *, cudaStream_t);
int trimul_gate_bwd(int, int64_t, int, const void *, int64_t, const float *, const float *, void *,
                    int64_t, float *, float *, cudaStream_t);
size_t trimul_gate_bwd_ws(int64_t, int);
size_t outgate_bwd_ws(int64_t, int64_t);
int outgate_fwd(int, int64_t, int64_t, const float *, const void *, int64_t, const void *,
                int64_t, float *, cudaStream_t);
int outgate_bwd(int, int64_t, int64_t, const float *, const void *, int64_t, const void *,
                int64_t, void *, int64_t, void *, int64_t, float *, float *, float *,
                cudaStream_t);
int relu_bwd(int, int64_t, const void *, const void *, void *, cudaStream_t);
int relu_bwd_colsum(int64_t, int64_t, const void *, const void *, void *, float *, float *,
                    cudaStream_t);
int sq_mean(int64_t, const float *, float *, float *, void *, cudaStream_t);
int add(int64_t, const float *, const float *, float *, cudaStream_t);
int div_scalar(int64_t, const float *, float, float *, cudaStream_t);
int split_bf16(int64_t, int64_t, const float *, int64_t, void *, int64_t, void *, int64_t, void *,
               int64_t, cudaStream_t);

static bool use_skinny(const evo_gemm_desc *d) {
  return !d->force_simt && gemm_skinny_accepts(d);
}
static bool use_tc(const evo_gemm_desc *d) {
  return !d->force_simt && !gemm_skinny_accepts(d) && gemm_tc_accepts(d);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("EVO_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace evo

using namespace evo;

#define CHECK_DT(x) EVO_REQUIRE(valid_dtype(x), EVO_EARG, "%s: bad dtype %d", __func__, (int)(x))
#define CHECK_PTR(p) EVO_REQUIRE((p) != nullptr, EVO_EARG, "%s: %s is NULL", __func__, #p)

extern "C" {

const char *evo_last_error(void) { return g_err; }
int evo_version(void) { return 1; }
int64_t evo_launch_count(void) { return g_launches.load(); }
int evo_tc_available(void) { return tc::encode_fn() != nullptr ? 1 : 0; }
int64_t evo_backend_count(int b) {
  return (b >= 0 && b < EVO_BK_COUNT) ? g_backend[b].load() : -1;
}
int evo_last_backend(void) { return g_last_backend; }
void evo_set_strict_tc(int on) { g_strict_tc.store(on ? 1 : 0); }
int evo_get_strict_tc(void) { return g_strict_tc.load(); }

size_t evo_gemm_workspace_bytes(const evo_gemm_desc *d) {
  if (!d) return 0;
  if (use_skinny(d)) return gemm_skinny_workspace(d);
  return use_tc(d) ? gemm_tc_workspace(d) : gemm_simt_workspace(d);
}

int evo_gemm(const evo_gemm_desc *d, void *stream) {
  CHECK_PTR(d);
  CHECK_DT(d->dtype_ab);
  CHECK_DT(d->dtype_c);
  EVO_REQUIRE(d->M >= 0 && d->N >= 0 && d->K >= 0 && d->B1 >= 1 && d->B2 >= 1, EVO_EDIM,
              "evo_gemm: bad sizes M=%lld N=%lld K=%lld B=%lldx%lld", (long long)d->M,
              (long long)d->N, (long long)d->K, (long long)d->B1, (long long)d->B2);
  EVO_REQUIRE(d->epilogue >= EVO_EPI_NONE && d->epilogue <= EVO_EPI_SIGMOID_FROM, EVO_EARG,
              "evo_gemm: bad epilogue %d", d->epilogue);
  EVO_REQUIRE(!d->accumulate || d->dtype_c == EVO_F32, EVO_EARG,
              "evo_gemm: accumulate needs an fp32 C");
  if (d->M == 0 || d->N == 0) return EVO_OK;
  CHECK_PTR(d->C.ptr);
  if (d->K > 0) {
    CHECK_PTR(d->A.ptr);
    CHECK_PTR(d->B.ptr);
  }
  cudaStream_t st = as_stream(stream);
  if (use_skinny(d) && d->K > 0) {
    note_backend(EVO_BK_GEMM_SKINNY);
    return gemm_skinny(d, st);
  }
  if (use_tc(d)) {
    int rc = gemm_tc(d, st);
    if (rc != EVO_EUNSUP) {
      note_backend(EVO_BK_GEMM_TC);
      return rc;
    }
  }
  EVO_REQUIRE(!(g_strict_tc.load() && d->dtype_ab == EVO_BF16 && !d->force_simt), EVO_EUNSUP,
              "evo_gemm: bf16 M=%lld N=%lld K=%lld B=%lldx%lld (A rs=%lld cs=%lld, B rs=%lld "
              "cs=%lld, epi=%d bias=%d) is not taken by the tensor-core kernel and strict "
              "tensor-core mode forbids the SIMT fallback",
              (long long)d->M, (long long)d->N, (long long)d->K, (long long)d->B1,
              (long long)d->B2, (long long)d->A.rs, (long long)d->A.cs, (long long)d->B.rs,
              (long long)d->B.cs, d->epilogue, d->bias ? 1 : 0);
  note_backend(EVO_BK_GEMM_SIMT);
  return gemm_simt(d, st);
}

int evo_layernorm_fwd(int dtype_x, int dtype_y, int64_t rows, int cols, const void *x,
                      int64_t x_rs, int64_t x_cs, const float *gamma, const float *beta, void *y,
                      int64_t y_rs, float *mean, float *rstd, float eps, void *stream) {
  CHECK_DT(dtype_x);
  CHECK_DT(dtype_y);
  EVO_REQUIRE(rows >= 0 && cols >= 1, EVO_EDIM, "evo_layernorm_fwd: rows=%lld cols=%d",
              (long long)rows, cols);
  EVO_REQUIRE(eps > 0.f, EVO_EARG, "evo_layernorm_fwd: eps must be > 0");
  if (rows == 0) return EVO_OK;
  CHECK_PTR(x); CHECK_PTR(gamma); CHECK_PTR(beta); CHECK_PTR(y); CHECK_PTR(mean); CHECK_PTR(rstd);
  return layernorm_fwd(dtype_x, dtype_y, rows, cols, x, x_rs, x_cs, gamma, beta, y, y_rs, mean,
                       rstd, eps, as_stream(stream));
}

int evo_layernorm_fwd_split(int64_t rows, int cols, const float *x, const float *gamma,
                            const float *beta, void *y3, float *mean, float *rstd, float eps,
                            void *stream) {
  EVO_REQUIRE(rows >= 0 && cols >= 1, EVO_EDIM, "evo_layernorm_fwd_split: rows=%lld cols=%d",
              (long long)rows, cols);
  EVO_REQUIRE(eps > 0.f, EVO_EARG, "evo_layernorm_fwd_split: eps must be > 0");
  if (rows == 0) return EVO_OK;
  CHECK_PTR(x); CHECK_PTR(gamma); CHECK_PTR(beta); CHECK_PTR(y3); CHECK_PTR(mean); CHECK_PTR(rstd);
  return layernorm_fwd_split(rows, cols, x, gamma, beta, y3, mean, rstd, eps, as_stream(stream));
}

size_t evo_layernorm_bwd_workspace_bytes(int64_t rows, int cols) {
  return layernorm_bwd_ws(rows, cols);
}

int evo_layernorm_bwd(int dtype_dy, int dtype_x, int dtype_dx, int64_t rows, int cols,
                      const void *dy, int64_t dy_rs, const void *x, int64_t x_rs, int64_t x_cs,
                      const float *mean, const float *rstd, const float *gamma, const float *dres,
                      void *dx, int64_t dx_rs, int64_t dx_cs, float *dgamma, float *dbeta,
                      int accumulate_params, void *workspace, size_t workspace_bytes,
                      void *stream) {
  CHECK_DT(dtype_dy);
  CHECK_DT(dtype_x);
  CHECK_DT(dtype_dx);
  EVO_REQUIRE(rows >= 0 && cols >= 1, EVO_EDIM, "evo_layernorm_bwd: rows=%lld cols=%d",
              (long long)rows, cols);
  if (rows == 0) return EVO_OK;
  CHECK_PTR(dy); CHECK_PTR(x); CHECK_PTR(mean); CHECK_PTR(rstd); CHECK_PTR(gamma); CHECK_PTR(dx);
  return layernorm_bwd(dtype_dy, dtype_x, dtype_dx, rows, cols, dy, dy_rs, x, x_rs, x_cs, mean,
                       rstd, gamma, dres, dx, dx_rs, dx_cs, dgamma, dbeta, accumulate_params,
                       workspace, workspace_bytes, as_stream(stream));
}

int evo_layernorm_bwd_ex(int dtype_x, int64_t rows, int cols, const float *dy, const void *x,
                         const float *mean, const float *rstd, const float *gamma,
                         const float *dres, float *dx, void *dx_act, float *dgamma, float *dbeta,
                         float *dx_colsum, void *workspace, size_t workspace_bytes,
                         void *stream) {
  CHECK_DT(dtype_x);
  EVO_REQUIRE(rows >= 0 && cols >= 1, EVO_EDIM, "evo_layernorm_bwd_ex: rows=%lld cols=%d",
              (long long)rows, cols);
  if (rows == 0) return EVO_OK;
  CHECK_PTR(dy); CHECK_PTR(x); CHECK_PTR(mean); CHECK_PTR(rstd); CHECK_PTR(gamma); CHECK_PTR(dx);
  return layernorm_bwd_ex(rows, cols, dy, x, dtype_x, mean, rstd, gamma, dres, dx, dx_act, dgamma,
                          dbeta, dx_colsum, workspace, workspace_bytes, as_stream(stream));
}

int evo_layernorm_bwd_proj(int64_t rows, int cols, const float *dy, const float *x,
                           const float *mean, const float *rstd, const float *gamma,
                           const float *beta, const float *dres, const float *dproj, int64_t p_rs,
                           const void *Wp, int nh, float *dx, void *dx_act, float *dgamma,
                           float *dbeta, float *dx_colsum, float *dWp, void *workspace,
                           size_t workspace_bytes, void *stream) {
  EVO_REQUIRE(rows >= 0 && cols >= 1, EVO_EDIM, "evo_layernorm_bwd_proj: rows=%lld cols=%d",
              (long long)rows, cols);
  if (rows == 0) return EVO_OK;
  CHECK_PTR(x); CHECK_PTR(mean); CHECK_PTR(rstd); CHECK_PTR(gamma); CHECK_PTR(beta);
  CHECK_PTR(dproj); CHECK_PTR(Wp); CHECK_PTR(dx); CHECK_PTR(dWp);
  return layernorm_bwd_proj(rows, cols, dy, x, mean, rstd, gamma, beta, dres, dproj, p_rs, Wp, nh,
                            dx, dx_act, dgamma, dbeta, dx_colsum, dWp, workspace,
                            workspace_bytes, as_stream(stream));
}

static int check_attn(const evo_attn_desc *d, bool bwd) {
  CHECK_PTR(d);
  CHECK_DT(d->dtype);
  EVO_REQUIRE(d->nb >= 0 && d->H >= 1 && d->L >= 1 && d->D >= 1, EVO_EDIM,
              "attention: bad sizes nb=%lld H=%d L=%d D=%d", (long long)d->nb, d->H, d->L, d->D);
  EVO_REQUIRE(d->nb <= 65535, EVO_EDIM, "attention: nb=%lld > 65535", (long long)d->nb);
  CHECK_PTR(d->q); CHECK_PTR(d->k); CHECK_PTR(d->v); CHECK_PTR(d->g);
  CHECK_PTR(d->o); CHECK_PTR(d->lse);
  if (!bwd) CHECK_PTR(d->gm);
  if (bwd) {
    CHECK_PTR(d->dgm); CHECK_PTR(d->dq); CHECK_PTR(d->dk); CHECK_PTR(d->dv); CHECK_PTR(d->dgpre);
  }
  return EVO_OK;
}

int evo_attention_fwd(const evo_attn_desc *d, void *stream) {
  int rc = check_attn(d, false);
  if (rc != EVO_OK || d->nb == 0) return rc;
  if (attention_tc_accepts(d)) {
    rc = attention_tc_fwd(d, as_stream(stream));
    if (rc != EVO_EUNSUP) {
      note_backend(EVO_BK_ATTN_TC);
      return rc;
    }
  }
  EVO_REQUIRE(!(g_strict_tc.load() && d->dtype == EVO_BF16), EVO_EUNSUP,
              "evo_attention_fwd: bf16 nb=%lld H=%d L=%d D=%d is not taken by the tensor-core "
              "kernel and strict tensor-core mode forbids the SIMT fallback",
              (long long)d->nb, d->H, d->L, d->D);
  note_backend(EVO_BK_ATTN_SIMT);
  return attention_simt_fwd(d, as_stream(stream));
}

size_t evo_attention_bwd_workspace_bytes(const evo_attn_desc *d) {
  if (!d) return 0;
  return std::max(attention_simt_bwd_ws(d), attention_tc_bwd_ws(d));
}

int evo_attention_bwd(const evo_attn_desc *d, void *stream) {
  int rc = check_attn(d, true);
  if (rc != EVO_OK || d->nb == 0) return rc;
  if (attention_tc_accepts(d)) {
    rc = attention_tc_bwd(d, as_stream(stream));
    if (rc != EVO_EUNSUP) {
      note_backend(EVO_BK_ATTN_TC);
      return rc;
    }
  }
  EVO_REQUIRE(!(g_strict_tc.load() && d->dtype == EVO_BF16), EVO_EUNSUP,
              "evo_attention_bwd: bf16 nb=%lld H=%d L=%d D=%d is not taken by the tensor-core "
              "kernel and strict tensor-core mode forbids the SIMT fallback",
              (long long)d->nb, d->H, d->L, d->D);
  note_backend(EVO_BK_ATTN_SIMT);
  return attention_simt_bwd(d, as_stream(stream));
}

int evo_reduce_lead(int dtype_src, int64_t nb, int64_t n1, int64_t n2, const void *src,
                    float *dst, int64_t d_s1, int64_t d_s2, int accumulate, void *stream) {
  CHECK_DT(dtype_src);
  EVO_REQUIRE(nb >= 0 && n1 >= 0 && n2 >= 0, EVO_EDIM, "evo_reduce_lead: negative size");
  if (n1 * n2 == 0) return EVO_OK;
  CHECK_PTR(dst);
  if (nb > 0) CHECK_PTR(src);
  return reduce_lead(dtype_src, nb, n1, n2, src, dst, d_s1, d_s2, accumulate, as_stream(stream));
}

size_t evo_colsum_workspace_bytes(int64_t cols) { return (size_t)256 * cols * sizeof(float); }

int evo_colsum(int dtype_src, int64_t rows, int64_t cols, const void *src, int64_t rs,
               float *dst, int accumulate, void *workspace, size_t workspace_bytes,
               void *stream) {
  CHECK_DT(dtype_src);
  EVO_REQUIRE(rows >= 0 && cols >= 0, EVO_EDIM, "evo_colsum: negative size");
  if (cols == 0) return EVO_OK;
  CHECK_PTR(dst);
  if (rows == 0) {
    if (!accumulate) cudaMemsetAsync(dst, 0, cols * sizeof(float), as_stream(stream));
    return EVO_OK;
  }
  CHECK_PTR(src);
  EVO_REQUIRE(workspace && workspace_bytes >= evo_colsum_workspace_bytes(cols), EVO_EARG,
              "evo_colsum: workspace too small");
  return colsum(dtype_src, rows, cols, src, rs, dst, accumulate,
                reinterpret_cast<float *>(workspace), as_stream(stream));
}

int evo_copy2d(int dtype_src, int dtype_dst, int64_t rows, int64_t cols, const void *src,
               int64_t s_rs, int64_t s_cs, void *dst, int64_t d_rs, int64_t d_cs, void *stream) {
  CHECK_DT(dtype_src);
  CHECK_DT(dtype_dst);
  EVO_REQUIRE(rows >= 0 && cols >= 0, EVO_EDIM, "evo_copy2d: negative size");
  if (rows * cols == 0) return EVO_OK;
  CHECK_PTR(src); CHECK_PTR(dst);
  return copy2d(dtype_src, dtype_dst, rows, cols, src, s_rs, s_cs, dst, d_rs, d_cs,
                as_stream(stream));
}

int evo_copy3d(int dtype_src, int dtype_dst, int64_t n0, int64_t rows, int64_t cols,
               const void *src, int64_t s_bs, int64_t s_rs, int64_t s_cs, void *dst, int64_t d_bs,
               int64_t d_rs, int64_t d_cs, void *stream) {
  CHECK_DT(dtype_src);
  CHECK_DT(dtype_dst);
  EVO_REQUIRE(n0 >= 0 && rows >= 0 && cols >= 0, EVO_EDIM, "evo_copy3d: negative size");
  if (n0 * rows * cols == 0) return EVO_OK;
  CHECK_PTR(src); CHECK_PTR(dst);
  return copy3d(dtype_src, dtype_dst, n0, rows, cols, src, s_bs, s_rs, s_cs, dst, d_bs, d_rs,
                d_cs, as_stream(stream));
}

int evo_zero(void *ptr, size_t bytes, void *stream) {
  if (bytes == 0) return EVO_OK;
  CHECK_PTR(ptr);
  const cudaError_t e = cudaMemsetAsync(ptr, 0, bytes, as_stream(stream));
  EVO_REQUIRE(e == cudaSuccess, EVO_ECUDA, "evo_zero: %s", cudaGetErrorString(e));
  return EVO_OK;
}

int evo_mul2d(int dtype_a, int dtype_b, int dtype_out, int64_t rows, int64_t cols, const void *a,
              int64_t a_rs, const void *b, int64_t b_rs, void *out, int64_t o_rs, void *stream) {
  CHECK_DT(dtype_a); CHECK_DT(dtype_b); CHECK_DT(dtype_out);
  if (rows * cols == 0) return EVO_OK;
  CHECK_PTR(a); CHECK_PTR(b); CHECK_PTR(out);
  return mul2d(dtype_a, dtype_b, dtype_out, rows, cols, a, a_rs, b, b_rs, out, o_rs,
               as_stream(stream));
}

int evo_trimul_gate_fwd(int dtype, int64_t rows, int c, const void *proj, int64_t ldp,
                        void *a_cf, void *b_cf, void *stream) {
  CHECK_DT(dtype);
  EVO_REQUIRE(c >= 1 && c <= 256 && ldp >= 4 * c, EVO_EDIM, "evo_trimul_gate_fwd: c=%d ldp=%lld",
              c, (long long)ldp);
  if (rows == 0) return EVO_OK;
  CHECK_PTR(proj); CHECK_PTR(a_cf); CHECK_PTR(b_cf);
  return trimul_gate_fwd(dtype, rows, c, proj, ldp, a_cf, b_cf, as_stream(stream));
}

size_t evo_trimul_gate_bwd_workspace_bytes(int64_t rows, int c) {
  return trimul_gate_bwd_ws(rows, c);
}

int evo_trimul_gate_bwd(int dtype, int64_t rows, int c, const void *proj, int64_t ldp,
                        const float *da_cf, const float *db_cf, void *dproj, int64_t ldd,
                        float *colsum, void *workspace, size_t workspace_bytes, void *stream) {
  CHECK_DT(dtype);
  EVO_REQUIRE(c >= 1 && c <= 256 && ldp >= 4 * c && ldd >= 4 * c, EVO_EDIM,
              "evo_trimul_gate_bwd: c=%d", c);
  if (rows == 0) return EVO_OK;
  CHECK_PTR(proj); CHECK_PTR(da_cf); CHECK_PTR(db_cf); CHECK_PTR(dproj);
  EVO_REQUIRE(!colsum || (workspace && workspace_bytes >= trimul_gate_bwd_ws(rows, c)), EVO_EARG,
              "evo_trimul_gate_bwd: workspace too small for the column sums");
  return trimul_gate_bwd(dtype, rows, c, proj, ldp, da_cf, db_cf, dproj, ldd, colsum,
                         reinterpret_cast<float *>(workspace), as_stream(stream));
}

int evo_outgate_fwd(int dtype, int64_t rows, int64_t cols, const float *z, const void *g,
                    int64_t g_rs, const void *o, int64_t o_rs, float *znew, void *stream) {
  CHECK_DT(dtype);
  if (rows * cols == 0) return EVO_OK;
  CHECK_PTR(z); CHECK_PTR(g); CHECK_PTR(o); CHECK_PTR(znew);
  return outgate_fwd(dtype, rows, cols, z, g, g_rs, o, o_rs, znew, as_stream(stream));
}

size_t evo_outgate_bwd_workspace_bytes(int64_t rows, int64_t cols) {
  return outgate_bwd_ws(rows, cols);
}

int evo_outgate_bwd(int dtype, int64_t rows, int64_t cols, const float *dz, const void *g,
                    int64_t g_rs, const void *o, int64_t o_rs, void *do_, int64_t do_rs,
                    void *dgpre, int64_t dg_rs, float *do_colsum, float *dg_colsum,
                    void *workspace, size_t workspace_bytes, void *stream) {
  CHECK_DT(dtype);
  if (rows * cols == 0) return EVO_OK;
  CHECK_PTR(dz); CHECK_PTR(g); CHECK_PTR(o); CHECK_PTR(do_); CHECK_PTR(dgpre);
  EVO_REQUIRE(!(do_colsum || dg_colsum) ||
                  (workspace && workspace_bytes >= outgate_bwd_ws(rows, cols)),
              EVO_EARG, "evo_outgate_bwd: workspace too small for the column sums");
  return outgate_bwd(dtype, rows, cols, dz, g, g_rs, o, o_rs, do_, do_rs, dgpre, dg_rs,
                     do_colsum, dg_colsum, reinterpret_cast<float *>(workspace),
                     as_stream(stream));
}

int evo_relu_bwd(int dtype, int64_t n, const void *dh, const void *h, void *dpre, void *stream) {
  CHECK_DT(dtype);
  if (n == 0) return EVO_OK;
  CHECK_PTR(dh); CHECK_PTR(h); CHECK_PTR(dpre);
  return relu_bwd(dtype, n, dh, h, dpre, as_stream(stream));
}

int evo_relu_bwd_colsum(int64_t rows, int64_t cols, const void *dh, const void *h, void *dpre,
                        float *colsum_dst, void *workspace, size_t workspace_bytes,
                        void *stream) {
  EVO_REQUIRE(rows >= 0 && cols >= 1, EVO_EDIM, "evo_relu_bwd_colsum: rows=%lld cols=%lld",
              (long long)rows, (long long)cols);
  if (rows == 0) return EVO_OK;
  CHECK_PTR(dh); CHECK_PTR(h); CHECK_PTR(dpre); CHECK_PTR(colsum_dst);
  EVO_REQUIRE(workspace && workspace_bytes >= evo_colsum_workspace_bytes(cols), EVO_EARG,
              "evo_relu_bwd_colsum: workspace too small");
  return relu_bwd_colsum(rows, cols, dh, h, dpre, colsum_dst, reinterpret_cast<float *>(workspace),
                         as_stream(stream));
}

int evo_sq_mean(int64_t n, const float *x, float *out, float *dx, void *workspace,
                void *stream) {
  EVO_REQUIRE(n > 0, EVO_EDIM, "evo_sq_mean: n must be > 0");
  CHECK_PTR(x); CHECK_PTR(out); CHECK_PTR(workspace);
  return sq_mean(n, x, out, dx, workspace, as_stream(stream));
}

int evo_add(int64_t n, const float *a, const float *b, float *out, void *stream) {
  if (n == 0) return EVO_OK;
  CHECK_PTR(a); CHECK_PTR(b); CHECK_PTR(out);
  return add(n, a, b, out, as_stream(stream));
}

int evo_div_scalar(int64_t n, const float *x, float d, float *out, void *stream) {
  if (n == 0) return EVO_OK;
  CHECK_PTR(x); CHECK_PTR(out);
  return div_scalar(n, x, d, out, as_stream(stream));
}

int evo_split_bf16(int64_t rows, int64_t cols, const float *x, int64_t x_rs, void *hi,
                   int64_t h_rs, void *lo, int64_t l_rs, void *hi2, int64_t h2_rs, void *stream) {
  EVO_REQUIRE(rows >= 0 && cols >= 0, EVO_EDIM, "evo_split_bf16: negative size");
  if (rows * cols == 0) return EVO_OK;
  CHECK_PTR(x); CHECK_PTR(hi); CHECK_PTR(lo);
  return split_bf16(rows, cols, x, x_rs, hi, h_rs, lo, l_rs, hi2, h2_rs, as_stream(stream));
}

}  // extern "C"
