// GEMM epilogue shared by the SIMT and tcgen05 kernels and the split-K
// reducer (order fixed by include/evo_b200.h: alpha, bias, relu|sigmoid,
// residual, accumulate).
#pragma once
#include "common.cuh"

namespace evo {

struct EpiArgs {
  void *C;
  IdxMap cmap;
  int64_t c_b1, c_b2;
  int dtype_c;
  int epi, epi_col0, accumulate;
  const float *bias, *residual;
  float alpha;
};

__device__ __forceinline__ float epi_value(const EpiArgs &e, int64_t n, float acc) {
  float v = e.alpha * acc;
  if (e.bias) v += e.bias[n];
  if (e.epi == EVO_EPI_RELU) v = fmaxf(v, 0.f);
  else if (e.epi == EVO_EPI_SIGMOID_FROM && n >= e.epi_col0) v = sigmoidf_stable(v);
  return v;
}

// Store one finished value (after epi_value) at element offset `off`.
__device__ __forceinline__ void epi_store(const EpiArgs &e, int64_t off, float v) {
  if (e.residual) v += e.residual[off];
  if (e.dtype_c == EVO_F32) {
    float *c = reinterpret_cast<float *>(e.C);
    c[off] = e.accumulate ? c[off] + v : v;
  } else {
    bf16 *c = reinterpret_cast<bf16 *>(e.C);
    c[off] = __float2bfloat16_rn(e.accumulate ? __bfloat162float(c[off]) + v : v);
  }
}

inline EpiArgs epi_args_of(const evo_gemm_desc *d) {
  EpiArgs e;
  e.C = d->C.ptr;
  e.cmap = idxmap_of(d->C);
  e.c_b1 = d->C.bs1;
  e.c_b2 = d->C.bs2;
  e.dtype_c = d->dtype_c;
  e.epi = d->epilogue;
  e.epi_col0 = d->epi_col0;
  e.accumulate = d->accumulate;
  e.bias = d->bias;
  e.residual = d->residual;
  e.alpha = d->alpha;
  return e;
}

// Sum split-K partials [split][B1*B2][M][N] (fixed order) and apply the
// epilogue.  Partials already carry no alpha.
int gemm_splitk_reduce(const evo_gemm_desc *d, int split, const float *partial,
                       cudaStream_t st);

}  // namespace evo
