#pragma once
#include "common.cuh"

namespace evo {
int gemm_simt(const evo_gemm_desc *d, cudaStream_t st);
size_t gemm_simt_workspace(const evo_gemm_desc *d);
// tcgen05/TMA path; returns EVO_EUNSUP when the shape/layout is not taken.
int gemm_tc(const evo_gemm_desc *d, cudaStream_t st);
bool gemm_tc_accepts(const evo_gemm_desc *d);
size_t gemm_tc_workspace(const evo_gemm_desc *d);
// bandwidth-bound skinny shapes (N <= 16, K <= 16, or tiny M*N with huge K)
bool gemm_skinny_accepts(const evo_gemm_desc *d);
size_t gemm_skinny_workspace(const evo_gemm_desc *d);
int gemm_skinny(const evo_gemm_desc *d, cudaStream_t st);
}  // namespace evo
