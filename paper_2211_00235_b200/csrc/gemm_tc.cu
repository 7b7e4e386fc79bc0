// placeholder: the tcgen05/TMA GEMM lands in the next milestone
#include "gemm.cuh"
namespace evo {
bool gemm_tc_accepts(const evo_gemm_desc *) { return false; }
size_t gemm_tc_workspace(const evo_gemm_desc *) { return 0; }
int gemm_tc(const evo_gemm_desc *, cudaStream_t) { return EVO_EUNSUP; }
}  // namespace evo
