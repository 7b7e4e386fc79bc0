// placeholder: the tensor-core attention lands in a later milestone
#include "common.cuh"
namespace evo {
bool attention_tc_accepts(const evo_attn_desc *) { return false; }
size_t attention_tc_bwd_ws(const evo_attn_desc *) { return 0; }
int attention_tc_fwd(const evo_attn_desc *, cudaStream_t) { return EVO_EUNSUP; }
int attention_tc_bwd(const evo_attn_desc *, cudaStream_t) { return EVO_EUNSUP; }
}  // namespace evo
