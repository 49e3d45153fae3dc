// tc_kernels.cu — tcgen05 kernels (placeholder until the TMEM/TMA kernels land).
#include "tc_kernels.cuh"

namespace evo {
namespace tc {

bool device_supported() { return false; }
size_t fwd_scratch_bytes(const evo_attn_desc*) { return 0; }
size_t bwd_scratch_bytes(const evo_attn_desc*) { return 0; }

evo_status fwd(const evo_attn_desc*, const Shape&, const void*, const void*, const void*, void*,
               float*, void*, cudaStream_t, int*, std::string* err) {
  *err = "tcgen05 forward not built";
  return EVO_ERR_UNSUPPORTED;
}

evo_status bwd(const evo_attn_desc*, const Shape&, const void*, const void*, const void*,
               const void*, const float*, const float*, void*, void*, void*, float*, float*,
               void*, cudaStream_t, int*, std::string* err) {
  *err = "tcgen05 backward not built";
  return EVO_ERR_UNSUPPORTED;
}

}  // namespace tc
}  // namespace evo
