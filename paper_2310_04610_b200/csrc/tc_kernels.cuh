// tc_kernels.cuh — tcgen05 (sm_100a tensor core) kernels: host-side entry points.
#pragma once
#include <string>

#include "common.cuh"

namespace evo {
namespace tc {

bool device_supported();
size_t fwd_scratch_bytes(const evo_attn_desc* d);
size_t bwd_scratch_bytes(const evo_attn_desc* d);
bool bwd_available(const evo_attn_desc* d);

evo_status fwd(const evo_attn_desc* d, const Shape& s, const void* q, const void* k, const void* v,
               void* o, float* lse, void* workspace, cudaStream_t st, int* launches,
               std::string* err);

evo_status bwd(const evo_attn_desc* d, const Shape& s, const void* dout, const void* q,
               const void* k, const void* v, const void* o, const float* lse, const float* delta, void* dq,
               void* dk, void* dv, float* dbias1, float* dbias2, void* scratch, cudaStream_t st,
               int* launches, std::string* err);

}  // namespace tc
}  // namespace evo
