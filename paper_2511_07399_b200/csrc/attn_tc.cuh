// tensor-core attention (placeholder until the kernel lands).
#pragma once
#include <string>
#include "kernels.cuh"
namespace sdv2 {
inline bool tc_attn_enabled() { return false; }
inline bool tc_attention(cudaStream_t, const AttnArgs&, const TickDesc*, int, int, int, std::string* err) {
  *err = "tc attention not built"; return false; }
}  // namespace sdv2
