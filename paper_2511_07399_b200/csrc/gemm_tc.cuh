// tcgen05 GEMM (placeholder until the tensor-core kernel lands).
#pragma once
#include <string>
#include "kernels.cuh"
namespace sdv2 {
struct TmaGemmPlan { int unused = 0; };
inline bool tc_gemm_enabled() { return false; }
inline bool tc_gemm_plan(TmaGemmPlan&, std::string*) { return true; }
inline bool tc_gemm(cudaStream_t, const TmaGemmPlan&, const void*, const void*, int, int, int, int, const EpiArgs&,
                    std::string* err) { *err = "tc gemm not built"; return false; }
}  // namespace sdv2
