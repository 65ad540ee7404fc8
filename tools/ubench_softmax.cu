// Cycles per softmax half-row (64 scores -> bf16 P + row sum) with 2 warps per SMSP, as
// in the attention kernel; isolates the exp section from the pipeline.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_softmax tools/ubench_softmax.cu -lcuda
#include <cstdio>
#include "../paper_2511_07399_b200/csrc/kernels.cuh"
#include "../paper_2511_07399_b200/csrc/gemm_tc.cuh"
#include "../paper_2511_07399_b200/csrc/attn_tc.cuh"

using namespace sdv2;

template <bool POLY>
__global__ void __launch_bounds__(256, 1) bench(float* out, long long* cyc, float scale) {
  float sv[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) sv[i] = -float((threadIdx.x * 7 + i * 13) % 97) * 0.05f;
  uint32_t sink = 0;
  float l = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < 1000; ++it) {
    uint32_t pk[32];
    const float m = float(it & 7) * 1e-3f;
    const uint64_t sc2 = f2pack(scale, scale), nm2 = f2pack(-m, -m);
    l += p_row<64, POLY>(sv, pk, sc2, nm2);
#pragma unroll
    for (int i = 0; i < 32; ++i) sink ^= pk[i];
    __syncwarp();
  }
  const long long t1 = clock64();
  out[blockIdx.x * 256 + threadIdx.x] = l + float(sink & 1);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&cyc, 148 * 8);
  long long h;
  bench<false><<<148, 256>>>(out, cyc, 0.1f);
  bench<false><<<148, 256>>>(out, cyc, 0.1f);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("MUFU only : %.0f cycles per 64-score half-row (2 warps/SMSP)\n", h / 1000.0);
  bench<true><<<148, 256>>>(out, cyc, 0.1f);
  bench<true><<<148, 256>>>(out, cyc, 0.1f);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("3/8 poly  : %.0f cycles per 64-score half-row (2 warps/SMSP)\n", h / 1000.0);
  return 0;
}
