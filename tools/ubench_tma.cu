// L2 -> SM TMA streaming bandwidth on sm_100a (one CTA per SM, a 6-stage ring of 32 KB
// tiles, consumer releases immediately).  `share` CTAs read the same tile sequence at the
// same time (attention: the query tiles of a head share K/V; GEMM: M tiles share W).
// Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma tools/ubench_tma.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_2511_07399_b200/csrc/tc_common.cuh"

using namespace sdv2;
constexpr int kMaxStages = 6, kTileRows = 128, kTileBytes = kTileRows * 128 * 2;   // 128 x 128 bf16 (2 boxes)

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int tiles, int share,
                                                int rows_total, long long* cyc, int kStages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kMaxStages * kTileBytes);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    tc::fence_barrier_init();
  }
  __syncthreads();
  const int group = blockIdx.x / share;   // CTAs of a group stream the same rows
  const int ngroups = (gridDim.x + share - 1) / share;
  const long long t0 = clock64();
  if (warp == 0) {
    for (int i = 0; i < tiles; ++i) {
      const int st = i % kStages;
      tc::mbar_wait(empty + st, ((i / kStages) & 1) ^ 1);
      if (tc::elect_one()) {
        tc::mbar_expect_tx(full + st, kTileBytes);
        const int row = int(((long long)(i * ngroups + group) * kTileRows) % rows_total);
        tc::tma_load_2d(smem + st * kTileBytes, &tm, full + st, 0, row);
        tc::tma_load_2d(smem + st * kTileBytes + kTileBytes / 2, &tm, full + st, 64, row);
      }
      __syncwarp();
    }
  } else {
    for (int i = 0; i < tiles; ++i) {
      const int st = i % kStages;
      tc::mbar_wait(full + st, (i / kStages) & 1);
      if (tc::elect_one()) tc::mbar_arrive(empty + st);
      __syncwarp();
    }
    if (threadIdx.x == 32) cyc[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(fn);
  const int smem = kMaxStages * kTileBytes + 1024 + 256;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  for (long long mb : {32LL, 96LL, 1024LL}) {   // working set: L2-resident ... HBM
    const int rows = int(mb * 1024 * 1024 / 256);
    void* buf;
    cudaMalloc(&buf, size_t(rows) * 256);
    cudaMemset(buf, 0, size_t(rows) * 256);
    CUtensorMap tm;
    const cuuint64_t dims[2] = {128, cuuint64_t(rows)};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {64, kTileRows};
    const cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int cfg = 0; cfg < 9; ++cfg) {
      const int share = cfg < 4 ? (int[]){1, 2, 4, 13}[cfg] : 13;
      const int stages = cfg < 4 ? 6 : (int[]){1, 2, 3, 4, 5}[cfg - 4];
      const int tiles = 2000;
      stream<<<148, 64, smem>>>(tm, tiles, share, rows, cyc, stages);
      stream<<<148, 64, smem>>>(tm, tiles, share, rows, cyc, stages);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bpc = double(tiles) * kTileBytes / mx;
      printf("working set %5lld MB, %2d CTAs share each tile, %d x 32 KB in flight: %6.1f B/cycle/SM (%.1f TB/s "
             "@1.9GHz), latency %5.0f cycles\n",
             mb, share, stages, bpc, bpc * 148 * 1.9e9 / 1e12, stages * double(kTileBytes) / bpc);
    }
    cudaFree(buf);
  }
  return 0;
}
