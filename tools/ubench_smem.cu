// Does TMA / bulk-copy traffic into shared memory slow the tensor pipe's shared-memory
// operand reads?  One CTA per SM: warp 4 issues tcgen05.mma 128x128x16 (8 per iteration,
// SS = A and B from smem, TS = A from TMEM), warp 0 optionally streams 32 KB bulk copies
// (L2-resident source) into smem at the same time.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_smem_bin tools/ubench_smem.cu
#include <cstdio>
#include <cstdlib>
#include "../paper_2511_07399_b200/csrc/tc_common.cuh"
using namespace sdv2;
constexpr int kIters = 2000;

template <int mode>
__global__ void __launch_bounds__(160, 1) ub(const uint8_t* src, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                  // 32 KB
  uint8_t* sB = smem + 32768;          // 32 KB
  uint8_t* sD = smem + 65536;          // 2 x 32 KB copy destination
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 131072);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 8);
  volatile int* done = reinterpret_cast<volatile int*>(bars + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool ts = mode == 2 || mode == 3, copies = mode == 1 || mode == 3 || mode >= 4, mma = mode != 4 && mode < 9;
  // modes 9 / 10: copies alone, every SM streaming its own data: 9 = a 256 KB region per SM
  // (37 MB total, L2-resident after the first pass), 10 = a 6.4 MB region per SM (948 MB, HBM)
  const size_t region = mode == 9 ? (size_t(256) << 10) : mode == 10 ? (size_t(6400) << 10) : 65536;
  const uint8_t* mysrc = mode >= 9 ? src + region * blockIdx.x : src;
  // modes 5..8: SS variants: D column 0 or 256, accumulate from the second MMA of each
  // iteration (k > 0) or always after the first overall ((it | k) > 0)
  const uint32_t dcol = (mode == 5 || mode == 7) ? 0u : 256u;
  const bool acc_iter = mode == 5 || mode == 6;
  if (threadIdx.x == 0) {
    tc::mbar_init(bars + 0, 1);
    tc::mbar_init(bars + 1, 1);
    tc::mbar_init(bars + 2, 1);
    *done = 0;
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 4 && mma) {
    const uint32_t qa = tc::smem_u32(sA), ka = tc::smem_u32(sB);
    const uint32_t idS = tc::idesc_bf16(128, 128);
    long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * (128 * 128) + (k & 3) * 32;
          if (ts)
            tc::mma_bf16_ts(tmem + 256, tmem + k * 8, tc::sw128_kmajor_desc(ka + off), idS, (it | k) > 0);
          else if (mode >= 5)
            tc::mma_bf16(tmem + dcol, tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + off), idS,
                         acc_iter ? (k > 0) : ((it | k) > 0));
          else
            tc::mma_bf16(tmem + 256, tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + off), idS, (it | k) > 0);
        }
      }
      __syncwarp();
    }
    if (tc::elect_one()) {
      tc::mma_commit(bars + 2);
      tc::mbar_wait(bars + 2, 0);
      out[blockIdx.x * 4 + 0] = clock64() - t0;
      *done = 1;
    }
    __syncwarp();
  } else if (warp == 0 && copies) {
    long long t0 = clock64(), n = 0;
    const int maxn = mode == 4 || mode >= 9 ? 4000 : 1 << 30;
    while (n < maxn && !*done) {
      const int b = int(n & 1);
      if (n >= 2) tc::mbar_wait(bars + b, uint32_t(((n - 2) >> 1) & 1));
      if (lane == 0) {
        tc::mbar_expect_tx(bars + b, 32768);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];" ::"r"(
                         tc::smem_u32(sD + b * 32768)),
                     "l"(mysrc + (size_t(n) * 32768) % region), "r"(tc::smem_u32(bars + b))
                     : "memory");
      }
      __syncwarp();
      ++n;
    }
    if (n >= 1) tc::mbar_wait(bars + ((n - 1) & 1), uint32_t(((n - 1) >> 1) & 1));
    if (n >= 2) tc::mbar_wait(bars + ((n - 2) & 1), uint32_t(((n - 2) >> 1) & 1));
    if (lane == 0) {
      out[blockIdx.x * 4 + 1] = clock64() - t0;
      out[blockIdx.x * 4 + 2] = n;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

int main(int argc, char** argv) {
  const int grid = argc > 1 ? atoi(argv[1]) : 148;
  long long* d;
  uint8_t* src;
  cudaMalloc(&d, sizeof(long long) * 4 * 1024);
  const size_t srcb = size_t(6400) << 10;
  cudaMalloc(&src, srcb * 148);
  cudaMemset(src, 0, srcb * 148);
  const int smem = 131072 + 1024 + 256;
  void (*ks[11])(const uint8_t*, long long*) = {ub<0>, ub<1>, ub<2>, ub<3>, ub<4>, ub<5>, ub<6>, ub<7>, ub<8>, ub<9>, ub<10>};
  for (auto k : ks) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"8 SS MMA alone", "8 SS MMA + bulk copies", "8 TS MMA alone", "8 TS MMA + bulk copies",
                         "bulk copies alone", "SS D@0 acc k>0", "SS D@256 acc k>0", "SS D@0 acc always",
                         "SS D@256 acc always", "copies, own 256 KB per SM", "copies, own 6.4 MB per SM"};
  for (int mode = 0; mode < 11; ++mode) {
    for (int rep = 0; rep < 2; ++rep) ks[mode]<<<grid, 160, smem>>>(src, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    long long h[4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double mma_cyc = mode == 4 ? 0 : double(h[0]) / kIters;
    const double copy_bpc = (mode == 1 || mode == 3 || mode == 4 || mode >= 9) && h[1] > 0 ? double(h[2]) * 32768.0 / double(h[1]) : 0;
    printf("mode %d %-26s MMA %7.1f cycles / 8 MMAs   copies %6.1f B/cycle\n", mode, names[mode], mma_cyc, copy_bpc);
  }
  return 0;
}
