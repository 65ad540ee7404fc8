// Microbenchmark of the tcgen05 / mbarrier hand-off latencies the attention pipeline is
// built from (one CTA per SM, cycles per iteration).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_tc tools/ubench_tc.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include "../paper_2511_07399_b200/csrc/tc_common.cuh"

using namespace sdv2;

constexpr int kIters = 2000;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, %1;\n\t"
      "@px mov.s32 %0, 1;\n\t}"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

// mode 0: commit (no MMA) -> softmax wait -> arrive -> MMA-thread wait   (hand-off round trip)
// mode 1: mode 0 + 8 SS MMAs 128x128x16 before the commit               (+ S = QK^T latency)
// mode 2: mode 0 + softmax tcgen05.st x32 + wait before arrive
// mode 3: mode 0 + softmax 2x tcgen05.ld x32 + wait before arrive
// mode 4: MMA thread alone: 8 SS MMAs + commit + wait, serial           (MMA batch latency)
// mode 5: MMA thread alone: 8 SS MMAs + commit per iteration, no wait    (SS throughput)
// mode 6: MMA thread alone: 8 TS MMAs (A from TMEM) + commit, no wait     (TS throughput)
// mode 7: mode 5 with N = 256 (one 128x256 MMA per K step, 8 per iteration)
// mode 8: mode 5 without the per-iteration commit (one commit at the end)
// mode 9: mode 7 without the per-iteration commit
// mode 10: mode 8 with N = 64;  mode 11: N = 192
// mode 12: mode 8 alternating between 2 accumulators; mode 13: 4 accumulators (N = 128)
// mode 14: mode 9 (N = 256) alternating between 2 accumulators
// mode 15 / 16: mode 8 / 9 issued by the whole converged warp through elect.sync
// mode 17: mode 15 with one elect.sync around the 8 MMAs (not one per MMA)
// mode 18: mode 17 with N = 64
// mode 19: mode 17 with 8 TS MMAs (A = P from TMEM, N = 128: the attention PV step)
// mode 20: mode 17 with 8 SS (S into columns 0..127) then 8 TS (O += P V, P read from
//          columns 0..63): the attention's S / PV alternation, 16 MMAs per iteration
__global__ void __launch_bounds__(160, 1) ubench(int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // 128 x 128 bf16, two 64-col SW128 chunks (32 KB)
  uint8_t* sB = smem + 32768;       // 256 x 128 bf16 (64 KB)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 32768 + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(bars + 0, 1);   // s (MMA -> softmax)
    tc::mbar_init(bars + 1, 4);   // p (softmax -> MMA)
    tc::mbar_init(bars + 2, 1);   // self
    tc::mbar_init(bars + 3, 1);   // sink for throughput-mode commits
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *slot;
  const int NN = (mode == 7 || mode == 9 || mode == 14 || mode == 16) ? 256 : (mode == 10 || mode == 18) ? 64 : mode == 11 ? 192 : 128;
  const int nacc = (mode == 12 || mode == 14) ? 2 : mode == 13 ? 4 : 1;
  const uint32_t idS = tc::idesc_bf16(128, NN);
  const uint32_t idO = tc::idesc_bf16(128, 128, true);
  long long t0 = clock64();
  if (warp == 4 && (mode == 17 || mode == 18 || mode == 19 || mode == 20)) {
    const uint32_t qa = tc::smem_u32(sA), ka = tc::smem_u32(sB);
    for (int it = 0; it < kIters; ++it) {
      if (elect_one()) {
        if (mode != 19) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t off = (k >> 2) * (128 * 128) + (k & 3) * 32;
            const uint32_t koff = (k >> 2) * (NN * 128) + (k & 3) * 32;
            tc::mma_bf16(tmem, tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + koff), idS, k > 0);
          }
        }
        if (mode >= 19) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tc::mma_bf16_ts(tmem + 256, tmem + (k >> 2) * 64 + (k & 3) * 8, tc::sw128_mnmajor_desc(ka + k * 2048, 128 * 128),
                            idO, (it | k) > 0);
        }
      }
      __syncwarp();
    }
    if (elect_one()) {
      tc::mma_commit(bars + 2);
      tc::mbar_wait(bars + 2, 0);
      out[blockIdx.x * 2 + 0] = clock64() - t0;
    }
    __syncwarp();
  } else if (warp == 4 && mode >= 15) {
    const uint32_t qa = tc::smem_u32(sA), ka = tc::smem_u32(sB);
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k >> 2) * (128 * 128) + (k & 3) * 32;
        const uint32_t koff = (k >> 2) * (NN * 128) + (k & 3) * 32;
        if (elect_one())
          tc::mma_bf16(tmem, tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + koff), idS, k > 0);
        __syncwarp();
      }
    }
    if (elect_one()) {
      tc::mma_commit(bars + 2);
      tc::mbar_wait(bars + 2, 0);
      out[blockIdx.x * 2 + 0] = clock64() - t0;
    }
    __syncwarp();
  } else if (warp == 4) {
    if (lane == 0) {
      const uint32_t qa = tc::smem_u32(sA), ka = tc::smem_u32(sB);
      for (int it = 0; it < kIters; ++it) {
        if (mode == 1 || mode >= 4) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t off = (k >> 2) * (128 * 128) + (k & 3) * 32;
            const uint32_t koff = (k >> 2) * (NN * 128) + (k & 3) * 32;
            if (mode == 6)
              tc::mma_bf16_ts(tmem + 256, tmem + k * 8, tc::sw128_mnmajor_desc(ka + k * 2048, 128 * 128), idO, k > 0);
            else
              tc::mma_bf16(tmem + (k % nacc) * (512 / nacc), tc::sw128_kmajor_desc(qa + off),
                           tc::sw128_kmajor_desc(ka + koff), idS, k >= nacc);
          }
        }
        if (mode <= 3) {
          tc::mma_commit(bars + 0);
          tc::mbar_wait(bars + 1, it & 1);
          tc::tc_fence_after();
        } else if (mode == 4) {
          tc::mma_commit(bars + 2);
          tc::mbar_wait(bars + 2, it & 1);
        } else if (mode <= 7) {
          tc::mma_commit(bars + 3);
        }
      }
      if (mode >= 5) {
        tc::mma_commit(bars + 2);
        tc::mbar_wait(bars + 2, 0);
      }
      out[blockIdx.x * 2 + 0] = clock64() - t0;
    }
  } else if (mode <= 3) {
    const uint32_t lo = uint32_t(warp * 32) << 16;
    for (int it = 0; it < kIters; ++it) {
      tc::mbar_wait(bars + 0, it & 1);
      tc::tc_fence_after();
      if (mode == 2) {
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = uint32_t(it + i);
        tc::tmem_st32(tmem + lo, z);
        tc::tmem_st_wait();
      } else if (mode == 3) {
        uint32_t r0[32], r1[32];
        tc::tmem_ld32(tmem + lo, r0);
        tc::tmem_ld32(tmem + lo + 32, r1);
        tc::tmem_ld_wait();
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) x ^= r0[i] ^ r1[i];
        if (x == 0x12345678u) out[1] = x;
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bars + 1);
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
  const int grid = argc > 1 ? atoi(argv[1]) : 1;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 2 * 1024);
  const int smem = 32768 + 65536 + 1024 + 256;
  cudaFuncSetAttribute(ubench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"handoff commit->wait->arrive->wait", "  + 8 SS MMA 128x128x16",
                         "  + tcgen05.st x32 + wait", "  + 2x tcgen05.ld x32 + wait",
                         "8 SS MMA + commit + wait (latency)", "8 SS MMA N=128 throughput",
                         "8 TS MMA N=128 throughput", "8 SS MMA N=256 throughput",
                         "8 SS MMA N=128, no commits", "8 SS MMA N=256, no commits",
                         "8 SS MMA N=64, no commits", "8 SS MMA N=192, no commits",
                         "8 SS MMA N=128, 2 accumulators", "8 SS MMA N=128, 4 accumulators",
                         "8 SS MMA N=256, 2 accumulators", "8 SS MMA N=128, warp + elect",
                         "8 SS MMA N=256, warp + elect", "8 SS MMA N=128, one elect", "8 SS MMA N=64, one elect",
                         "8 TS MMA N=128, one elect", "8 SS + 8 TS (S, PV), one elect"};
  for (int mode = 0; mode < 21; ++mode) {
    for (int rep = 0; rep < 2; ++rep) ubench<<<grid, 160, smem>>>(mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d %-40s %8.1f cycles/iter\n", mode, names[mode], double(h[0]) / kIters);
  }
  return 0;
}
