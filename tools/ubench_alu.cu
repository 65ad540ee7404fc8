// Per-SM issue throughput of the softmax instruction mix (warp instructions per cycle per
// SM) on sm_100a: MUFU.EX2, F2FP bf16x2 pack, FFMA2, FFMA, PRMT, FMNMX.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_alu tools/ubench_alu.cu
#include <cstdio>
#include <cstdint>

constexpr int kIters = 4096;

template <int OP>
__global__ void alu(float* out, float seed, long long* cyc) {
  float a[8];
  uint32_t u[8];
  uint64_t d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = seed * (i + 1) + threadIdx.x * 1e-3f;
    u[i] = __float_as_uint(a[i]);
    asm("mov.b64 %0, {%1, %2};" : "=l"(d[i]) : "f"(a[i]), "f"(a[i] * 0.5f));
  }
  const uint64_t c2 = d[0];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %0;" : "+r"(u[i]) : "f"(a[i]));
      if (OP == 2) asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %1;" : "+l"(d[i]) : "l"(c2));
      if (OP == 3) asm volatile("fma.rn.ftz.f32 %0, %0, %1, %1;" : "+f"(a[i]) : "f"(seed));
      if (OP == 4) asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      if (OP == 5) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(seed));
      if (OP == 6) asm volatile("add.rn.ftz.f32x2 %0, %0, %1;" : "+l"(d[i]) : "l"(c2));
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += a[i] + __uint_as_float(u[i]) + __uint_as_float(uint32_t(d[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, float* out, long long* cyc, int threads) {
  alu<OP><<<148, threads>>>(out, 1.0001f, cyc);
  alu<OP><<<148, threads>>>(out, 1.0001f, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double warp_instr = double(kIters) * 8 * threads / 32;
  printf("%-22s threads %4d: %6.3f warp-instr/cycle/SM (%5.2f cycles per warp-instr per SMSP)\n", name, threads,
         warp_instr / h, 4.0 * h / warp_instr);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int th : {128, 512}) {
    run<0>("MUFU.EX2", out, cyc, th);
    run<1>("F2FP.BF16 pack", out, cyc, th);
    run<2>("FFMA2", out, cyc, th);
    run<3>("FFMA", out, cyc, th);
    run<4>("PRMT", out, cyc, th);
    run<5>("FMNMX", out, cyc, th);
    run<6>("FADD2", out, cyc, th);
  }
  return 0;
}
