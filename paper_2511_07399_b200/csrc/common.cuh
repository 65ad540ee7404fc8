// Device helpers shared by the sm_100a kernels (no method arithmetic here).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sdv2 {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// Programmatic dependent launch: wait for the upstream grid (its writes visible) and
// allow the downstream grid to be scheduled.  Every kernel launched with PDL calls
// pdl_wait() before its first access to data produced (or still read) upstream, and
// before any early return (so completion order is preserved).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Philox4x32-10 (Salmon et al., SC'11), same counter layout as the oracle:
// key = (seed lo, seed hi), counter = (X, j, e/4, 0).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// eps_{X,j}[e]: Box–Muller in fp64 on (w0,w1) for e%4 in {0,1}, (w2,w3) for {2,3};
// cos for even e%4, sin for odd (reading Q21).
__device__ __forceinline__ double gauss_noise(uint64_t seed, uint32_t X, uint32_t j, uint32_t e) {
  const uint4 w = philox4x32_10(make_uint4(X, j, e >> 2, 0u),
                                make_uint2(uint32_t(seed & 0xffffffffu), uint32_t(seed >> 32)));
  const uint32_t q = e & 3u;
  const uint32_t a = q < 2 ? w.x : w.z;
  const uint32_t b = q < 2 ? w.y : w.w;
  const double u1 = (double(a) + 0.5) * 2.3283064365386963e-10;
  const double u2 = (double(b) + 0.5) * 2.3283064365386963e-10;
  const double rad = sqrt(-2.0 * log(u1));
  const double ang = 6.283185307179586 * u2;
  return (q & 1u) ? rad * sin(ang) : rad * cos(ang);
}

}  // namespace sdv2
