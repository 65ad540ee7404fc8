// Causal 3D convolution on the tensor cores (Stream-VAE stand-in, SURVEY.md §8(f) N1;
// "Stream-VAE processes short video chunks (e.g., 4 frames) and caches
// intermediate features within each 3D convolution to maintain temporal coherence").
//
//   y[t, h, w, co] = b[co] + sum_{kt, kh, kw, ci} W[co, kt, kh, kw, ci] x[t + kt, h + kh - 1, w + kw - 1, ci]
//   (+ r[t, h, w, co]),  kernel 3 x 3 x 3, spatial padding 1 (zeros), causal in time:
//   the input buffer holds 2 cached frames of the previous chunk in front of the chunk's
//   frames (zeros before the first chunk), so output frame t reads buffer frames t..t+2.
//
// Implicit GEMM, no im2col buffer: M = output pixels (tiles of 128 consecutive w of one
// (t, h) row), N = output channels, K = 27 taps x Cin.  The A tile of k-block (tap, 64-channel
// block) is ONE 4D TMA box {64 ch, 128 w, 1 h, 1 t} at the tap-shifted coordinates of the
// channels-last input [T][H][W][C]; TMA zero-fills the out-of-bounds w = -1 / W and
// h = -1 / H rows, which is exactly the spatial zero padding.  B = weights [Cout][27 Cin]
// K-major.  tcgen05.mma M=128 N=BN K=16 into a double-buffered TMEM accumulator, epilogue
// bias (+ residual) -> bf16 channels-last.  The K order is fixed (taps, then channels), so
// a chunked (streamed) run and a whole-sequence run give bit-identical frames.
// Warp roles (256 threads): 0 TMA, 1 MMA, 2 TMEM alloc, 4..7 epilogue.
#pragma once
#include <string>

#include "gemm_tc.cuh"

namespace sdv2 {

constexpr int kConvThreads = 256;
constexpr int kConvBM = 128;

struct ConvArgs {
  int T, H, W;          // output frames / height / width (input buffer has T + 2 frames)
  int Cin, Cout;        // stored channels (multiples of 64 / 32)
  int BN;               // output-channel tile (multiple of 32, <= 256, divides Cout)
  const float* bias;    // [Cout]
  const bf16* res;      // [T][H][W][Cout] or nullptr
  bf16* out;            // [T][H][W][Cout]
};

__host__ __device__ inline int conv_stages(int BN) {
  const int st = (kGemmSmem - 2048 - 256 * 4) / (kGemmSmemA + BN * kGemmBK * 2);
  return st > kGemmMaxStages ? kGemmMaxStages : st;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kConvThreads, 1) conv3d_tc_kernel(const __grid_constant__ CUtensorMap tmX,
                                                           const __grid_constant__ CUtensorMap tmW, ConvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int BN = a.BN;
  const int kStages = conv_stages(BN);
  const int kSmemB = BN * kGemmBK * 2;
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kGemmSmemA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kSmemB);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sBias = reinterpret_cast<float*>(tmem_slot + 4);   // [BN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WB = (a.W + kConvBM - 1) / kConvBM;
  const int num_m = a.T * a.H * WB, num_n = a.Cout / BN;
  const int tiles = num_m * num_n;
  const int CB = a.Cin / kGemmBK;
  const int KB = 27 * CB;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmX);
    tc::tma_prefetch_desc(&tmW);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(tfull + s, 1);
      tc::mbar_init(tempty + s, 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  pdl_wait();
  pdl_trigger();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t bytes = uint32_t(kGemmSmemA + kSmemB);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m = t % num_m, nb = t / num_m;
      const int wb = m % WB, h = (m / WB) % a.H, tt = m / (WB * a.H);
      for (int kb = 0; kb < KB; ++kb) {
        const int tap = kb / CB, cb = kb % CB;
        const int kt = tap / 9, kh = (tap / 3) % 3, kw = tap % 3;
        tc::mbar_wait(empty + stage, phase ^ 1);
        if (tc::elect_one()) {
          tc::mbar_expect_tx(full + stage, bytes);
          tma_load_4d(sA + stage * kGemmSmemA, &tmX, full + stage, cb * kGemmBK, wb * kConvBM + kw - 1, h + kh - 1,
                      tt + kt);
          tc::tma_load_2d(sB + stage * kSmemB, &tmW, full + stage, kb * kGemmBK, nb * BN);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = tc::idesc_bf16(kConvBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      tc::mbar_wait(tempty + acc, acc_phase ^ 1);
      tc::tc_fence_after();
      const uint32_t d_tmem = tmem + uint32_t(acc * BN);
      for (int kb = 0; kb < KB; ++kb) {
        tc::mbar_wait(full + stage, phase);
        tc::tc_fence_after();
        const uint32_t a0 = tc::smem_u32(sA + stage * kGemmSmemA);
        const uint32_t b0 = tc::smem_u32(sB + stage * kSmemB);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            tc::mma_bf16(d_tmem, tc::sw128_kmajor_desc(a0 + k * 32), tc::sw128_kmajor_desc(b0 + k * 32), idesc,
                         (kb | k) != 0);
          tc::mma_commit(empty + stage);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (tc::elect_one()) tc::mma_commit(tfull + acc);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m = t % num_m, nb = t / num_m;
      const int wb = m % WB, h = (m / WB) % a.H, tt = m / (WB * a.H);
      asm volatile("bar.sync 1, 128;" ::: "memory");            // previous tile's bias readers done
      for (int i = threadIdx.x - 128; i < BN; i += 128) sBias[i] = a.bias[nb * BN + i];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc::mbar_wait(tfull + acc, acc_phase);
      tc::tc_fence_after();
      const int w = wb * kConvBM + row;
      const size_t pix = (size_t(tt) * a.H + h) * a.W + (w < a.W ? w : 0);
      const uint32_t tbase = tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tbase + c, v);
        tc::tmem_ld_wait_dep(v);
        if (w < a.W) {
          const int co = nb * BN + c;
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) + sBias[c + i];
          if (a.res) {
            const uint4* rp = reinterpret_cast<const uint4*>(a.res + pix * a.Cout + co);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 u = rp[j];
              const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 x2 = __bfloat1622float2(b2[k]);
                f[j * 8 + 2 * k] += x2.x;
                f[j * 8 + 2 * k + 1] += x2.y;
              }
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
            pk[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          uint4* op = reinterpret_cast<uint4*>(a.out + pix * a.Cout + co);
#pragma unroll
          for (int j = 0; j < 4; ++j) op[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tempty + acc);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// 4D bf16 map over a channels-last buffer [T][H][W][C]: box {64 ch, 128 w, 1, 1}.
inline bool conv_map_x(PFN_encodeTiled enc, CUtensorMap* m, const void* ptr, int T, int H, int W, int C,
                       std::string* err) {
  const cuuint64_t dims[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(T)};
  const cuuint64_t strides[3] = {cuuint64_t(C) * 2, cuuint64_t(W) * C * 2, cuuint64_t(H) * W * C * 2};
  const cuuint32_t box[4] = {64, kConvBM, 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "conv input map encode failed (" + std::to_string(int(r)) + ")";
    return false;
  }
  return true;
}

inline bool conv_attr() {
  return cudaFuncSetAttribute(conv3d_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem) == cudaSuccess;
}

inline int conv_pick_bn(int Cout) {
  for (int bn : {256, 192, 128, 96, 64, 32})
    if (Cout % bn == 0) return bn;
  return 0;
}

// x: input buffer [T + 2][H][W][Cin] (two causal cache frames first), w: [Cout][27 Cin].
inline bool tc_conv3d(cudaStream_t s, PFN_encodeTiled enc, int num_sms, const void* x, const void* w, const ConvArgs& a_in,
                      std::string* err, bool pdl = false) {
  ConvArgs a = a_in;
  if (a.Cin % 64 || a.Cout % 32) {
    *err = "conv3d: Cin % 64 or Cout % 32";
    return false;
  }
  a.BN = conv_pick_bn(a.Cout);
  CUtensorMap mx, mw;
  if (!conv_map_x(enc, &mx, x, a.T + 2, a.H, a.W, a.Cin, err)) return false;
  {
    const cuuint64_t dims[2] = {cuuint64_t(27) * a.Cin, cuuint64_t(a.Cout)};
    const cuuint64_t strides[1] = {cuuint64_t(27) * a.Cin * 2};
    const cuuint32_t box[2] = {64, cuuint32_t(a.BN)};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&mw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      *err = "conv weight map encode failed";
      return false;
    }
  }
  const int tiles = a.T * a.H * ((a.W + kConvBM - 1) / kConvBM) * (a.Cout / a.BN);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles < num_sms ? tiles : num_sms);
  cfg.blockDim = dim3(kConvThreads);
  cfg.dynamicSmemBytes = kGemmSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, conv3d_tc_kernel, mx, mw, a);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("conv3d_tc launch: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

}  // namespace sdv2
