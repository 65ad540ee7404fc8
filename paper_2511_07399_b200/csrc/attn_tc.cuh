// tcgen05 attention of the chunk queries over the [sink || rolling window] KV lane
// (SURVEY.md §8(a) a7, P:183 FlashAttention-style O(BT) memory, P:472 rolling cache)
// and over the prompt K/V (a9 cross-attention).
//
// One CTA = (entry e, head h, 128 query rows).  Keys are one contiguous row range
// of the lane (valid slots are always a prefix, so no gather and no slot mask; only
// the ragged key tail is masked).  Per 128-key tile j:
//   S_j = Q K_j^T        tcgen05.mma M=128 N=128 K=hd, A=Q (smem), B=K_j (smem), D in TMEM
//   softmax              4 warps, one query row per thread (tcgen05.ld S), exp2, running
//                        max / sum; P_j -> smem (bf16, 128-byte swizzle = UMMA K-major A)
//   O += P_j V_j         tcgen05.mma M=128 N=hd K=128, B = V_j MN-major, O stays in TMEM
// S is double-buffered in TMEM so S_{j+1}, S_{j+2} run on the tensor core while the
// softmax warps work on S_j.  O is rescaled in TMEM only when a row max grows by more
// than 2^8 (lazy rescale; P <= 256 keeps bf16 and fp32 sums safe).
// Warp roles (192 threads): 0 TMA, 1 MMA issuer, 2..5 softmax / correction / epilogue.
#pragma once
#include <string>
#include <unordered_map>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace sdv2 {

constexpr int kAttnBQ = 128, kAttnBKV = 128;

template <int HD>
struct AttnSmem {
  static constexpr int Q = kAttnBQ * HD * 2;          // 32 KB (hd 128)
  static constexpr int KV = kAttnBKV * HD * 2;        // one K or V tile
  static constexpr int P = kAttnBQ * kAttnBKV * 2;    // 32 KB
  static constexpr int total = Q + 4 * KV + P + 1024 + 512;
};

struct AttnTcArgs {
  int L;               // query rows per entry
  int q_row_base;      // always 0 (q buffer row e*L)
  int kv_row0;         // row of lane 0 / version 0 of this block in the K/V map
  int kv_lane_rows;    // rows between lanes (self) or prompt versions (cross)
  int cross;
  int Lk_cross;
  int col0;            // unused
  float scale_log2;    // log2(e) / sqrt(hd)
  void* o;
  int ldo;
};

__device__ __forceinline__ void tmem_ld32_f(uint32_t taddr, float (&f)[32]) {
  uint32_t r[32];
  tc::tmem_ld32(taddr, r);
  tc::tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(r[i]);
}

template <int HD>
__global__ void __launch_bounds__(192, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                         const __grid_constant__ CUtensorMap tmK,
                                                         const __grid_constant__ CUtensorMap tmV, AttnTcArgs a,
                                                         const TickDesc* __restrict__ td) {
  using SM = AttnSmem<HD>;
  constexpr int NCH = HD / 64;              // 64-column chunks of the head dim
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + SM::Q;                 // 2 stages
  uint8_t* sV = sK + 2 * SM::KV;            // 2 stages
  uint8_t* sP = sV + 2 * SM::KV;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + SM::P);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;   // [2]
  uint64_t* s_empty = bar + 11; // [2]
  uint64_t* p_full = bar + 13;
  uint64_t* p_empty = bar + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int e = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * kAttnBQ;
  const EntryDesc& E = td->e[e];
  if (!E.active || q0 >= a.L) return;
  const int Lk = a.cross ? a.Lk_cross : E.nvalid * a.L;
  const int kv_row = a.kv_row0 + (a.cross ? (E.pver & 1) : e) * a.kv_lane_rows;
  const int J = (Lk + kAttnBKV - 1) / kAttnBKV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(k_full + s, 1);
      tc::mbar_init(k_empty + s, 1);
      tc::mbar_init(v_full + s, 1);
      tc::mbar_init(v_empty + s, 1);
      tc::mbar_init(s_full + s, 1);
      tc::mbar_init(s_empty + s, 4);
    }
    tc::mbar_init(p_full, 4);
    tc::mbar_init(p_empty, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128u};
  const uint32_t tO = tmem + 256u;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const int col = h * HD;
      tc::mbar_expect_tx(q_full, SM::Q);
      for (int c = 0; c < NCH; ++c)
        tc::tma_load_2d(sQ + c * (kAttnBQ * 128), &tmQ, q_full, col + c * 64, a.q_row_base + e * a.L + q0);
      for (int j = 0; j < J; ++j) {
        const int s = j & 1;
        const uint32_t ph = ((j >> 1) & 1) ^ 1;
        tc::mbar_wait(k_empty + s, ph);
        tc::mbar_expect_tx(k_full + s, SM::KV);
        for (int c = 0; c < NCH; ++c)
          tc::tma_load_2d(sK + s * SM::KV + c * (kAttnBKV * 128), &tmK, k_full + s, col + c * 64,
                          kv_row + j * kAttnBKV);
        tc::mbar_wait(v_empty + s, ph);
        tc::mbar_expect_tx(v_full + s, SM::KV);
        for (int c = 0; c < NCH; ++c)
          tc::tma_load_2d(sV + s * SM::KV + c * (kAttnBKV * 128), &tmV, v_full + s, col + c * 64,
                          kv_row + j * kAttnBKV);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idS = tc::idesc_bf16(kAttnBQ, kAttnBKV);
      const uint32_t idO = tc::idesc_bf16(kAttnBQ, HD, true);
      const uint32_t qa = tc::smem_u32(sQ), pa = tc::smem_u32(sP);
      auto issue_S = [&](int j) {
        const int s = j & 1;
        tc::mbar_wait(k_full + s, (j >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t ka = tc::smem_u32(sK + s * SM::KV);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (kAttnBQ * 128) + (k & 3) * 32;
          const uint32_t koff = (k >> 2) * (kAttnBKV * 128) + (k & 3) * 32;
          tc::mma_bf16(tS[s], tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + koff), idS, k > 0);
        }
        tc::mma_commit(k_empty + s);
        tc::mma_commit(s_full + s);
      };
      tc::mbar_wait(q_full, 0);
      issue_S(0);
      if (J > 1) issue_S(1);
      for (int j = 0; j < J; ++j) {
        const int s = j & 1;
        tc::mbar_wait(p_full, j & 1);
        tc::mbar_wait(v_full + s, (j >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t va = tc::smem_u32(sV + s * SM::KV);
#pragma unroll
        for (int k = 0; k < kAttnBKV / 16; ++k) {
          const uint32_t poff = (k >> 2) * (kAttnBQ * 128) + (k & 3) * 32;
          tc::mma_bf16(tO, tc::sw128_kmajor_desc(pa + poff),
                       tc::sw128_mnmajor_desc(va + k * 2048, kAttnBKV * 128), idO, (j | k) != 0);
        }
        tc::mma_commit(v_empty + s);
        tc::mma_commit(p_empty);
        if (j + 2 < J) {
          tc::mbar_wait(s_empty + s, (j >> 1) & 1);
          issue_S(j + 2);
        }
      }
    }
  } else {
    // ------------------------------------------------ softmax / correction / epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    float m_used = -INFINITY;   // max the current P / O are relative to (log2 domain)
    float l = 0.f;
    for (int j = 0; j < J; ++j) {
      const int s = j & 1;
      tc::mbar_wait(s_full + s, (j >> 1) & 1);
      tc::tc_fence_after();
      float sv[kAttnBKV];
#pragma unroll
      for (int c = 0; c < kAttnBKV / 32; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(tS[s] + lane_off + c * 32, r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[i]);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(s_empty + s);
      const int kvalid = Lk - j * kAttnBKV;
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < kAttnBKV; ++i) {
        sv[i] = (i < kvalid) ? sv[i] * a.scale_log2 : -INFINITY;
        mx = fmaxf(mx, sv[i]);
      }
      // wait until PV_{j-1} finished: P smem free and O stable in TMEM
      if (j > 0) tc::mbar_wait(p_empty, (j - 1) & 1);
      tc::tc_fence_after();
      if (mx > m_used + 8.f) {
        const float m_new = mx;
        if (j > 0) {
          const float alpha = exp2f(m_used - m_new);
          l *= alpha;
#pragma unroll
          for (int c = 0; c < HD / 16; ++c) {
            uint32_t r[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15])
                : "r"(tO + lane_off + c * 16));
            tc::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tc::tmem_st16(tO + lane_off + c * 16, r);
          }
          tc::tmem_st_wait();
        }
        m_used = m_new;
      }
      // P = exp2(s - m_used) -> bf16, 128-byte swizzled K-major rows
      float rs = 0.f;
      uint8_t* prow_base = sP + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
      for (int g = 0; g < kAttnBKV / 8; ++g) {
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float p0 = exp2f(sv[g * 8 + 2 * u] - m_used);
          const float p1 = exp2f(sv[g * 8 + 2 * u + 1] - m_used);
          rs += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          pk[u] = *reinterpret_cast<uint32_t*>(&b2);
        }
        const int chunk = g >> 3, unit = g & 7;
        uint8_t* dst = prow_base + chunk * (kAttnBQ * 128) + ((unit ^ (row & 7)) << 4);
        *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      l += rs;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full);
    }
    // epilogue: wait for the last PV, O / l -> bf16
    tc::mbar_wait(p_empty, (J - 1) & 1);
    tc::tc_fence_after();
    const float inv = 1.f / l;
    const int qr = q0 + row;
    bf16* orow = reinterpret_cast<bf16*>(a.o) + size_t(e * a.L + qr) * a.ldo + h * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t r[32];
      tc::tmem_ld32(tO + lane_off + c * 32, r);
      tc::tmem_ld_wait();
      if (qr < a.L) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[2 * i]) * inv, __uint_as_float(r[2 * i + 1]) * inv);
          pk[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          reinterpret_cast<uint4*>(orow + c * 32)[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side
struct AttnPlan {
  PFN_encodeTiled encode = nullptr;
  std::unordered_map<std::string, CUtensorMap> maps;
  bool ready = false;
};

inline bool tc_attn_enabled() { return true; }

inline bool attn_plan_init(AttnPlan& p, PFN_encodeTiled enc) {
  p.encode = enc;
  cudaFuncSetAttribute(attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<128>::total);
  cudaFuncSetAttribute(attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<64>::total);
  p.ready = true;
  return true;
}

// 2D bf16 map over [rows, ld] with a (64 x box_rows) box, 128-byte swizzle.
inline const CUtensorMap* attn_map(AttnPlan& p, const void* base, long long rows, int ld, int box_rows,
                                   std::string* err) {
  const std::string key = std::to_string(reinterpret_cast<uintptr_t>(base)) + ":" + std::to_string(rows) + ":" +
                          std::to_string(ld) + ":" + std::to_string(box_rows);
  auto it = p.maps.find(key);
  if (it != p.maps.end()) return &it->second;
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(ld), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
  const cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = p.encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "attn map encode failed (" + std::to_string(int(r)) + ")";
    return nullptr;
  }
  return &(p.maps.emplace(key, m).first->second);
}

// q: [q_rows, ldq] bf16; K/V maps over whole buffers [kv_rows, ldk]; grid over
// (q tiles, heads, entries).
inline bool tc_attention(cudaStream_t s, AttnPlan& p, const void* q, long long q_rows, const void* Kbase,
                         const void* Vbase, long long kv_rows, int d, int hd, int H, int n_entries,
                         const AttnTcArgs& a, const TickDesc* td, std::string* err) {
  const CUtensorMap* mq = attn_map(p, q, q_rows, d, kAttnBQ, err);
  const CUtensorMap* mk = attn_map(p, Kbase, kv_rows, d, kAttnBKV, err);
  const CUtensorMap* mv = attn_map(p, Vbase, kv_rows, d, kAttnBKV, err);
  if (!mq || !mk || !mv) return false;
  dim3 grid((a.L + kAttnBQ - 1) / kAttnBQ, H, n_entries);
  if (hd == 128)
    attn_tc_kernel<128><<<grid, 192, AttnSmem<128>::total, s>>>(*mq, *mk, *mv, a, td);
  else
    attn_tc_kernel<64><<<grid, 192, AttnSmem<64>::total, s>>>(*mq, *mk, *mv, a, td);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("attn_tc launch: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

}  // namespace sdv2
