// tcgen05 cross-attention over the prompt K/V (model card C.5 step 6:
// o_c = softmax(q_c K_c^T / sqrt(hd)) V_c per head, K_c / V_c computed once per prompt,
// P:189).  The prompt has Lk <= 512 keys (L_txt = 512 at every large config), so the whole
// S row of a 128-query tile fits TMEM and the softmax is exact and single-pass in its
// statistics: the row max over all Lk keys is known before any exponential, so there is
// no online rescale, no running-max exchange per tile and no split / merge of a unit
// across CTAs (the general kernel's stream-K pieces cost more than the 4 key tiles here).
//
// Unit = (entry, head, 128-query tile), persistent CTAs (one per SM) walk units u, u + G,
// ...; units of full query tiles come first and the ragged last tiles (L % 128 valid rows)
// last, so the second partial wave (156 units on 148 SMs at 1.3B 480p n = 1) holds the
// cheapest units.  Per unit, J = ceil(Lk / 128) <= 4 key tiles:
//   TMEM: S slots 0..2 at columns [0, 384), O at [384, 384 + hd).  S_0, S_1, S_2 land in
//   slots 0..2; with J = 4 the softmax warps copy S_0 to registers in the max pass and
//   free slot 0 for S_3.  Max pass over all tiles (row max exchanged once between the two
//   key-half warps of a row), then the exponential pass writes P (bf16, over its own S
//   columns) tile by tile and each PV_t MMA starts as soon as P_t is in TMEM; P_0 (from
//   registers) goes into slot 0 after PV_3 has read P_3 there.
// Warp roles (320 threads): 0 TMA (one Q tile, one 5-stage K/V ring: K_0..K_{J-1} then
// V_0..V_{J-1}), 1 MMA issuer, 2..9 softmax / epilogue (TMEM lane quarter x key half).
#pragma once
#include "attn_tc.cuh"

namespace sdv2 {

constexpr int kXattnThreads = 320;
constexpr int kXattnKV = 5;          // K/V ring stages: K_0..K_3 and V_0 in flight at unit start
constexpr int kXattnMaxJ = 4;        // key tiles per unit (Lk <= 512)

template <int HD>
struct XattnSmem {
  static constexpr int Q = kAttnBQ * HD * 2;
  static constexpr int KV = kAttnBKV * HD * 2;
  static constexpr int O = kAttnBQ * HD * 2;   // bf16 output tile staged for the TMA store
  // no alignment pad: the __align__(1024) extern block starts 1024-aligned (checked)
  static constexpr int total = Q + kXattnKV * KV + O + 512 + 2 * 1024 + 64;
};

struct XattnArgs {
  int L;              // query rows per entry
  int H, QT;          // heads, query tiles per entry (ceil(L / 128))
  int n_entries;      // active entries (prefix)
  int Lk;             // prompt keys (<= 512)
  int kv_row0;        // row of this block's slot 0 in the K/V maps
  int kv_slot_rows;   // rows between prompt slots (EntryDesc::xslot)
  float scale_log2;   // log2(e) / sqrt(hd)
  void* o;            // [rows, ldo] bf16
  int ldo;
  // Fused cross-q RMS (C.5 step 6, q_c = g_cq RMS_d(q)): when rowsq != nullptr, q holds the
  // raw projection, rowsq[row] its sum of squares over d, and the prompt K the gain-folded
  // K_c * g_cq; scores of row r are scaled by rsqrt(rowsq[r] / d + eps).
  const float* rowsq;   // [rows][nparts] partial sums of squares (d / 32 per row)
  int nparts;
  float inv_d, eps;
  long long* trace;     // test hook only: CTA wall stamps (globaltimer ns) [4096 + cta * 8 + event]
};

// test hook: 0 entry, 1 set up (after the PDL wait), 2 first Q landed (MMA warp), 3 first
// S landed (softmax), 4 unit 0's P done, 5 unit 0's epilogue done, 6 last epilogue done, 7 exit
#define XATTN_STAMP(ev)                                                                     \
  do {                                                                                      \
    if (a.trace != nullptr && blockIdx.x < 1024) {                                          \
      unsigned long long t_;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
      a.trace[4096 + blockIdx.x * 8 + (ev)] = (long long)t_;                                \
    }                                                                                       \
  } while (0)

// unit u -> (entry, head, query tile): full tiles first, then the ragged last tiles
__device__ __forceinline__ void xattn_unit(const XattnArgs& a, int u, int& e, int& h, int& qt) {
  const int QF = a.L / kAttnBQ;                       // full query tiles per entry
  const int nfull = a.n_entries * a.H * QF;
  if (u < nfull) {
    e = u / (a.H * QF);
    const int r = u % (a.H * QF);
    h = r / QF;
    qt = r % QF;
  } else {
    const int v = u - nfull;
    e = v / a.H;
    h = v % a.H;
    qt = QF;
  }
}

template <int HD>
__global__ void __launch_bounds__(kXattnThreads, 1) xattn_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                            const __grid_constant__ CUtensorMap tmK,
                                                            const __grid_constant__ CUtensorMap tmV,
                                                            const __grid_constant__ CUtensorMap tmO, XattnArgs a,
                                                            const TickDesc* __restrict__ td) {
  using SM = XattnSmem<HD>;
  constexpr int NCH = HD / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // one Q tile (a CTA rarely owns two units)
  uint8_t* sKV = sQ + SM::Q;                  // kXattnKV stages
  uint8_t* sO = sKV + kXattnKV * SM::KV;      // [HD / 64 boxes][128 rows][128 B], 128-byte swizzle
  uint64_t* bar = reinterpret_cast<uint64_t*>(sO + SM::O);
  if (smem != smem_raw) __trap();             // the budget has no alignment pad
  uint64_t* q_full = bar;                     // [2]
  uint64_t* q_empty = bar + 2;                // [2]
  uint64_t* kv_full = bar + 4;                // [kXattnKV]
  uint64_t* kv_empty = kv_full + kXattnKV;    // [kXattnKV]
  uint64_t* s_full = kv_empty + kXattnKV;     // [4] by key tile
  uint64_t* p_full = s_full + 4;              // [4] by key tile (8 softmax warps)
  uint64_t* pv_done = p_full + 4;             // [4] by key tile
  uint64_t* s0_free = pv_done + 4;            // softmax copied S_0 to registers (J = 4)
  uint64_t* o_empty = s0_free + 1;            // epilogue read O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);
  float* xm = reinterpret_cast<float*>(bar + 64);   // [2 halves][128] row max exchange
  float* xl = xm + 256;                              // [2 halves][128] row sum exchange

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  if (threadIdx.x == 0) XATTN_STAMP(0);
  const int QF = a.L / kAttnBQ;
  const int units = a.n_entries * a.H * (QF + (a.L % kAttnBQ ? 1 : 0));
  const int J = (a.Lk + kAttnBKV - 1) / kAttnBKV;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(q_full + i, 1);
      tc::mbar_init(q_empty + i, 1);
    }
    for (int i = 0; i < kXattnKV; ++i) {
      tc::mbar_init(kv_full + i, 1);
      tc::mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(s_full + i, 1);
      tc::mbar_init(p_full + i, 8);
      tc::mbar_init(pv_done + i, 1);
    }
    tc::mbar_init(s0_free, 8);
    tc::mbar_init(o_empty, 8);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  pdl_wait();      // q is produced upstream; prompt K/V may have been rewritten by a switch
  pdl_trigger();
  if (threadIdx.x == 0) XATTN_STAMP(1);
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 384u;
  auto tS = [&](int slot) { return tmem + uint32_t(slot) * 128u; };
  auto slot_of = [&](int t) { return t == 3 ? 0 : t; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int kvi = 0, ui = 0;
    for (int u = c; u < units; u += G, ++ui) {
      int e, h, qt;
      xattn_unit(a, u, e, h, qt);
      const int col = h * HD;
      const int kv_row = a.kv_row0 + td->e[e].xslot * a.kv_slot_rows;
      const int qs = 0;
      tc::mbar_wait(q_empty, (ui & 1) ^ 1);
      if (tc::elect_one()) {
        tc::mbar_expect_tx(q_full + qs, SM::Q);
        for (int ch = 0; ch < NCH; ++ch)
          tc::tma_load_2d(sQ + qs * SM::Q + ch * (kAttnBQ * 128), &tmQ, q_full + qs, col + ch * 64,
                          e * a.L + qt * kAttnBQ);
      }
      __syncwarp();
      for (int kv = 0; kv < 2; ++kv) {            // K_0..K_{J-1}, then V_0..V_{J-1}
        const CUtensorMap* map = kv ? &tmV : &tmK;
        for (int t = 0; t < J; ++t, ++kvi) {
          const int st = kvi % kXattnKV;
          tc::mbar_wait(kv_empty + st, ((kvi / kXattnKV) & 1) ^ 1);
          if (tc::elect_one()) {
            tc::mbar_expect_tx(kv_full + st, SM::KV);
            for (int ch = 0; ch < NCH; ++ch)
              tc::tma_load_2d(sKV + st * SM::KV + ch * (kAttnBKV * 128), map, kv_full + st, col + ch * 64,
                              kv_row + t * kAttnBKV);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idS = tc::idesc_bf16(kAttnBQ, kAttnBKV);
    const uint32_t idO = tc::idesc_bf16(kAttnBQ, HD, true);
    int kvi = 0, ui = 0;
    for (int u = c; u < units; u += G, ++ui) {
      const uint32_t ph = ui & 1;
      const int qs = 0;
      tc::mbar_wait(q_full, ui & 1);
      if (ui == 0 && lane == 0) XATTN_STAMP(2);
      const uint32_t qa = tc::smem_u32(sQ + qs * SM::Q);
      // S_t = Q K_t^T (S_3 into slot 0 once the softmax copied S_0 out)
      for (int t = 0; t < J; ++t, ++kvi) {
        const int st = kvi % kXattnKV;
        if (t == 3) tc::mbar_wait(s0_free, ph);
        tc::mbar_wait(kv_full + st, (kvi / kXattnKV) & 1);
        tc::tc_fence_after();
        const uint32_t ka = tc::smem_u32(sKV + st * SM::KV);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t off = (k >> 2) * (kAttnBQ * 128) + (k & 3) * 32;
            tc::mma_bf16(tS(slot_of(t)), tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + off), idS, k > 0);
          }
          tc::mma_commit(kv_empty + st);
          tc::mma_commit(s_full + t);
          if (t == J - 1) tc::mma_commit(q_empty + qs);
        }
        __syncwarp();
      }
      // O = sum_t P_t V_t in the softmax's P order (tile 0 last when J = 4)
      tc::mbar_wait(o_empty, ph ^ 1);
      for (int i = 0; i < J; ++i) {
        const int t = J == 4 ? (i == 0 ? 3 : (i == 3 ? 0 : i)) : i;   // 3, 1, 2, 0
        const int st = (kvi + t) % kXattnKV;                           // V_t's ring stage
        tc::mbar_wait(kv_full + st, ((kvi + t) / kXattnKV) & 1);
        tc::mbar_wait(p_full + t, ph);
        tc::tc_fence_after();
        const uint32_t va = tc::smem_u32(sKV + st * SM::KV);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tc::mma_bf16_ts(tO, tS(slot_of(t)) + (k >> 2) * 64 + (k & 3) * 8,
                            tc::sw128_mnmajor_desc(va + k * 2048, kAttnBKV * 128), idO, (i | k) != 0);
          tc::mma_commit(kv_empty + st);
          tc::mma_commit(pv_done + t);
        }
        __syncwarp();
      }
      kvi += J;
    }
  } else {
    // ------------------------------------------------ softmax / epilogue (8 warps)
    constexpr int HC = kAttnBKV / 2;        // S columns of a tile per thread (key half)
    constexpr int HO = HD / 2;              // O columns per thread in the epilogue
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory"); };
    int ui = 0;
    for (int u = c; u < units; u += G, ++ui) {
      int e, h, qt;
      xattn_unit(a, u, e, h, qt);
      const uint32_t ph = ui & 1;
      // per-row softmax scale (the fused q RMS factor, 1 without the fusion)
      const int qrow = qt * kAttnBQ + row;
      float rscale = a.scale_log2;
      if (a.rowsq) {   // sum the row's per-32-column partials in column order (deterministic)
        // nparts = d / 32 is a multiple of 4: independent 16-byte loads, fixed summation order
        const float4* rp = reinterpret_cast<const float4*>(a.rowsq + size_t(e * a.L + (qrow < a.L ? qrow : a.L - 1)) * a.nparts);
        float ssq = 0.f;
#pragma unroll 8
        for (int i = 0; i < a.nparts / 4; ++i) {
          const float4 v4 = __ldg(rp + i);
          ssq += (v4.x + v4.y) + (v4.z + v4.w);
        }
        rscale *= rsqrtf(ssq * a.inv_d + a.eps);
      }
      const uint64_t sc2 = f2pack(rscale, rscale);
      // ---- max pass (S_0 kept in registers when slot 0 is needed for S_3)
      float s0[HC];
      float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int t = 0; t < J; ++t) {
        tc::mbar_wait(s_full + t, ph);
        if (ui == 0 && t == 0 && warp == 2 && lane == 0) XATTN_STAMP(3);
        tc::tc_fence_after();
        float sv[HC];
        {
          uint32_t r[HC];
#pragma unroll
          for (int cc = 0; cc < HC / 32; ++cc)
            tc::tmem_ld32(tS(slot_of(t)) + lane_off + half * HC + cc * 32,
                          *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < HC; ++i) sv[i] = __uint_as_float(r[i]);
        }
        const int kvalid = a.Lk - t * kAttnBKV - half * HC;
        if (kvalid < HC) {
#pragma unroll
          for (int i = 0; i < HC; ++i) sv[i] = i < kvalid ? sv[i] : -INFINITY;
        }
#pragma unroll
        for (int i = 0; i < HC; i += 8) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mq[k] = fmax3(mq[k], sv[i + 2 * k], sv[i + 2 * k + 1]);
        }
        if (t == 0 && J == 4) {
#pragma unroll
          for (int i = 0; i < HC; ++i) s0[i] = sv[i];
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(s0_free);
        }
      }
      float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * rscale;
      xm[half * 128 + row] = mx;
      pair_sync();
      mx = fmaxf(mx, xm[(half ^ 1) * 128 + row]);
      const float msub = mx == -INFINITY ? 0.f : mx;   // rows with no valid key (never: Lk >= 1)
      const uint64_t nm2 = f2pack(-msub, -msub);
      // ---- exponential pass: P_t (bf16) over its own S columns, PV_t right behind it
      float l = 0.f;
      for (int i = 0; i < J; ++i) {
        const int t = J == 4 ? (i == 0 ? 3 : (i == 3 ? 0 : i)) : i;
        float sv[HC];
        if (t == 0 && J == 4) {
#pragma unroll
          for (int k = 0; k < HC; ++k) sv[k] = s0[k];
          tc::mbar_wait(pv_done + 3, ph);   // PV_3 read P_3 in slot 0
          tc::tc_fence_after();
        } else {
          uint32_t r[HC];
#pragma unroll
          for (int cc = 0; cc < HC / 32; ++cc)
            tc::tmem_ld32(tS(slot_of(t)) + lane_off + half * HC + cc * 32,
                          *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
          tc::tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < HC; ++k) sv[k] = __uint_as_float(r[k]);
        }
        const int kvalid = a.Lk - t * kAttnBKV - half * HC;
        uint32_t pk[HC / 2];
        float rs;
        if (kvalid >= HC) {
          rs = p_row<HC, true>(sv, pk, sc2, nm2);
        } else {
#pragma unroll
          for (int k = 0; k < HC; ++k) sv[k] = k < kvalid ? sv[k] : -INFINITY;
          rs = p_row<HC, false>(sv, pk, sc2, nm2);
        }
        l += rs;
        tc::tmem_st32(tS(slot_of(t)) + lane_off + half * HC, pk);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full + t);
      }
      // ---- epilogue: O / (l_half0 + l_half1) -> bf16
      if (ui == 0 && warp == 2 && lane == 0) XATTN_STAMP(4);
      xl[half * 128 + row] = l;
      const int tl = J == 4 ? 0 : J - 1;     // last PV issued
      tc::mbar_wait(pv_done + tl, ph);
      tc::tc_fence_after();
      pair_sync();
      const float inv = 1.f / (l + xl[(half ^ 1) * 128 + row]);
      // the row's HO columns -> the staged tile (box = 64 columns x 128 rows, 16-byte
      // granule g of row r at g ^ (r & 7)); rows >= L are clipped by the 3D map's bounds
#pragma unroll
      for (int cc = 0; cc < HO / 32; ++cc) {
        uint32_t r0[32];
        tc::tmem_ld32(tO + lane_off + half * HO + cc * 32, r0);
        tc::tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r0[2 * i]) * inv, __uint_as_float(r0[2 * i + 1]) * inv);
          pk[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        const int c0 = half * HO + cc * 32;                  // first column of the 32
        const uint32_t box = tc::smem_u32(sO + (c0 >> 6) * (kAttnBQ * 128)) + row * 128;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int g = ((c0 & 63) >> 3) + i;
          tc::st_shared_v4(box + ((g ^ (row & 7)) << 4), make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
        }
      }
      tc::fence_proxy_async_smem();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (warp == 2 && lane == 0) {
#pragma unroll
        for (int b = 0; b < HD / 64; ++b) tc::tma_store_3d(&tmO, sO + b * (kAttnBQ * 128), h * HD + b * 64, qt * kAttnBQ, e);
        tc::tma_store_commit_wait_read();   // staged tile reusable by this CTA's next unit
      }
      tc::tc_fence_before();
      pair_sync();                          // xm / xl reusable by the next unit
      if (lane == 0) tc::mbar_arrive(o_empty);
      if (warp == 2 && lane == 0) XATTN_STAMP(ui == 0 ? 5 : 6);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (warp == 2 && lane == 0) tc::tma_store_wait_all();
  if (threadIdx.x == 0) XATTN_STAMP(7);
}

// 3D bf16 map over the output [entries][L][ld] with (64 x 128 x 1) boxes, 128-byte swizzle:
// a 128-row tile of entry e ending past row L is clipped at the entry's end.
inline const CUtensorMap* xattn_out_map(AttnPlan& p, const void* base, int entries, int L, int ld, std::string* err) {
  const std::string key = "o3:" + std::to_string(reinterpret_cast<uintptr_t>(base)) + ":" + std::to_string(entries) +
                          ":" + std::to_string(L) + ":" + std::to_string(ld);
  auto it = p.maps.find(key);
  if (it != p.maps.end()) return &it->second;
  CUtensorMap m;
  const cuuint64_t dims[3] = {cuuint64_t(ld), cuuint64_t(L), cuuint64_t(entries)};
  const cuuint64_t strides[2] = {cuuint64_t(ld) * 2, cuuint64_t(L) * ld * 2};
  const cuuint32_t box[3] = {64, cuuint32_t(kAttnBQ), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = p.encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "xattn output map encode failed (" + std::to_string(int(r)) + ")";
    return nullptr;
  }
  return &(p.maps.emplace(key, m).first->second);
}

inline bool xattn_plan_init() {
  return cudaFuncSetAttribute(xattn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              XattnSmem<128>::total) == cudaSuccess &&
         cudaFuncSetAttribute(xattn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              XattnSmem<64>::total) == cudaSuccess;
}

// q: [q_rows, d] bf16; K / V maps over the whole prompt buffers [kv_rows, d].
inline bool tc_cross_attention(cudaStream_t s, AttnPlan& p, const void* q, long long q_rows, const void* Kbase,
                               const void* Vbase, long long kv_rows, int d, int hd, const XattnArgs& a,
                               const TickDesc* td, std::string* err, bool pdl = false) {
  if (a.Lk < 1 || a.Lk > kXattnMaxJ * kAttnBKV || (hd != 64 && hd != 128)) {
    *err = "cross attention: Lk must be in [1, 512], head dim 64 or 128";
    return false;
  }
  const CUtensorMap* mq = attn_map(p, q, q_rows, d, kAttnBQ, err);
  const CUtensorMap* mk = attn_map(p, Kbase, kv_rows, d, kAttnBKV, err);
  const CUtensorMap* mv = attn_map(p, Vbase, kv_rows, d, kAttnBKV, err);
  const CUtensorMap* mo = xattn_out_map(p, a.o, int(q_rows / a.L), a.L, a.ldo, err);
  if (!mq || !mk || !mv || !mo) return false;
  const int units = a.n_entries * a.H * a.QT;
  const int G = units < p.num_sms ? units : p.num_sms;
  if (G < 1) return true;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kXattnThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e;
  if (hd == 128) {
    cfg.dynamicSmemBytes = XattnSmem<128>::total;
    e = cudaLaunchKernelEx(&cfg, xattn_tc_kernel<128>, *mq, *mk, *mv, *mo, a, td);
  } else {
    cfg.dynamicSmemBytes = XattnSmem<64>::total;
    e = cudaLaunchKernelEx(&cfg, xattn_tc_kernel<64>, *mq, *mk, *mv, *mo, a, td);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("xattn_tc launch: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

}  // namespace sdv2
