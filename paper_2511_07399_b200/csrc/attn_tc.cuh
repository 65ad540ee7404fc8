// tcgen05 attention of the chunk queries over the [sink || rolling window] KV lane
// (SURVEY.md §8(a) a7, P:183 FlashAttention-style O(BT) memory, P:472 rolling cache)
// and over the prompt K/V (a9 cross-attention).
//
// Work unit = (entry e, head h, 128-query tile).  Keys are one contiguous row range of
// the lane (valid slots are always a prefix, so no gather and no slot mask; only the
// ragged key tail is masked).  The (unit, 128-key tile) space is split evenly over
// exactly one CTA per SM ("stream-K"): a CTA walks its contiguous tile range, which
// covers whole units in the middle and at most one partial unit at each end; partial
// units leave (unnormalised O, running max, sum) in a scratch slot and are merged by
// attn_combine_kernel in a fixed CTA order (deterministic).  This removes the wave
// quantisation of 156 units on 148 SMs (1.3B, 480p, n = 1).
//
// Per key tile g:  S_g = Q K_g^T (tcgen05.mma M=128 N=128 K=hd, D in TMEM, double
// buffered) -> softmax (4 warps, one query row per thread, tcgen05.ld, exp2, lazy
// rescale of O in TMEM when the row max grows by > 2^8) -> P_g (bf16, 128-byte
// swizzled smem = UMMA K-major A) -> O += P_g V_g (tcgen05.mma N=hd, V MN-major).
// Warp roles (192 threads): 0 TMA, 1 MMA issuer, 2..5 softmax / correction / epilogue.
#pragma once
#include <string>
#include <unordered_map>

#include <cuda_fp16.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace sdv2 {

constexpr int kAttnBQ = 128, kAttnBKV = 128;

template <int HD>
struct AttnSmem {
  static constexpr int Q = kAttnBQ * HD * 2;          // 32 KB (hd 128)
  static constexpr int KV = kAttnBKV * HD * 2;        // one K or V tile
  static constexpr int P = kAttnBQ * kAttnBKV * 2;    // 32 KB
  static constexpr int KS = 3, VS = 2;               // K / V ring stages
  static constexpr int total = Q + (KS + VS) * KV + 1024 + 256 + 512 * 4 + 64;
};

struct AttnTcArgs {
  int L;               // query rows per entry
  int kv_row0;         // row of lane 0 / version 0 of this block in the K/V map
  int kv_lane_rows;    // rows between lanes (self) or prompt versions (cross)
  int cross;
  int Lk_cross;
  float scale_log2;    // log2(e) / sqrt(hd)
  void* o;
  int ldo;
  int H, QT;           // heads, query tiles per entry
  int n_entries;       // entries covered (active prefix)
  float* part_o;       // [G][2][128][HD] fp32 partial (unnormalised) O
  float* part_ml;      // [G][2][128][2] running max (log2 domain), sum
  int per_unit;        // 1: one CTA per unit (grid = units, no merge); 0: stream-K
};

// Stream-K geometry shared by the attention and the combine kernels.
struct AttnGeo {
  long long off[kMaxSteps + 1];   // tile offset of entry e's first unit
  int J[kMaxSteps];               // key tiles per unit of entry e
  long long T;                    // total tiles
  __device__ void init(const AttnTcArgs& a, const TickDesc* td) {
    off[0] = 0;
    for (int e = 0; e < kMaxSteps; ++e) {
      int j = 0;
      if (e < a.n_entries && td->e[e].active) {
        const int Lk = a.cross ? a.Lk_cross : td->e[e].nvalid * a.L;
        j = (Lk + kAttnBKV - 1) / kAttnBKV;
      }
      J[e] = j;
      off[e + 1] = off[e] + (long long)a.H * a.QT * j;
    }
    T = off[kMaxSteps];
  }
  // unit containing global tile g -> (e, unit-in-entry w, tile j)
  __device__ void locate(long long g, int& e, int& w, int& j) const {
    e = 0;
    while (e < kMaxSteps - 1 && g >= off[e + 1]) ++e;
    const long long r = g - off[e];
    w = int(r / J[e]);
    j = int(r % J[e]);
  }
  __device__ long long start(int c, int G) const { return (T * c) / G; }
  __device__ int cta_of(long long g, int G) const { return int(((g + 1) * G + T - 1) / T) - 1; }
};

constexpr int kAttnThreads = 352;   // warp 0 TMA Q+K, 1 MMA, 2..9 softmax (two key halves), 10 TMA V

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Two exp2 per MUFU op: the softmax probabilities are rounded to bf16 (8-bit mantissa)
// for the PV MMA anyway; fp16 arguments (x <= 8 after the lazy-rescale threshold) lose
// precision only for terms below 2^-16 of the row maximum.
__device__ __forceinline__ float2 ex2x2(float x0, float x1) {
  uint32_t in, out;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(in) : "f"(x1), "f"(x0));
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(out) : "r"(in));
  __half2 h = *reinterpret_cast<__half2*>(&out);
  return __half22float2(h);
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                         const __grid_constant__ CUtensorMap tmK,
                                                         const __grid_constant__ CUtensorMap tmV, AttnTcArgs a,
                                                         const TickDesc* __restrict__ td) {
  using SM = AttnSmem<HD>;
  constexpr int NCH = HD / 64;              // 64-column chunks of the head dim
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  constexpr int KS = SM::KS, VS = SM::VS;
  uint8_t* sK = sQ + SM::Q;                 // KS stages
  uint8_t* sV = sK + KS * SM::KV;           // VS stages
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + VS * SM::KV);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* o_empty = bar + 2;
  // p_full / p_empty are indexed [S buffer][key half]: with the softmax running ahead of
  // the PV MMAs, per-buffer barriers never get more than one phase ahead of a waiter
  // (parity waits stay unambiguous).
  uint64_t* p_full = bar + 3;    // [2][2] P of (buffer, half) written (4 softmax warps)
  uint64_t* p_empty = bar + 7;   // [2][2] PV of (buffer, half) done
  uint64_t* s_full = bar + 11;   // [2]
  uint64_t* k_full = bar + 13;   // [KS]
  uint64_t* k_empty = bar + 16;  // [KS]
  uint64_t* v_full = bar + 19;   // [VS]
  uint64_t* v_empty = bar + 21;  // [VS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 23);
  float* xch = reinterpret_cast<float*>(bar + 24);   // [2 halves][128] (max, sum) exchange at segment end

  pdl_wait();      // q, K/V lanes and o are produced / consumed by the neighbouring kernels
  pdl_trigger();
  AttnGeo geo;
  geo.init(a, td);
  const int G = gridDim.x, c = blockIdx.x;
  long long t0, t1;
  if (a.per_unit) {
    const int e = c / (a.H * a.QT), w = c % (a.H * a.QT);
    if (e >= kMaxSteps || geo.J[e] == 0) return;
    t0 = geo.off[e] + (long long)w * geo.J[e];
    t1 = t0 + geo.J[e];
  } else {
    t0 = geo.start(c, G);
    t1 = geo.start(c + 1, G);
  }
  if (t0 >= t1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    tc::mbar_init(o_empty, 8);
    for (int s = 0; s < KS; ++s) {
      tc::mbar_init(k_full + s, 1);
      tc::mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < VS; ++s) {
      tc::mbar_init(v_full + s, 1);
      tc::mbar_init(v_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) tc::mbar_init(s_full + s, 1);
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(p_full + i, 4);
      tc::mbar_init(p_empty + i, 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128u};
  // Each key half (64 of the 128 keys of a tile) has its own O accumulator and running
  // max, so the two softmax warpgroups never synchronise per tile; they are merged once
  // per unit.  TMEM: S0 | S1 | O_half0 | O_half1 (128 columns each).
  const uint32_t tO2[2] = {tmem + 256u, tmem + 384u};

  // Segment iteration: [gs, ge) of global tiles inside one unit.
  struct Seg {
    int e, h, q0, jb, je, J;
    long long ge;
  };
  auto seg_at = [&](long long g) {
    Seg s;
    int w, j;
    geo.locate(g, s.e, w, j);
    s.h = w / a.QT;
    s.q0 = (w % a.QT) * kAttnBQ;
    s.J = geo.J[s.e];
    s.jb = j;
    const long long unit_end = g - j + s.J;
    s.ge = unit_end < t1 ? unit_end : t1;
    s.je = j + int(s.ge - g);
    return s;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      long long g = t0;
      int gi = 0, sg = 0;   // local tile counter, segment counter
      while (g < t1) {
        const Seg s = seg_at(g);
        const int col = s.h * HD;
        const int kv_row = a.kv_row0 + (a.cross ? (td->e[s.e].pver & 1) : s.e) * a.kv_lane_rows;
        if (sg > 0) tc::mbar_wait(q_empty, (sg - 1) & 1);
        tc::mbar_expect_tx(q_full, SM::Q);
        for (int ch = 0; ch < NCH; ++ch)
          tc::tma_load_2d(sQ + ch * (kAttnBQ * 128), &tmQ, q_full, col + ch * 64, s.e * a.L + s.q0);
        for (int j = s.jb; j < s.je; ++j, ++gi) {
          const int st = gi % KS;
          tc::mbar_wait(k_empty + st, ((gi / KS) & 1) ^ 1);
          tc::mbar_expect_tx(k_full + st, SM::KV);
          for (int ch = 0; ch < NCH; ++ch)
            tc::tma_load_2d(sK + st * SM::KV + ch * (kAttnBKV * 128), &tmK, k_full + st, col + ch * 64,
                            kv_row + j * kAttnBKV);
        }
        g = s.ge;
        ++sg;
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ TMA producer (V)
    // V tiles are consumed one MMA phase later than K: an own producer keeps the K
    // prefetch from waiting on V slots.
    if (lane == 0) {
      long long g = t0;
      int gi = 0;
      while (g < t1) {
        const Seg s = seg_at(g);
        const int col = s.h * HD;
        const int kv_row = a.kv_row0 + (a.cross ? (td->e[s.e].pver & 1) : s.e) * a.kv_lane_rows;
        for (int j = s.jb; j < s.je; ++j, ++gi) {
          const int st = gi % VS;
          tc::mbar_wait(v_empty + st, ((gi / VS) & 1) ^ 1);
          tc::mbar_expect_tx(v_full + st, SM::KV);
          for (int ch = 0; ch < NCH; ++ch)
            tc::tma_load_2d(sV + st * SM::KV + ch * (kAttnBKV * 128), &tmV, v_full + st, col + ch * 64,
                            kv_row + j * kAttnBKV);
        }
        g = s.ge;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idS = tc::idesc_bf16(kAttnBQ, kAttnBKV);
      const uint32_t idO = tc::idesc_bf16(kAttnBQ, HD, true);
      const uint32_t qa = tc::smem_u32(sQ);
      auto issue_S = [&](int gg) {     // gg = local tile counter
        const int st = gg & 1;         // S / P TMEM buffer
        const int ks = gg % KS;        // K smem stage
        // S_gg reuses the TMEM buffer of tile gg-2, whose P was consumed by PV_{gg-2}:
        // issued earlier by this thread, and tcgen05 MMAs execute in issue order.
        tc::mbar_wait(k_full + ks, (gg / KS) & 1);
        tc::tc_fence_after();
        const uint32_t ka = tc::smem_u32(sK + ks * SM::KV);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (kAttnBQ * 128) + (k & 3) * 32;
          const uint32_t koff = (k >> 2) * (kAttnBKV * 128) + (k & 3) * 32;
          tc::mma_bf16(tS[st], tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + koff), idS, k > 0);
        }
        tc::mma_commit(k_empty + ks);
        tc::mma_commit(s_full + st);
      };
      long long g = t0;
      int gi = 0, sg = 0;
      while (g < t1) {
        const Seg s = seg_at(g);
        const int nt = s.je - s.jb;
        tc::mbar_wait(q_full, sg & 1);
        issue_S(gi);
        if (nt > 1) issue_S(gi + 1);
        for (int t = 0; t < nt; ++t) {
          const int gt = gi + t;
          tc::mbar_wait(v_full + (gt % VS), (gt / VS) & 1);
          if (t == 0 && sg > 0) tc::mbar_wait(o_empty, (sg - 1) & 1);
          const uint32_t va = tc::smem_u32(sV + (gt % VS) * SM::KV);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {   // O_h += P[:, 64h : 64h+64] V[64h : 64h+64, :]
            tc::mbar_wait(p_full + (gt & 1) * 2 + hh, (gt >> 1) & 1);
            tc::tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k) {   // A = P_half from TMEM (bf16 pairs, 8 columns per K=16)
              tc::mma_bf16_ts(tO2[hh], tS[gt & 1] + hh * 64 + k * 8,
                              tc::sw128_mnmajor_desc(va + (hh * 4 + k) * 2048, kAttnBKV * 128), idO, (t | k) != 0);
            }
            tc::mma_commit(p_empty + (gt & 1) * 2 + hh);
          }
          tc::mma_commit(v_empty + (gt % VS));
          if (t + 2 < nt) issue_S(gt + 2);
        }
        tc::mma_commit(q_empty);
        gi += nt;
        g = s.ge;
        ++sg;
      }
    }
  } else if (warp <= 9) {
    // ------------------------------------------------ softmax / correction / epilogue
    // 8 warps: TMEM lane quarter = warp & 3 (row), column half = (warp - 2) / 4.
    constexpr int HC = kAttnBKV / 2;            // S columns per thread
    constexpr int HO = HD / 2;                  // O columns per thread
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    long long g = t0;
    int gi = 0, sg = 0;
    while (g < t1) {
      const Seg s = seg_at(g);
      const int nt = s.je - s.jb;
      const int Lk = a.cross ? a.Lk_cross : td->e[s.e].nvalid * a.L;
      float m_used = -INFINITY;   // max the current P / O are relative to (log2 domain)
      float l = 0.f;              // this half's share of the row sum
      for (int t = 0; t < nt; ++t) {
        const int gt = gi + t;
        const int st = gt & 1;
        tc::mbar_wait(s_full + st, (gt >> 1) & 1);
        tc::tc_fence_after();
        float sv[HC];
#pragma unroll
        for (int cc = 0; cc < HC / 32; ++cc) {
          uint32_t r[32];
          tc::tmem_ld32(tS[st] + lane_off + half * HC + cc * 32, r);
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[cc * 32 + i] = __uint_as_float(r[i]);
        }
        const int kvalid = Lk - (s.jb + t) * kAttnBKV - half * HC;
        float mx = -INFINITY;
        if (kvalid >= HC) {
#pragma unroll
          for (int i = 0; i < HC; ++i) mx = fmaxf(mx, sv[i]);
        } else {
#pragma unroll
          for (int i = 0; i < HC; ++i) {
            sv[i] = (i < kvalid) ? sv[i] : -INFINITY;
            mx = fmaxf(mx, sv[i]);
          }
        }
        mx *= a.scale_log2;
        // P_t lands in S buffer t&1 (not the one PV_{t-1} reads), so the softmax runs ahead
        // of the PV MMAs; only an O rescale needs PV_{t-1} of this half to be complete.
        if (mx > m_used + 8.f) {
          const float m_new = mx;
          if (t > 0) {     // rescale this half's O row (all HD columns) in TMEM
            tc::mbar_wait(p_empty + ((gt - 1) & 1) * 2 + half, ((gt - 1) >> 1) & 1);
            tc::tc_fence_after();
            const float alpha = ex2(m_used - m_new);
            l *= alpha;
#pragma unroll
            for (int cc = 0; cc < HD / 16; ++cc) {
              uint32_t r[16];
              const uint32_t ta = tO2[half] + lane_off + cc * 16;
              asm volatile(
                  "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                  "[%16];"
                  : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                    "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                    "=r"(r[15])
                  : "r"(ta));
              tc::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
              tc::tmem_st16(ta, r);
            }
            tc::tmem_st_wait();
          }
          m_used = m_new;
        }
        // P = exp2(s * scale - m_used) -> bf16 pairs written over this half's own S columns
        // in TMEM (A operand of the PV MMA); a half with no valid key yet writes P = 0
        const float msub = m_used == -INFINITY ? 0.f : m_used;
        float rs = 0.f;
        uint32_t pk[HC / 2];
#pragma unroll
        for (int i = 0; i < HC / 2; ++i) {
          const float2 pp = ex2x2(fmaf(sv[2 * i], a.scale_log2, -msub), fmaf(sv[2 * i + 1], a.scale_log2, -msub));
          rs += pp.x + pp.y;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(pp.x, pp.y);
          pk[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        tc::tmem_st32(tS[st] + lane_off + half * HC, pk);
        tc::tmem_st_wait();
        l += rs;
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full + (gt & 1) * 2 + half);
      }
      // end of segment: wait for this half's last PV; exchange (m, l) with the other half
      const int gl = gi + nt - 1;   // last tile of the segment
      tc::mbar_wait(p_empty + (gl & 1) * 2 + half, (gl >> 1) & 1);
      xch[half * 256 + row] = m_used;
      xch[half * 256 + 128 + row] = l;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      tc::mbar_wait(p_empty + (gl & 1) * 2 + (half ^ 1), (gl >> 1) & 1);   // other half's O complete too
      tc::tc_fence_after();
      const float m0 = xch[row], l0 = xch[128 + row], m1 = xch[256 + row], l1 = xch[384 + row];
      const float M = fmaxf(m0, m1);
      const float w0 = m0 == -INFINITY ? 0.f : ex2(m0 - M), w1 = m1 == -INFINITY ? 0.f : ex2(m1 - M);
      const float lt = l0 * w0 + l1 * w1;
      const bool full = (s.jb == 0 && s.je == s.J);
      const int slot = (g == t0) ? 0 : 1;
      const int qr = s.q0 + row;
      const float inv = full ? 1.f / lt : 1.f;
      const float c0w = w0 * inv, c1w = w1 * inv;
      bf16* orow = reinterpret_cast<bf16*>(a.o) + size_t(s.e * a.L + qr) * a.ldo + s.h * HD + half * HO;
      float* prow = a.part_o + ((size_t(c) * 2 + slot) * kAttnBQ + row) * HD + half * HO;
#pragma unroll
      for (int cc = 0; cc < HO / 32; ++cc) {
        uint32_t r0[32], r1[32];
        tc::tmem_ld32(tO2[0] + lane_off + half * HO + cc * 32, r0);
        tc::tmem_ld32(tO2[1] + lane_off + half * HO + cc * 32, r1);
        tc::tmem_ld_wait();
        float o[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r0[i]) * c0w + __uint_as_float(r1[i]) * c1w;
        if (full) {
          if (qr < a.L) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              __nv_bfloat162 b2 = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
              pk[i] = *reinterpret_cast<uint32_t*>(&b2);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(orow + cc * 32)[i] =
                  make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(prow + cc * 32)[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        }
      }
      if (!full && half == 0) {
        float* ml = a.part_ml + ((size_t(c) * 2 + slot) * kAttnBQ + row) * 2;
        ml[0] = M;
        ml[1] = lt;
      }
      tc::tc_fence_before();
      asm volatile("bar.sync 1, 256;" ::: "memory");   // xch reusable, both halves done with O
      if (lane == 0) tc::mbar_arrive(o_empty);
      gi += nt;
      g = s.ge;
      ++sg;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// Merge the partial units (split between consecutive CTAs) in CTA order:
// O = sum_k 2^(m_k - M) O_k / sum_k 2^(m_k - M) l_k.  One CTA per unit; a warp per row,
// lanes across the head dim (coalesced 512 B row reads).
template <int HD>
__global__ void __launch_bounds__(256) attn_combine_kernel(AttnTcArgs a, const TickDesc* __restrict__ td, int G) {
  pdl_wait();
  pdl_trigger();
  constexpr int PL = HD / 32;   // columns per lane
  AttnGeo geo;
  geo.init(a, td);
  const int u = blockIdx.x;
  const int e = u / (a.H * a.QT), w = u % (a.H * a.QT);
  if (e >= a.n_entries || geo.J[e] == 0) return;
  const long long off = geo.off[e] + (long long)w * geo.J[e];
  const int cf = geo.cta_of(off, G), cl = geo.cta_of(off + geo.J[e] - 1, G);
  if (a.per_unit || cf == cl) return;   // one CTA covered the whole unit and wrote the final output
  const int h = w / a.QT, q0 = (w % a.QT) * kAttnBQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot_f = geo.start(cf, G) < off ? 1 : 0;
  for (int row = warp; row < kAttnBQ; row += 8) {
    const int qr = q0 + row;
    if (qr >= a.L) break;
    float M = -INFINITY;
    for (int cc = cf; cc <= cl; ++cc) {
      const int slot = cc == cf ? slot_f : 0;
      M = fmaxf(M, a.part_ml[((size_t(cc) * 2 + slot) * kAttnBQ + row) * 2]);
    }
    float den = 0.f, acc[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) acc[i] = 0.f;
    for (int cc = cf; cc <= cl; ++cc) {
      const int slot = cc == cf ? slot_f : 0;
      const size_t base = (size_t(cc) * 2 + slot) * kAttnBQ + row;
      const float wgt = exp2f(a.part_ml[base * 2] - M);
      den += wgt * a.part_ml[base * 2 + 1];
      const float* po = a.part_o + base * HD + lane * PL;
#pragma unroll
      for (int i = 0; i < PL; ++i) acc[i] += wgt * po[i];
    }
    const float inv = 1.f / den;
    bf16* orow = reinterpret_cast<bf16*>(a.o) + size_t(e * a.L + qr) * a.ldo + h * HD + lane * PL;
#pragma unroll
    for (int i = 0; i < PL; i += 2) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[i] * inv, acc[i + 1] * inv);
      *reinterpret_cast<__nv_bfloat162*>(orow + i) = b2;
    }
  }
}

// ------------------------------------------------------------------ host side
struct AttnPlan {
  PFN_encodeTiled encode = nullptr;
  int num_sms = 148;
  std::unordered_map<std::string, CUtensorMap> maps;
  bool ready = false;
};

inline bool tc_attn_enabled() { return true; }

// Stream-K (even tile split + merge) vs one CTA per unit: compare rounds of tiles,
// charging each unit boundary / merge about one tile of fixed cost.
inline int attn_pick_per_unit(long long units, long long tiles, int num_sms) {
  const long long J = units ? (tiles + units - 1) / units : 1;
  if (J <= 8) return 1;     // short key ranges (cross-attention): merge cost dominates
  const double per_unit = double((units + num_sms - 1) / num_sms) * double(J + 1);
  const double streamk = double((tiles + num_sms - 1) / num_sms) + 4.0;
  return per_unit <= streamk ? 1 : 0;
}

inline bool attn_plan_init(AttnPlan& p, PFN_encodeTiled enc, int num_sms) {
  p.encode = enc;
  p.num_sms = num_sms;
  cudaFuncSetAttribute(attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<128>::total);
  cudaFuncSetAttribute(attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<64>::total);
  p.ready = true;
  return true;
}

// Scratch for the partial units: [num_sms][2][128][hd] fp32 + [num_sms][2][128][2].
inline size_t attn_scratch_floats(int num_sms, int hd) {
  return size_t(num_sms) * 2 * kAttnBQ * hd + size_t(num_sms) * 2 * kAttnBQ * 2;
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

// q: [q_rows, d] bf16; K/V maps over whole buffers [kv_rows, d].  `total_tiles_hint`
// (host estimate of the unit x key-tile space) only sizes the grid: min(SMs, tiles).
inline bool tc_attention(cudaStream_t s, AttnPlan& p, const void* q, long long q_rows, const void* Kbase,
                         const void* Vbase, long long kv_rows, int d, int hd, long long total_tiles_hint,
                         const AttnTcArgs& a, const TickDesc* td, std::string* err, bool pdl = false) {
  const CUtensorMap* mq = attn_map(p, q, q_rows, d, kAttnBQ, err);
  const CUtensorMap* mk = attn_map(p, Kbase, kv_rows, d, kAttnBKV, err);
  const CUtensorMap* mv = attn_map(p, Vbase, kv_rows, d, kAttnBKV, err);
  if (!mq || !mk || !mv) return false;
  const int units = a.n_entries * a.H * a.QT;
  const int G = a.per_unit ? units : int(total_tiles_hint < p.num_sms ? total_tiles_hint : p.num_sms);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kAttnThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e;
  cfg.gridDim = dim3(G);
  cfg.dynamicSmemBytes = hd == 128 ? AttnSmem<128>::total : AttnSmem<64>::total;
  e = hd == 128 ? cudaLaunchKernelEx(&cfg, attn_tc_kernel<128>, *mq, *mk, *mv, a, td)
                : cudaLaunchKernelEx(&cfg, attn_tc_kernel<64>, *mq, *mk, *mv, a, td);
  if (e == cudaSuccess && !a.per_unit) {
    cfg.gridDim = dim3(units);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    e = hd == 128 ? cudaLaunchKernelEx(&cfg, attn_combine_kernel<128>, a, td, G)
                  : cudaLaunchKernelEx(&cfg, attn_combine_kernel<64>, a, td, G);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("attn_tc launch: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

}  // namespace sdv2
