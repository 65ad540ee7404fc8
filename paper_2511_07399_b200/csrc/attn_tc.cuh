// tcgen05 attention of the chunk queries over the [sink || rolling window] KV lane
// (SURVEY.md §8(a) a7, P:183 FlashAttention-style O(BT) memory, P:472 rolling cache)
// and over the prompt K/V (a9 cross-attention).
//
// Work unit = (entry e, head h, 128-query tile).  Keys are one contiguous row range of
// the lane (valid slots are always a prefix, so no gather and no slot mask; only the
// ragged key tail is masked).  The (unit, 128-key tile) space is split evenly over
// exactly one CTA per SM ("stream-K"): a CTA owns a contiguous tile range, whole units
// in the middle and at most one piece of a unit at each end.  Ranges are walked from
// the end, so a unit shared by CTAs c' < c is first handed on by c' ((O, m, l) piece in
// a scratch slot + release flag) and last finished by c, which merges the pieces in CTA
// order (deterministic) and writes the output: no separate merge kernel.  This removes
// the wave quantisation of 156 units on 148 SMs (1.3B, 480p, n = 1).
//
// Per key tile t:  S_t = Q K_t^T (tcgen05.mma M=128 N=128 K=hd into one of 3 rotating
// TMEM slots) -> softmax (8 warps: TMEM lane quarter x key half; the two warps of a row
// agree on the row max each tile; exp2 on the MUFU plus a degree-3 polynomial on the
// FMA pipe; lazy rescale of O in TMEM when the max grows by > 2^8) -> P_t (bf16,
// written over S_t in TMEM) -> O += P_t V_t (tcgen05.mma, A from TMEM, V MN-major).
// Warp roles (352 threads): 0 TMA Q/K, 10 TMA V, 1 MMA issuer, 2..9 softmax / epilogue.
#pragma once
#include <string>
#include <unordered_map>

#include <cuda_fp16.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace sdv2 {

constexpr int kAttnBQ = 128, kAttnBKV = 128;

template <int HD, int CL = 1>
struct AttnSmem {
  static constexpr int Q = kAttnBQ * HD * 2;          // 32 KB (hd 128)
  static constexpr int KV = kAttnBKV * HD * 2 / CL;   // one K or V tile (CTA pair: this CTA's half)
  static constexpr int P = kAttnBQ * kAttnBKV * 2;    // 32 KB
  // K / V ring stages.  V is consumed a softmax later than K and its loads see ~2800
  // cycles of latency under load (tools/attn_trace.py): the deeper ring goes to V.
  // A CTA pair holds half of every K / V tile per CTA: twice the stages in the same space.
  static constexpr int KS = CL == 2 ? 4 : 2, VS = CL == 2 ? 4 : 3;
  static constexpr int total = Q + (KS + VS) * KV + 1024 + 256 + 768 * 4 + 64;
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
  float* part_o;       // [G][2 halves][HD/8 granules][128 rows][4] fp32 partial (unnormalised) O
  float* part_ml;      // [G][128][2] running max (log2 domain), sum
  int* flags;          // [G] partial ready (1), reset by the CTA that merges it
  int per_unit;        // 1: one CTA per unit (grid = units, no merge); 0: stream-K
  int rr;              // stream-K only: deal whole units round-robin first (R = units / CTAs
                       // full rounds), stream-K split only the tiles of the last partial round
  int dbg;             // test hook only (pipeline timing): bit 0 skips the softmax math,
                       // bit 1 the MMAs, bit 2 the K/V loads, bit 3 the PV MMAs, bit 4 the
                       // S MMAs; 0 in the product path
  long long* trace;    // test hook only: per-tile clock64 stamps of CTA 0 (nullptr = off)
};

// Pipeline trace (test hook): stamp event `ev` of local tile `t` (CTA 0, first 256 tiles).
#define ATTN_TRACE(ev, t)                                                  \
  do {                                                                     \
    if (a.trace != nullptr && blockIdx.x == 0 && lane == 0 && (t) < 256)   \
      a.trace[(t) * 16 + (ev)] = clock64();                                \
  } while (0)

// Stream-K geometry of the attention kernel.
struct AttnGeo {
  long long off[kMaxEntries + 1];   // tile offset of entry e's first unit
  int J[kMaxEntries];               // key tiles per unit of entry e
  long long T;                    // total tiles
  int QP;                         // query-tile groups per head (CL query tiles per group)
  long long ubase[kMaxEntries + 1]; // first unit of entry e
  long long Tr = 0;               // first tile of the stream-K split (after R whole rounds)
  int R = 0;                      // whole-unit rounds dealt round-robin
  __device__ void init(const AttnTcArgs& a, const TickDesc* td, int CL) {
    QP = (a.QT + CL - 1) / CL;
    off[0] = 0;
    for (int e = 0; e < kMaxEntries; ++e) {
      int j = 0;
      if (e < a.n_entries && td->e[e].active) {
        const int Lk = a.cross ? a.Lk_cross : td->e[e].nvalid * a.L;
        j = (Lk + kAttnBKV - 1) / kAttnBKV;
      }
      J[e] = j;
      off[e + 1] = off[e] + (long long)a.H * QP * j;
    }
    T = off[kMaxEntries];
    ubase[0] = 0;
    for (int e = 0; e < kMaxEntries; ++e) ubase[e + 1] = ubase[e] + (J[e] > 0 ? (long long)a.H * QP : 0);
  }
  // Hybrid schedule over G CTAs: R = units / G rounds of whole units (unit c + k G for CTA
  // c: the G concurrently running units are consecutive, so they share a few heads' K/V in
  // L2), then the tiles of the remaining units split evenly (stream-K).
  // One round is always left to the split, so the split covers >= G units: every CTA gets
  // a non-empty range (the merge waits on every CTA between a unit's first and last
  // owner) and a unit is cut into at most two pieces (cheap merges).
  __device__ void plan(bool rr, int G) {
    R = rr ? int(ubase[kMaxEntries] / G) - 1 : 0;
    if (R < 0) R = 0;
    Tr = R > 0 ? unit_lo((long long)R * G) : 0;
  }
  __device__ long long unit_lo(long long u) const {   // first tile of unit u (u <= units)
    int e = 0;
    while (e < kMaxEntries - 1 && u >= ubase[e + 1]) ++e;
    return u >= ubase[kMaxEntries] ? T : off[e] + (u - ubase[e]) * J[e];
  }
  // unit containing global tile g -> (e, unit-in-entry w, tile j)
  __device__ void locate(long long g, int& e, int& w, int& j) const {
    e = 0;
    while (e < kMaxEntries - 1 && g >= off[e + 1]) ++e;
    const long long r = g - off[e];
    w = int(r / J[e]);
    j = int(r % J[e]);
  }
  // stream-K split of the tiles [Tr, T)
  __device__ long long start(int c, int G) const { return Tr + ((T - Tr) * c) / G; }
  __device__ int cta_of(long long g, int G) const {
    const long long Ts = T - Tr;
    return int(((g - Tr + 1) * G + Ts - 1) / Ts) - 1;
  }
};

constexpr int kAttnThreads = 352;   // warp 0 TMA Q+K, 1 MMA, 2..9 softmax (two key halves), 10 TMA V

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Three-input max (sm_100 FMNMX3): the row-max pass in one instruction per two scores.
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2): two softmax elements per instruction.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2unpack(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for a pair on the FMA / ALU pipes instead of the MUFU (which would otherwise pace
// the softmax at one ex2 per element): x = n + f with n = rint(x) (magic-number add),
// 2^f on [-1/2, 1/2] by a degree-3 minimax polynomial (max rel. error 7.5e-5, far below
// the bf16 rounding of P), and n added into the exponent field.  x is clamped at -126 so
// the exponent never wraps; callers use it only on tiles with no masked (-inf) key.
__device__ __forceinline__ float2 ex2_poly2(uint64_t x2) {
  float2 x = f2unpack(x2);
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const uint64_t magic = f2pack(12582912.f, 12582912.f);   // 1.5 * 2^23
  const uint64_t xc = f2pack(x.x, x.y);
  const uint64_t t = fadd2(xc, magic);
  const uint64_t f = fsub2(xc, fsub2(t, magic));
  uint64_t p = ffma2(f2pack(0.0551716685f, 0.0551716685f), f, f2pack(0.242611155f, 0.242611155f));
  p = ffma2(p, f, f2pack(0.693260968f, 0.693260968f));
  p = ffma2(p, f, f2pack(0.999928057f, 0.999928057f));
  const float2 pv = f2unpack(p), tv = f2unpack(t);
  return make_float2(__uint_as_float(__float_as_uint(pv.x) + (__float_as_uint(tv.x) << 23)),
                     __uint_as_float(__float_as_uint(pv.y) + (__float_as_uint(tv.y) << 23)));
}

// Pairs i with bit (i % 8) set use the FMA-pipe polynomial: 0x44 = {2, 6}, 1/4 of them
// (0x00 / 0x44 / 0xA4 / 0xAA measured 87.3 / 84.7 / 85.5 / 84.4 us on the 1.3B self-attention)
#ifndef SDV2_ATTN_POLY_MASK
#define SDV2_ATTN_POLY_MASK 0x44
#endif
// P = 2^(s * scale - m) for one thread's HC scores -> bf16 pairs in pk, returns the row
// sum.  POLY: pairs with i % 8 in {2, 5, 7} (3/8) use ex2_poly2 instead of the MUFU.
template <int HC, bool POLY>
__device__ __forceinline__ float p_row(const float* sv, uint32_t* pk, uint64_t sc2, uint64_t nm2) {
  uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};   // packed row-sum chains (0.0f bits)
#pragma unroll
  for (int i = 0; i < HC / 2; ++i) {
    const uint64_t x2 = ffma2(f2pack(sv[2 * i], sv[2 * i + 1]), sc2, nm2);
    float2 pp;
    if (POLY && ((SDV2_ATTN_POLY_MASK >> (i & 7)) & 1)) {
      pp = ex2_poly2(x2);
    } else {
      const float2 x = f2unpack(x2);
      pp = make_float2(ex2(x.x), ex2(x.y));
    }
    acc[i & 3] = fadd2(acc[i & 3], f2pack(pp.x, pp.y));
    __nv_bfloat162 b2 = __floats2bfloat162_rn(pp.x, pp.y);
    pk[i] = *reinterpret_cast<uint32_t*>(&b2);
  }
  const float2 s01 = f2unpack(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
  return s01.x + s01.y;
}

// CL = CTAs per cluster along the query tiles of one head (1 or 2).  CL = 2 is a CTA
// pair (tcgen05 cta_group::2, head dim 128): the two CTAs take adjacent query tiles of
// one head and walk the same key tiles; each loads half of every K tile (64 keys) and
// half of every V tile (64 head-dim columns), and the even CTA issues M = 256 MMAs that
// read both halves in place.  Per SM the K/V stream halves (32 KB per 128 x 128 tile
// instead of 64 KB), so the loads stay ahead of the tensor pipe (tools/attn_trace.py
// showed single-CTA K/V loads queueing ~2.8-4.6k cycles).
template <int HD, int CL>
__global__ void __launch_bounds__(kAttnThreads, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                         const __grid_constant__ CUtensorMap tmK,
                                                         const __grid_constant__ CUtensorMap tmV, AttnTcArgs a,
                                                         const TickDesc* __restrict__ td) {
  static_assert(CL == 1 || HD == 128, "CTA-pair attention needs head dim 128");
  using SM = AttnSmem<HD, CL>;
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
  uint64_t* o_empty = bar + 2;   // O read out by the 8 softmax warps at a segment end
  // S / P TMEM buffers rotate over 3 slots (tile gt uses slot gt % 3, phase (gt / 3) & 1):
  // S_{t+2} is issued before PV_t, so the tensor pipe never waits on the softmax of the
  // tile it has just finished.  No waiter can fall two phases behind (S_{t+3} needs PV_t,
  // which needs P_t).
  uint64_t* s_full = bar + 3;    // [3] S ready (MMA commit)
  uint64_t* p_full = bar + 6;    // [3] P written (8 softmax warps)
  uint64_t* pv_done = bar + 9;   // [3] PV complete (MMA commit)
  uint64_t* k_full = bar + 12;       // [KS]
  uint64_t* k_empty = k_full + KS;   // [KS]
  uint64_t* v_full = k_empty + KS;   // [VS]
  uint64_t* v_empty = v_full + VS;   // [VS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + VS);
  float* xm = reinterpret_cast<float*>(bar + 32);   // [2 tile parity][2 halves][128] row-max exchange
  float* xl = xm + 512;                             // [2 halves][128] row-sum exchange at segment end

  // test hook: CTA-level wall stamps (globaltimer ns) [4096 + cta * 4 + {0 entry, 1 set up,
  // 2 first S issued, 3 exit}]
#define ATTN_CTA_STAMP(ev)                                                                  \
  do {                                                                                      \
    if (a.trace != nullptr && blockIdx.x < 1024) {                                          \
      unsigned long long t_;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
      a.trace[4096 + blockIdx.x * 4 + (ev)] = (long long)t_;                                \
    }                                                                                       \
  } while (0)
  if (threadIdx.x == 0) ATTN_CTA_STAMP(0);
  AttnGeo geo;
  geo.init(a, td, CL);
  const int G = gridDim.x / CL, c = blockIdx.x / CL;   // cluster (query-tile group) index
  const int cr = CL > 1 ? int(tc::cluster_ctarank()) : 0;
  const uint16_t mc_mask = uint16_t((1u << CL) - 1);
  long long t0, t1;
  if (a.per_unit) {
    const int e = c / (a.H * geo.QP), w = c % (a.H * geo.QP);
    if (e >= kMaxEntries || geo.J[e] == 0) return;
    t0 = geo.off[e] + (long long)w * geo.J[e];
    t1 = t0 + geo.J[e];
  } else {
    geo.plan(a.rr != 0, G);
    t0 = geo.start(c, G);
    t1 = geo.start(c + 1, G);
  }
  if (t0 >= t1 && geo.R == 0) return;
  // Work ranges of this CTA, each walked from its end: range 0 = its stream-K tile range,
  // ranges 1..R = its whole units c + (r - 1) G.  seg_before clamps to the current t0.
  const long long tail_lo = t0, tail_hi = t1;
  const int nrg = 1 + geo.R;
  auto range_of = [&](int rg, long long& lo, long long& hi) {
    if (rg == 0) {
      lo = tail_lo;
      hi = tail_hi;
    } else {
      const long long u = c + (long long)(rg - 1) * G;
      lo = geo.unit_lo(u);
      hi = geo.unit_lo(u + 1);
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    tc::mbar_init(o_empty, 8 * CL);      // pair: both CTAs' softmax warps (on the even CTA)
    for (int s = 0; s < KS; ++s) {
      tc::mbar_init(k_full + s, 1);
      tc::mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < VS; ++s) {
      tc::mbar_init(v_full + s, 1);
      tc::mbar_init(v_empty + s, 1);
    }
    for (int i = 0; i < 3; ++i) {
      tc::mbar_init(s_full + i, 1);
      tc::mbar_init(p_full + i, 8 * CL);
      tc::mbar_init(pv_done + i, 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0) {
    if (CL > 1) tc::tmem_alloc_cg2(tmem_slot, 512);
    else tc::tmem_alloc(tmem_slot, 512);
  }
  tc::tc_fence_before();
  if (CL > 1) tc::cluster_sync();   // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc::tc_fence_after();
  // Barrier init, descriptor prefetch and TMEM allocation above overlap the upstream
  // kernel's tail (PDL; the upstream is an element-wise kernel that holds no TMEM).
  pdl_wait();      // q, K/V lanes and o are produced / consumed by the neighbouring kernels
  pdl_trigger();
  if (threadIdx.x == 0) ATTN_CTA_STAMP(1);
  const uint32_t tmem = *tmem_slot;
  // TMEM: O (HD columns) | S0 | S1 | S2 (128 fp32 columns each, from column 128).  One O
  // accumulator per row: the two softmax warps of a row (key halves) agree on the row
  // max every tile through a shared-memory exchange.
  const uint32_t tO = tmem;
  auto tS = [&](int b) { return tmem + 128u + uint32_t(b) * 128u; };

  // Segment iteration: [gs, ge) of global tiles inside one unit.
  // Segment = the part of one unit inside [t0, t1).  Segments are visited from the END
  // of the range: a unit shared with the previous CTA (whose range ends inside it) is
  // then produced first over there and finished last here, where its pieces are merged.
  struct Seg {
    int e, h, q0, jb, je, J;
    long long gs, ustart;   // first global tile of the segment / of its unit
  };
  auto seg_before = [&](long long ge_) {   // segment ending at global tile ge_ (exclusive)
    Seg s;
    int w, j;
    geo.locate(ge_ - 1, s.e, w, j);
    s.h = w / geo.QP;
    s.q0 = ((w % geo.QP) * CL + cr) * kAttnBQ;
    s.J = geo.J[s.e];
    s.je = j + 1;
    s.ustart = ge_ - 1 - j;
    s.gs = s.ustart > t0 ? s.ustart : t0;
    s.jb = int(s.gs - s.ustart);
    return s;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    {   // whole warp walks the loop; one elected lane issues
      long long g = t1;
      int gi = 0, sg = 0;   // local tile counter, segment counter
      for (int rg = 0; rg < nrg; ++rg) {
        range_of(rg, t0, g);
        while (g > t0) {
          const Seg s = seg_before(g);
          const int col = s.h * HD;
          const int kv_row = a.kv_row0 + (a.cross ? td->e[s.e].xslot : s.e) * a.kv_lane_rows;
          if (sg > 0) tc::mbar_wait(q_empty, (sg - 1) & 1);
          if (tc::elect_one()) {
            if (CL > 1) {   // both CTAs' Q land on the even CTA's barrier
              if (cr == 0) tc::mbar_expect_tx(q_full, 2 * SM::Q);
              for (int ch = 0; ch < NCH; ++ch)
                tc::tma_load_2d_cg2(sQ + ch * (kAttnBQ * 128), &tmQ, tc::mapa_shared(q_full, 0), col + ch * 64,
                                    s.e * a.L + s.q0);
            } else {
              tc::mbar_expect_tx(q_full, SM::Q);
              for (int ch = 0; ch < NCH; ++ch)
                tc::tma_load_2d(sQ + ch * (kAttnBQ * 128), &tmQ, q_full, col + ch * 64, s.e * a.L + s.q0);
            }
          }
          __syncwarp();
          for (int j = s.jb; j < s.je; ++j, ++gi) {
            const int st = gi % KS;
            tc::mbar_wait(k_empty + st, ((gi / KS) & 1) ^ 1);
            ATTN_TRACE(8, gi);
            if (tc::elect_one()) {
              if (a.dbg & 4) {
                tc::mbar_arrive(k_full + st);
              } else if (CL > 1) {   // this CTA's 64 keys x 128 dims, counted on the even CTA
                if (cr == 0) tc::mbar_expect_tx(k_full + st, 2 * SM::KV);
                for (int ch = 0; ch < NCH; ++ch)
                  tc::tma_load_2d_cg2(sK + st * SM::KV + ch * (kAttnBKV / 2 * 128), &tmK, tc::mapa_shared(k_full + st, 0),
                                      col + ch * 64, kv_row + j * kAttnBKV + cr * (kAttnBKV / 2));
              } else {
                tc::mbar_expect_tx(k_full + st, SM::KV);
                for (int ch = 0; ch < NCH; ++ch)
                  tc::tma_load_2d(sK + st * SM::KV + ch * (kAttnBKV * 128), &tmK, k_full + st, col + ch * 64,
                                  kv_row + j * kAttnBKV);
              }
            }
            __syncwarp();
          }
          g = s.gs;
          ++sg;
        }
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ TMA producer (V)
    // V tiles are consumed one MMA phase later than K: an own producer keeps the K
    // prefetch from waiting on V slots.
    {
      long long g = t1;
      int gi = 0;
      for (int rg = 0; rg < nrg; ++rg) {
        range_of(rg, t0, g);
        while (g > t0) {
          const Seg s = seg_before(g);
          const int col = s.h * HD;
          const int kv_row = a.kv_row0 + (a.cross ? td->e[s.e].xslot : s.e) * a.kv_lane_rows;
          for (int j = s.jb; j < s.je; ++j, ++gi) {
            const int st = gi % VS;
            tc::mbar_wait(v_empty + st, ((gi / VS) & 1) ^ 1);
            ATTN_TRACE(9, gi);
            if (tc::elect_one()) {
              if (a.dbg & 4) {
                tc::mbar_arrive(v_full + st);
              } else if (CL > 1) {   // 128 keys x this CTA's 64 head-dim columns
                if (cr == 0) tc::mbar_expect_tx(v_full + st, 2 * SM::KV);
                tc::tma_load_2d_cg2(sV + st * SM::KV, &tmV, tc::mapa_shared(v_full + st, 0), col + cr * 64,
                                    kv_row + j * kAttnBKV);
              } else {
                tc::mbar_expect_tx(v_full + st, SM::KV);
                for (int ch = 0; ch < NCH; ++ch)
                  tc::tma_load_2d(sV + st * SM::KV + ch * (kAttnBKV * 128), &tmV, v_full + st, col + ch * 64,
                                  kv_row + j * kAttnBKV);
              }
            }
            __syncwarp();
          }
          g = s.gs;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (cr == 0) {   // whole warp walks the loop; one elected lane issues (see tc::elect_one)
      const uint32_t idS = tc::idesc_bf16(kAttnBQ * CL, kAttnBKV);
      const uint32_t idO = tc::idesc_bf16(kAttnBQ * CL, HD, true);
      const uint32_t qa = tc::smem_u32(sQ);
      auto commit = [&](uint64_t* bar) {   // pair: arrive on the barrier in both CTAs
        if (CL > 1) tc::mma_commit_cg2_mc(bar, mc_mask);
        else tc::mma_commit(bar);
      };
      auto issue_S = [&](int gg) {     // gg = local tile counter
        const int b = gg % 3;          // S / P TMEM slot: last read by PV_{gg-3}, issued earlier
        const int ks = gg % KS;        // K smem stage
        tc::mbar_wait(k_full + ks, (gg / KS) & 1);
        ATTN_TRACE(3, gg);
        if (gg == 0 && lane == 0) ATTN_CTA_STAMP(2);
        tc::tc_fence_after();
        const uint32_t ka = tc::smem_u32(sK + ks * SM::KV);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t off = (k >> 2) * (kAttnBQ * 128) + (k & 3) * 32;
            const uint32_t koff = (k >> 2) * (kAttnBKV / CL * 128) + (k & 3) * 32;
            if (!(a.dbg & 18)) {
              if (CL > 1)
                tc::mma_bf16_cg2(tS(b), tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + koff), idS, k > 0);
              else
                tc::mma_bf16(tS(b), tc::sw128_kmajor_desc(qa + off), tc::sw128_kmajor_desc(ka + koff), idS, k > 0);
            }
          }
          commit(k_empty + ks);
          commit(s_full + b);
        }
        __syncwarp();
      };
      long long g = t1;
      int gi = 0, sg = 0;
      for (int rg = 0; rg < nrg; ++rg) {
        range_of(rg, t0, g);
        while (g > t0) {
          const Seg s = seg_before(g);
          const int nt = s.je - s.jb;
          tc::mbar_wait(q_full, sg & 1);
          auto release_q = [&]() {   // last S of the segment issued: Q smem reusable once it lands
            if (tc::elect_one()) commit(q_empty);
            __syncwarp();
          };
          issue_S(gi);
          if (nt > 1) issue_S(gi + 1);
          if (nt <= 2) release_q();
          for (int t = 0; t < nt; ++t) {
            const int gt = gi + t;
            if (t + 2 < nt) {
              issue_S(gt + 2);
              if (t + 3 == nt) release_q();
            }
            tc::mbar_wait(v_full + (gt % VS), (gt / VS) & 1);
            ATTN_TRACE(0, gt);
            if (t == 0 && sg > 0) tc::mbar_wait(o_empty, (sg - 1) & 1);
            tc::mbar_wait(p_full + gt % 3, (gt / 3) & 1);
            ATTN_TRACE(1, gt);
            tc::tc_fence_after();
            const uint32_t va = tc::smem_u32(sV + (gt % VS) * SM::KV);
            if (tc::elect_one()) {
  #pragma unroll
              for (int k = 0; k < 8; ++k) {   // O += P V; A = P from TMEM (bf16 pairs, 8 columns per K=16):
                                              // keys 64h..64h+63 sit in slot columns [64h, 64h+32)
                if (!(a.dbg & 10)) {
                  if (CL > 1)   // B = this CTA's 64 head-dim columns of V (one 64-wide block)
                    tc::mma_bf16_ts_cg2(tO, tS(gt % 3) + (k >> 2) * 64 + (k & 3) * 8,
                                        tc::sw128_mnmajor_desc(va + k * 2048, kAttnBKV * 128), idO, (t | k) != 0);
                  else
                    tc::mma_bf16_ts(tO, tS(gt % 3) + (k >> 2) * 64 + (k & 3) * 8,
                                    tc::sw128_mnmajor_desc(va + k * 2048, kAttnBKV * 128), idO, (t | k) != 0);
                }
              }
              commit(v_empty + (gt % VS));
              commit(pv_done + gt % 3);
            }
            __syncwarp();
          }
          gi += nt;
          g = s.gs;
          ++sg;
        }
      }
    }
  } else if (warp <= 9) {
    // ------------------------------------------------ softmax / correction / epilogue
    // 8 warps: TMEM lane quarter = warp & 3 (row), key half = (warp - 2) / 4.  The two
    // warps of a row quarter (same SMSP) exchange their half-row maxima every tile.
    constexpr int HC = kAttnBKV / 2;            // S columns per thread
    constexpr int HO = HD / 2;                  // O columns per thread (rescale, epilogue)
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory"); };
    auto arrive_lead = [&](uint64_t* bar) {   // barriers the MMA issuer waits on live in the even CTA
      if (CL > 1) tc::mbar_arrive_cluster(tc::mapa_shared(bar, 0));
      else tc::mbar_arrive(bar);
    };
    long long g = t1;
    int gi = 0, sg = 0;
    for (int rg = 0; rg < nrg; ++rg) {
      range_of(rg, t0, g);
      while (g > t0) {
        const Seg s = seg_before(g);
        const int nt = s.je - s.jb;
        const int Lk = a.cross ? a.Lk_cross : td->e[s.e].nvalid * a.L;
        float m_used = -INFINITY;   // row max the current P / O are relative to (log2 domain)
        float l = 0.f;              // this half's share of the row sum
        for (int t = 0; t < nt; ++t) {
          const int gt = gi + t;
          const int b = gt % 3;
          tc::mbar_wait(s_full + b, (gt / 3) & 1);
          if (quarter == 0) ATTN_TRACE(4 + 2 * half, gt);
          tc::tc_fence_after();
          if (a.dbg & 1) {   // timing experiment: no softmax work, P = 0
            uint32_t z[32];
  #pragma unroll
            for (int i = 0; i < 32; ++i) z[i] = 0u;
            tc::tmem_st32(tS(b) + lane_off + half * HC, z);
            tc::tmem_st_wait();
            l = 1.f;
            m_used = 0.f;
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_lead(p_full + b);
            if (quarter == 0) ATTN_TRACE(5 + 2 * half, gt);
            continue;
          }
          float sv[HC];
          {
            uint32_t r[HC];
  #pragma unroll
            for (int cc = 0; cc < HC / 32; ++cc)
              tc::tmem_ld32(tS(b) + lane_off + half * HC + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
            tc::tmem_ld_wait();
  #pragma unroll
            for (int i = 0; i < HC; ++i) sv[i] = __uint_as_float(r[i]);
          }
          if (quarter == 0) ATTN_TRACE(10 + 2 * half, gt);
          const int kvalid = Lk - (s.jb + t) * kAttnBKV - half * HC;
          const bool full_tile = kvalid >= HC;
          if (!full_tile) {
  #pragma unroll
            for (int i = 0; i < HC; ++i) sv[i] = (i < kvalid) ? sv[i] : -INFINITY;
          }
          float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};   // 4 independent chains
  #pragma unroll
          for (int i = 0; i < HC; i += 8) {
  #pragma unroll
            for (int k = 0; k < 4; ++k) mq[k] = fmax3(mq[k], sv[i + 2 * k], sv[i + 2 * k + 1]);
          }
          float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * a.scale_log2;
          // row max over both key halves (both warps then take the same rescale decision)
          xm[((gt & 1) * 2 + half) * 128 + row] = mx;
          pair_sync();
          mx = fmaxf(mx, xm[((gt & 1) * 2 + (half ^ 1)) * 128 + row]);
          if (quarter == 0) ATTN_TRACE(11 + 2 * half, gt);
          // lazy rescale: P / O stay relative to m_used until the max grows by > 2^8.  The
          // decision is WARP-UNIFORM: the TMEM accesses below are .sync.aligned (every lane of
          // the warp must execute them), so when any row of the warp needs it, every row
          // rescales to max(m_used, mx) (alpha = 1 for a row whose max did not grow).  The two
          // key-half warps of a row quarter hold the same rows and exchanged maxima, so they
          // take the same decision.  (A per-row branch here hung the kernel when the rows of
          // one warp disagreed: found on a 10k-chunk long-horizon run.)
          if (__any_sync(0xffffffffu, mx > m_used + 8.f)) {
            const float m_new = fmaxf(m_used, mx);
            if (t > 0) {     // O row (this half's HD/2 columns) *= 2^(m_used - m_new) once PV_{t-1} landed
              tc::mbar_wait(pv_done + (gt - 1) % 3, ((gt - 1) / 3) & 1);
              tc::tc_fence_after();
              const float alpha = m_used == -INFINITY ? 0.f : ex2(m_used - m_new);
              l *= alpha;
  #pragma unroll
              for (int cc = 0; cc < HO / 16; ++cc) {
                uint32_t r[16];
                const uint32_t ta = tO + lane_off + half * HO + cc * 16;
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
          // P = exp2(s * scale - m_used) -> bf16 pairs over this half's own S columns (A
          // operand of the PV MMA); a row with no valid key yet writes P = 0
          const float msub = m_used == -INFINITY ? 0.f : m_used;
          const uint64_t sc2 = f2pack(a.scale_log2, a.scale_log2), nm2 = f2pack(-msub, -msub);
          uint32_t pk[HC / 2];
          // full tiles move a share of the exponentials to the FMA pipe (the MUFU alone would
          // need 8 cycles per warp instruction x 64 per half-row: the MMA time of a tile)
          const float rs = full_tile ? p_row<HC, true>(sv, pk, sc2, nm2) : p_row<HC, false>(sv, pk, sc2, nm2);
          tc::tmem_st32(tS(b) + lane_off + half * HC, pk);
          tc::tmem_st_wait();
          l += rs;
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_lead(p_full + b);
          if (quarter == 0) ATTN_TRACE(5 + 2 * half, gt);
        }
        // end of segment: last PV landed -> O / (l_half0 + l_half1), this half's columns
        const int gl = gi + nt - 1;   // last tile of the segment
        xl[half * 128 + row] = l;
        tc::mbar_wait(pv_done + gl % 3, (gl / 3) & 1);
        tc::tc_fence_after();
        pair_sync();
        const float lt = l + xl[(half ^ 1) * 128 + row];
        const bool partial = s.je < s.J;               // head / middle piece of a unit: hand on
        const bool finisher = !partial && s.jb > 0;    // tail piece: merge the earlier pieces
        const int slot = c * CL + cr;
        const int qr = s.q0 + row;
        // partial layout [slot][half][granule j][row][4]: a warp moves 32 rows x 16 B at once
        auto part_at = [&](int sl, int j) {
          return reinterpret_cast<float4*>(a.part_o) + (size_t(sl * 2 + half) * (HO / 4) + j) * kAttnBQ + row;
        };
        int c_first = c;
        float wown = 1.f, den = lt, Mfin = m_used;
        if (finisher) {   // pieces of this unit from CTAs c_first .. c-1 (their first-visited segment)
          c_first = geo.cta_of(s.ustart, G);
          if (warp == 2 && lane == 0) {
            for (int cc = c_first; cc < c; ++cc) {
              const int* f = a.flags + cc * CL + cr;
              int v = 0;
              do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
              } while (v == 0);
            }
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          float M = m_used;
          for (int cc = c_first; cc < c; ++cc) M = fmaxf(M, __ldcg(a.part_ml + (size_t(cc * CL + cr) * kAttnBQ + row) * 2));
          Mfin = M;
          wown = m_used == -INFINITY ? 0.f : ex2(m_used - M);
          den = lt * wown;
          for (int cc = c_first; cc < c; ++cc) {
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(a.part_ml) + size_t(cc * CL + cr) * kAttnBQ + row);
            den += (ml.x == -INFINITY ? 0.f : ex2(ml.x - M)) * ml.y;
          }
        }
        const float inv = partial ? 1.f : 1.f / den;
        bf16* orow = reinterpret_cast<bf16*>(a.o) + size_t(s.e * a.L + qr) * a.ldo + s.h * HD + half * HO;
  #pragma unroll
        for (int cc = 0; cc < HO / 32; ++cc) {
          uint32_t r0[32];
          tc::tmem_ld32(tO + lane_off + half * HO + cc * 32, r0);
          tc::tmem_ld_wait();
          float o[32];
          if (partial) {
  #pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              __stcg(part_at(slot, cc * 8 + jj), make_float4(__uint_as_float(r0[4 * jj]), __uint_as_float(r0[4 * jj + 1]),
                                                            __uint_as_float(r0[4 * jj + 2]),
                                                            __uint_as_float(r0[4 * jj + 3])));
            continue;
          }
  #pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r0[i]) * wown;
          if (finisher) {
            const float M = Mfin;
            for (int k = c_first; k < c; ++k) {
              const float mk = __ldcg(a.part_ml + (size_t(k * CL + cr) * kAttnBQ + row) * 2);
              const float wk = mk == -INFINITY ? 0.f : ex2(mk - M);
  #pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const float4 p4 = __ldcg(part_at(k * CL + cr, cc * 8 + jj));
                o[4 * jj] += wk * p4.x;
                o[4 * jj + 1] += wk * p4.y;
                o[4 * jj + 2] += wk * p4.z;
                o[4 * jj + 3] += wk * p4.w;
              }
            }
          }
          if (qr < a.L) {
            uint32_t pk[16];
  #pragma unroll
            for (int i = 0; i < 16; ++i) {
              __nv_bfloat162 b2 = __floats2bfloat162_rn(o[2 * i] * inv, o[2 * i + 1] * inv);
              pk[i] = *reinterpret_cast<uint32_t*>(&b2);
            }
  #pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(orow + cc * 32)[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
        if (partial) {   // publish the piece: (m, l) of the row, then one release of the flag
          if (half == 0) __stcg(reinterpret_cast<float2*>(a.part_ml) + size_t(slot) * kAttnBQ + row, make_float2(m_used, lt));
          __threadfence();
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (warp == 2 && lane == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(a.flags + slot), "r"(1) : "memory");
        }
        if (finisher) {   // merged: re-arm the contributors' flags for the next launch
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (warp == 2 && lane == 0)
            for (int cc = c_first; cc < c; ++cc) a.flags[cc * CL + cr] = 0;
        }
        tc::tc_fence_before();
        pair_sync();   // xl reusable
        if (lane == 0) arrive_lead(o_empty);
        gi += nt;
        g = s.gs;
        ++sg;
      }
    }
  }
  tc::tc_fence_before();
  if (CL > 1) tc::cluster_sync();   // no CTA exits while its peer may still multicast into it
  else __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    if (CL > 1) tc::tmem_dealloc_cg2(tmem, 512);
    else tc::tmem_dealloc(tmem, 512);
  }
  if (threadIdx.x == 0) ATTN_CTA_STAMP(3);
}

// ------------------------------------------------------------------ host side
struct AttnPlan {
  PFN_encodeTiled encode = nullptr;
  int num_sms = 148;
  std::unordered_map<std::string, CUtensorMap> maps;
  bool ready = false;
  int* flags = nullptr;   // [num_sms] split-unit hand-off flags (zero between launches)
};

inline bool tc_attn_enabled() { return true; }

// Stream-K (even tile split, in-kernel merge of split units) vs one CTA per unit: one
// CTA per unit whenever the units fit in one wave (nothing to merge), else stream-K
// (measured: 156 cross-attention units of 4 key tiles 19.1 us stream-K vs 20.6 us in
// two waves; self-attention 86 vs 135 us).
inline int attn_pick_per_unit(long long units, long long tiles, int num_sms) {
  (void)tiles;
  return units <= num_sms ? 1 : 0;
}

// Hybrid stream-K (whole units round-robin, then an even split of the last partial
// round) is the schedule; rr = 0 (the plain even split of all tiles) stays reachable
// through the kernel-level test hook only.
constexpr int kAttnRR = 1;
inline int attn_rr() { return kAttnRR; }

// CTA-pair attention (cluster 2) was measured neutral at the 1.3B shapes and slower at
// 14B (84 vs 57 ms/step): single-CTA units.
constexpr int kAttnCluster = 1;
inline int attn_cluster() { return kAttnCluster; }

// flags: [num_sms] ints of caller-owned device memory (the handle carves them from
// its workspace and zeroes them once; the kernel leaves them zero after every launch).
inline bool attn_plan_init(AttnPlan& p, PFN_encodeTiled enc, int num_sms, int* flags) {
  p.encode = enc;
  p.num_sms = num_sms;
  if (!flags) return false;
  if (cudaFuncSetAttribute(attn_tc_kernel<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<128>::total) != cudaSuccess ||
      cudaFuncSetAttribute(attn_tc_kernel<64, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<64>::total) != cudaSuccess ||
      cudaFuncSetAttribute(attn_tc_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<128, 2>::total) != cudaSuccess)
    return false;
  p.flags = flags;
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
                         const AttnTcArgs& a_in, const TickDesc* td, std::string* err, bool pdl = false) {
  AttnTcArgs a = a_in;
  a.flags = p.flags;
  const CUtensorMap* mq = attn_map(p, q, q_rows, d, kAttnBQ, err);
  const int CL = hd == 128 ? attn_cluster() : 1;
  // pair: K boxes of 64 keys x 64 dims, V boxes of 128 keys x 64 dims (one half each)
  const CUtensorMap* mk = attn_map(p, Kbase, kv_rows, d, kAttnBKV / CL, err);
  const CUtensorMap* mv = attn_map(p, Vbase, kv_rows, d, kAttnBKV, err);
  if (!mq || !mk || !mv) return false;
  const int QP = (a.QT + CL - 1) / CL;
  const long long units = (long long)a.n_entries * a.H * QP;                   // query-tile groups
  const long long tiles = total_tiles_hint * QP / (a.QT > 0 ? a.QT : 1);       // group x key tiles
  const int slots = p.num_sms / CL;
  const int G = a.per_unit ? int(units) : int(tiles < slots ? tiles : slots);  // clusters
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kAttnThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e;
  cfg.gridDim = dim3(G * CL);
  cfg.dynamicSmemBytes = CL == 2 ? AttnSmem<128, 2>::total : hd == 128 ? AttnSmem<128>::total : AttnSmem<64>::total;
  if (CL == 2)
    e = hd == 128 ? cudaLaunchKernelEx(&cfg, attn_tc_kernel<128, 2>, *mq, *mk, *mv, a, td)
                  : cudaErrorInvalidValue;
  else
    e = hd == 128 ? cudaLaunchKernelEx(&cfg, attn_tc_kernel<128, 1>, *mq, *mk, *mv, a, td)
                  : cudaLaunchKernelEx(&cfg, attn_tc_kernel<64, 1>, *mq, *mk, *mv, a, td);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("attn_tc launch: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

}  // namespace sdv2
