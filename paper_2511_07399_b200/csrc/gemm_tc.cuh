// tcgen05 GEMM for the DiT projections:
//   C[M, N] = A[M, K] . W[N, K]^T + b, bf16 operands, fp32 accumulation in TMEM,
// fused epilogues (bf16 store / GELU-tanh / gated fp32 residual / fp32 residual).
//
// Design (B200-first): persistent CTAs (one per SM), warp-specialised:
//   warp 0      TMA producer (A box 64x128, W box 64xBN, 128-byte swizzle, 4-stage ring)
//   warp 1      MMA issuer: one thread issues tcgen05.mma M=128, N=BN, K=16
//   warp 2      TMEM allocator (2 accumulator buffers x BN columns)
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns -> epilogue -> global
// The accumulator is double-buffered in TMEM so the epilogue of tile i overlaps the
// MMAs of tile i+1.  BN is a runtime parameter (multiple of 32, <= 256) chosen per
// GEMM shape by the host to balance tiles over the 148 SMs (M = 1560 is awkward).
// The K reduction order is fixed (64-wide blocks, ascending), independent of M and
// of the tile shape, so results are batch invariant.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <string>
#include <algorithm>
#include <unordered_map>
#include <utility>
#include <vector>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace sdv2 {

constexpr int kGemmBM = 128, kGemmBK = 64, kGemmMaxStages = 8, kGemmMaxBN = 256;
constexpr int kGemmSmemA = kGemmBM * kGemmBK * 2;        // 16 KB
constexpr int kGemmSmem = 227 * 1024;                    // whole SM: as many stages as fit
// 4 control warps + kGemmEpiWG epilogue warpgroups (each drains every kGemmEpiWG-th
// 32-column chunk of the accumulator).  Measured on the 1.3B step (tools/ab.sh): 2
// warpgroups 451 fps, 3 (128-register cap) 446, 4 (96 registers, spills) 415.
#ifndef SDV2_GEMM_EPI_WG
#define SDV2_GEMM_EPI_WG 2
#endif
constexpr int kGemmEpiWG = SDV2_GEMM_EPI_WG;
constexpr int kGemmEpiThreads = 128 * kGemmEpiWG;
constexpr int kGemmThreads = 128 + kGemmEpiThreads;

// Stages of the TMA->MMA ring for a tile width: the ring must cover the L2/HBM latency
// (about 1-2 us) at the MMA rate, so use all of shared memory.
constexpr int kGemmEpiVec = 3 * kGemmMaxBN * 4 + 4 * kGemmEpiWG * 2048;   // bias + 2 gate vectors per tile, 2 KB store staging per epilogue warp
// BNl = W rows held per CTA (BN, or BN / 2 for a CTA pair).
__host__ __device__ inline int gemm_stages(int BN, bool res_tma, int BNl) {
  const int xs = res_tma ? BN * kGemmBM * 4 : 0;     // staged fp32 residual tile
  const int st = (kGemmSmem - 1024 - 512 - kGemmEpiVec - xs) / (kGemmSmemA + BNl * kGemmBK * 2);
  return st > kGemmMaxStages ? kGemmMaxStages : st;
}
// Residual epilogues (x += g (acc + b), x += acc + b): 1 = the epilogue stages only the
// update in shared memory and a TMA reduce-add applies it to x at L2 (no x tile fetched
// into shared memory, no read-modify-write there); 0 = x tile fetched, updated in shared
// memory, stored back.
#ifndef SDV2_GEMM_XRED
#define SDV2_GEMM_XRED 1
#endif
constexpr bool kGemmXRed = SDV2_GEMM_XRED != 0;
constexpr int kResMaxBN = 192;   // residual epilogues: keep >= 3 stages next to the x tile

// Pipeline trace (test hook): event `ev` of k-block / tile index `i` of CTA 0 and 1
// (CTA 1 at +4096): [i * 8 + ev], i < 512.
// CTA wall stamps (globaltimer ns, test hook): [8192 + cta * 4 + {0 entry, 1 set up,
// 2 first tile's accumulator complete (epilogue saw it), 3 exit}].
#define GEMM_CTA_STAMP(ev)                                                              \
  do {                                                                                  \
    if (ep.trace != nullptr && blockIdx.x < 1024) {                                     \
      unsigned long long t_;                                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
      ep.trace[8192 + blockIdx.x * 4 + (ev)] = (long long)t_;                           \
    }                                                                                   \
  } while (0)
#define GEMM_TRACE(ev, i)                                                               \
  do {                                                                                  \
    if (ep.trace != nullptr && blockIdx.x < 2 && (i) < 512)                             \
      ep.trace[blockIdx.x * 4096 + (i) * 8 + (ev)] = clock64();                         \
  } while (0)

// sbias: the chunk's 32 bias values (shared memory, staged per tile).  bf16 outputs go
// through a per-warp 2 KB staging buffer (XOR-swizzled 16 B granules, conflict-free)
// and leave as 8 rows x 64 B per store instruction instead of 32 scattered rows.
// Every lane of the warp must call it (rows >= M are computed but not stored).
template <int EPI, typename TOut>
__device__ __forceinline__ void gemm_epilogue_chunk(const EpiArgs& ep, int r, int M, int c0, int N,
                                                    const uint32_t (&v)[32], const float* sbias, uint4* stage,
                                                    int lane, int r_warp0) {
  if (c0 + 32 <= N) {
    float acc[32];
    const uint32_t sb = tc::smem_u32(sbias);
#pragma unroll
    for (int i = 0; i < 32; i += 4) {   // bias add on the packed f32x2 pipe
      const float4 b = tc::ld_shared_f4(sb + i * 4);
      const float2 s0 = __fadd2_rn(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), make_float2(b.x, b.y));
      const float2 s1 =
          __fadd2_rn(make_float2(__uint_as_float(v[i + 2]), __uint_as_float(v[i + 3])), make_float2(b.z, b.w));
      acc[i] = s0.x;
      acc[i + 1] = s0.y;
      acc[i + 2] = s1.x;
      acc[i + 3] = s1.y;
    }
    if (EPI == EPI_STORE || EPI == EPI_GELU || EPI == EPI_STORE_RSQ) {
      if constexpr (sizeof(TOut) == 2) {
        uint32_t pk[16];
        float ssq = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float2 a = make_float2(acc[2 * i], acc[2 * i + 1]);
          if (EPI == EPI_GELU && !(ep.dbg & 2)) a = gelu_tanh_fast2(a);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(a.x, a.y);
          pk[i] = *reinterpret_cast<uint32_t*>(&h2);
          if (EPI == EPI_STORE_RSQ) {   // of the stored (bf16) values, as the unfused RMS kernel read them
            const float2 b = __bfloat1622float2(h2);
            ssq += b.x * b.x + b.y * b.y;
          }
        }
        // one partial per (row, 32-column chunk), summed in fixed order by the consumer
        // (no atomics: the bits do not depend on the order CTAs finish)
        if (EPI == EPI_STORE_RSQ && r < M) ep.rowsq[size_t(r) * (N / 32) + c0 / 32] = ssq;
        if (ep.dbg & 8) {   // test hook: each thread stores its row segment directly
          if (r < M) {
            uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<TOut*>(ep.out) + size_t(r) * ep.ldo + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
          return;
        }
        const uint32_t st0 = tc::smem_u32(stage);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          tc::st_shared_v4(st0 + (lane * 4 + (j ^ ((lane >> 1) & 3))) * 16,
                           make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = i * 8 + (lane >> 2), seg = lane & 3;
          const uint4 w = tc::ld_shared_v4(st0 + (rr * 4 + (seg ^ ((rr >> 1) & 3))) * 16);
          if (r_warp0 + rr < M && !(ep.dbg & 1))
            *reinterpret_cast<uint4*>(reinterpret_cast<TOut*>(ep.out) + size_t(r_warp0 + rr) * ep.ldo + c0 + seg * 8) = w;
        }
        __syncwarp();
      } else {
        if (r < M) {
          TOut* o = reinterpret_cast<TOut*>(ep.out) + size_t(r) * ep.ldo + c0;
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = from_f<TOut>(EPI == EPI_GELU ? gelu_tanh(acc[i]) : acc[i]);
        }
      }
    } else if (r < M) {
      // Residual epilogues: issue every load (x row segment, gate vectors through the
      // read-only path) before the first store, so the 8 x 16 B round trips overlap
      // instead of serialising on possible aliasing between x and the gate pointers.
      float* x = reinterpret_cast<float*>(ep.out) + size_t(r) * ep.ldo + c0;
      float4 xv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) xv[i] = __ldcg(reinterpret_cast<const float4*>(x) + i);
      if (EPI == EPI_RES_GATE) {
        const int e = r / ep.L;
        const float4* gm = reinterpret_cast<const float4*>(ep.mod + ep.gate_row * N + c0);
        const float4* ge = reinterpret_cast<const float4*>(ep.e0 + size_t(e) * 6 * N + ep.gate_row * N + c0);
        float4 ga[8], gb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          ga[i] = __ldg(gm + i);
          gb[i] = __ldg(ge + i);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          xv[i].x += (ga[i].x + gb[i].x) * acc[4 * i];
          xv[i].y += (ga[i].y + gb[i].y) * acc[4 * i + 1];
          xv[i].z += (ga[i].z + gb[i].z) * acc[4 * i + 2];
          xv[i].w += (ga[i].w + gb[i].w) * acc[4 * i + 3];
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          xv[i].x += acc[4 * i];
          xv[i].y += acc[4 * i + 1];
          xv[i].z += acc[4 * i + 2];
          xv[i].w += acc[4 * i + 3];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) reinterpret_cast<float4*>(x)[i] = xv[i];
    }
  } else if (r < M) {
    for (int i = 0; i < 32; ++i)
      if (c0 + i < N) epi_store<TOut, EPI>(ep, r, c0 + i, N, __uint_as_float(v[i]));
  }
}

// Stream-K (sk = 1): the tiles x k-blocks iteration space is split evenly over the
// clusters (contiguous unit ranges), so M = 1560 shapes with few output tiles still keep
// every SM on full-width tiles.  A cluster whose range ends inside a tile writes that
// partial accumulator to its workspace slot and raises its flag; the cluster holding
// the tile's last k-block adds the earlier partials (ascending cluster order: a fixed,
// deterministic reduction order for a given shape) before the epilogue.  Each cluster
// walks its range from the END, so partials are produced first and consumed last.
struct GemmSk {
  int on;
  int x_late;     // residual epilogues, one tile per cluster: stage the x tile in the (then
                  // idle) operand ring after the last MMA instead of a dedicated buffer
  float* ws;      // [slot = cluster * MC + rank][BN / 32][8][128 rows][4] fp32 partials
  int* flags;     // [slot] 1 = partial ready (reset to 0 by its consumer)
};
constexpr int kGemmSkSlotFloats = kGemmMaxBN * kGemmBM;   // 128 KB per slot

struct GemmSeg {
  int t, kb0, kb1;   // tile, k-block range [kb0, kb1)
};
struct GemmSegIter {
  int sk, KB, tiles, cid, ncl, t_next;
  long long u0, cur;
  __device__ void init(int sk_, int KB_, int tiles_, int cid_, int ncl_) {
    sk = sk_;
    KB = KB_;
    tiles = tiles_;
    cid = cid_;
    ncl = ncl_;
    t_next = cid;
    const long long U = (long long)tiles * KB;
    u0 = U * cid / ncl;
    cur = U * (cid + 1) / ncl;
  }
  __device__ bool next(GemmSeg& g) {
    if (!sk) {
      if (t_next >= tiles) return false;
      g.t = t_next;
      g.kb0 = 0;
      g.kb1 = KB;
      t_next += ncl;
      return true;
    }
    if (cur <= u0) return false;
    const long long e = cur;
    const int t = int((e - 1) / KB);
    const long long ts = (long long)t * KB;
    const long long b = ts > u0 ? ts : u0;
    g.t = t;
    g.kb0 = int(b - ts);
    g.kb1 = int(e - ts);
    cur = b;
    return true;
  }
  // cluster whose range holds unit u (same split as init)
  __device__ int cluster_of(long long u) const {
    const long long U = (long long)tiles * KB;
    return int(((u + 1) * ncl + U - 1) / U) - 1;
  }
};

// MC = CTAs per cluster along M (1 or 2).  MC = 2 is a CTA pair (tcgen05 cta_group::2):
// the two CTAs hold consecutive m-blocks (A rows) and one half each of the BN W rows;
// the even CTA issues M = 256 MMAs that read both halves in place and accumulate 128
// rows into each CTA's TMEM.  Every SM then pulls 16 KB + BN * 64 B per k-block instead
// of 16 KB + BN * 128 B: the 128 x 256 single-CTA tile needs ~94 B/cycle/SM at the MMA
// rate, above the ~63-85 B/cycle/SM the L2 delivers (tools/ubench_tma), the pair ~62.
template <int EPI, typename TOut, int MC>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         const __grid_constant__ CUtensorMap tmX, int M, int N, int K,
                                                         int BN, EpiArgs ep, GemmSk sk) {
  // Residual epilogues stage the fp32 x tile in shared memory: TMA load issued as soon
  // as the epilogue warps reach the tile (overlapping the mainloop), in-place update,
  // TMA store.  128-byte swizzled 32-column boxes keep the row-per-thread smem accesses
  // conflict-light.
  constexpr bool kResTMA = (EPI == EPI_RES_GATE || EPI == EPI_RES);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int BNl = BN / MC;                  // W rows held by this CTA
  const bool x_late = kResTMA && sk.x_late;   // x tile lives in the operand ring (see GemmSk)
  const int kStages = gemm_stages(BN, kResTMA && !x_late, BNl);
  const int kSmemB = BNl * kGemmBK * 2;     // multiple of 1024 (BNl multiple of 16... 8 rows x 128 B)
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kGemmSmemA;
  uint8_t* sX = x_late ? smem : sB + kStages * kSmemB;   // [BN/32][128 rows][32 fp32], 16 KB per box
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kSmemB + (kResTMA && !x_late ? BN * kGemmBM * 4 : 0));
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* x_full = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_full + 1);
  float* sBias = reinterpret_cast<float*>(x_full + 2);   // [BN] bias, then [2][BN] gate sums
  float* sGate = sBias + kGemmMaxBN;
  uint4* sStage = reinterpret_cast<uint4*>(sGate + 2 * kGemmMaxBN);   // [epilogue warps][128] x 16 B

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + kGemmBM - 1) / kGemmBM, num_n = (N + BN - 1) / BN;
  const int num_mg = (num_m + MC - 1) / MC;                 // m-block groups (one per cluster tile)
  const int tiles = num_mg * num_n;
  const int kblocks = K / kGemmBK;
  const int cr = MC > 1 ? int(tc::cluster_ctarank()) : 0;
  const int cid = blockIdx.x / MC, ncl = gridDim.x / MC;
  const uint16_t mc_mask = uint16_t((1u << MC) - 1);
  GemmSegIter segs;
  segs.init(sk.on, kblocks, tiles, cid, ncl);
  if (threadIdx.x == 0) {
    GEMM_CTA_STAMP(0);
    pdl_trigger();
  }

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full + s, 1);        // pair: the even CTA's barrier counts both CTAs' bytes
      tc::mbar_init(empty + s, 1);       // pair: released by the even CTA's multicast commit
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(tfull + s, 1);
      tc::mbar_init(tempty + s, 4 * kGemmEpiWG * MC); // pair: both CTAs' epilogue warps free the accumulator
    }
    tc::mbar_init(x_full, 1);
    if (kResTMA) tc::tma_prefetch_desc(&tmX);
    tc::fence_barrier_init();
  }
  if (warp == 2) {
    if (MC > 1) tc::tmem_alloc_cg2(tmem_slot, 512);
    else tc::tmem_alloc(tmem_slot, 512);
  }
  tc::tc_fence_before();
  if (MC > 1) tc::cluster_sync();   // peer barriers initialised before any multicast
  else __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) GEMM_CTA_STAMP(1);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    {   // whole warp walks the loop; one elected lane issues (see tc::elect_one)
      int stage = 0;
      uint32_t phase = 0;
      // bytes landing on the stage's full barrier (pair: both CTAs' A and W halves)
      const uint32_t bytes = MC * (uint32_t(kGemmSmemA) + uint32_t(BNl) * kGemmBK * 2);
      auto load_a = [&](int st, int kb, int mb) {
        if (MC > 1)
          tc::tma_load_2d_cg2(sA + st * kGemmSmemA, &tmA, tc::mapa_shared(full + st, 0), kb * kGemmBK, mb * kGemmBM);
        else
          tc::tma_load_2d(sA + st * kGemmSmemA, &tmA, full + st, kb * kGemmBK, mb * kGemmBM);
      };
      auto load_w = [&](int st, int kb, int nb) {
        if (MC > 1)
          tc::tma_load_2d_cg2(sB + st * kSmemB, &tmB, tc::mapa_shared(full + st, 0), kb * kGemmBK,
                              nb * BN + cr * BNl);
        else
          tc::tma_load_2d(sB + st * kSmemB, &tmB, full + st, kb * kGemmBK, nb * BN);
      };
      // Weights never change: prefetch the first ring of W tiles before waiting for the
      // upstream kernel (PDL), then stream the activations.
      int pre = 0;
      GemmSegIter it = segs;
      GemmSeg g0;
      if (it.next(g0)) {
        const int nb0 = g0.t / num_mg;
        pre = g0.kb1 - g0.kb0 < kStages ? g0.kb1 - g0.kb0 : kStages;
        if (tc::elect_one()) {
          for (int i = 0; i < pre; ++i) {
            if (cr == 0) tc::mbar_expect_tx(full + i, bytes);   // pair: the even CTA counts both
            load_w(i, g0.kb0 + i, nb0);
          }
        }
        __syncwarp();
      }
      pdl_wait();
      int kg = 0;   // k-blocks loaded by this CTA (trace index)
      it = segs;
      GemmSeg g;
      while (it.next(g)) {
        const int t = g.t;
        const int mb = (t % num_mg) * MC + cr, nb = t / num_mg;
        for (int kb = g.kb0; kb < g.kb1; ++kb, ++kg) {
          if (pre > 0) {   // first tile, W already in flight for this stage
            if (tc::elect_one()) load_a(stage, kb, mb);
            --pre;
          } else {
            tc::mbar_wait(empty + stage, phase ^ 1);
            if (lane == 0) GEMM_TRACE(0, kg);
            if (tc::elect_one()) {
              if (cr == 0) tc::mbar_expect_tx(full + stage, bytes);
              load_a(stage, kb, mb);
              load_w(stage, kb, nb);
            }
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (cr == 0) {   // whole warp walks the loop; one elected lane issues (see tc::elect_one)
      const uint32_t idesc = tc::idesc_bf16(kGemmBM * MC, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int kg = 0, nt = 0;
      GemmSegIter it = segs;
      GemmSeg g;
      for (; it.next(g); ++nt) {
        tc::mbar_wait(tempty + acc, acc_phase ^ 1);
        if (lane == 0) GEMM_TRACE(2, nt);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(acc * BN);
        for (int kb = g.kb0; kb < g.kb1; ++kb, ++kg) {
          tc::mbar_wait(full + stage, phase);
          if (lane == 0) GEMM_TRACE(1, kg);
          tc::tc_fence_after();
          const uint32_t a0 = tc::smem_u32(sA + stage * kGemmSmemA);
          const uint32_t b0 = tc::smem_u32(sB + stage * kSmemB);
          if (tc::elect_one()) {
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k) {
              if (MC > 1)
                tc::mma_bf16_cg2(d_tmem, tc::sw128_kmajor_desc(a0 + k * 32), tc::sw128_kmajor_desc(b0 + k * 32), idesc,
                                 (kb - g.kb0 | k) != 0);
              else
                tc::mma_bf16(d_tmem, tc::sw128_kmajor_desc(a0 + k * 32), tc::sw128_kmajor_desc(b0 + k * 32), idesc,
                             (kb - g.kb0 | k) != 0);
            }
            if (MC > 1) tc::mma_commit_cg2_mc(empty + stage, mc_mask);
            else tc::mma_commit(empty + stage);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (tc::elect_one()) {
          if (MC > 1) tc::mma_commit_cg2_mc(tfull + acc, mc_mask);
          else tc::mma_commit(tfull + acc);
        }
        if (lane == 0) GEMM_TRACE(3, nt);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    pdl_wait();                         // epilogue reads x / gates produced upstream
    const int q = warp & 3;             // TMEM lane quarter accessible by this warp
    const int wg = (warp - 4) >> 2;     // epilogue warpgroup: 32-column chunks c % kGemmEpiWG == wg
    const bool leader = (warp == 4 && lane == 0);
    const int row = q * 32 + lane;      // row inside the tile
    int acc = 0;
    uint32_t acc_phase = 0;
    int nt = 0, nx = 0;                 // segments / residual tiles done by this CTA
    GemmSegIter it = segs;
    GemmSeg g;
    for (; it.next(g); ++nt) {
      const int t = g.t;
      const int mb = (t % num_mg) * MC + cr, nb = t / num_mg;
      const bool partial = g.kb1 < kblocks;        // stream-K: hand the partial sum on
      const bool fixup = !partial && g.kb0 > 0;    // stream-K: add the earlier partials
      const int c_first = fixup ? it.cluster_of((long long)t * kblocks) : cid;
      float* ws_mine = sk.ws + size_t(cid * MC + cr) * kGemmSkSlotFloats;
      if (kResTMA && !kGemmXRed && !x_late && !partial && leader) {   // fetch the residual tile while the MMAs run
        tc::mbar_expect_tx(x_full, uint32_t(BN) * kGemmBM * 4);
        for (int c = 0; c < BN; c += 32)
          tc::tma_load_2d(sX + (c / 32) * (kGemmBM * 128), &tmX, x_full, nb * BN + c, mb * kGemmBM);
      }
      // stage the tile's bias (and gate = mod + e0 rows of the tile's entries) in shared
      // memory while the MMAs run: the per-chunk loop then only waits on TMEM
      const int row0 = mb * kGemmBM;
      const int e_lo = (row0 < M ? row0 : M - 1) / ep.L;
      const int e_hi = ((row0 + kGemmBM - 1) < M ? row0 + kGemmBM - 1 : M - 1) / ep.L;
      const bool gate_smem = EPI == EPI_RES_GATE && e_hi <= e_lo + 1;
      asm volatile("bar.sync 3, %0;" ::"n"(kGemmEpiThreads) : "memory");   // previous tile's readers done
      for (int i = threadIdx.x - 128; i < (partial ? 0 : BN); i += kGemmEpiThreads) {
        const int col = nb * BN + i;
        const bool ok = col < N;
        sBias[i] = ok ? ep.bias[col] : 0.f;
        if (EPI == EPI_RES_GATE && gate_smem) {
          const float gm = ok ? ep.mod[ep.gate_row * N + col] : 0.f;
          sGate[i] = ok ? gm + ep.e0[size_t(e_lo) * 6 * N + ep.gate_row * N + col] : 0.f;
          if (e_hi > e_lo) sGate[kGemmMaxBN + i] = ok ? gm + ep.e0[size_t(e_hi) * 6 * N + ep.gate_row * N + col] : 0.f;
        }
      }
      if (fixup && threadIdx.x == 128) {   // earlier clusters' partials of this tile are ready
        for (int cc = c_first; cc < cid; ++cc) {
          const int* f = sk.flags + cc * MC + cr;
          int v = 0;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
          } while (v == 0);
        }
      }
      asm volatile("bar.sync 3, %0;" ::"n"(kGemmEpiThreads) : "memory");
      tc::mbar_wait(tfull + acc, acc_phase);
      if (warp == 4 && lane == 0) GEMM_TRACE(4, nt);
      if (warp == 4 && lane == 0 && nt == 0) GEMM_CTA_STAMP(2);
      tc::tc_fence_after();
      const int r = mb * kGemmBM + row;
      const float* gsm = sGate + ((r < M ? r : M - 1) / ep.L > e_lo ? kGemmMaxBN : 0);
      if (kResTMA && !kGemmXRed && x_late && !partial && leader) {   // last MMA done: the operand ring is free
        // (fetching each box earlier, as the last MMAs release the ring stages, measured
        // 1.3 % slower on the step: the x boxes then compete with the last operand loads)
        tc::mbar_expect_tx(x_full, uint32_t(BN) * kGemmBM * 4);
        for (int c = 0; c < BN; c += 32)
          tc::tma_load_2d(sX + (c / 32) * (kGemmBM * 128), &tmX, x_full, nb * BN + c, mb * kGemmBM);
      }
      if (kResTMA && !kGemmXRed && !partial) tc::mbar_wait(x_full, (nx++) & 1);
      const uint32_t tbase = tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
      auto chunk = [&](const uint32_t(&v0)[32], int c) {
        if (partial) {   // [chunk][j][row][4]: a warp stores 32 rows x 16 B contiguously
          float4* dst = reinterpret_cast<float4*>(ws_mine) + size_t(c / 32) * 8 * kGemmBM + row;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(dst + j * kGemmBM, make_float4(__uint_as_float(v0[4 * j]), __uint_as_float(v0[4 * j + 1]),
                                                  __uint_as_float(v0[4 * j + 2]), __uint_as_float(v0[4 * j + 3])));
          return;
        }
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = v0[i];
        if (fixup) {
          float a[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) a[i] = 0.f;
          for (int cc = c_first; cc < cid; ++cc) {   // partials in cluster (= k) order, then this tail
            const float4* src = reinterpret_cast<const float4*>(sk.ws + size_t(cc * MC + cr) * kGemmSkSlotFloats) +
                                size_t(c / 32) * 8 * kGemmBM + row;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 p = __ldcg(src + j * kGemmBM);
              a[4 * j] += p.x;
              a[4 * j + 1] += p.y;
              a[4 * j + 2] += p.z;
              a[4 * j + 3] += p.w;
            }
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(a[i] + __uint_as_float(v[i]));
        }
        const int c0 = nb * BN + c;
        if (kResTMA) {
          if (c0 + 32 <= N) {
            const uint32_t xrow = tc::smem_u32(sX + (c / 32) * (kGemmBM * 128) + (row >> 3) * 1024 + (row & 7) * 128);
            const uint32_t bias4 = tc::smem_u32(sBias + c), gs = tc::smem_u32(gsm + c);
            const float4* gm = reinterpret_cast<const float4*>(ep.mod + ep.gate_row * N + c0);
            const float4* ge =
                reinterpret_cast<const float4*>(ep.e0 + size_t(r < M ? r / ep.L : 0) * 6 * N + ep.gate_row * N + c0);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t px = xrow + ((u ^ (row & 7)) << 4);
              // x += g * (acc + b) on the packed f32x2 pipe (reduce-add: only the update is
              // staged, x stays zero here)
              const float4 xv = kGemmXRed ? make_float4(0.f, 0.f, 0.f, 0.f) : tc::ld_shared_f4(px);
              const float4 bb = tc::ld_shared_f4(bias4 + u * 16);
              float2 a01 = __fadd2_rn(make_float2(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1])),
                                      make_float2(bb.x, bb.y));
              float2 a23 = __fadd2_rn(make_float2(__uint_as_float(v[4 * u + 2]), __uint_as_float(v[4 * u + 3])),
                                      make_float2(bb.z, bb.w));
              float2 x01, x23;
              if (EPI == EPI_RES_GATE) {
                float4 g;
                if (gate_smem) {
                  g = tc::ld_shared_f4(gs + u * 16);
                } else {
                  const float4 ga = __ldg(gm + u), gb = __ldg(ge + u);
                  g = make_float4(ga.x + gb.x, ga.y + gb.y, ga.z + gb.z, ga.w + gb.w);
                }
                x01 = __ffma2_rn(make_float2(g.x, g.y), a01, make_float2(xv.x, xv.y));
                x23 = __ffma2_rn(make_float2(g.z, g.w), a23, make_float2(xv.z, xv.w));
              } else {
                x01 = __fadd2_rn(make_float2(xv.x, xv.y), a01);
                x23 = __fadd2_rn(make_float2(xv.z, xv.w), a23);
              }
              tc::st_shared_v4(px, make_uint4(__float_as_uint(x01.x), __float_as_uint(x01.y), __float_as_uint(x23.x),
                                              __float_as_uint(x23.y)));
            }
          }
        } else if (c0 < N) {
          gemm_epilogue_chunk<EPI, TOut>(ep, r, M, c0, N, v, sBias + c, sStage + (warp - 4) * 128, lane,
                                         mb * kGemmBM + q * 32);
        }
      };
      // two TMEM chunks in flight: the next 32 columns load while this chunk is processed
      // one 32-column TMEM load in flight per warp (keeping a second one in flight measured
      // no faster and costs the 32 registers a third epilogue warpgroup needs)
      constexpr int CS = 32 * kGemmEpiWG;   // column stride between this warpgroup's chunks
      for (int c = wg * 32; c < BN; c += CS) {
        uint32_t va[32];
        tc::tmem_ld32(tbase + c, va);
        tc::tmem_ld_wait_dep(va);
        if (warp == 4 && lane == 0 && c == 0) GEMM_TRACE(6, nt);
        chunk(va, c);
        if (warp == 4 && lane == 0 && c == 0) GEMM_TRACE(7, nt);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (MC > 1) tc::mbar_arrive_cluster(tc::mapa_shared(tempty + acc, 0));
        else tc::mbar_arrive(tempty + acc);
      }
      if (partial) {   // publish: every thread's stores, then one release of the flag
        __threadfence();
        asm volatile("bar.sync 3, %0;" ::"n"(kGemmEpiThreads) : "memory");
        if (threadIdx.x == 128)
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sk.flags + cid * MC + cr), "r"(1) : "memory");
      }
      if (fixup) {     // consumed: re-arm the contributors' flags for the next launch
        asm volatile("bar.sync 3, %0;" ::"n"(kGemmEpiThreads) : "memory");
        if (threadIdx.x == 128)
          for (int cc = c_first; cc < cid; ++cc) sk.flags[cc * MC + cr] = 0;
      }
      if (kResTMA && !partial) {
        tc::fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the TMA store
        asm volatile("bar.sync 2, %0;" ::"n"(kGemmEpiThreads) : "memory");
        if (leader) {
          for (int c = 0; c < BN; c += 32) {
            if (kGemmXRed) tc::tma_reduce_add_2d(&tmX, sX + (c / 32) * (kGemmBM * 128), nb * BN + c, mb * kGemmBM);
            else tc::tma_store_2d(&tmX, sX + (c / 32) * (kGemmBM * 128), nb * BN + c, mb * kGemmBM);
          }
          tc::tma_store_commit_wait_read();   // smem reusable for the next tile's load
        }
      }
      if (warp == 4 && lane == 0) GEMM_TRACE(5, nt);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (kResTMA && leader) tc::tma_store_wait_all();
  }
  tc::tc_fence_before();
  if (MC > 1) tc::cluster_sync();   // no CTA exits while its peer may still multicast into it
  else __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    if (MC > 1) tc::tmem_dealloc_cg2(tmem, 512);
    else tc::tmem_dealloc(tmem, 512);
  }
  if (threadIdx.x == 0) GEMM_CTA_STAMP(3);
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct GemmCfg {
  int MC, BN, SK;   // cluster size (1 or CTA pair), tile width, stream-K
  int XE = 0;       // residual epilogue with one tile per cluster: fetch the x tile into its
                    // own buffer while the MMAs run (fewer stages) instead of into the
                    // operand ring after the last MMA
};

struct TmaGemmPlan {
  PFN_encodeTiled encode = nullptr;
  int num_sms = 148;
  std::unordered_map<std::string, CUtensorMap> maps;
  std::unordered_map<std::string, GemmCfg> tuned;   // "M:N:K:epi" -> configuration
  float* sk_ws = nullptr;                           // stream-K partial slots [num_sms][128 KB]
  int* sk_flags = nullptr;                          // [num_sms], zero between launches
};

inline bool tc_gemm_enabled() { return true; }

template <int EPI, typename TOut, int MC>
inline void gemm_set_attr() {
  cudaFuncSetAttribute(gemm_tc_kernel<EPI, TOut, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem);
}

inline bool tc_gemm_plan(TmaGemmPlan& p, std::string* err) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  p.encode = reinterpret_cast<PFN_encodeTiled>(fn);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p.num_sms, cudaDevAttrMultiProcessorCount, dev);
  gemm_set_attr<EPI_STORE, bf16, 1>(); gemm_set_attr<EPI_STORE, bf16, 2>();
  gemm_set_attr<EPI_GELU, bf16, 1>(); gemm_set_attr<EPI_GELU, bf16, 2>();
  gemm_set_attr<EPI_RES_GATE, bf16, 1>(); gemm_set_attr<EPI_RES_GATE, bf16, 2>();
  gemm_set_attr<EPI_RES, bf16, 1>(); gemm_set_attr<EPI_RES, bf16, 2>();
  gemm_set_attr<EPI_STORE, float, 1>(); gemm_set_attr<EPI_STORE, float, 2>();
  gemm_set_attr<EPI_STORE_RSQ, bf16, 1>(); gemm_set_attr<EPI_STORE_RSQ, bf16, 2>();
  return true;
}

// 2D bf16 K-major tensor map [rows, K] with a (64 x box_rows) box, 128-byte swizzle.
inline bool tc_make_map(TmaGemmPlan& p, CUtensorMap* m, const void* ptr, int rows, int K, int box_rows,
                        std::string* err) {
  const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(K) * 2};
  const cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = p.encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")";
    return false;
  }
  return true;
}

// fp32 [rows, ld] residual map, 32-column x 128-row boxes, 128-byte swizzle.
inline const CUtensorMap* tc_map_res(TmaGemmPlan& p, const void* ptr, int rows, int cols, int ld, std::string* err) {
  const std::string key = "res:" + std::to_string(reinterpret_cast<uintptr_t>(ptr)) + ":" + std::to_string(rows) +
                          ":" + std::to_string(cols) + ":" + std::to_string(ld);
  auto it = p.maps.find(key);
  if (it != p.maps.end()) return &it->second;
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  const cuuint32_t box[2] = {32, uint32_t(kGemmBM)};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = p.encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (residual) failed (" + std::to_string(int(r)) + ")";
    return nullptr;
  }
  return &(p.maps.emplace(key, m).first->second);
}

inline const CUtensorMap* tc_map(TmaGemmPlan& p, const void* ptr, int rows, int K, int box_rows, std::string* err) {
  const std::string key = std::to_string(reinterpret_cast<uintptr_t>(ptr)) + ":" + std::to_string(rows) + ":" +
                          std::to_string(K) + ":" + std::to_string(box_rows);
  auto it = p.maps.find(key);
  if (it != p.maps.end()) return &it->second;
  CUtensorMap m;
  if (!tc_make_map(p, &m, ptr, rows, K, box_rows, err)) return nullptr;
  return &(p.maps.emplace(key, m).first->second);
}

// Tile width N chosen to balance (M/128/MC) x (N/BN) cluster tiles over the SMs:
// maximise useful-column fraction x useful-row fraction x wave efficiency.
inline int tc_pick_bn(int M, int N, int sms, int MC, int max_bn = 256) {
  const int num_m = (M + kGemmBM - 1) / kGemmBM;
  const int num_mg = (num_m + MC - 1) / MC;
  const int slots = sms / MC;
  int best = 256;
  double best_eff = -1.0;
  for (int bn = max_bn; bn >= 64; bn -= 32) {
    const int num_n = (N + bn - 1) / bn;
    const int tiles = num_mg * num_n;
    const int waves = (tiles + slots - 1) / slots;
    const double eff = double(N) / double(num_n * bn) * double(num_m) / double(num_mg * MC) * double(tiles) /
                       double(waves * slots);
    if (eff > best_eff + 1e-3) {   // prefer wider tiles on ties
      best_eff = eff;
      best = bn;
    }
  }
  return best;
}

// PDL for the projection GEMMs (set per call by the library; thread-local so the
// kernel-level test hook launches without it).
inline bool& gemm_pdl_flag() {
  static thread_local bool f = false;
  return f;
}

template <int EPI, typename TOut, int MC>
inline cudaError_t gemm_launch(cudaStream_t s, int grid, const CUtensorMap& ma, const CUtensorMap& mb,
                               const CUtensorMap& mx, int M, int N, int K, int BN, const EpiArgs& ep,
                               const GemmSk& sk) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = kGemmSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = gemm_pdl_flag() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<EPI, TOut, MC>, ma, mb, mx, M, N, K, BN, ep, sk);
}

template <int MC>
inline cudaError_t gemm_dispatch(cudaStream_t s, int grid, const CUtensorMap& ma, const CUtensorMap& mb,
                                 const CUtensorMap& mx, int M, int N, int K, int BN, int epi, const EpiArgs& ep,
                                 const GemmSk& sk) {
  switch (epi) {
    case EPI_STORE: return gemm_launch<EPI_STORE, bf16, MC>(s, grid, ma, mb, mx, M, N, K, BN, ep, sk);
    case EPI_GELU: return gemm_launch<EPI_GELU, bf16, MC>(s, grid, ma, mb, mx, M, N, K, BN, ep, sk);
    case EPI_RES_GATE: return gemm_launch<EPI_RES_GATE, bf16, MC>(s, grid, ma, mb, mx, M, N, K, BN, ep, sk);
    case EPI_STORE_F32: return gemm_launch<EPI_STORE, float, MC>(s, grid, ma, mb, mx, M, N, K, BN, ep, sk);
    case EPI_STORE_RSQ: return gemm_launch<EPI_STORE_RSQ, bf16, MC>(s, grid, ma, mb, mx, M, N, K, BN, ep, sk);
    default: return gemm_launch<EPI_RES, bf16, MC>(s, grid, ma, mb, mx, M, N, K, BN, ep, sk);
  }
}

inline std::string gemm_key(int M, int N, int K, int epi) {
  return std::to_string(M) + ":" + std::to_string(N) + ":" + std::to_string(K) + ":" + std::to_string(epi);
}

// One launch with an explicit (cluster size, tile width, stream-K) configuration.
inline bool tc_gemm_cfg(cudaStream_t s, TmaGemmPlan& p, const void* A, const void* W, int M, int N, int K, int epi,
                        const EpiArgs& ep, const GemmCfg& gc, std::string* err) {
  const int MC = gc.MC, BN = gc.BN;
  const int num_m = (M + kGemmBM - 1) / kGemmBM;
  const bool res = (epi == EPI_RES_GATE || epi == EPI_RES);
  const CUtensorMap* ma = tc_map(p, A, M, K, kGemmBM, err);
  const CUtensorMap* mb = tc_map(p, W, N, K, BN / MC, err);
  if (!ma || !mb) return false;
  const CUtensorMap* mx = res ? tc_map_res(p, ep.out, M, N, ep.ldo, err) : ma;
  if (!mx) return false;
  const int tiles = ((num_m + MC - 1) / MC) * ((N + BN - 1) / BN);
  const long long work = gc.SK ? (long long)tiles * (K / kGemmBK) : tiles;   // stream-K: tile x k-block units
  const int slots = p.num_sms / MC;
  const int grid = MC * int(work < slots ? work : slots);
  // residual x tile staged in the operand ring when no cluster gets a second tile
  if (gc.SK && (!p.sk_ws || !p.sk_flags)) {
    *err = "tc_gemm: stream-K needs the (test-hook) partial workspace";
    return false;
  }
  const GemmSk sk{gc.SK, (!gc.SK && !gc.XE && tiles <= slots) ? 1 : 0, p.sk_ws, p.sk_flags};
  cudaError_t e = MC == 2 ? gemm_dispatch<2>(s, grid, *ma, *mb, *mx, M, N, K, BN, epi, ep, sk)
                          : gemm_dispatch<1>(s, grid, *ma, *mb, *mx, M, N, K, BN, epi, ep, sk);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("gemm_tc launch: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

inline bool tc_gemm_check(int N, int K, int epi, std::string* err) {
  if (K % kGemmBK != 0 || N % 16 != 0) {
    *err = "tc_gemm: K % 64 or N % 16";
    return false;
  }
  if ((epi == EPI_RES_GATE || epi == EPI_RES) && N % 32 != 0) {
    *err = "tc_gemm: residual epilogue needs N % 32 == 0";
    return false;
  }
  return true;
}

// Default configuration from the tile-balance model (used when a shape was not tuned).
inline GemmCfg tc_gemm_default_cfg(const TmaGemmPlan& p, int M, int N, int epi) {
  const int num_m = (M + kGemmBM - 1) / kGemmBM;
  GemmCfg c;
  (void)num_m;
  c.MC = 1;
  c.SK = 0;
  const bool res = (epi == EPI_RES_GATE || epi == EPI_RES);
  const int max_bn = res ? kResMaxBN : 256;
  c.BN = c.SK ? std::min(max_bn, (N + 31) / 32 * 32) : tc_pick_bn(M, N, p.num_sms, c.MC, max_bn);
  return c;
}

inline bool tc_gemm(cudaStream_t s, TmaGemmPlan& p, const void* A, const void* W, int M, int N, int K, int epi,
                    const EpiArgs& ep, std::string* err, int a_rows_alloc = 0) {
  (void)a_rows_alloc;
  if (!tc_gemm_check(N, K, epi, err)) return false;
  auto it = p.tuned.find(gemm_key(M, N, K, epi));
  const GemmCfg gc = it != p.tuned.end() ? it->second : tc_gemm_default_cfg(p, M, N, epi);
  return tc_gemm_cfg(s, p, A, W, M, N, K, epi, ep, gc, err);
}

// Create-time autotuning of one GEMM shape on the real buffers: every (MC = 1, 2) x
// tile width (x early residual fetch), by CUDA-event time.  Every candidate reduces
// each output element over K in the same order (one CTA / CTA pair walks all k-blocks
// of its tile in order; no split-K), so the choice changes speed, never bits:
// tests/test_gpu_kernels.py::test_gemm_configs_bitwise_identical runs every candidate.
// Stream-K (ordered partial fix-up) changes the reduction order and is kept out of the
// product path (it was never the fastest at the DiT shapes).  The timed launches cycle through the weights of the different
// local blocks (Ws[0..nW)) so, as in a real step, the weights stream from HBM instead
// of sitting in L2 after the first launch.
// The configurations the tuner chooses from (also listed by the test hook).
inline std::vector<GemmCfg> tc_gemm_candidates(const TmaGemmPlan& p, int M, int N, int epi) {
  const int num_m = (M + kGemmBM - 1) / kGemmBM;
  const bool res = (epi == EPI_RES_GATE || epi == EPI_RES);
  std::vector<GemmCfg> cands;
  const int max_bn = std::min(res ? kResMaxBN : 256, (N + 31) / 32 * 32);
  for (int MC = 1; MC <= (num_m >= 2 ? 2 : 1); ++MC) {
    const int slots = p.num_sms / MC;
    for (int bn = max_bn; bn >= std::min(64, max_bn); bn -= 32) {   // narrow N (head): BN = 32
      cands.push_back({MC, bn, 0});
      if (res && ((num_m + MC - 1) / MC) * ((N + bn - 1) / bn) <= slots) cands.push_back({MC, bn, 0, 1});
    }
  }
  return cands;
}

inline bool tc_gemm_tune(cudaStream_t s, TmaGemmPlan& p, const void* A, const void* const* Ws, int nW, int M, int N,
                         int K, int epi, const EpiArgs& ep, std::string* err) {
  if (!tc_gemm_check(N, K, epi, err)) return false;
  const std::string key = gemm_key(M, N, K, epi);
  if (p.tuned.count(key)) return true;
  const std::vector<GemmCfg> cands = tc_gemm_candidates(p, M, N, epi);
  if (cands.empty()) {
    *err = "gemm tune: no candidate configuration";
    return false;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  GemmCfg best_cfg = cands.front();
  // each candidate: 8 launches replayed from a CUDA graph (device time only; a host
  // launch loop would be host-bound for the short M = 1560 GEMMs and rank noise)
  constexpr int kReps = 8;
  for (auto& c : cands) {
    for (int i = 0; i < 2; ++i)
      if (!tc_gemm_cfg(s, p, A, Ws[i % nW], M, N, K, epi, ep, c, err)) return false;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool ok = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    for (int i = 0; ok && i < kReps; ++i) ok = tc_gemm_cfg(s, p, A, Ws[i % nW], M, N, K, epi, ep, c, err);
    if (cudaStreamEndCapture(s, &graph) != cudaSuccess || !ok ||
        cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      *err = "gemm tune: graph capture failed";
      return false;
    }
    cudaGraphLaunch(exec, s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(exec, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (getenv("SDV2_VERBOSE") && atoi(getenv("SDV2_VERBOSE")) > 1)
      fprintf(stderr, "  cand MC=%d BN=%d SK=%d XE=%d %.1f us\n", c.MC, c.BN, c.SK, c.XE, ms * 1e3f / kReps);
    if (ms < best) {
      best = ms;
      best_cfg = c;
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  p.tuned[key] = best_cfg;
  if (getenv("SDV2_VERBOSE"))
    fprintf(stderr, "sdv2 gemm tune M=%d N=%d K=%d epi=%d -> MC=%d BN=%d SK=%d XE=%d (%.1f us)\n", M, N, K, epi,
            best_cfg.MC, best_cfg.BN, best_cfg.SK, best_cfg.XE, best * 1e3f / kReps);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace sdv2
