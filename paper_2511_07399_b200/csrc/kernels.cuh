// Fused elementwise kernels and fp32-SIMT parity kernels of the hot path.
//
// Every kernel cites the model-card step it implements (SURVEY.md §8(c) C.1–C.8,
// stream algorithm O3–O5) and through it the paper passage.  Activation type TA is
// float (fp32 parity path) or bf16 (tensor-core path); the residual stream x,
// latents, sigma and time embeddings are fp32 on both paths (reading R8/Q29).
#pragma once
#include <type_traits>

#include "common.cuh"
#include "ctl.h"

namespace sdv2 {

// ----------------------------------------------------------------------------
// Motion-aware noise controller + step-0 blend (O4), rank 0, 1 CTA.
// ----------------------------------------------------------------------------
struct CtrlState {
  double ds[64];        // last motion values (ring, index nd % 64)
  long long nd;         // number of d values pushed
  double s;             // s_{X-1} before admission, s_X after
  double d_hat;
  double s_table[64];   // s_X for X % 64 (sigma of later steps, R5)
  int has_prev;
  int pad;
};

struct StreamCfg {
  float t[kMaxSteps];   // timesteps
  int n;                // steps
  int k;                // motion window k (k+1 values)
  float sigma_m, s_min, s_max, lam;
  unsigned long long seed;
};

__device__ __forceinline__ float sigma_of(const CtrlState* st, const StreamCfg& cfg, int X, int j) {
  // sigma_{X,j} = s_X * t_j / t_0 in fp64, rounded once to fp32 (R5)
  return float(st->s_table[X & 63] * double(cfg.t[j]) / double(cfg.t[0]));
}

// Sigma of every entry on ranks that do not run the controller is carried in the
// packet; rank 0 also needs the ring-closure latents assembled: entry e >= B (step j >= 1
// of stream e % B) continues ring slot e - B of the previous micro-step.
__global__ void assemble_kernel(const float* __restrict__ ring_in, float* __restrict__ lat, const TickDesc* td,
                                int n_entries, int B, int CTHW) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.y + B;
  if (e >= n_entries || !td->e[e].active) return;
  const float4* src = reinterpret_cast<const float4*>(ring_in + size_t(e - B) * CTHW);
  float4* dst = reinterpret_cast<float4*>(lat + size_t(e) * CTHW);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < CTHW / 4; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// ----------------------------------------------------------------------------
// Time conditioning (C.2): sinusoid(1000 sigma) in fp64, then GEMVs.
// ----------------------------------------------------------------------------
__global__ void sinusoid_kernel(const float* __restrict__ sig, float* __restrict__ emb, int n, int dim) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.x;
  const int half = dim / 2;
  const double t = 1000.0 * double(sig[e]);
  for (int k = threadIdx.x; k < half; k += blockDim.x) {
    const double arg = t * pow(10000.0, -double(k) / double(half));
    emb[e * dim + k] = float(cos(arg));
    emb[e * dim + half + k] = float(sin(arg));
  }
}

// y = g * y / sqrt(mean(y^2) + eps) over the full row (C.4 RMS_g; cross-attention q and
// prompt K).  One warp per row.
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(256) rms_rows_kernel(const TIn* __restrict__ y, TOut* __restrict__ out,
                                                       const float* __restrict__ g, int rows, int d, int ld_in,
                                                       float eps) {
  pdl_wait();
  pdl_trigger();
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const TIn* yr = y + size_t(r) * ld_in;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = to_f(yr[c]);
    ss += v * v;
  }
  const float inv = rsqrtf(warp_sum(ss) / float(d) + eps);
  for (int c = lane; c < d; c += 32) out[size_t(r) * d + c] = from_f<TOut>(g[c] * to_f(yr[c]) * inv);
}

// ----------------------------------------------------------------------------
// q/k RMSNorm + 3D RoPE + KV lane write (+ sink refresh copy) (C.5 steps 2–4, C.6,
// O3).  Row r = entry e (lane j = e) token tau.  Reads qkv [rows, 3d]; writes q~ to
// qout [rows, d]; k~ and v to the lane's write slot; for each refreshed sink i also
// k~ at the sink's anchor temporal positions i T' + f and v, into slot i.
// RoPE: interleaved pairs; per head the first ct pairs are temporal, then ch height,
// then cw width; cos/sin tables come from fp64 on the host.
// ----------------------------------------------------------------------------
struct RopeTabs {
  const float* ct_cos; const float* ct_sin;   // [(2 T_off + 1)][ct], row = pos + T_off
  const float* ch_cos; const float* ch_sin;   // [hn][ch]
  const float* cw_cos; const float* cw_sin;   // [wn][cw]
  int ct, ch, cw, t_off;
};

__device__ __forceinline__ void rope_cs(const RopeTabs& R, int pair, int pt, int ph, int pw, float& c, float& s) {
  if (pair < R.ct) {
    c = R.ct_cos[(pt + R.t_off) * R.ct + pair];
    s = R.ct_sin[(pt + R.t_off) * R.ct + pair];
  } else if (pair < R.ct + R.ch) {
    c = R.ch_cos[ph * R.ch + pair - R.ct];
    s = R.ch_sin[ph * R.ch + pair - R.ct];
  } else {
    c = R.cw_cos[pw * R.cw + pair - R.ct - R.ch];
    s = R.cw_sin[pw * R.cw + pair - R.ct - R.ch];
  }
}

// RoPE phase re-base (R3): every ring slot of a re-basing lane, in every local
// block, is rotated on its temporal pairs by R(-T_reset).  Grid: (token-rows, lane);
// n = lanes per block (B n).
template <typename TA>
__global__ void __launch_bounds__(256) rebase_kernel(TA* __restrict__ K, const TickDesc* __restrict__ td, RopeTabs R,
                                                     int nblocks, int n, int S, int m, int W, int L, int d, int hd,
                                                     int T_reset) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.y;
  if (!td->e[j].active || !td->e[j].rebase) return;
  const size_t rows = size_t(nblocks) * W * L;
  const int half = hd / 2;
  for (size_t row = blockIdx.x * 8 + (threadIdx.x >> 5); row < rows; row += size_t(gridDim.x) * 8) {
    const int b = int(row / (size_t(W) * L));
    const int rem = int(row % (size_t(W) * L));
    const int s = m + rem / L, tau = rem % L;
    TA* kr = K + ((((size_t(b) * n + j) * S + s) * L) + tau) * d;
    for (int p = threadIdx.x & 31; p < d / 2; p += 32) {
      const int pair = p % half;
      if (pair >= R.ct) continue;
      const float cs = R.ct_cos[(-T_reset + R.t_off) * R.ct + pair];
      const float sn = R.ct_sin[(-T_reset + R.t_off) * R.ct + pair];
      const float k0 = to_f(kr[2 * p]), k1 = to_f(kr[2 * p + 1]);
      kr[2 * p] = from_f<TA>(k0 * cs - k1 * sn);
      kr[2 * p + 1] = from_f<TA>(k0 * sn + k1 * cs);
    }
  }
}

// ----------------------------------------------------------------------------
// fp32-SIMT GEMM with the hot-path epilogues: C = A W^T + b.
//   EPI_STORE: out (TOut) = acc + b
//   EPI_GELU:  out (TOut) = GELU_tanh(acc + b)                       (FFN1, C.4)
//   EPI_RES_GATE: x[r,c] += (mod[g][c] + e0[e][g][c]) (acc + b)        (O / FFN2, C.5 5/8)
//   EPI_RES:   x[r,c] += acc + b                                       (cross-O, C.5 7)
// 64x64 tile, 256 threads (4x4 each), BK = 16.
// ----------------------------------------------------------------------------
enum { EPI_STORE = 0, EPI_GELU = 1, EPI_RES_GATE = 2, EPI_RES = 3, EPI_STORE_F32 = 4, EPI_STORE_RSQ = 5 };

struct EpiArgs {
  void* out;            // TOut* (STORE/GELU) or float* x (RES*)
  int ldo;
  const float* bias;
  const float* mod;     // block modulation [6, d] (RES_GATE)
  const float* e0;      // [n, 6, d] (RES_GATE)
  int gate_row;         // 2 (g1) or 5 (g2)
  int L;                // rows per entry
  float* rowsq;         // EPI_STORE_RSQ: [M][N / 32] sums of squares of the stored bf16 row, per 32 columns
  long long* trace;     // test hook only (tc GEMM): clock64 stamps of CTA 0 / 1, nullptr = off
  int dbg;              // test hook only (tc GEMM epilogue timing): bit 0 no global stores,
                        // bit 1 no GELU, bit 2 one TMEM load in flight; 0 in the product path
};

__device__ __forceinline__ float gelu_tanh(float z) {
  return 0.5f * z * (1.f + tanhf(0.7978845608028654f * (z + 0.044715f * z * z * z)));
}
// bf16-output variant: tanh.approx (MUFU, rel. error ~2^-11, below the bf16 rounding)
__device__ __forceinline__ float gelu_tanh_fast(float z) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.7978845608028654f * (z + 0.044715f * z * z * z)));
  return 0.5f * z * (1.f + t);
}

// Packed pair variant (sm_100 f32x2 FMA pipe): 0.5 z (1 + tanh(z (c + 0.044715 c z^2))).
__device__ __forceinline__ float2 gelu_tanh_fast2(float2 z) {
  const float c = 0.7978845608028654f;
  const float2 u = __fmul2_rn(z, z);
  const float2 p = __ffma2_rn(u, make_float2(0.044715f * c, 0.044715f * c), make_float2(c, c));
  const float2 a = __fmul2_rn(z, p);
  float2 t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t.x) : "f"(a.x));
  asm("tanh.approx.f32 %0, %1;" : "=f"(t.y) : "f"(a.y));
  const float2 h = __fmul2_rn(z, make_float2(0.5f, 0.5f));
  return __ffma2_rn(h, t, h);
}

template <typename TOut, int EPI>
__device__ __forceinline__ void epi_store(const EpiArgs& ep, int r, int c, int N, float acc) {
  const float v = acc + ep.bias[c];
  if (EPI == EPI_STORE) {
    reinterpret_cast<TOut*>(ep.out)[size_t(r) * ep.ldo + c] = from_f<TOut>(v);
  } else if (EPI == EPI_GELU) {
    reinterpret_cast<TOut*>(ep.out)[size_t(r) * ep.ldo + c] = from_f<TOut>(gelu_tanh(v));
  } else if (EPI == EPI_RES_GATE) {
    const int e = r / ep.L;
    const float g = ep.mod[ep.gate_row * N + c] + ep.e0[size_t(e) * 6 * N + ep.gate_row * N + c];
    float* x = reinterpret_cast<float*>(ep.out) + size_t(r) * ep.ldo + c;
    *x = *x + g * v;
  } else {
    float* x = reinterpret_cast<float*>(ep.out) + size_t(r) * ep.ldo + c;
    *x = *x + v;
  }
}

template <typename TIn, typename TW, typename TOut, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const TIn* __restrict__ A, const TW* __restrict__ Wt, int M,
                                                        int N, int K, int lda, int ldw, EpiArgs ep) {
  pdl_wait();
  pdl_trigger();
  __shared__ float As[16][64 + 4];
  __shared__ float Ws[16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int rr = i / 16, kk = i % 16;
      const int gr = m0 + rr, gk = k0 + kk;
      As[kk][rr] = (gr < M && gk < K) ? to_f(A[size_t(gr) * lda + gk]) : 0.f;
      const int gn = n0 + rr;
      Ws[kk][rr] = (gn < N && gk < K) ? to_f(Wt[size_t(gn) * ldw + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i) b[i] = Ws[kk][tx * 4 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fmaf(a[i], b[jj], acc[i][jj]);
    }
    __syncthreads();
  }
  const int c4 = n0 + tx * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
    if (r >= M) continue;
    if constexpr (EPI == EPI_STORE && std::is_same<TOut, float>::value) {
      if ((ep.ldo & 3) == 0 && c4 + 3 < N) {   // a 16-byte store per row and thread
        const float4 b = *reinterpret_cast<const float4*>(ep.bias + c4);
        *reinterpret_cast<float4*>(static_cast<float*>(ep.out) + size_t(r) * ep.ldo + c4) =
            make_float4(acc[i][0] + b.x, acc[i][1] + b.y, acc[i][2] + b.z, acc[i][3] + b.w);
        continue;
      }
    }
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int c = c4 + jj;
      if (c < N) epi_store<TOut, EPI>(ep, r, c, N, acc[i][jj]);
    }
  }
}

// ----------------------------------------------------------------------------
// SIMT attention (parity path; C.5 step 4 / 6): per (entry, head, 16-query tile),
// online softmax over key tiles of 64.  Self-attention: keys are the valid prefix of
// the entry's lane (nvalid * L rows); cross-attention: the prompt K/V of the entry's
// prompt version.  Slot order is irrelevant to softmax, so the lane is one
// contiguous key range.
// ----------------------------------------------------------------------------
struct AttnArgs {
  const void* q; int ldq;            // [rows, ldq], head h at column h*hd
  const void* K; const void* V;      // base pointers
  size_t kv_lane_stride;             // elements between lanes (self) or prompt versions (cross)
  int ldk;
  void* o; int ldo;
  int L;                             // query rows per entry
  int cross;                         // 0: keys = lane e, nvalid*L rows; 1: keys = prompt slot xslot, Lk rows
  int Lk_cross;
  float scale;
};

template <typename TA, int HD>
__global__ void __launch_bounds__(128) attn_simt_kernel(AttnArgs a, const TickDesc* __restrict__ td) {
  pdl_wait();
  pdl_trigger();
  constexpr int QT = 16, KT = HD == 128 ? 32 : 64;
  __shared__ float qs[QT][HD + 1];
  __shared__ float ks[KT][HD + 1];
  __shared__ float vs[KT][HD + 1];
  __shared__ float ps[QT][KT + 1];
  __shared__ float m_s[QT], l_s[QT], alpha_s[QT];
  const int e = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * QT;
  const EntryDesc& E = td->e[e];
  if (!E.active || q0 >= a.L) return;
  const int tid = threadIdx.x;
  const TA* Q = reinterpret_cast<const TA*>(a.q);
  const TA* Kb = reinterpret_cast<const TA*>(a.K);
  const TA* Vb = reinterpret_cast<const TA*>(a.V);
  int Lk;
  size_t kv_off;
  if (a.cross) {
    Lk = a.Lk_cross;
    kv_off = size_t(E.xslot) * a.kv_lane_stride;
  } else {
    Lk = E.nvalid * a.L;
    kv_off = size_t(e) * a.kv_lane_stride;
  }
  for (int i = tid; i < QT * HD; i += 128) {
    const int rr = i / HD, c = i % HD;
    const int qr = q0 + rr;
    qs[rr][c] = qr < a.L ? to_f(Q[size_t(e * a.L + qr) * a.ldq + h * HD + c]) : 0.f;
  }
  if (tid < QT) {
    m_s[tid] = -INFINITY;
    l_s[tid] = 0.f;
  }
  float oacc[QT * HD / 128];
#pragma unroll
  for (int i = 0; i < QT * HD / 128; ++i) oacc[i] = 0.f;
  __syncthreads();
  for (int k0 = 0; k0 < Lk; k0 += KT) {
    for (int i = tid; i < KT * HD; i += 128) {
      const int rr = i / HD, c = i % HD;
      const int kr = k0 + rr;
      const size_t off = kv_off + size_t(kr) * a.ldk + h * HD + c;
      ks[rr][c] = kr < Lk ? to_f(Kb[off]) : 0.f;
      vs[rr][c] = kr < Lk ? to_f(Vb[off]) : 0.f;
    }
    __syncthreads();
    for (int i = tid; i < QT * KT; i += 128) {
      const int rr = i / KT, cc = i % KT;
      float s = 0.f;
#pragma unroll 8
      for (int c = 0; c < HD; ++c) s = fmaf(qs[rr][c], ks[cc][c], s);
      ps[rr][cc] = (k0 + cc < Lk) ? s * a.scale : -INFINITY;
    }
    __syncthreads();
    {
      // 8 threads per query row: running max / sum
      const int rr = tid / 8, sub = tid % 8;
      float mx = -INFINITY;
      for (int cc = sub; cc < KT; cc += 8) mx = fmaxf(mx, ps[rr][cc]);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mnew = fmaxf(m_s[rr], mx);
      float sum = 0.f;
      for (int cc = sub; cc < KT; cc += 8) {
        const float p = expf(ps[rr][cc] - mnew);
        ps[rr][cc] = p;
        sum += p;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      __syncwarp();
      if (sub == 0) {
        const float al = expf(m_s[rr] - mnew);
        alpha_s[rr] = al;
        l_s[rr] = l_s[rr] * al + sum;
        m_s[rr] = mnew;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < QT * HD / 128; ++i) {
      const int idx = tid + i * 128;
      const int rr = idx / HD, c = idx % HD;
      float s = oacc[i] * alpha_s[rr];
      for (int cc = 0; cc < KT; ++cc) s = fmaf(ps[rr][cc], vs[cc][c], s);
      oacc[i] = s;
    }
    __syncthreads();
  }
  TA* O = reinterpret_cast<TA*>(a.o);
#pragma unroll
  for (int i = 0; i < QT * HD / 128; ++i) {
    const int idx = tid + i * 128;
    const int rr = idx / HD, c = idx % HD;
    if (q0 + rr < a.L) O[size_t(e * a.L + q0 + rr) * a.ldo + h * HD + c] = from_f<TA>(oacc[i] / l_s[rr]);
  }
}

}  // namespace sdv2
