// Fused elementwise kernels and fp32-SIMT parity kernels of the hot path.
//
// Every kernel cites the model-card step it implements (SURVEY.md §8(c) C.1–C.8,
// stream algorithm O3–O5) and through it the paper passage.  Activation type TA is
// float (fp32 parity path) or bf16 (tensor-core path); the residual stream x,
// latents, sigma and time embeddings are fp32 on both paths (reading R8/Q29).
#pragma once
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

__global__ void __launch_bounds__(1024) noise_ctl_kernel(const float* __restrict__ chunk, float* prev,
                                                         CtrlState* st, float* lat0, float* sig, float* sign,
                                                         const TickDesc* td, StreamCfg cfg, int CHW, int HW,
                                                         int T) {
  __shared__ double red[32];
  __shared__ double s_s;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int C = CHW / (HW * T);
  const int X = td->e[0].X;
  for (int f = 0; f < T; ++f) {
    // d = sqrt(sum (v_f - v_prev)^2 / (C H W)) with fp64 accumulation
    double acc = 0.0;
    for (int i = tid; i < C * HW; i += nt) {
      const int c = i / HW, p = i % HW;
      const double dv = double(chunk[(c * T + f) * HW + p]) - double(prev[i]);
      acc += dv * dv;
    }
    acc = warp_sum_d(acc);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid < 32) {
      double v = tid < (nt >> 5) ? red[tid] : 0.0;
      v = warp_sum_d(v);
      if (tid == 0) {
        const double d = st->has_prev ? sqrt(v / double(C * HW)) : 0.0;   // d = 0 at frame 0 (Q15)
        st->ds[st->nd & 63] = d;
        st->nd += 1;
      }
    }
    __syncthreads();
    for (int i = tid; i < C * HW; i += nt) {
      const int c = i / HW, p = i % HW;
      prev[i] = chunk[(c * T + f) * HW + p];
    }
    if (tid == 0) st->has_prev = 1;
    __syncthreads();
  }
  if (tid == 0) {
    // d_hat = clip(max over the last k+1 values / sigma, 0, 1) (Q13)
    double mx = 0.0;
    const long long lo = st->nd - (cfg.k + 1) > 0 ? st->nd - (cfg.k + 1) : 0;
    for (long long i = lo; i < st->nd; ++i) mx = fmax(mx, st->ds[i & 63]);
    double dh = mx / double(cfg.sigma_m);
    dh = fmin(fmax(dh, 0.0), 1.0);
    // s_X = lam [s_max - (s_max - s_min) d_hat] + (1 - lam) s_{X-1}
    const double lam = double(cfg.lam);
    const double s = lam * (double(cfg.s_max) - (double(cfg.s_max) - double(cfg.s_min)) * dh) + (1.0 - lam) * st->s;
    st->s = s;
    st->d_hat = dh;
    st->s_table[X & 63] = s;
    s_s = s;
    for (int e = 0; e < cfg.n; ++e) {
      const EntryDesc& E = td->e[e];
      if (!E.active) continue;
      sig[e] = sigma_of(st, cfg, E.X, E.j);
      sign[e] = (E.j + 1 < cfg.n) ? sigma_of(st, cfg, E.X, E.j + 1) : 0.f;
    }
  }
  __syncthreads();
  // x_{X,0} = (1 - sigma_{X,0}) v_X + sigma_{X,0} eps_{X,0}   (O4)
  const float s0 = float(s_s * double(cfg.t[0]) / double(cfg.t[0]));
  for (int i = tid; i < CHW; i += nt) {
    const float eps = float(gauss_noise(cfg.seed, uint32_t(X), 0u, uint32_t(i)));
    lat0[i] = (1.f - s0) * chunk[i] + s0 * eps;
  }
}

// Sigma of every entry on ranks that do not run the controller is carried in the
// packet; rank 0 also needs the ring-closure latents assembled: lat[j] = ring_in[j-1].
__global__ void assemble_kernel(const float* __restrict__ ring_in, float* __restrict__ lat, const TickDesc* td,
                                int n, int CTHW) {
  const int j = blockIdx.y + 1;
  if (j >= n || !td->e[j].active) return;
  const float4* src = reinterpret_cast<const float4*>(ring_in + size_t(j - 1) * CTHW);
  float4* dst = reinterpret_cast<float4*>(lat + size_t(j) * CTHW);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < CTHW / 4; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// ----------------------------------------------------------------------------
// Patchify + patch embedding (C.1): x_tau = W_pe u_tau + b_pe, u_tau[c*4+a*2+b] =
// v[c, f, 2i+a, 2jj+b].  fp32 SIMT (K = 4C is tiny).  One CTA per 16 tokens.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) patch_embed_kernel(const float* __restrict__ lat, const float* __restrict__ Wpe,
                                                          const float* __restrict__ bpe, float* __restrict__ x,
                                                          int rows, int L, int d, int C, int T, int h, int w) {
  extern __shared__ float u_s[];   // [16][4C]
  const int P = 4 * C;
  const int r0 = blockIdx.x * 16;
  const int hn = h / 2, wn = w / 2;
  for (int i = threadIdx.x; i < 16 * P; i += blockDim.x) {
    const int rr = i / P, k = i % P;
    const int r = r0 + rr;
    float v = 0.f;
    if (r < rows) {
      const int e = r / L, tau = r % L;
      const int f = tau / (hn * wn), ii = (tau / wn) % hn, jj = tau % wn;
      const int c = k / 4, a = (k / 2) % 2, b = k % 2;
      v = lat[size_t(e) * C * T * h * w + ((size_t(c) * T + f) * h + 2 * ii + a) * w + 2 * jj + b];
    }
    u_s[i] = v;
  }
  __syncthreads();
  for (int col = threadIdx.x; col < d; col += blockDim.x) {
    float acc[16];
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) acc[rr] = 0.f;
    for (int k = 0; k < P; ++k) {
      const float wv = Wpe[size_t(col) * P + k];
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) acc[rr] += wv * u_s[rr * P + k];
    }
    const float b = bpe[col];
#pragma unroll
    for (int rr = 0; rr < 16; ++rr)
      if (r0 + rr < rows) x[size_t(r0 + rr) * d + col] = acc[rr] + b;
  }
}

// ----------------------------------------------------------------------------
// Time conditioning (C.2): sinusoid(1000 sigma) in fp64, then GEMVs.
// ----------------------------------------------------------------------------
__global__ void sinusoid_kernel(const float* __restrict__ sig, float* __restrict__ emb, int n, int dim) {
  const int e = blockIdx.x;
  const int half = dim / 2;
  const double t = 1000.0 * double(sig[e]);
  for (int k = threadIdx.x; k < half; k += blockDim.x) {
    const double arg = t * pow(10000.0, -double(k) / double(half));
    emb[e * dim + k] = float(cos(arg));
    emb[e * dim + half + k] = float(sin(arg));
  }
}

// out[e][r] = sum_k W[r,k] act(in[e][k]) + b[r]; act = SiLU if pre_silu.  One warp per row.
template <typename TW>
__global__ void __launch_bounds__(256) gemv_kernel(const TW* __restrict__ W, const float* __restrict__ b,
                                                   const float* __restrict__ in, float* __restrict__ out, int n,
                                                   int R, int Kd, int pre_silu) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  float acc[kMaxSteps];
#pragma unroll
  for (int e = 0; e < kMaxSteps; ++e) acc[e] = 0.f;
  const TW* wr = W + size_t(warp) * Kd;
  for (int k = lane; k < Kd; k += 32) {
    const float wv = to_f(wr[k]);
#pragma unroll
    for (int e = 0; e < kMaxSteps; ++e) {
      if (e < n) {
        float z = in[size_t(e) * Kd + k];
        if (pre_silu) z = z / (1.f + expf(-z));
        acc[e] += wv * z;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < kMaxSteps; ++e) {
    if (e < n) {
      const float s = warp_sum(acc[e]);
      if (lane == 0) out[size_t(e) * R + warp] = s + b[warp];
    }
  }
}

// ----------------------------------------------------------------------------
// adaLN norm + modulate (C.5 steps 1, 6, 8): out = N(x) * (a0 + A) + B.
//   mode 0: A = mod[sc] + e0[e][sc], B = mod[sh] + e0[e][sh], a0 = 1   (norm1 / norm2)
//   mode 1: A = gamma, B = beta, a0 = 0                                (norm3, affine)
// N = RMSNorm (center = 0) or affine-free LayerNorm (center = 1), eps inside the sqrt.
// One warp per row, fp32 statistics.
// ----------------------------------------------------------------------------
template <typename TA>
__global__ void __launch_bounds__(256) norm_mod_kernel(const float* __restrict__ x, TA* __restrict__ out, int rows,
                                                       int d, int L, int mode, const float* __restrict__ mod,
                                                       const float* __restrict__ e0, int sc_row, int sh_row,
                                                       const float* __restrict__ gamma,
                                                       const float* __restrict__ beta, float eps, int center) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + size_t(r) * d;
  float mu = 0.f;
  if (center) {
    float s = 0.f;
    for (int c = lane * 4; c < d; c += 128) {
      const float4 v = *reinterpret_cast<const float4*>(xr + c);
      s += v.x + v.y + v.z + v.w;
    }
    mu = warp_sum(s) / float(d);
  }
  float ss = 0.f;
  for (int c = lane * 4; c < d; c += 128) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    const float a = v.x - mu, b = v.y - mu, cc = v.z - mu, dd = v.w - mu;
    ss += a * a + b * b + cc * cc + dd * dd;
  }
  const float inv = rsqrtf(warp_sum(ss) / float(d) + eps);
  const int e = r / L;
  TA* orow = out + size_t(r) * d;
  for (int c = lane * 4; c < d; c += 128) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cc = c + q;
      float A, B, a0;
      if (mode == 0) {
        A = mod[sc_row * d + cc] + e0[size_t(e) * 6 * d + sc_row * d + cc];
        B = mod[sh_row * d + cc] + e0[size_t(e) * 6 * d + sh_row * d + cc];
        a0 = 1.f;
      } else {
        A = gamma[cc];
        B = beta[cc];
        a0 = 0.f;
      }
      orow[cc] = from_f<TA>((xv[q] - mu) * inv * (a0 + A) + B);
    }
  }
}

// y = g * y / sqrt(mean(y^2) + eps) over the full row (C.4 RMS_g; cross-attention q and
// prompt K).  One warp per row.
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(256) rms_rows_kernel(const TIn* __restrict__ y, TOut* __restrict__ out,
                                                       const float* __restrict__ g, int rows, int d, int ld_in,
                                                       float eps) {
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

template <typename TA>
__global__ void __launch_bounds__(256) qkv_post_kernel(const TA* __restrict__ qkv, TA* __restrict__ qout,
                                                       TA* __restrict__ Kc, TA* __restrict__ Vc,
                                                       const float* __restrict__ gq, const float* __restrict__ gk,
                                                       const TickDesc* __restrict__ td, RopeTabs R, int rows, int d,
                                                       int hd, int L, int hn, int wn, int T, int S, float eps) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int e = r / L, tau = r % L;
  const EntryDesc& E = td->e[e];
  const int f = tau / (hn * wn), ph = (tau / wn) % hn, pw = tau % wn;
  const TA* qr = qkv + size_t(r) * 3 * d;
  const TA* kr = qr + d;
  const TA* vr = qr + 2 * d;
  float sq = 0.f, sk = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float a = to_f(qr[c]), b = to_f(kr[c]);
    sq += a * a;
    sk += b * b;
  }
  const float iq = rsqrtf(warp_sum(sq) / float(d) + eps);
  const float ik = rsqrtf(warp_sum(sk) / float(d) + eps);
  const size_t lane_base = size_t(e) * S * L * d;   // lane j = e
  const int pt = E.pos[f];
  const int half = hd / 2;
  for (int p = lane; p < d / 2; p += 32) {
    const int c0 = 2 * p, pair = p % half;
    float cs, sn;
    rope_cs(R, pair, pt, ph, pw, cs, sn);
    const float q0 = gq[c0] * to_f(qr[c0]) * iq, q1 = gq[c0 + 1] * to_f(qr[c0 + 1]) * iq;
    qout[size_t(r) * d + c0] = from_f<TA>(q0 * cs - q1 * sn);
    qout[size_t(r) * d + c0 + 1] = from_f<TA>(q0 * sn + q1 * cs);
    const float k0 = gk[c0] * to_f(kr[c0]) * ik, k1 = gk[c0 + 1] * to_f(kr[c0 + 1]) * ik;
    const size_t o = lane_base + (size_t(E.write_slot) * L + tau) * d + c0;
    Kc[o] = from_f<TA>(k0 * cs - k1 * sn);
    Kc[o + 1] = from_f<TA>(k0 * sn + k1 * cs);
    Vc[o] = vr[c0];
    Vc[o + 1] = vr[c0 + 1];
    if (E.refresh_mask) {
      for (int i = 0; i < 32; ++i) {
        if (!(E.refresh_mask & (1 << i))) continue;
        float ca, sa;
        rope_cs(R, pair, i * T + f, ph, pw, ca, sa);   // anchored at i T' + f (Q10)
        const size_t oi = lane_base + (size_t(i) * L + tau) * d + c0;
        Kc[oi] = from_f<TA>(k0 * ca - k1 * sa);
        Kc[oi + 1] = from_f<TA>(k0 * sa + k1 * ca);
        Vc[oi] = vr[c0];
        Vc[oi + 1] = vr[c0 + 1];
      }
    }
  }
}

// RoPE phase re-base (R3): every ring slot of a re-basing lane, in every local
// block, is rotated on its temporal pairs by R(-T_reset).  Grid: (token-rows, lane).
template <typename TA>
__global__ void __launch_bounds__(256) rebase_kernel(TA* __restrict__ K, const TickDesc* __restrict__ td, RopeTabs R,
                                                     int nblocks, int n, int S, int m, int W, int L, int d, int hd,
                                                     int T_reset) {
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
enum { EPI_STORE = 0, EPI_GELU = 1, EPI_RES_GATE = 2, EPI_RES = 3 };

struct EpiArgs {
  void* out;            // TOut* (STORE/GELU) or float* x (RES*)
  int ldo;
  const float* bias;
  const float* mod;     // block modulation [6, d] (RES_GATE)
  const float* e0;      // [n, 6, d] (RES_GATE)
  int gate_row;         // 2 (g1) or 5 (g2)
  int L;                // rows per entry
};

__device__ __forceinline__ float gelu_tanh(float z) {
  return 0.5f * z * (1.f + tanhf(0.7978845608028654f * (z + 0.044715f * z * z * z)));
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
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int r = m0 + ty * 4 + i, c = n0 + tx * 4 + jj;
      if (r < M && c < N) epi_store<TOut, EPI>(ep, r, c, N, acc[i][jj]);
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
  int cross;                         // 0: keys = lane e, nvalid*L rows; 1: keys = version pver, Lk rows
  int Lk_cross;
  float scale;
};

template <typename TA, int HD>
__global__ void __launch_bounds__(128) attn_simt_kernel(AttnArgs a, const TickDesc* __restrict__ td) {
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
    kv_off = size_t(E.pver & 1) * a.kv_lane_stride;
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

// ----------------------------------------------------------------------------
// Head + unpatchify + flow-matching x0 + output / re-noise (C.7, C.8, O5), fp32.
// One warp per token row: (sh, sc) = mod_h + e[e]; y = (N(x)(1+sc)+sh) W_h^T + b_h;
// v_hat[c, f, 2i+a, 2jj+b] = y[(a*2+b) C + c]; x0 = x_sigma - sigma v_hat; the last
// step writes the clean output, other steps write (1 - s') x0 + s' eps_{X,j+1} into
// the ring-closure buffer slot j.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) head_kernel(const float* __restrict__ x, const float* __restrict__ e_emb,
                                                   const float* __restrict__ head_mod, const float* __restrict__ Wh,
                                                   const float* __restrict__ bh, const float* __restrict__ lat,
                                                   const float* __restrict__ sig, const float* __restrict__ sign,
                                                   float* __restrict__ out, float* __restrict__ ring_out,
                                                   const TickDesc* __restrict__ td, int rows, int d, int L, int C,
                                                   int T, int h, int w, int n, float eps, int center,
                                                   unsigned long long seed) {
  extern __shared__ float a_s[];   // [8 warps][d]
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + wid;
  if (r >= rows) return;
  const int e = r / L, tau = r % L;
  const EntryDesc& E = td->e[e];
  if (!E.active) return;
  const float* xr = x + size_t(r) * d;
  float mu = 0.f;
  if (center) {
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s += xr[c];
    mu = warp_sum(s) / float(d);
  }
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = xr[c] - mu;
    ss += v * v;
  }
  const float inv = rsqrtf(warp_sum(ss) / float(d) + eps);
  float* as = a_s + wid * d;
  for (int c = lane; c < d; c += 32) {
    const float sh = head_mod[c] + e_emb[size_t(e) * d + c];
    const float sc = head_mod[d + c] + e_emb[size_t(e) * d + c];
    as[c] = (xr[c] - mu) * inv * (1.f + sc) + sh;
  }
  __syncwarp();
  const int P = 4 * C;
  const int hn = h / 2, wn = w / 2;
  const int f = tau / (hn * wn), ii = (tau / wn) % hn, jj = tau % wn;
  const size_t CTHW = size_t(C) * T * h * w;
  for (int p = lane; p < P; p += 32) {
    float acc = 0.f;
    const float* wr = Wh + size_t(p) * d;
    for (int c = 0; c < d; ++c) acc = fmaf(wr[c], as[c], acc);
    const float y = acc + bh[p];
    const int ab = p / C, ch = p % C, a = ab / 2, b = ab % 2;
    const size_t idx = ((size_t(ch) * T + f) * h + 2 * ii + a) * w + 2 * jj + b;
    const float x0 = lat[size_t(e) * CTHW + idx] - sig[e] * y;
    if (E.j == n - 1) {
      out[idx] = x0;
    } else {
      const float s1 = sign[e];
      const float eps1 = float(gauss_noise(seed, uint32_t(E.X), uint32_t(E.j + 1), uint32_t(idx)));
      ring_out[size_t(E.j) * CTHW + idx] = (1.f - s1) * x0 + s1 * eps1;
    }
  }
}

}  // namespace sdv2
