// Fused memory-bound kernels of the hot path (SURVEY.md §8(a) a1–a4, a6, a12), written
// for HBM bandwidth: rows are held in registers (one load of every input), 16-byte
// vector loads/stores, row statistics reduced with warp shuffles + a small smem
// exchange, and the per-element work spread over many CTAs.
#pragma once
#include "common.cuh"
#include "ctl.h"
#include "kernels.cuh"

namespace sdv2 {

constexpr int kRowThreads = 128;          // threads cooperating on one row

// Block-wide (kRowThreads) sum of two values; `red` = smem [2][kRowThreads/32].
__device__ __forceinline__ void row_sum2(float& a, float& b, float* red, int sub) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = (threadIdx.x % kRowThreads) >> 5, lane = threadIdx.x & 31;
  float* rr = red + sub * 2 * (kRowThreads / 32);
  if (lane == 0) {
    rr[w] = a;
    rr[kRowThreads / 32 + w] = b;
  }
  __syncthreads();
  a = 0.f;
  b = 0.f;
#pragma unroll
  for (int i = 0; i < kRowThreads / 32; ++i) {
    a += rr[i];
    b += rr[kRowThreads / 32 + i];
  }
}

__device__ __forceinline__ void store4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void store4(bf16* p, float a, float b, float c, float d) {
  __nv_bfloat162 x = __floats2bfloat162_rn(a, b), y = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&x);
  u.y = *reinterpret_cast<uint32_t*>(&y);
  *reinterpret_cast<uint2*>(p) = u;
}

// ----------------------------------------------------------------------------
// Norm + modulate (C.5 steps 1/6/8, C.7 head):
//   out = N(x) * (a0 + modA[sc] + eA[e][sc]) + (modA[sh] + eA[e][sh])
// adaLN (a0 = 1): modA = block modulation [6,d], eA = e0 [n,6d] (estride 6d) or the
// head's mod_h [2,d] + e [n,d] (estride d, same vector for shift and scale);
// affine norm3 (a0 = 0): modA = gamma at sc, beta at sh, eA = nullptr.
// 2 rows per 256-thread CTA, the row in registers.
// ----------------------------------------------------------------------------
struct ModArgs {
  const float* modA; int sc_off, sh_off;
  const float* eA; int estride, esc_off, esh_off;
  float a0;
  float* zero_rows = nullptr;   // if set, zero_rows[r] = 0 for every row (a downstream GEMM's atomic row sums)
};

template <typename TA, int NV>
__global__ void __launch_bounds__(256) norm_mod2_kernel(const float* __restrict__ x, TA* __restrict__ out, int rows,
                                                        int d, int L, ModArgs m, float eps, int center) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[2][2][2 * (kRowThreads / 32)];
  const int sub = threadIdx.x / kRowThreads, t = threadIdx.x % kRowThreads;
  const int r = blockIdx.x * 2 + sub;
  const bool ok = r < rows;
  const float* xr = x + size_t(ok ? r : 0) * d;
  const int e = (ok ? r : 0) / L;
  float4 v[NV], A[NV], B[NV];
  float s = 0.f, ss = 0.f;
  // every load is issued up front: the row of x and the modulation vectors (scale,
  // shift, per-entry offsets) do not depend on each other, one memory round trip total
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * kRowThreads + t) * 4;
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    A[i] = B[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < d && ok) {
      v[i] = __ldcg(reinterpret_cast<const float4*>(xr + c));
      A[i] = __ldg(reinterpret_cast<const float4*>(m.modA + m.sc_off + c));
      B[i] = __ldg(reinterpret_cast<const float4*>(m.modA + m.sh_off + c));
      if (m.eA) {
        const float4 ea = __ldg(reinterpret_cast<const float4*>(m.eA + size_t(e) * m.estride + m.esc_off + c));
        const float4 eb = __ldg(reinterpret_cast<const float4*>(m.eA + size_t(e) * m.estride + m.esh_off + c));
        A[i].x += ea.x; A[i].y += ea.y; A[i].z += ea.z; A[i].w += ea.w;
        B[i].x += eb.x; B[i].y += eb.y; B[i].z += eb.z; B[i].w += eb.w;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) s += v[i].x + v[i].y + v[i].z + v[i].w;
  float mu = 0.f;
  if (center) {   // two-pass LayerNorm statistics (row in registers)
    float dummy = 0.f;
    row_sum2(s, dummy, &red[0][0][0], sub);
    mu = s / float(d);
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * kRowThreads + t) * 4;
    if (c < d) {
      const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
      ss += a0 * a0 + a1 * a1 + a2 * a2 + a3 * a3;
    }
  }
  float dummy2 = 0.f;
  row_sum2(ss, dummy2, &red[1][0][0], sub);
  const float inv = rsqrtf(ss / float(d) + eps);
  if (!ok) return;
  if (m.zero_rows && t == 0) m.zero_rows[r] = 0.f;
  TA* orow = out + size_t(r) * d;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * kRowThreads + t) * 4;
    if (c < d)
      store4(orow + c, (v[i].x - mu) * inv * (m.a0 + A[i].x) + B[i].x, (v[i].y - mu) * inv * (m.a0 + A[i].y) + B[i].y,
             (v[i].z - mu) * inv * (m.a0 + A[i].z) + B[i].z, (v[i].w - mu) * inv * (m.a0 + A[i].w) + B[i].w);
  }
}

// ----------------------------------------------------------------------------
// 16-byte units of 8 activations (bf16) or 4 (fp32): helpers for the row kernels.
// ----------------------------------------------------------------------------
template <typename TA> struct Unit;
template <> struct Unit<bf16> {
  static constexpr int N = 8;
  __device__ static void load(const bf16* p, float (&f)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ static void store(bf16* p, const float (&f)[8]) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = u;
  }
  __device__ static void copy(bf16* dst, const bf16* src) {
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
  }
};
template <> struct Unit<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* p, float (&f)[4]) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
  __device__ static void store(float* p, const float (&f)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
  __device__ static void copy(float* dst, const float* src) {
    *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
  }
};

// ----------------------------------------------------------------------------
// q/k RMSNorm + 3D RoPE + KV lane write + sink refresh copy (C.5 2–4, C.6, O3).
// 2 rows per CTA; each thread holds <= kMaxU units of q and k.
// ----------------------------------------------------------------------------
template <typename TA, int kMaxU>
__global__ void __launch_bounds__(256) qkv_post2_kernel(const TA* __restrict__ qkv, TA* __restrict__ qout,
                                                        TA* __restrict__ Kc, TA* __restrict__ Vc,
                                                        const float* __restrict__ gq, const float* __restrict__ gk,
                                                        const TickDesc* __restrict__ td, RopeTabs R, int rows, int d,
                                                        int hd, int L, int hn, int wn, int T, int S, float eps) {
  using U = Unit<TA>;
  constexpr int UN = U::N;
  __shared__ float red[2][2 * (kRowThreads / 32)];
  const int sub = threadIdx.x / kRowThreads, t = threadIdx.x % kRowThreads;
  const int r = blockIdx.x * 2 + sub;
  const bool ok = r < rows;
  const int rr = ok ? r : 0;
  const TA* qr = qkv + size_t(rr) * 3 * d;
  const TA* kr = qr + d;
  const TA* vr = qr + 2 * d;
  const int units = d / UN;
  // everything that does not depend on the row statistics is loaded before the
  // reduction (q, k, v, the gains, the entry's positions and the RoPE table entries):
  // the kernel is latency-bound at 2 rows per CTA, so one round trip instead of three
  const int e = rr / L, tau = rr % L;
  const int f = tau / (hn * wn), ph = (tau / wn) % hn, pw = tau % wn;
  const EntryDesc& E = td->e[e];
  const int pt = E.pos[f];
  constexpr bool kPre = kMaxU <= 3;   // wide rows (d = 5120): gains / RoPE loaded late (registers)
  constexpr int kP = kPre ? kMaxU : 1;
  float q[kMaxU][UN], k[kMaxU][UN], vv[kMaxU][UN], gqv[kP][UN], gkv[kP][UN];
  float cs[kP][UN / 2], sn[kP][UN / 2];
  float sq = 0.f, sk = 0.f;
  const int half = hd / 2;
  // the gains, the tick descriptor's positions and the RoPE tables are not produced by
  // the upstream kernel: their loads (a dependent chain) run before the PDL wait
  if constexpr (kPre) {
#pragma unroll
    for (int i = 0; i < kMaxU; ++i) {
      const int u = i * kRowThreads + t;
      if (u < units && ok) {
        const int c0 = u * UN;
#pragma unroll
        for (int j = 0; j < UN; j += 4) {
          const float4 a4 = __ldg(reinterpret_cast<const float4*>(gq + c0 + j));
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(gk + c0 + j));
          gqv[i][j] = a4.x; gqv[i][j + 1] = a4.y; gqv[i][j + 2] = a4.z; gqv[i][j + 3] = a4.w;
          gkv[i][j] = b4.x; gkv[i][j + 1] = b4.y; gkv[i][j + 2] = b4.z; gkv[i][j + 3] = b4.w;
        }
#pragma unroll
        for (int j = 0; j < UN; j += 2) rope_cs(R, ((c0 + j) >> 1) % half, pt, ph, pw, cs[i][j / 2], sn[i][j / 2]);
      }
    }
  }
  pdl_wait();
  pdl_trigger();
#pragma unroll
  for (int i = 0; i < kMaxU; ++i) {
    const int u = i * kRowThreads + t;
    if (u < units && ok) {
      const int c0 = u * UN;
      U::load(qr + c0, q[i]);
      U::load(kr + c0, k[i]);
      U::load(vr + c0, vv[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxU; ++i) {
    const int u = i * kRowThreads + t;
    if (u < units && ok) {
#pragma unroll
      for (int j = 0; j < UN; ++j) {
        sq += q[i][j] * q[i][j];
        sk += k[i][j] * k[i][j];
      }
    }
  }
  row_sum2(sq, sk, &red[0][0], sub);
  if (!ok) return;
  const float iq = rsqrtf(sq / float(d) + eps), ik = rsqrtf(sk / float(d) + eps);
  const size_t lane_base = size_t(e) * S * L * d;
  const size_t wrow = lane_base + (size_t(E.write_slot) * L + tau) * d;
#pragma unroll
  for (int i = 0; i < kMaxU; ++i) {
    const int u = i * kRowThreads + t;
    if (u >= units) continue;
    const int c0 = u * UN;
    float qo[UN], ko[UN], kn[UN];
#pragma unroll
    for (int j = 0; j < UN; j += 2) {
      float c_, s_, gq0, gq1, gk0, gk1;
      if constexpr (kPre) {
        c_ = cs[i][j / 2];
        s_ = sn[i][j / 2];
        gq0 = gqv[i][j]; gq1 = gqv[i][j + 1]; gk0 = gkv[i][j]; gk1 = gkv[i][j + 1];
      } else {
        rope_cs(R, ((c0 + j) >> 1) % half, pt, ph, pw, c_, s_);
        gq0 = __ldg(gq + c0 + j); gq1 = __ldg(gq + c0 + j + 1);
        gk0 = __ldg(gk + c0 + j); gk1 = __ldg(gk + c0 + j + 1);
      }
      const float q0 = gq0 * q[i][j] * iq, q1 = gq1 * q[i][j + 1] * iq;
      const float k0 = gk0 * k[i][j] * ik, k1 = gk1 * k[i][j + 1] * ik;
      qo[j] = q0 * c_ - q1 * s_;
      qo[j + 1] = q0 * s_ + q1 * c_;
      ko[j] = k0 * c_ - k1 * s_;
      ko[j + 1] = k0 * s_ + k1 * c_;
      kn[j] = k0;
      kn[j + 1] = k1;
    }
    U::store(qout + size_t(rr) * d + c0, qo);
    U::store(Kc + wrow + c0, ko);
    U::store(Vc + wrow + c0, vv[i]);
    if (E.refresh_mask) {
      for (int s = 0; s < 32; ++s) {
        if (!(E.refresh_mask & (1 << s))) continue;
        float ka[UN];
#pragma unroll
        for (int j = 0; j < UN; j += 2) {
          const int pair = ((c0 + j) >> 1) % half;
          float cs, sn;
          rope_cs(R, pair, s * T + f, ph, pw, cs, sn);   // anchored at s T' + f (Q10)
          ka[j] = kn[j] * cs - kn[j + 1] * sn;
          ka[j + 1] = kn[j] * sn + kn[j + 1] * cs;
        }
        const size_t srow = lane_base + (size_t(s) * L + tau) * d;
        U::store(Kc + srow + c0, ka);
        U::store(Vc + srow + c0, vv[i]);
      }
    }
  }
}

// y = g * y / sqrt(mean(y^2) + eps) (C.4 RMS_g, cross-attention q), in place.
template <typename TA, int kMaxU>
__global__ void __launch_bounds__(256) rms_rows2_kernel(TA* __restrict__ y, const float* __restrict__ g, int rows, int d,
                                                        float eps) {
  pdl_wait();
  pdl_trigger();
  using U = Unit<TA>;
  constexpr int UN = U::N;
  __shared__ float red[2][2 * (kRowThreads / 32)];
  const int sub = threadIdx.x / kRowThreads, t = threadIdx.x % kRowThreads;
  const int r = blockIdx.x * 2 + sub;
  const bool ok = r < rows;
  TA* yr = y + size_t(ok ? r : 0) * d;
  const int units = d / UN;
  float v[kMaxU][UN], gv[kMaxU][UN];
  float ss = 0.f, dummy = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxU; ++i) {
    const int u = i * kRowThreads + t;
    if (u < units && ok) {
      U::load(yr + u * UN, v[i]);
#pragma unroll
      for (int j = 0; j < UN; j += 4) {
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(g + u * UN + j));
        gv[i][j] = g4.x; gv[i][j + 1] = g4.y; gv[i][j + 2] = g4.z; gv[i][j + 3] = g4.w;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxU; ++i) {
    const int u = i * kRowThreads + t;
    if (u < units && ok) {
#pragma unroll
      for (int j = 0; j < UN; ++j) ss += v[i][j] * v[i][j];
    }
  }
  row_sum2(ss, dummy, &red[0][0], sub);
  if (!ok) return;
  const float inv = rsqrtf(ss / float(d) + eps);
#pragma unroll
  for (int i = 0; i < kMaxU; ++i) {
    const int u = i * kRowThreads + t;
    if (u < units) {
#pragma unroll
      for (int j = 0; j < UN; ++j) v[i][j] = gv[i][j] * v[i][j] * inv;
      U::store(yr + u * UN, v[i]);
    }
  }
}

// ----------------------------------------------------------------------------
// Motion-aware noise controller: per-frame d (fp64 accumulation), window
// max over the last k+1 values, clip, EMA s_X, sigma of every entry of the stream (R5).
// chunk / prev / st point at stream 0's; CTHW = chunk stride.
// ----------------------------------------------------------------------------
// Grid (kMotionSlices, B): CTA c of stream b owns a contiguous slice of the frame's C HW
// values; per frame it writes its fp64 partial sum of squared differences and moves its
// slice of the frame into prev; the last CTA of the stream to finish (arrival counter)
// sums the partials in slice order (deterministic) and runs the controller update.
constexpr int kMotionSlices = 32;
__global__ void __launch_bounds__(256) motion_kernel(const float* __restrict__ chunk_all, float* prev_all,
                                                     CtrlState* st_all, float* sig, float* sign, const TickDesc* td,
                                                     StreamCfg cfg, int CHW, int HW, int T, int n_entries,
                                                     double* part, unsigned* arrive) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[8];
  __shared__ bool last;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int b = blockIdx.y, c = blockIdx.x, P = gridDim.x;
  const float* chunk = chunk_all + size_t(b) * CHW;
  const int C = CHW / (HW * T);
  const int n4 = C * HW / 4;                        // float4 per frame (C HW % 4 == 0)
  const int i0 = int((long long)n4 * c / P), i1 = int((long long)n4 * (c + 1) / P);
  float* prev = prev_all + size_t(b) * C * HW;
  CtrlState* st = st_all + b;
  for (int f = 0; f < T; ++f) {
    double acc = 0.0;
    for (int q = i0 + tid; q < i1; q += nt) {
      const int i = q * 4;
      // frame f of channel c is contiguous
      const int ch = i / HW, p = i % HW;
      const float4 a = *reinterpret_cast<const float4*>(chunk + (size_t(ch) * T + f) * HW + p);
      const float4 v = *reinterpret_cast<const float4*>(prev + i);
      const double d0 = double(a.x) - double(v.x), d1 = double(a.y) - double(v.y);
      const double d2 = double(a.z) - double(v.z), d3 = double(a.w) - double(v.w);
      acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
      *reinterpret_cast<float4*>(prev + i) = a;      // this frame is the next one's previous
    }
    acc = warp_sum_d(acc);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double v = 0.0;
      for (int w = 0; w < (nt >> 5); ++w) v += red[w];
      part[(size_t(b) * kMaxFrames + f) * kMotionSlices + c] = v;
    }
    __syncthreads();
  }
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(arrive + b, 1u) == unsigned(P - 1);
  }
  __syncthreads();
  if (!last || tid != 0) return;
  __threadfence();
  arrive[b] = 0u;   // re-armed for the next call
  const int X = td->e[b].X;
  for (int f = 0; f < T; ++f) {
    double v = 0.0;
    for (int k = 0; k < P; ++k) v += __ldcg(part + (size_t(b) * kMaxFrames + f) * kMotionSlices + k);
    const double dd = st->has_prev ? sqrt(v / double(C * HW)) : 0.0;   // d = 0 at frame 0 (Q15)
    st->ds[st->nd & 63] = dd;
    st->nd += 1;
    st->has_prev = 1;
  }
  {
    double mx = 0.0;
    const long long lo = st->nd - (cfg.k + 1) > 0 ? st->nd - (cfg.k + 1) : 0;
    for (long long i = lo; i < st->nd; ++i) mx = fmax(mx, st->ds[i & 63]);
    double dh = mx / double(cfg.sigma_m);
    dh = fmin(fmax(dh, 0.0), 1.0);
    const double lam = double(cfg.lam);
    const double s = lam * (double(cfg.s_max) - (double(cfg.s_max) - double(cfg.s_min)) * dh) + (1.0 - lam) * st->s;
    st->s = s;
    st->d_hat = dh;
    st->s_table[X & 63] = s;
    for (int e = 0; e < n_entries; ++e) {
      const EntryDesc& E = td->e[e];
      if (!E.active || E.stream != b) continue;
      sig[e] = sigma_of(st, cfg, E.X, E.j);
      sign[e] = (E.j + 1 < cfg.n) ? sigma_of(st, cfg, E.X, E.j + 1) : 0.f;
    }
  }
}

// Philox key of stream b: (seed_lo, seed_hi + b) (noise source Q21).
__device__ __forceinline__ unsigned long long stream_key(unsigned long long seed, int b) {
  return seed + (static_cast<unsigned long long>(b) << 32);
}

// x_{X,0} = (1 - sigma_{X,0}) v_X + sigma_{X,0} eps_{X,0}  (O4), all SMs; grid.y = stream
// b, whose step-0 entry is e = b.
__global__ void __launch_bounds__(256) blend_kernel(const float* __restrict__ chunk, float* __restrict__ lat0,
                                                    const float* __restrict__ sig, const TickDesc* __restrict__ td,
                                                    unsigned long long seed, int CTHW) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  const int X = td->e[b].X;
  const float s0 = sig[b];
  const unsigned long long key = stream_key(seed, b);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < CTHW; i += gridDim.x * blockDim.x) {
    const float eps = float(gauss_noise(key, uint32_t(X), 0u, uint32_t(i)));
    lat0[size_t(b) * CTHW + i] = (1.f - s0) * chunk[size_t(b) * CTHW + i] + s0 * eps;
  }
}

// Patchify (C.1): u[r, c*4 + a*2 + b] = v_e[c, f, 2i+a, 2jj+b], fp32.
__global__ void patchify_kernel(const float* __restrict__ lat, float* __restrict__ u, int rows, int L, int C, int T,
                                int h, int w) {
  pdl_wait();
  pdl_trigger();
  const int P = 4 * C, hn = h / 2, wn = w / 2;
  const size_t CTHW = size_t(C) * T * h * w;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * P; i += gridDim.x * blockDim.x) {
    const int r = i / P, k = i % P;
    const int e = r / L, tau = r % L;
    const int f = tau / (hn * wn), ii = (tau / wn) % hn, jj = tau % wn;
    const int c = k / 4, a = (k / 2) % 2, b = k % 2;
    u[i] = lat[size_t(e) * CTHW + ((size_t(c) * T + f) * h + 2 * ii + a) * w + 2 * jj + b];
  }
}

// Head tail (C.7, C.8, O5): v_hat[c, f, 2i+a, 2jj+b] = y[tau][(a*2+b) C + c]; x0 = x_sigma -
// sigma v_hat; the last step writes the clean output of its stream b (out[b]), the
// others (1 - s') x0 + s' eps_{X,j+1} into ring-closure slot e (= j B + b; consumed as
// entry e + B at the next micro-step).  One thread per latent element, all SMs.
__global__ void __launch_bounds__(256) flow_kernel(const float* __restrict__ y, const float* __restrict__ lat,
                                                   const float* __restrict__ sig, const float* __restrict__ sign,
                                                   float* __restrict__ out, float* __restrict__ ring_out,
                                                   const TickDesc* __restrict__ td, int n_act, int L, int C, int T,
                                                   int h, int w, int n, unsigned long long seed) {
  pdl_wait();
  pdl_trigger();
  const int P = 4 * C, hn = h / 2, wn = w / 2;
  const int CTHW = C * T * h * w;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_act * CTHW; i += gridDim.x * blockDim.x) {
    const int e = i / CTHW, idx = i % CTHW;
    const EntryDesc& E = td->e[e];
    if (!E.active) continue;
    const int xx = idx % w, yy = (idx / w) % h, f = (idx / (w * h)) % T, c = idx / (w * h * T);
    const int tau = f * hn * wn + (yy >> 1) * wn + (xx >> 1);
    const int p = ((yy & 1) * 2 + (xx & 1)) * C + c;
    const float x0 = lat[size_t(e) * CTHW + idx] - sig[e] * y[size_t(e * L + tau) * P + p];
    if (E.j == n - 1) {
      out[size_t(E.stream) * CTHW + idx] = x0;
    } else {
      const float s1 = sign[e];
      const float eps1 = float(gauss_noise(stream_key(seed, E.stream), uint32_t(E.X), uint32_t(E.j + 1), uint32_t(idx)));
      ring_out[size_t(e) * CTHW + idx] = (1.f - s1) * x0 + s1 * eps1;
    }
  }
}

// out[e][r] = W[r,:] . act(in[e,:]) + b[r], act = SiLU if pre_silu; the activated input
// vectors are staged once per CTA in smem; 8 warps x 4 rows per CTA.  The 4 rows of a warp
// are walked together with 16-byte weight loads (4 fp32 / 8 bf16 per lane and row), so
// each lane keeps 4 independent loads in flight; a scalar loop covers Kd % (32 x vec).
template <typename TW> struct GemvVec;
template <> struct GemvVec<float> {
  static constexpr int V = 4;
  __device__ static void load(const float* p, float (&w)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  }
};
template <> struct GemvVec<bf16> {
  static constexpr int V = 8;
  __device__ static void load(const bf16* p, float (&w)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 t = __bfloat1622float2(h[i]);
      w[2 * i] = t.x;
      w[2 * i + 1] = t.y;
    }
  }
};

template <typename TW, int NMAX = kMaxEntries>
__global__ void __launch_bounds__(256) gemv2_kernel(const TW* __restrict__ W, const float* __restrict__ b,
                                                    const float* __restrict__ in, float* __restrict__ out, int n,
                                                    int R, int Kd, int pre_silu) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float xs[];   // [n][Kd]
  for (int i = threadIdx.x; i < n * Kd; i += blockDim.x) {
    float z = in[i];
    if (pre_silu) z = z / (1.f + expf(-z));
    xs[i] = z;
  }
  __syncthreads();
  constexpr int V = GemvVec<TW>::V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = (blockIdx.x * 8 + warp) * 4;
  if (rb >= R) return;
  float acc[4][NMAX];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
#pragma unroll
    for (int e = 0; e < NMAX; ++e) acc[rr][e] = 0.f;
  const int kvec = (Kd / (32 * V)) * (32 * V);
  for (int k = lane * V; k < kvec; k += 32 * V) {
    float w[4][V];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int r = rb + rr < R ? rb + rr : R - 1;
      GemvVec<TW>::load(W + size_t(r) * Kd + k, w[rr]);
    }
#pragma unroll
    for (int e = 0; e < NMAX; ++e) {
      if (e < n) {
        float xv[V];
#pragma unroll
        for (int j = 0; j < V; ++j) xv[j] = xs[e * Kd + k + j];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int j = 0; j < V; ++j) acc[rr][e] += w[rr][j] * xv[j];
      }
    }
  }
  for (int k = kvec + lane; k < Kd; k += 32) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int r = rb + rr < R ? rb + rr : R - 1;
      const float wv = to_f(W[size_t(r) * Kd + k]);
#pragma unroll
      for (int e = 0; e < NMAX; ++e)
        if (e < n) acc[rr][e] += wv * xs[e * Kd + k];
    }
  }
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = rb + rr;
    if (r >= R) break;
#pragma unroll
    for (int e = 0; e < NMAX; ++e) {
      if (e < n) {
        const float s = warp_sum(acc[rr][e]);
        if (lane == 0) out[size_t(e) * R + r] = s + b[r];
      }
    }
  }
}

}  // namespace sdv2
