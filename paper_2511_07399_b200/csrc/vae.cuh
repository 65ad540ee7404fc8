// Stream-VAE stand-in ("Stream-VAE processes short
// video chunks (e.g., 4 frames) and caches intermediate features within each 3D
// convolution"), the first / last stage extras of the pipeline.
//
// Wan2.1-VAE-shaped (channels 96 / 192 / 384, 16 latent channels, 4 video frames per latent
// frame): every 3x3x3 conv is causal in time and runs on the tensor cores as an implicit
// GEMM over its own input buffer [T + 2][H][W][C] whose first two frames are the cache of
// the previous chunk (conv_tc.cuh); RMS + SiLU, 2x2 (x2) average pooling and nearest
// upsampling are channels-last elementwise kernels that write straight into the next
// conv's buffer.  Activations are bf16 channels-last with channels padded to multiples of
// 64 (96 -> 128; padded channels stay exactly zero), fp32 accumulation.
// Layer order (identical to the oracle's reading, oracle/vae.py, written independently):
//   encoder conv_in 3->c1, res(c1), pool 2x2, conv c1->c2, res(c2), pool 2x2x2, conv c2->c3,
//           res(c3), pool 2x2x2, res(c3), RMS-SiLU, conv c3->16
//   decoder conv_in 16->c3, res(c3), up x2x2x2, conv c3->c3, res(c3), up x2x2x2, conv c3->c2,
//           res(c2), up 2x2, conv c2->c1, res(c1), RMS-SiLU, conv c1->3
//   res(c) = x + conv(RMS-SiLU(conv(RMS-SiLU(x))))
#pragma once
#include <string>
#include <vector>

#include "conv_tc.cuh"

namespace sdv2 {

inline int vae_cs(int c) { return (c + 63) / 64 * 64; }   // stored channels

// RMS over the logical channels + gain + SiLU, one warp per pixel: in [P][Cs_in] -> out
// [P][Cs_out] (channels >= C of out are never written: they stay zero).
__global__ void __launch_bounds__(256) vae_norm_silu_kernel(const bf16* __restrict__ in, int cs_in, bf16* __restrict__ out,
                                                           int cs_out, const float* __restrict__ g, long long P, int C,
                                                           float eps) {
  pdl_wait();
  pdl_trigger();
  const long long p = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= P) return;
  const bf16* x = in + p * cs_in;
  float v[12];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < C ? __bfloat162float(x[c]) : 0.f;
    ss += v[i] * v[i];
  }
  const float inv = rsqrtf(warp_sum(ss) / float(C) + eps);
  bf16* y = out + p * cs_out;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const int c = lane + 32 * i;
    if (c < C) {
      const float z = g[c] * v[i] * inv;
      y[c] = __float2bfloat16_rn(z / (1.f + __expf(-z)));
    }
  }
}

// Average of 2x2 pixels (and of tf frames): in [T][H][W][Cs] -> out [T/tf][H/2][W/2][Cs].
__global__ void vae_pool_kernel(const bf16* __restrict__ in, bf16* __restrict__ out, int T, int H, int W, int Cs,
                                int tf) {
  pdl_wait();
  pdl_trigger();
  const int To = T / tf, Ho = H / 2, Wo = W / 2;
  const long long n = (long long)To * Ho * Wo * (Cs / 2);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c2 = int(i % (Cs / 2));
    long long r = i / (Cs / 2);
    const int wo = int(r % Wo);
    r /= Wo;
    const int ho = int(r % Ho);
    const int to = int(r / Ho);
    float ax = 0.f, ay = 0.f;
    for (int dt = 0; dt < tf; ++dt)
      for (int dh = 0; dh < 2; ++dh)
        for (int dw = 0; dw < 2; ++dw) {
          const size_t src = ((size_t(to * tf + dt) * H + 2 * ho + dh) * W + 2 * wo + dw) * Cs + 2 * c2;
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(in + src));
          ax += f.x;
          ay += f.y;
        }
    const float s = 1.f / float(4 * tf);
    *reinterpret_cast<__nv_bfloat162*>(out + ((size_t(to) * Ho + ho) * Wo + wo) * Cs + 2 * c2) =
        __floats2bfloat162_rn(ax * s, ay * s);
  }
}

// Nearest upsampling: in [T][H][W][Cs] -> out [T*tf][2H][2W][Cs].
__global__ void vae_up_kernel(const bf16* __restrict__ in, bf16* __restrict__ out, int T, int H, int W, int Cs, int tf) {
  pdl_wait();
  pdl_trigger();
  const int To = T * tf, Ho = 2 * H, Wo = 2 * W, C8 = Cs / 8;
  const long long n = (long long)To * Ho * Wo * C8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c8 = int(i % C8);
    long long r = i / C8;
    const int wo = int(r % Wo);
    r /= Wo;
    const int ho = int(r % Ho);
    const int to = int(r / Ho);
    const uint4 v = *reinterpret_cast<const uint4*>(in + ((size_t(to / tf) * H + ho / 2) * W + wo / 2) * Cs + 8 * c8);
    *reinterpret_cast<uint4*>(out + ((size_t(to) * Ho + ho) * Wo + wo) * Cs + 8 * c8) = v;
  }
}

// fp32 [C][T][H][W] (video chunk or latent) <-> bf16 channels-last [T][H][W][Cs].
__global__ void vae_cf_to_cl_kernel(const float* __restrict__ in, bf16* __restrict__ out, int C, int T, int H, int W,
                                    int Cs) {
  pdl_wait();
  pdl_trigger();
  const long long n = (long long)C * T * H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int w = int(i % W);
    long long r = i / W;
    const int h = int(r % H);
    r /= H;
    const int t = int(r % T);
    const int c = int(r / T);
    out[((size_t(t) * H + h) * W + w) * Cs + c] = __float2bfloat16_rn(in[i]);
  }
}
__global__ void vae_cl_to_cf_kernel(const bf16* __restrict__ in, float* __restrict__ out, int C, int T, int H, int W,
                                    int Cs) {
  pdl_wait();
  pdl_trigger();
  const long long n = (long long)C * T * H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int w = int(i % W);
    long long r = i / W;
    const int h = int(r % H);
    r /= H;
    const int t = int(r % T);
    const int c = int(r / T);
    out[i] = __bfloat162float(in[((size_t(t) * H + h) * W + w) * Cs + c]);
  }
}

// ------------------------------------------------------------------ host side
struct VaeAct {        // plain activation [T][H][W][Cs]
  bf16* p = nullptr;
  int T = 0, H = 0, W = 0, C = 0, Cs = 0;
  size_t frame() const { return size_t(H) * W * Cs; }
  long long pixels() const { return (long long)T * H * W; }
};

struct VaeConv {       // causal conv with its input buffer [T + 2][H][W][Cs_in] (2 cache frames first)
  bf16* in = nullptr;
  bf16* w = nullptr;   // [Cs_out][27 Cs_in]
  float* b = nullptr;  // [Cs_out]
  int T = 0, H = 0, W = 0, Cin = 0, Cout = 0;
  VaeAct in_frames() const {   // the chunk's frames inside the buffer
    VaeAct a;
    a.p = in + 2 * size_t(H) * W * vae_cs(Cin);
    a.T = T; a.H = H; a.W = W; a.C = Cin; a.Cs = vae_cs(Cin);
    return a;
  }
};

struct VaeRes {
  VaeConv c1, c2;
  float *n1 = nullptr, *n2 = nullptr;
  VaeAct tmp;          // output of c1
};

}  // namespace sdv2

struct sdv2_vae {
  sdv2_vae_desc d;
  int H = 0, W = 0, h = 0, w = 0;
  int c1 = 0, c2 = 0, c3 = 0, cl = 0, cv = 3;
  cudaStream_t stream = nullptr;
  sdv2::PFN_encodeTiled enc = nullptr;
  int num_sms = 148;
  std::string err;
  size_t ws_bytes = 0;
  // encoder
  sdv2::VaeConv e_in, e_c2, e_c3, e_out;
  sdv2::VaeRes e_r1, e_r2, e_r3, e_r4;
  sdv2::VaeAct ex[8];
  float* e_nout = nullptr;
  // decoder
  sdv2::VaeConv d_in, d_c2, d_c3, d_c4, d_out;
  sdv2::VaeRes d_r1, d_r2, d_r3, d_r4;
  sdv2::VaeAct dx[9];
  float* d_nout = nullptr;
  float* vid_stage = nullptr;   // [3][4][H][W] fp32
  float* lat_stage = nullptr;   // [cl][1][h][w] fp32
  std::vector<sdv2::VaeConv*> convs_enc, convs_dec;
  int64_t launches = 0;
};

namespace sdv2 {

struct VaeCarver {
  char* base;
  size_t off = 0;
  explicit VaeCarver(void* b) : base(b ? static_cast<char*>(b) : reinterpret_cast<char*>(uintptr_t(1) << 20)) {}
  template <typename T>
  T* take(size_t n) {
    off = (off + 1023) & ~size_t(1023);
    T* p = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
};

inline void vae_conv_carve(VaeCarver& cv, VaeConv& c, int T, int H, int W, int Cin, int Cout) {
  c.T = T; c.H = H; c.W = W; c.Cin = Cin; c.Cout = Cout;
  c.in = cv.take<bf16>(size_t(T + 2) * H * W * vae_cs(Cin));
  c.w = cv.take<bf16>(size_t(vae_cs(Cout)) * 27 * vae_cs(Cin));
  c.b = cv.take<float>(vae_cs(Cout));
}
inline VaeAct vae_act_carve(VaeCarver& cv, int T, int H, int W, int C) {
  VaeAct a;
  a.T = T; a.H = H; a.W = W; a.C = C; a.Cs = vae_cs(C);
  a.p = cv.take<bf16>(size_t(T) * H * W * a.Cs);
  return a;
}
inline void vae_res_carve(VaeCarver& cv, VaeRes& r, int T, int H, int W, int C) {
  vae_conv_carve(cv, r.c1, T, H, W, C, C);
  vae_conv_carve(cv, r.c2, T, H, W, C, C);
  r.n1 = cv.take<float>(C);
  r.n2 = cv.take<float>(C);
  r.tmp = vae_act_carve(cv, T, H, W, C);
}

// Workspace layout for the video H x W (4 frames per chunk) and the latent H/8 x W/8.
inline size_t vae_carve(sdv2_vae* v, void* base) {
  VaeCarver cv(base);
  const int H = v->H, W = v->W, c1 = v->c1, c2 = v->c2, c3 = v->c3, cl = v->cl, cvd = v->cv;
  // encoder: 4 frames at H x W, 4 at H/2, 2 at H/4, 1 at H/8
  vae_conv_carve(cv, v->e_in, 4, H, W, cvd, c1);
  v->ex[0] = vae_act_carve(cv, 4, H, W, c1);
  vae_res_carve(cv, v->e_r1, 4, H, W, c1);
  v->ex[1] = vae_act_carve(cv, 4, H, W, c1);
  vae_conv_carve(cv, v->e_c2, 4, H / 2, W / 2, c1, c2);
  v->ex[2] = vae_act_carve(cv, 4, H / 2, W / 2, c2);
  vae_res_carve(cv, v->e_r2, 4, H / 2, W / 2, c2);
  v->ex[3] = vae_act_carve(cv, 4, H / 2, W / 2, c2);
  vae_conv_carve(cv, v->e_c3, 2, H / 4, W / 4, c2, c3);
  v->ex[4] = vae_act_carve(cv, 2, H / 4, W / 4, c3);
  vae_res_carve(cv, v->e_r3, 2, H / 4, W / 4, c3);
  v->ex[5] = vae_act_carve(cv, 2, H / 4, W / 4, c3);
  v->ex[6] = vae_act_carve(cv, 1, H / 8, W / 8, c3);
  vae_res_carve(cv, v->e_r4, 1, H / 8, W / 8, c3);
  v->ex[7] = vae_act_carve(cv, 1, H / 8, W / 8, c3);
  v->e_nout = cv.take<float>(c3);
  vae_conv_carve(cv, v->e_out, 1, H / 8, W / 8, c3, cl);
  // decoder: 1 frame at H/8, 2 at H/4, 4 at H/2, 4 at H
  vae_conv_carve(cv, v->d_in, 1, H / 8, W / 8, cl, c3);
  v->dx[0] = vae_act_carve(cv, 1, H / 8, W / 8, c3);
  vae_res_carve(cv, v->d_r1, 1, H / 8, W / 8, c3);
  v->dx[1] = vae_act_carve(cv, 1, H / 8, W / 8, c3);
  vae_conv_carve(cv, v->d_c2, 2, H / 4, W / 4, c3, c3);
  v->dx[2] = vae_act_carve(cv, 2, H / 4, W / 4, c3);
  vae_res_carve(cv, v->d_r2, 2, H / 4, W / 4, c3);
  v->dx[3] = vae_act_carve(cv, 2, H / 4, W / 4, c3);
  vae_conv_carve(cv, v->d_c3, 4, H / 2, W / 2, c3, c2);
  v->dx[4] = vae_act_carve(cv, 4, H / 2, W / 2, c2);
  vae_res_carve(cv, v->d_r3, 4, H / 2, W / 2, c2);
  v->dx[5] = vae_act_carve(cv, 4, H / 2, W / 2, c2);
  vae_conv_carve(cv, v->d_c4, 4, H, W, c2, c1);
  v->dx[6] = vae_act_carve(cv, 4, H, W, c1);
  vae_res_carve(cv, v->d_r4, 4, H, W, c1);
  v->dx[7] = vae_act_carve(cv, 4, H, W, c1);
  v->d_nout = cv.take<float>(c1);
  vae_conv_carve(cv, v->d_out, 4, H, W, c1, cvd);
  v->dx[8] = vae_act_carve(cv, 4, H, W, cvd);
  v->vid_stage = cv.take<float>(size_t(cvd) * 4 * H * W);
  v->lat_stage = cv.take<float>(size_t(cl) * (H / 8) * (W / 8));
  v->convs_enc = {&v->e_in, &v->e_r1.c1, &v->e_r1.c2, &v->e_c2, &v->e_r2.c1, &v->e_r2.c2, &v->e_c3,
                  &v->e_r3.c1, &v->e_r3.c2, &v->e_r4.c1, &v->e_r4.c2, &v->e_out};
  v->convs_dec = {&v->d_in, &v->d_r1.c1, &v->d_r1.c2, &v->d_c2, &v->d_r2.c1, &v->d_r2.c2, &v->d_c3,
                  &v->d_r3.c1, &v->d_r3.c2, &v->d_c4, &v->d_r4.c1, &v->d_r4.c2, &v->d_out};
  return cv.off + 1024;
}

}  // namespace sdv2

namespace sdv2 {

#define VK(call)                                                          \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess) {                                              \
      v->err = std::string(#call) + ": " + cudaGetErrorString(e_);        \
      return SDV2_E_CUDA;                                                 \
    }                                                                     \
  } while (0)

inline int vae_grid(long long n) { return int(std::min<long long>((n + 255) / 256, 148LL * 16)); }

// copy the last two input frames of the previous chunk to the front (the causal cache)
inline sdv2_status vae_shift(sdv2_vae* v, const VaeConv& c) {
  const size_t fr = size_t(c.H) * c.W * vae_cs(c.Cin) * sizeof(bf16);
  if (c.T >= 2) {
    VK(cudaMemcpyAsync(c.in, reinterpret_cast<char*>(c.in) + c.T * fr, 2 * fr, cudaMemcpyDeviceToDevice, v->stream));
  } else {   // T = 1: frames 1, 2 -> 0, 1 (non-overlapping one at a time)
    VK(cudaMemcpyAsync(c.in, reinterpret_cast<char*>(c.in) + fr, fr, cudaMemcpyDeviceToDevice, v->stream));
    VK(cudaMemcpyAsync(reinterpret_cast<char*>(c.in) + fr, reinterpret_cast<char*>(c.in) + 2 * fr, fr,
                       cudaMemcpyDeviceToDevice, v->stream));
  }
  return SDV2_OK;
}

inline sdv2_status vae_conv(sdv2_vae* v, const VaeConv& c, const VaeAct& out, const VaeAct* res) {
  ConvArgs a{};
  a.T = c.T; a.H = c.H; a.W = c.W;
  a.Cin = vae_cs(c.Cin);
  a.Cout = vae_cs(c.Cout);
  a.bias = c.b;
  a.res = res ? res->p : nullptr;
  a.out = out.p;
  ++v->launches;
  if (!tc_conv3d(v->stream, v->enc, v->num_sms, c.in, c.w, a, &v->err)) return SDV2_E_CUDA;
  return SDV2_OK;
}

inline sdv2_status vae_norm(sdv2_vae* v, const VaeAct& x, const float* g, const VaeAct& dst) {
  const long long P = x.pixels();
  vae_norm_silu_kernel<<<int((P + 7) / 8), 256, 0, v->stream>>>(x.p, x.Cs, dst.p, dst.Cs, g, P, x.C, v->d.eps);
  ++v->launches;
  VK(cudaGetLastError());
  return SDV2_OK;
}

#define VTRY(x)                        \
  do {                                 \
    sdv2_status s_ = (x);              \
    if (s_ != SDV2_OK) return s_;      \
  } while (0)

inline sdv2_status vae_res(sdv2_vae* v, const VaeRes& r, const VaeAct& x, const VaeAct& out) {
  VTRY(vae_norm(v, x, r.n1, r.c1.in_frames()));
  VTRY(vae_conv(v, r.c1, r.tmp, nullptr));
  VTRY(vae_norm(v, r.tmp, r.n2, r.c2.in_frames()));
  return vae_conv(v, r.c2, out, &x);
}

inline sdv2_status vae_pool(sdv2_vae* v, const VaeAct& x, const VaeAct& dst, int tf) {
  const long long n = (long long)(x.T / tf) * (x.H / 2) * (x.W / 2) * (x.Cs / 2);
  vae_pool_kernel<<<vae_grid(n), 256, 0, v->stream>>>(x.p, dst.p, x.T, x.H, x.W, x.Cs, tf);
  ++v->launches;
  VK(cudaGetLastError());
  return SDV2_OK;
}

inline sdv2_status vae_up(sdv2_vae* v, const VaeAct& x, const VaeAct& dst, int tf) {
  const long long n = (long long)(x.T * tf) * (2 * x.H) * (2 * x.W) * (x.Cs / 8);
  vae_up_kernel<<<vae_grid(n), 256, 0, v->stream>>>(x.p, dst.p, x.T, x.H, x.W, x.Cs, tf);
  ++v->launches;
  VK(cudaGetLastError());
  return SDV2_OK;
}

// pack a logical conv weight [co][3][3][3][ci] + bias (fp32, host or device) into the padded
// bf16 K-major layout [Cs_out][27][Cs_in]
inline sdv2_status vae_load_conv(sdv2_vae* v, VaeConv& c, const void* w, const void* b) {
  const int co = c.Cout, ci = c.Cin, cso = vae_cs(co), csi = vae_cs(ci);
  std::vector<float> hw(size_t(co) * 27 * ci), hb(co);
  VK(cudaMemcpy(hw.data(), w, hw.size() * 4, cudaMemcpyDefault));
  VK(cudaMemcpy(hb.data(), b, hb.size() * 4, cudaMemcpyDefault));
  std::vector<bf16> pw(size_t(cso) * 27 * csi, __float2bfloat16_rn(0.f));
  std::vector<float> pb(cso, 0.f);
  for (int o = 0; o < co; ++o) {
    pb[o] = hb[o];
    for (int tap = 0; tap < 27; ++tap)
      for (int i = 0; i < ci; ++i)
        pw[(size_t(o) * 27 + tap) * csi + i] = __float2bfloat16_rn(hw[(size_t(o) * 27 + tap) * ci + i]);
  }
  VK(cudaMemcpy(c.w, pw.data(), pw.size() * sizeof(bf16), cudaMemcpyHostToDevice));
  VK(cudaMemcpy(c.b, pb.data(), pb.size() * 4, cudaMemcpyHostToDevice));
  return SDV2_OK;
}

inline sdv2_status vae_load_vec(sdv2_vae* v, float* dst, const void* src, int n) {
  VK(cudaMemcpy(dst, src, size_t(n) * 4, cudaMemcpyDefault));
  return SDV2_OK;
}

inline sdv2_status vae_fill(sdv2_vae* v, const sdv2_vae_desc* d) {
  if (!d) return SDV2_E_INVALID;
  v->d = *d;
  v->H = d->video_h;
  v->W = d->video_w;
  v->c1 = d->dims[0]; v->c2 = d->dims[1]; v->c3 = d->dims[2];
  v->cl = d->latent_channels;
  v->cv = 3;
  if (v->H < 8 || v->W < 8 || v->H % 8 || v->W % 8) return SDV2_E_SHAPE;
  for (int c : {v->c1, v->c2, v->c3, v->cl})
    if (c < 1 || c > 384) return SDV2_E_SHAPE;
  v->h = v->H / 8;
  v->w = v->W / 8;
  return SDV2_OK;
}

}  // namespace sdv2

extern "C" {

size_t sdv2_vae_workspace_bytes(const sdv2_vae_desc* d) {
  sdv2_vae tmp;
  if (sdv2::vae_fill(&tmp, d) != SDV2_OK) return 0;
  return sdv2::vae_carve(&tmp, nullptr);
}

sdv2_status sdv2_vae_create(const sdv2_vae_desc* d, const sdv2_weights* wts, void* workspace, size_t bytes,
                            int device, void* stream, sdv2_vae** out) {
  using namespace sdv2;
  if (!out) return SDV2_E_INVALID;
  *out = nullptr;
  auto* v = new sdv2_vae();
  sdv2_status s = vae_fill(v, d);
  if (s != SDV2_OK) {
    delete v;
    return s;
  }
  const size_t need = vae_carve(v, nullptr);
  if (!workspace || bytes < need) {
    delete v;
    return SDV2_E_WORKSPACE;
  }
  char* base = static_cast<char*>(workspace);
  const size_t adj = (1024 - (reinterpret_cast<uintptr_t>(base) & 1023)) & 1023;
  if (bytes < need + adj) {
    delete v;
    return SDV2_E_WORKSPACE;
  }
  *out = v;   // returned even on failure below (sdv2_vae_last_error, then destroy)
  if (cudaSetDevice(device) != cudaSuccess) return SDV2_E_CUDA;
  v->stream = static_cast<cudaStream_t>(stream);
  v->ws_bytes = bytes;
  vae_carve(v, base + adj);
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      v->err = "cuTensorMapEncodeTiled unavailable";
      return SDV2_E_CUDA;
    }
    v->enc = reinterpret_cast<PFN_encodeTiled>(fn);
    cudaDeviceGetAttribute(&v->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (!conv_attr()) {
      v->err = "conv3d kernel attribute";
      return SDV2_E_CUDA;
    }
  }
  if (cudaMemsetAsync(base + adj, 0, need - 1024, v->stream) != cudaSuccess) return SDV2_E_CUDA;
  // weights in the order of the layer list: conv (w, b); res (n1, c1.w, c1.b, n2, c2.w, c2.b); norm (g)
  if (!wts || !wts->tensors) return SDV2_E_INVALID;
  const void* const* T = wts->tensors;
  int i = 0;
  auto conv = [&](VaeConv& c) -> sdv2_status {
    if (i + 2 > wts->count) return SDV2_E_INVALID;
    sdv2_status st = vae_load_conv(v, c, T[i], T[i + 1]);
    i += 2;
    return st;
  };
  auto res = [&](VaeRes& r) -> sdv2_status {
    if (i + 6 > wts->count) return SDV2_E_INVALID;
    VTRY(vae_load_vec(v, r.n1, T[i], r.c1.Cin));
    VTRY(vae_load_conv(v, r.c1, T[i + 1], T[i + 2]));
    VTRY(vae_load_vec(v, r.n2, T[i + 3], r.c2.Cin));
    VTRY(vae_load_conv(v, r.c2, T[i + 4], T[i + 5]));
    i += 6;
    return SDV2_OK;
  };
  auto norm = [&](float* g, int c) -> sdv2_status {
    if (i + 1 > wts->count) return SDV2_E_INVALID;
    return vae_load_vec(v, g, T[i++], c);
  };
  VTRY(conv(v->e_in)); VTRY(res(v->e_r1)); VTRY(conv(v->e_c2)); VTRY(res(v->e_r2)); VTRY(conv(v->e_c3));
  VTRY(res(v->e_r3)); VTRY(res(v->e_r4)); VTRY(norm(v->e_nout, v->c3)); VTRY(conv(v->e_out));
  VTRY(conv(v->d_in)); VTRY(res(v->d_r1)); VTRY(conv(v->d_c2)); VTRY(res(v->d_r2)); VTRY(conv(v->d_c3));
  VTRY(res(v->d_r3)); VTRY(conv(v->d_c4)); VTRY(res(v->d_r4)); VTRY(norm(v->d_nout, v->c1)); VTRY(conv(v->d_out));
  if (i != wts->count) {
    v->err = "weight count mismatch: expected " + std::to_string(i);
    return SDV2_E_INVALID;
  }
  if (cudaStreamSynchronize(v->stream) != cudaSuccess) return SDV2_E_CUDA;
  return SDV2_OK;
}

sdv2_status sdv2_vae_reset(sdv2_vae* v) {
  using namespace sdv2;
  if (!v) return SDV2_E_INVALID;
  for (auto* list : {&v->convs_enc, &v->convs_dec})
    for (VaeConv* c : *list)
      VK(cudaMemsetAsync(c->in, 0, size_t(c->T + 2) * c->H * c->W * vae_cs(c->Cin) * sizeof(bf16), v->stream));
  return SDV2_OK;
}

sdv2_status sdv2_vae_encode_chunk(sdv2_vae* v, const float* video, float* latent) {
  using namespace sdv2;
  if (!v || !video || !latent) return SDV2_E_INVALID;
  for (VaeConv* c : v->convs_enc) VTRY(vae_shift(v, *c));
  VK(cudaMemcpyAsync(v->vid_stage, video, size_t(3) * 4 * v->H * v->W * 4, cudaMemcpyDefault, v->stream));
  {
    const VaeAct dst = v->e_in.in_frames();
    const long long n = 3LL * 4 * v->H * v->W;
    vae_cf_to_cl_kernel<<<vae_grid(n), 256, 0, v->stream>>>(v->vid_stage, dst.p, 3, 4, v->H, v->W, dst.Cs);
    ++v->launches;
    VK(cudaGetLastError());
  }
  VTRY(vae_conv(v, v->e_in, v->ex[0], nullptr));
  VTRY(vae_res(v, v->e_r1, v->ex[0], v->ex[1]));
  VTRY(vae_pool(v, v->ex[1], v->e_c2.in_frames(), 1));
  VTRY(vae_conv(v, v->e_c2, v->ex[2], nullptr));
  VTRY(vae_res(v, v->e_r2, v->ex[2], v->ex[3]));
  VTRY(vae_pool(v, v->ex[3], v->e_c3.in_frames(), 2));
  VTRY(vae_conv(v, v->e_c3, v->ex[4], nullptr));
  VTRY(vae_res(v, v->e_r3, v->ex[4], v->ex[5]));
  VTRY(vae_pool(v, v->ex[5], v->ex[6], 2));
  VTRY(vae_res(v, v->e_r4, v->ex[6], v->ex[7]));
  VTRY(vae_norm(v, v->ex[7], v->e_nout, v->e_out.in_frames()));
  VaeAct y;
  y.p = v->dx[8].p;   // reuse: the decoder's output buffer is idle during an encode
  y.T = 1; y.H = v->h; y.W = v->w; y.C = v->cl; y.Cs = vae_cs(v->cl);
  VTRY(vae_conv(v, v->e_out, y, nullptr));
  {
    const long long n = (long long)v->cl * v->h * v->w;
    vae_cl_to_cf_kernel<<<vae_grid(n), 256, 0, v->stream>>>(y.p, v->lat_stage, v->cl, 1, v->h, v->w, y.Cs);
    ++v->launches;
    VK(cudaGetLastError());
  }
  VK(cudaMemcpyAsync(latent, v->lat_stage, size_t(v->cl) * v->h * v->w * 4, cudaMemcpyDefault, v->stream));
  return SDV2_OK;
}

sdv2_status sdv2_vae_decode_chunk(sdv2_vae* v, const float* latent, float* video) {
  using namespace sdv2;
  if (!v || !video || !latent) return SDV2_E_INVALID;
  for (VaeConv* c : v->convs_dec) VTRY(vae_shift(v, *c));
  VK(cudaMemcpyAsync(v->lat_stage, latent, size_t(v->cl) * v->h * v->w * 4, cudaMemcpyDefault, v->stream));
  {
    const VaeAct dst = v->d_in.in_frames();
    const long long n = (long long)v->cl * v->h * v->w;
    vae_cf_to_cl_kernel<<<vae_grid(n), 256, 0, v->stream>>>(v->lat_stage, dst.p, v->cl, 1, v->h, v->w, dst.Cs);
    ++v->launches;
    VK(cudaGetLastError());
  }
  VTRY(vae_conv(v, v->d_in, v->dx[0], nullptr));
  VTRY(vae_res(v, v->d_r1, v->dx[0], v->dx[1]));
  VTRY(vae_up(v, v->dx[1], v->d_c2.in_frames(), 2));
  VTRY(vae_conv(v, v->d_c2, v->dx[2], nullptr));
  VTRY(vae_res(v, v->d_r2, v->dx[2], v->dx[3]));
  VTRY(vae_up(v, v->dx[3], v->d_c3.in_frames(), 2));
  VTRY(vae_conv(v, v->d_c3, v->dx[4], nullptr));
  VTRY(vae_res(v, v->d_r3, v->dx[4], v->dx[5]));
  VTRY(vae_up(v, v->dx[5], v->d_c4.in_frames(), 1));
  VTRY(vae_conv(v, v->d_c4, v->dx[6], nullptr));
  VTRY(vae_res(v, v->d_r4, v->dx[6], v->dx[7]));
  VTRY(vae_norm(v, v->dx[7], v->d_nout, v->d_out.in_frames()));
  VTRY(vae_conv(v, v->d_out, v->dx[8], nullptr));
  {
    const long long n = 3LL * 4 * v->H * v->W;
    vae_cl_to_cf_kernel<<<vae_grid(n), 256, 0, v->stream>>>(v->dx[8].p, v->vid_stage, 3, 4, v->H, v->W, v->dx[8].Cs);
    ++v->launches;
    VK(cudaGetLastError());
  }
  VK(cudaMemcpyAsync(video, v->vid_stage, size_t(3) * 4 * v->H * v->W * 4, cudaMemcpyDefault, v->stream));
  return SDV2_OK;
}

int64_t sdv2_vae_launches(const sdv2_vae* v) { return v ? v->launches : 0; }
const char* sdv2_vae_last_error(const sdv2_vae* v) { return v ? v->err.c_str() : "null handle"; }

sdv2_status sdv2_vae_destroy(sdv2_vae* v) {
  if (!v) return SDV2_E_INVALID;
  if (v->stream || v->enc) cudaStreamSynchronize(v->stream);
  delete v;
  return SDV2_OK;
}

}  // extern "C"
