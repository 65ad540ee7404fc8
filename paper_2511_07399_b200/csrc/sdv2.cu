// libsdv2: C-ABI implementation (include/sdv2.h) — workspace carving, weight
// packing, prompt conditioning and the per-call stage-tick orchestration.
//
// One call = one stage-tick (reading R2 in DESIGN.md): this rank runs every active
// (chunk, step) entry of micro-batch `call` through its DiT blocks, all entries
// batched into the same GEMMs (Stream Batch, P:164 / P:227).  Rank 0 additionally
// runs the motion-aware noise controller, patch embedding and time
// conditioning; the last rank runs the head, x0 prediction and re-noising.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <type_traits>
#include <utility>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <map>

#include "../../include/sdv2.h"
#include "ctl.h"
#include "gemm_tc.cuh"
#include "attn_tc.cuh"
#include "xattn_tc.cuh"
#include "vae.cuh"
#include "elem.cuh"
#include "kernels.cuh"

using namespace sdv2;

namespace {

constexpr int kNumGlobal = 15;
constexpr int kNumBlockT = 27;
constexpr int kTdRing = 16;
constexpr int kMaxTOff = 4096 + 16;
constexpr int kMaxSMs = 160;

enum GlobalT { G_PATCH_W, G_PATCH_B, G_TXT1_W, G_TXT1_B, G_TXT2_W, G_TXT2_B, G_T1_W, G_T1_B, G_T2_W, G_T2_B,
               G_TP_W, G_TP_B, G_HEAD_MOD, G_HEAD_W, G_HEAD_B };
enum BlockT { B_MOD, B_WQ, B_BQ, B_WK, B_BK, B_WV, B_BV, B_WO, B_BO, B_GQ, B_GK, B_N3G, B_N3B, B_WCQ, B_BCQ,
              B_WCK, B_BCK, B_WCV, B_BCV, B_WCO, B_BCO, B_GCQ, B_GCK, B_W1, B_B1, B_W2, B_B2 };

struct Carver {
  char* base;
  size_t off = 0;
  // sizing mode (b == nullptr) carves from a dummy base; the pointers are never used
  explicit Carver(void* b) : base(b ? static_cast<char*>(b) : reinterpret_cast<char*>(uintptr_t(1) << 20)) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 1023) & ~size_t(1023);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
};

// Per-block packed weights (TW = float or bf16 for the matrices; vectors fp32).
struct BlockW {
  float* mod;                 // [6, d]
  void* wqkv; float* bqkv;    // [3d, d], [3d]
  void* wo; float* bo;
  float *gq, *gk, *n3g, *n3b;
  void* wcq; float* bcq;
  void* wck; float* bck;
  void* wcv; float* bcv;
  void* wco; float* bco;
  float *gcq, *gck;
  float* gkq;                 // [d] g_ck * g_cq: prompt K with the cross-q gain folded in (fused q RMS)
  void* w1; float* b1;        // [F, d]
  void* w2; float* b2;        // [d, F]
};

// Tick packet: the residual stream and everything a downstream stage needs.
struct Packet {
  float* x;     // [n L, d]
  float* e0;    // [n, 6d]
  float* e;     // [n, d]
  float* sig;   // [n]
  float* sign;  // [n]
  float* lat;   // [n, CTHW]
  size_t bytes;
  size_t nx = 0, ne0 = 0, ne = 0;   // element counts of x, e0, e
};

}  // namespace

struct sdv2_handle {
  sdv2_model_desc md;
  sdv2_geometry g;
  sdv2_precision prec;
  int K = 1, rank = 0, b0 = 0, b1 = 0, nb = 0;   // active global blocks [b0, b1); nb = resident count
  int r0 = 0;                                     // first resident (weights + KV carved) global block
  int a0 = 0, a1 = 0;                             // active range as resident-local indices
  int d, H, hd, F, C, T, hh, ww, L, n, m, W, S, Lt, Dt, CTHW, Mmax, P;
  int B = 1;                  // streams batched per call (SLO batch)
  int NE = 1;                 // entries per call = B n (entry e = j B + b = KV lane e)
  int hn, wn, ct, ch, cw;
  size_t ta;  // bytes per activation element
  cudaStream_t stream = nullptr;
  int device = 0;

  // workspace
  float* gw[kNumGlobal];      // global weights (fp32 except tp_w which is TW)
  void* tp_w;
  std::vector<BlockW> bw;
  char* packet_base;          // tick state (packet layout)
  Packet st;
  char* act_io[2][2];         // [in/out][parity]
  float* ring[2][2];          // [in/out][parity] ring-closure latents [B (n-1), CTHW]
  float* lat_in;              // staged caller chunks [B, CTHW]
  float* prev_frame;          // [B, C h w]
  float* out_stage;           // [B, CTHW]
  CtrlState* ctrl;            // [B]
  float* emb;                 // [B n, 256]
  float* u;                   // patchified tokens [Mmax, 4C] fp32
  float* yh;                  // head output [Mmax, 4C] fp32
  float* attn_part;           // stream-K attention partials
  float* rowsq;               // [Mmax][d / 32] partial sums of squares of the raw cross q rows (fused q RMS)
  int* attn_flags;            // [kMaxSMs] split-unit hand-off flags (zero between launches)
  void* head_w_tw;            // head weight [4C, d] TW
  float* t1;                  // [B n, d]
  void* a;                    // [Mmax, d] TA
  void* qkv;                  // [Mmax, 3d] TA
  void* q;                    // [Mmax, d] TA
  void* o;                    // [Mmax, d] TA
  void* hbuf;                 // [Mmax, F] TA
  float* staging;             // weight staging (aliases the activation scratch)
  size_t staging_elems;
  void* Kc; void* Vc;         // KV lanes [nb][B n][S][L][d] TA
  void* Kx; void* Vx;         // prompt K/V [B][2 versions][nb][Lt][d] TA
  float* prompt;              // [Lt, Dt]
  float* ctx;                 // [Lt, d]
  float* ctx_tmp;             // [Lt, d]
  float* rope;                // tables
  RopeTabs rt;
  TickDesc* td_dev;
  TickDesc* td_host = nullptr;   // pinned ring: [kTdRing] call descriptors, then [kTdRing] clean-pass ones
  // kv_mode 1 (clean re-run): the previous call's descriptor (its entries are re-run with
  // rebase cleared), the device copy the clean pass reads, sigma = 0 per entry
  TickDesc td_prev;
  bool td_prev_valid = false;
  TickDesc* td_clean_dev = nullptr;
  float* sig_zero = nullptr;
  double* motion_part = nullptr;      // [B][kMaxFrames][kMotionSlices] motion partial sums
  unsigned* motion_arrive = nullptr;  // [B] CTA arrival counters (zero between calls)
  cudaGraphExec_t clean_graph_exec[kMaxEntries + 1] = {};
  int64_t clean_graph_launches[kMaxEntries + 1] = {};
  cudaEvent_t td_ev[kTdRing];
  bool td_ev_used[kTdRing];
  size_t ws_bytes;

  // state
  Control ctl;
  bool stream_ready = false;
  StreamCfg scfg;
  int T_reset = 1;
  int pver[kMaxEntries] = {};                 // prompt version per stream
  float* tap = nullptr;
  sdv2_tick_info info;
  std::string err;
  TmaGemmPlan gplan;
  AttnPlan aplan;
  int64_t launches = 0;
  TickDesc* td_host_cur = nullptr;
  // CUDA graphs of the call body, keyed by (active entries, call parity)
  bool graphs = true;
  bool debug_sync = false;   // test hook: synchronise + log after every launch (graphs off)
  bool pdl = true;        // programmatic dependent launch (sdv2_exec_options.pdl): +2 % fps measured
  bool tune = true;       // create-time GEMM tile tuning (sdv2_exec_options.tune_gemms)
  bool l2_persist = true;    // sdv2_exec_options.l2_persist
  std::vector<int32_t> gemm_table;   // sdv2_exec_options.gemm_table (records of 8)
  int64_t last_switch_call[kMaxEntries];   // call index of stream b's last sdv2_set_prompt (-1: none)
  cudaGraphExec_t graph_exec[2 * (kMaxEntries + 1)] = {};
  int64_t graph_launches[2 * (kMaxEntries + 1)] = {};
  // profiling (sdv2_profile_enable): event pairs around each launch, per class
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  struct ProfRec { int cls; double flops; cudaEvent_t a, b; int blk; };
  std::vector<ProfRec> prof_recs;
  sdv2_profile prof_acc;
  std::vector<double> prof_blk_ms;     // [nb] summed block-span ms (class 4) per resident block
  std::vector<int64_t> prof_blk_n;
};

namespace {
// Profiling scope: records an event pair around the launches of one kernel class.
struct ProfScope {
  sdv2_handle* h;
  int cls;
  double flops;
  int blk;
  cudaEvent_t a = nullptr;
  ProfScope(sdv2_handle* h_, int c, double f, int blk_ = -1) : h(h_), cls(c), flops(f), blk(blk_) {
    if (!h->prof) return;
    if (h->ev_next + 2 > h->ev_pool.size()) {
      for (int i = 0; i < 256; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        h->ev_pool.push_back(e);
      }
    }
    a = h->ev_pool[h->ev_next++];
    cudaEventRecord(a, h->stream);
  }
  ~ProfScope() {
    if (!h->prof || !a) return;
    cudaEvent_t b = h->ev_pool[h->ev_next++];
    cudaEventRecord(b, h->stream);
    h->prof_recs.push_back({cls, flops, a, b, blk});
  }
};
}  // namespace

namespace {

// Point the packet fields at `base` (the layout is the same in every packet buffer).
void set_packet(sdv2_handle* h, char* base) {
  float* p = reinterpret_cast<float*>(base);
  h->st.x = p; p += h->st.nx;
  h->st.e0 = p; p += h->st.ne0;
  h->st.e = p; p += h->st.ne;
  h->st.sig = p; p += 64;
  h->st.sign = p; p += 64;
  h->st.lat = p;
}

// Where call parity `par` computes its packet: in place in the hand-off buffers, so no
// stage copies the packet (K = 1: the handle's own packet; rank 0: the outgoing buffer;
// ranks > 0: the received buffer, which is also what they send on).
char* packet_for(sdv2_handle* h, int par) {
  if (h->K == 1) return h->packet_base;
  return h->rank == 0 ? h->act_io[1][par] : h->act_io[0][par];
}

size_t carve(sdv2_handle* h, void* base) {
  Carver cv(base);
  const size_t TWb = h->prec == SDV2_BF16 ? 2 : 4;
  const int d = h->d, F = h->F, P = h->P;
  auto tw = [&](size_t cnt) -> void* { return cv.take<char>(cnt * TWb); };
  h->gw[G_PATCH_W] = cv.take<float>(size_t(d) * P);
  h->gw[G_PATCH_B] = cv.take<float>(d);
  h->gw[G_TXT1_W] = cv.take<float>(size_t(d) * h->Dt);
  h->gw[G_TXT1_B] = cv.take<float>(d);
  h->gw[G_TXT2_W] = cv.take<float>(size_t(d) * d);
  h->gw[G_TXT2_B] = cv.take<float>(d);
  h->gw[G_T1_W] = cv.take<float>(size_t(d) * h->md.freq_dim);
  h->gw[G_T1_B] = cv.take<float>(d);
  h->gw[G_T2_W] = cv.take<float>(size_t(d) * d);
  h->gw[G_T2_B] = cv.take<float>(d);
  h->gw[G_TP_W] = nullptr;
  h->tp_w = tw(size_t(6) * d * d);
  h->gw[G_TP_B] = cv.take<float>(6 * d);
  h->gw[G_HEAD_MOD] = cv.take<float>(2 * d);
  h->gw[G_HEAD_W] = cv.take<float>(size_t(P) * d);
  h->gw[G_HEAD_B] = cv.take<float>(P);
  h->head_w_tw = tw(size_t(P) * d);
  h->bw.assign(h->nb, BlockW{});
  for (int b = 0; b < h->nb; ++b) {
    BlockW& B = h->bw[b];
    B.mod = cv.take<float>(6 * d);
    B.wqkv = tw(size_t(3) * d * d); B.bqkv = cv.take<float>(3 * d);
    B.wo = tw(size_t(d) * d); B.bo = cv.take<float>(d);
    B.gq = cv.take<float>(d); B.gk = cv.take<float>(d);
    B.n3g = cv.take<float>(d); B.n3b = cv.take<float>(d);
    B.wcq = tw(size_t(d) * d); B.bcq = cv.take<float>(d);
    B.wck = tw(size_t(d) * d); B.bck = cv.take<float>(d);
    B.wcv = tw(size_t(d) * d); B.bcv = cv.take<float>(d);
    B.wco = tw(size_t(d) * d); B.bco = cv.take<float>(d);
    B.gcq = cv.take<float>(d); B.gck = cv.take<float>(d);
    B.gkq = cv.take<float>(d);
    B.w1 = tw(size_t(F) * d); B.b1 = cv.take<float>(F);
    B.w2 = tw(size_t(d) * F); B.b2 = cv.take<float>(d);
  }
  // packet (tick state) — contiguous so it can be shipped as one message
  {
    const size_t x = size_t(h->Mmax) * d, e0 = size_t(h->NE) * 6 * d, e = size_t(h->NE) * d,
                 lat = size_t(h->NE) * h->CTHW;
    const size_t sz = (x + e0 + e + 2 * 64 + lat) * 4;
    h->st.bytes = sz;
    h->st.nx = x; h->st.ne0 = e0; h->st.ne = e;
    h->packet_base = cv.take<char>(sz);
    set_packet(h, h->packet_base);
    for (int io = 0; io < 2; ++io)
      for (int par = 0; par < 2; ++par) h->act_io[io][par] = h->K > 1 ? cv.take<char>(sz) : nullptr;
  }
  const size_t ring_elems = size_t(h->n > 1 ? h->n - 1 : 1) * h->B * h->CTHW;
  for (int io = 0; io < 2; ++io)
    for (int par = 0; par < 2; ++par) h->ring[io][par] = cv.take<float>(ring_elems);
  h->lat_in = cv.take<float>(size_t(h->B) * h->CTHW);
  h->prev_frame = cv.take<float>(size_t(h->B) * h->C * h->hh * h->ww);
  h->out_stage = cv.take<float>(size_t(h->B) * h->CTHW);
  h->ctrl = cv.take<CtrlState>(h->B);
  h->emb = cv.take<float>(size_t(h->NE) * h->md.freq_dim);
  h->u = cv.take<float>(size_t(h->Mmax) * h->P);
  h->yh = cv.take<float>(size_t(h->Mmax) * h->P);
  h->attn_part = cv.take<float>(attn_scratch_floats(kMaxSMs, h->hd));
  h->rowsq = cv.take<float>(size_t(h->Mmax) * (h->d / 32));
  h->attn_flags = cv.take<int>(kMaxSMs);
  h->t1 = cv.take<float>(size_t(h->NE) * d);
  // activation scratch, aliased by the weight staging buffer during create
  {
    const size_t act = (size_t(h->Mmax) * d * 3 + size_t(h->Mmax) * 3 * d + size_t(h->Mmax) * F) * h->ta + 5 * 1024;
    size_t maxw = size_t(F) * d;
    maxw = std::max(maxw, size_t(6) * d * d);
    maxw = std::max(maxw, size_t(d) * h->Dt);
    const size_t stag = maxw * 4;
    const size_t sz = std::max(act, stag);
    char* s = cv.take<char>(sz);
    h->staging = reinterpret_cast<float*>(s);
    h->staging_elems = maxw;
    Carver sub(s);
    h->a = sub.take<char>(size_t(h->Mmax) * d * h->ta);
    h->qkv = sub.take<char>(size_t(h->Mmax) * 3 * d * h->ta);
    h->q = sub.take<char>(size_t(h->Mmax) * d * h->ta);
    h->o = sub.take<char>(size_t(h->Mmax) * d * h->ta);
    h->hbuf = sub.take<char>(size_t(h->Mmax) * F * h->ta);
  }
  const size_t kv = size_t(h->nb) * h->NE * h->S * h->L * d;
  h->Kc = cv.take<char>(kv * h->ta);
  h->Vc = cv.take<char>(kv * h->ta);
  const size_t px = size_t(2) * h->B * h->nb * h->Lt * d;
  h->Kx = cv.take<char>(px * h->ta);
  h->Vx = cv.take<char>(px * h->ta);
  h->prompt = cv.take<float>(size_t(h->Lt) * h->Dt);
  h->ctx = cv.take<float>(size_t(h->Lt) * d);
  h->ctx_tmp = cv.take<float>(size_t(h->Lt) * d);
  const size_t rope_elems = size_t(2 * kMaxTOff + 1) * h->ct * 2 + size_t(h->hn) * h->ch * 2 + size_t(h->wn) * h->cw * 2;
  h->rope = cv.take<float>(rope_elems);
  h->td_dev = cv.take<TickDesc>(1);
  h->td_clean_dev = cv.take<TickDesc>(1);
  h->motion_part = cv.take<double>(size_t(h->B) * kMaxFrames * kMotionSlices);
  h->motion_arrive = cv.take<unsigned>(h->B);
  h->sig_zero = cv.take<float>(kMaxEntries);
  return cv.off + 1024;
}

sdv2_status fill_dims(sdv2_handle* h, const sdv2_model_desc* md, const sdv2_geometry* g,
                      const sdv2_pipeline_desc* pp, sdv2_precision prec, std::string* why) {
  if (!md || !g) return SDV2_E_INVALID;
  h->md = *md;
  h->g = *g;
  h->prec = prec;
  if (prec != SDV2_FP32 && prec != SDV2_BF16) return SDV2_E_INVALID;
  if (md->num_blocks < 1 || md->dim < 1 || md->num_heads < 1 || md->ffn_dim < 1) return SDV2_E_SHAPE;
  if (md->dim % md->num_heads) { *why = "dim % num_heads != 0"; return SDV2_E_SHAPE; }
  h->d = md->dim; h->H = md->num_heads; h->hd = md->dim / md->num_heads; h->F = md->ffn_dim;
  if (h->hd % 2) { *why = "odd head_dim"; return SDV2_E_SHAPE; }
  if (h->hd != 64 && h->hd != 128) { *why = "head_dim must be 64 or 128"; return SDV2_E_UNSUPPORTED; }
  if (h->d % 128 || h->F % 64) { *why = "dim % 128 or ffn % 64"; return SDV2_E_UNSUPPORTED; }
  if (md->patch_t != 1 || md->patch_h != 2 || md->patch_w != 2) { *why = "patch must be (1,2,2)"; return SDV2_E_UNSUPPORTED; }
  if (md->freq_dim != 256 || md->text_len < 1 || md->text_dim < 1) return SDV2_E_SHAPE;
  if (g->latent_h % 2 || g->latent_w % 2 || g->latent_h < 2 || g->latent_w < 2) { *why = "latent not divisible by patch"; return SDV2_E_SHAPE; }
  if (g->window_chunks < 1 || g->sink_chunks < 0) { *why = "window_chunks < 1"; return SDV2_E_SHAPE; }
  if (g->chunk_frames < 1 || g->chunk_frames > kMaxFrames) return SDV2_E_SHAPE;
  if (g->steps < 1 || g->steps > kMaxSteps) return SDV2_E_SHAPE;
  if (g->streams < 1 || g->streams * g->steps > kMaxEntries) { *why = "streams * steps must be in [1, 16]"; return SDV2_E_SHAPE; }
  if (g->sink_chunks + g->window_chunks > kMaxSlots || g->sink_chunks > 31) return SDV2_E_SHAPE;
  if (g->kv_mode != 0 && g->kv_mode != 1) { *why = "kv_mode must be 0 or 1"; return SDV2_E_INVALID; }
  if (g->kv_mode == 1 && (g->steps != 1 || (pp && pp->world > 1))) {
    *why = "kv_mode 1 (clean re-run) needs steps == 1 and a single stage";
    return SDV2_E_UNSUPPORTED;
  }
  h->C = md->latent_channels; h->T = g->chunk_frames; h->hh = g->latent_h; h->ww = g->latent_w;
  h->hn = h->hh / 2; h->wn = h->ww / 2;
  h->L = h->T * h->hn * h->wn;
  h->n = g->steps; h->m = g->sink_chunks; h->W = g->window_chunks; h->S = h->m + h->W;
  h->Lt = md->text_len; h->Dt = md->text_dim;
  h->CTHW = h->C * h->T * h->hh * h->ww;
  if (h->CTHW % 4 || (h->hh * h->ww) % 4) return SDV2_E_SHAPE;
  h->B = g->streams;
  h->NE = h->B * h->n;
  h->Mmax = h->NE * h->L;
  h->P = 4 * h->C;
  const int c = h->hd / 2;
  h->ct = c - 2 * (c / 3); h->ch = c / 3; h->cw = c / 3;
  h->ta = prec == SDV2_BF16 ? 2 : 4;
  if (pp) {
    if (pp->world < 1 || pp->rank < 0 || pp->rank >= pp->world) return SDV2_E_INVALID;
    if (pp->world > md->num_blocks) { *why = "more stages than blocks"; return SDV2_E_INVALID; }
    if (pp->block_begin < 0 || pp->block_end > md->num_blocks || pp->block_begin >= pp->block_end) {
      *why = "bad block range";
      return SDV2_E_INVALID;
    }
    h->K = pp->world; h->rank = pp->rank; h->b0 = pp->block_begin; h->b1 = pp->block_end;
    if (pp->resident_begin == 0 && pp->resident_end == 0) {
      h->r0 = h->b0;
      h->nb = h->b1 - h->b0;
    } else {
      if (pp->resident_begin < 0 || pp->resident_end > md->num_blocks || pp->resident_begin > h->b0 ||
          pp->resident_end < h->b1) {
        *why = "resident range must contain the block range";
        return SDV2_E_INVALID;
      }
      h->r0 = pp->resident_begin;
      h->nb = pp->resident_end - pp->resident_begin;
    }
  } else {
    h->K = 1; h->rank = 0; h->b0 = 0; h->b1 = md->num_blocks;
    h->r0 = 0;
    h->nb = md->num_blocks;
  }
  h->a0 = h->b0 - h->r0;
  h->a1 = h->b1 - h->r0;
  // the control plane keeps the records of the last kRecRing admitted chunks; the oldest
  // in-flight entry is (n-1) K calls old
  if (int64_t(h->n - 1) * h->K + 1 > kRecRing) { *why = "(steps - 1) * world + 1 exceeds the chunk-record ring"; return SDV2_E_INVALID; }
  return SDV2_OK;
}

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      h->err = std::string(#call) + ": " + cudaGetErrorString(e_);            \
      return SDV2_E_CUDA;                                                     \
    }                                                                         \
  } while (0)

#define CKL()                                                                 \
  do {                                                                        \
    ++h->launches;                                                            \
    cudaError_t e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess) {                                                  \
      h->err = std::string("launch: ") + cudaGetErrorString(e_);              \
      return SDV2_E_CUDA;                                                     \
    }                                                                         \
    debug_sync_point(h, __LINE__);                                            \
  } while (0)

// Test hook (sdv2_debug_sync): every launch is followed by a stream synchronisation and a
// line on stderr, so a kernel that never completes is named by the last line printed.
inline void debug_sync_point(sdv2_handle* h, int line) {
  if (!h->debug_sync) return;
  fprintf(stderr, "sdv2 launch @%d\n", line);
  fflush(stderr);
  cudaStreamSynchronize(h->stream);
}

__global__ void mul_vec_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] * b[i];
}

template <typename T>
__global__ void convert_kernel(const float* __restrict__ src, T* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = from_f<T>(src[i]);
}

sdv2_status load_tensor(sdv2_handle* h, const void* src, void* dst, size_t elems, bool to_tw) {
  if (!src) {
    h->err = "null weight tensor";
    return SDV2_E_INVALID;
  }
  if (!to_tw || h->prec == SDV2_FP32) {
    CK(cudaMemcpyAsync(dst, src, elems * 4, cudaMemcpyDefault, h->stream));
    return SDV2_OK;
  }
  CK(cudaMemcpyAsync(h->staging, src, elems * 4, cudaMemcpyDefault, h->stream));
  convert_kernel<bf16><<<592, 256, 0, h->stream>>>(h->staging, static_cast<bf16*>(dst), elems);
  CKL();
  return SDV2_OK;
}

// ---------------------------------------------------------------- GEMM dispatch
template <typename TIn, typename TW, typename TOut>
sdv2_status gemm_simt(sdv2_handle* h, const TIn* A, const TW* W, int M, int N, int K, int lda, int epi,
                      const EpiArgs& ep) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  switch (epi) {
    case EPI_STORE: gemm_simt_kernel<TIn, TW, TOut, EPI_STORE><<<grid, 256, 0, h->stream>>>(A, W, M, N, K, lda, K, ep); break;
    case EPI_GELU: gemm_simt_kernel<TIn, TW, TOut, EPI_GELU><<<grid, 256, 0, h->stream>>>(A, W, M, N, K, lda, K, ep); break;
    case EPI_RES_GATE: gemm_simt_kernel<TIn, TW, TOut, EPI_RES_GATE><<<grid, 256, 0, h->stream>>>(A, W, M, N, K, lda, K, ep); break;
    default: gemm_simt_kernel<TIn, TW, TOut, EPI_RES><<<grid, 256, 0, h->stream>>>(A, W, M, N, K, lda, K, ep); break;
  }
  CKL();
  return SDV2_OK;
}

// Activation GEMM of the hot path: fp32 SIMT on the parity path, tcgen05 on bf16.
sdv2_status gemm_act(sdv2_handle* h, const void* A, const void* W, int M, int N, int K, int epi, const EpiArgs& ep) {
  ProfScope ps(h, 0, 2.0 * M * N * K);
  if (h->prec == SDV2_FP32)
    return gemm_simt<float, float, float>(h, static_cast<const float*>(A), static_cast<const float*>(W), M, N, K, K,
                                          epi, ep);
  if (tc_gemm_enabled()) {
    ++h->launches;
    gemm_pdl_flag() = h->pdl;
    const bool ok = tc_gemm(h->stream, h->gplan, A, W, M, N, K, epi, ep, &h->err);
    gemm_pdl_flag() = false;
    debug_sync_point(h, __LINE__ * 1000 + epi);
    return ok ? SDV2_OK : SDV2_E_CUDA;
  }
  return gemm_simt<bf16, bf16, bf16>(h, static_cast<const bf16*>(A), static_cast<const bf16*>(W), M, N, K, K, epi, ep);
}

// Cross-q RMS fused into the cross-Q GEMM epilogue (row sums of squares) and the
// cross-attention scores (per-row scale, gain folded into the prompt K): the bf16 path
// whenever the prompt fits the single-pass cross kernel.
inline bool fused_cross_rms(const sdv2_handle* h) { return h->prec == SDV2_BF16 && h->Lt <= kXattnMaxJ * kAttnBKV; }

sdv2_status attention(sdv2_handle* h, const AttnArgs& aa, int Mrows_entries, double flops, int bl) {
  ProfScope ps(h, aa.cross ? 2 : 1, flops);
  dim3 grid((h->L + 15) / 16, h->H, Mrows_entries);
  if (h->prec == SDV2_FP32) {
    if (h->hd == 64) attn_simt_kernel<float, 64><<<grid, 128, 0, h->stream>>>(aa, h->td_dev);
    else attn_simt_kernel<float, 128><<<grid, 128, 0, h->stream>>>(aa, h->td_dev);
  } else {
    if (aa.cross && h->Lt <= kXattnMaxJ * kAttnBKV) {
      // prompt keys fit one TMEM row: exact single-pass cross-attention (xattn_tc.cuh)
      ++h->launches;
      XattnArgs xa{};
      xa.L = h->L;
      xa.H = h->H;
      xa.QT = (h->L + kAttnBQ - 1) / kAttnBQ;
      xa.n_entries = Mrows_entries;
      xa.Lk = h->Lt;
      xa.kv_row0 = bl * 2 * h->B * h->Lt;      // prompt K/V [nb][2B slots][Lt][d]
      xa.kv_slot_rows = h->Lt;
      xa.scale_log2 = 1.4426950408889634f / sqrtf(float(h->hd));
      xa.o = aa.o;
      xa.ldo = aa.ldo;
      xa.rowsq = h->rowsq;
      xa.nparts = h->d / 32;
      xa.inv_d = 1.f / float(h->d);
      xa.eps = h->md.eps;
      const bool okx = tc_cross_attention(h->stream, h->aplan, aa.q, h->Mmax, h->Kx, h->Vx, 2LL * h->B * h->nb * h->Lt,
                                          h->d, h->hd, xa, h->td_dev, &h->err, h->pdl);
      debug_sync_point(h, __LINE__);
      return okx ? SDV2_OK : SDV2_E_CUDA;
    }
    if (tc_attn_enabled()) {
      ++h->launches;
      AttnTcArgs ta{};
      ta.L = h->L;
      ta.cross = aa.cross;
      ta.Lk_cross = aa.Lk_cross;
      ta.scale_log2 = 1.4426950408889634f / sqrtf(float(h->hd));
      ta.o = aa.o;
      ta.ldo = aa.ldo;
      ta.H = h->H;
      ta.QT = (h->L + kAttnBQ - 1) / kAttnBQ;
      ta.n_entries = Mrows_entries;
      ta.part_o = h->attn_part;
      ta.part_ml = h->attn_part + size_t(kMaxSMs) * 2 * kAttnBQ * h->hd;
      long long tiles = 0;
      for (int e = 0; e < Mrows_entries; ++e) {
        const int Lk = aa.cross ? aa.Lk_cross : h->td_host_cur->e[e].nvalid * h->L;
        tiles += (long long)ta.H * ta.QT * ((Lk + kAttnBKV - 1) / kAttnBKV);
      }
      {
        const int CL = h->hd == 128 ? attn_cluster() : 1, QP = (ta.QT + CL - 1) / CL;   // decide on query-tile groups
        ta.per_unit = attn_pick_per_unit((long long)Mrows_entries * ta.H * QP, tiles * QP / ta.QT,
                                         h->aplan.num_sms / CL);
        ta.rr = attn_rr();
      }
      const void *Kb, *Vb;
      long long kv_rows;
      if (aa.cross) {
        Kb = h->Kx; Vb = h->Vx;
        kv_rows = 2LL * h->B * h->nb * h->Lt;
        ta.kv_row0 = bl * 2 * h->B * h->Lt;     // prompt K/V [nb][2B slots][Lt][d]
        ta.kv_lane_rows = h->Lt;
      } else {
        Kb = h->Kc; Vb = h->Vc;
        kv_rows = (long long)h->nb * h->NE * h->S * h->L;
        ta.kv_row0 = bl * h->NE * h->S * h->L;
        ta.kv_lane_rows = h->S * h->L;
      }
      const bool oka = tc_attention(h->stream, h->aplan, aa.q, h->Mmax, Kb, Vb, kv_rows, h->d, h->hd, tiles, ta,
                                    h->td_dev, &h->err, h->pdl);
      if (h->debug_sync)
        fprintf(stderr, "sdv2 self-attn block %d per_unit %d tiles %lld units %d\n", bl, ta.per_unit, tiles,
                Mrows_entries * ta.H * ta.QT);
      debug_sync_point(h, __LINE__);
      return oka ? SDV2_OK : SDV2_E_CUDA;
    }
    if (h->hd == 64) attn_simt_kernel<bf16, 64><<<grid, 128, 0, h->stream>>>(aa, h->td_dev);
    else attn_simt_kernel<bf16, 128><<<grid, 128, 0, h->stream>>>(aa, h->td_dev);
  }
  CKL();
  return SDV2_OK;
}

// Every per-call kernel is launched with programmatic dependent launch (PDL): its
// prologue (barrier init, TMEM alloc, descriptor / weight prefetch) overlaps the tail of
// the previous kernel; each kernel executes griddepcontrol.wait before touching data
// produced upstream.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename TA>
sdv2_status launch_norm_args(sdv2_handle* h, int rows, const ModArgs& m) {
  const int nv = (h->d / 4 + kRowThreads - 1) / kRowThreads;
  if (nv <= 4)
    launch_k(h->pdl, norm_mod2_kernel<TA, 4>, dim3((rows + 1) / 2), dim3(256), 0, h->stream, h->st.x, static_cast<TA*>(h->a), rows, h->d, h->L,
                                                                    m, h->md.eps, h->md.norm_center);
  else
    launch_k(h->pdl, norm_mod2_kernel<TA, 16>, dim3((rows + 1) / 2), dim3(256), 0, h->stream, h->st.x, static_cast<TA*>(h->a), rows, h->d, h->L,
                                                                     m, h->md.eps, h->md.norm_center);
  CKL();
  return SDV2_OK;
}

// adaLN (mode 0: shift row sh_row, scale row sc_row of mod + e0[e]) or affine (mode 1).
template <typename TA>
sdv2_status launch_norm(sdv2_handle* h, int rows, int mode, const float* mod, int sc_row, int sh_row,
                        const float* gamma, const float* beta, float* zero_rows = nullptr) {
  ModArgs m{};
  m.zero_rows = zero_rows;
  if (mode == 0) {
    m.modA = mod; m.sc_off = sc_row * h->d; m.sh_off = sh_row * h->d;
    m.eA = h->st.e0; m.estride = 6 * h->d; m.esc_off = sc_row * h->d; m.esh_off = sh_row * h->d;
    m.a0 = 1.f;
  } else {
    m.modA = gamma; m.sc_off = 0;
    m.sh_off = int(beta - gamma);   // beta follows gamma in the workspace (carve order)
    m.eA = nullptr;
    m.a0 = 0.f;
  }
  return launch_norm_args<TA>(h, rows, m);
}

#define TRY(x)                        \
  do {                                \
    sdv2_status s_ = (x);             \
    if (s_ != SDV2_OK) return s_;     \
  } while (0)

// Drop every captured call graph (call bodies and clean passes): they bake in stream
// constants and the active block range.
void drop_graphs(sdv2_handle* h) {
  for (auto& g : h->graph_exec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  for (auto& g : h->clean_graph_exec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
}

template <typename TA>
sdv2_status run_block(sdv2_handle* h, int bl, int rows, int n_act) {
  const BlockW& B = h->bw[bl];
  const int d = h->d;
  EpiArgs ep{};
  ep.L = h->L;
  // 1. adaLN norm1 + modulate (shift row 0, scale row 1)
  TRY(launch_norm<TA>(h, rows, 0, B.mod, 1, 0, nullptr, nullptr));
  // 2. QKV projection
  ep.out = h->qkv; ep.ldo = 3 * d; ep.bias = B.bqkv;
  TRY(gemm_act(h, h->a, B.wqkv, rows, 3 * d, d, EPI_STORE, ep));
  // 3–4. q/k RMSNorm + RoPE + KV lane write
  const size_t lane_elems = size_t(h->NE) * h->S * h->L * d;
  TA* Kb = static_cast<TA*>(h->Kc) + bl * lane_elems;
  TA* Vb = static_cast<TA*>(h->Vc) + bl * lane_elems;
  {
    const int units_pt = (d / (16 / int(sizeof(TA))) + kRowThreads - 1) / kRowThreads;
    if (units_pt <= 2)
      launch_k(h->pdl, qkv_post2_kernel<TA, 2>, dim3((rows + 1) / 2), dim3(256), 0, h->stream, 
          static_cast<const TA*>(h->qkv), static_cast<TA*>(h->q), Kb, Vb, B.gq, B.gk, h->td_dev, h->rt, rows, d, h->hd,
          h->L, h->hn, h->wn, h->T, h->S, h->md.eps);
    else
      launch_k(h->pdl, qkv_post2_kernel<TA, 8>, dim3((rows + 1) / 2), dim3(256), 0, h->stream, 
          static_cast<const TA*>(h->qkv), static_cast<TA*>(h->q), Kb, Vb, B.gq, B.gk, h->td_dev, h->rt, rows, d, h->hd,
          h->L, h->hn, h->wn, h->T, h->S, h->md.eps);
    CKL();
  }
  // self-attention over the lane's valid prefix
  AttnArgs aa{};
  aa.q = h->q; aa.ldq = d; aa.K = Kb; aa.V = Vb; aa.kv_lane_stride = size_t(h->S) * h->L * d; aa.ldk = d;
  aa.o = h->o; aa.ldo = d; aa.L = h->L; aa.cross = 0; aa.scale = 1.f / sqrtf(float(h->hd));
  double fl_self = 0.0;
  for (int j = 0; j < n_act; ++j) fl_self += 4.0 * h->L * double(h->td_host_cur->e[j].nvalid) * h->L * d;
  TRY(attention(h, aa, n_act, fl_self, bl));
  // 5. out projection + gated residual (g1 = row 2)
  ep.out = h->st.x; ep.ldo = d; ep.bias = B.bo; ep.mod = B.mod; ep.e0 = h->st.e0; ep.gate_row = 2;
  TRY(gemm_act(h, h->o, B.wo, rows, d, d, EPI_RES_GATE, ep));
  // 6. cross-attention: affine norm3, q projection, RMS q (fused on the bf16 path: the
  //    GEMM epilogue sums q^2 per row, the cross kernel scales the scores, K carries g_cq)
  const bool fused = fused_cross_rms(h);
  TRY(launch_norm<TA>(h, rows, 1, nullptr, 0, 0, B.n3g, B.n3b));
  ep.out = h->q; ep.ldo = d; ep.bias = B.bcq; ep.rowsq = h->rowsq;
  TRY(gemm_act(h, h->a, B.wcq, rows, d, d, fused ? EPI_STORE_RSQ : EPI_STORE, ep));
  if (!fused) {
    const int units_pt = (d / (16 / int(sizeof(TA))) + kRowThreads - 1) / kRowThreads;
    if (units_pt <= 2)
      launch_k(h->pdl, rms_rows2_kernel<TA, 2>, dim3((rows + 1) / 2), dim3(256), 0, h->stream, static_cast<TA*>(h->q), B.gcq, rows, d, h->md.eps);
    else
      launch_k(h->pdl, rms_rows2_kernel<TA, 8>, dim3((rows + 1) / 2), dim3(256), 0, h->stream, static_cast<TA*>(h->q), B.gcq, rows, d, h->md.eps);
    CKL();
  }
  const size_t px = size_t(h->Lt) * d;
  aa.q = h->q; aa.K = static_cast<TA*>(h->Kx) + size_t(bl) * 2 * h->B * px;
  aa.V = static_cast<TA*>(h->Vx) + size_t(bl) * 2 * h->B * px;
  aa.kv_lane_stride = px; aa.cross = 1; aa.Lk_cross = h->Lt;
  TRY(attention(h, aa, n_act, 4.0 * double(rows) * h->Lt * d, bl));
  // 7. cross out projection, ungated residual
  ep.out = h->st.x; ep.ldo = d; ep.bias = B.bco;
  TRY(gemm_act(h, h->o, B.wco, rows, d, d, EPI_RES, ep));
  // 8. FFN: norm2 + modulate (shift row 3, scale row 4), GELU, gated residual (g2 = row 5)
  TRY(launch_norm<TA>(h, rows, 0, B.mod, 4, 3, nullptr, nullptr));
  ep.out = h->hbuf; ep.ldo = h->F; ep.bias = B.b1;
  TRY(gemm_act(h, h->a, B.w1, rows, h->F, d, EPI_GELU, ep));
  ep.out = h->st.x; ep.ldo = d; ep.bias = B.b2; ep.mod = B.mod; ep.e0 = h->st.e0; ep.gate_row = 5;
  TRY(gemm_act(h, h->hbuf, B.w2, rows, d, h->F, EPI_RES_GATE, ep));
  if (h->tap) CK(cudaMemcpyAsync(h->tap + size_t(bl - h->a0) * h->Mmax * d, h->st.x, size_t(rows) * d * 4,
                                 cudaMemcpyDeviceToDevice, h->stream));
  return SDV2_OK;
}

// Prompt conditioning (C.3): ctx = W_x2 GELU(W_x1 P + b) + b; per block K_c = RMS(ctx W_ck^T + b),
// V_c = ctx W_cv^T + b into prompt version slot `ver & 1`.
template <typename TA>
sdv2_status embed_prompt(sdv2_handle* h, const float* prompt_host, int b_stream, int ver) {
  const int d = h->d, Lt = h->Lt;
  CK(cudaMemcpyAsync(h->prompt, prompt_host, size_t(Lt) * h->Dt * 4, cudaMemcpyHostToDevice, h->stream));
  EpiArgs ep{};
  ep.out = h->ctx_tmp; ep.ldo = d; ep.bias = h->gw[G_TXT1_B];
  TRY((gemm_simt<float, float, float>(h, h->prompt, h->gw[G_TXT1_W], Lt, d, h->Dt, h->Dt, EPI_GELU, ep)));
  ep.out = h->ctx; ep.bias = h->gw[G_TXT2_B];
  TRY((gemm_simt<float, float, float>(h, h->ctx_tmp, h->gw[G_TXT2_W], Lt, d, d, d, EPI_STORE, ep)));
  const size_t px = size_t(Lt) * d;
  for (int b = 0; b < h->nb; ++b) {
    const BlockW& B = h->bw[b];
    const size_t slot = size_t(2 * b_stream + (ver & 1));   // EntryDesc::xslot
    TA* Kd = static_cast<TA*>(h->Kx) + (size_t(b) * 2 * h->B + slot) * px;
    TA* Vd = static_cast<TA*>(h->Vx) + (size_t(b) * 2 * h->B + slot) * px;
    ep.out = h->ctx_tmp; ep.bias = B.bck;
    TRY((gemm_simt<float, TA, float>(h, h->ctx, static_cast<const TA*>(B.wck), Lt, d, d, d, EPI_STORE, ep)));
    launch_k(h->pdl, rms_rows_kernel<float, TA>, dim3((Lt + 7) / 8), dim3(256), 0, h->stream, h->ctx_tmp, Kd,
             fused_cross_rms(h) ? B.gkq : B.gck, Lt, d, d, h->md.eps);
    CKL();
    ep.out = Vd; ep.bias = B.bcv;
    TRY((gemm_simt<float, TA, TA>(h, h->ctx, static_cast<const TA*>(B.wcv), Lt, d, d, d, EPI_STORE, ep)));
  }
  return SDV2_OK;
}

sdv2_status set_prompt_common(sdv2_handle* h, const float* prompt_host, int b_stream, int ver) {
  // h = mean-pooled prompt, fp64 (reading Q8)
  std::vector<double> mean(h->Dt, 0.0);
  for (int t = 0; t < h->Lt; ++t)
    for (int c = 0; c < h->Dt; ++c) mean[c] += double(prompt_host[size_t(t) * h->Dt + c]);
  double nrm = 0.0;
  for (int c = 0; c < h->Dt; ++c) {
    mean[c] /= double(h->Lt);
    nrm += mean[c] * mean[c];
  }
  if (!(nrm > 0.0)) {
    h->err = "zero-norm prompt mean";
    return SDV2_E_INVALID;
  }
  if (h->prec == SDV2_FP32) TRY(embed_prompt<float>(h, prompt_host, b_stream, ver));
  else TRY(embed_prompt<bf16>(h, prompt_host, b_stream, ver));
  h->ctl.set_prompt_mean(b_stream, mean, ver);
  return SDV2_OK;
}

// Device work of one call that depends only on (active entries, call parity): the
// part replayed from a CUDA graph.
template <typename TA>
sdv2_status tick_body(sdv2_handle* h, int na, int par) {
  const int rows = na * h->L;
  const bool first = h->rank == 0, last = h->rank == h->K - 1;
  if (first) {
    ProfScope ps(h, 5, 0.0);
    // motion-aware noise controller then the step-0 blend on all SMs
    launch_k(h->pdl, motion_kernel, dim3(kMotionSlices, h->B), dim3(256), 0, h->stream, h->lat_in, h->prev_frame, h->ctrl, h->st.sig, h->st.sign, h->td_dev,
             h->scfg, h->CTHW, h->hh * h->ww, h->T, h->NE, h->motion_part, h->motion_arrive);
    CKL();
    launch_k(h->pdl, blend_kernel, dim3((h->CTHW + 255) / 256, h->B), dim3(256), 0, h->stream, h->lat_in, h->st.lat, h->st.sig, h->td_dev,
             h->scfg.seed, h->CTHW);
    CKL();
    if (na > h->B) {
      // K = 1: the ring packet of call c-1 was written to ring[1][(c-1)&1] == ring[1][par^1]
      const float* rin = h->K == 1 ? h->ring[1][par ^ 1] : h->ring[0][par];
      launch_k(h->pdl, assemble_kernel, dim3(64, h->NE - h->B), dim3(256), 0, h->stream, rin, h->st.lat, h->td_dev, h->NE,
               h->B, h->CTHW);
      CKL();
    }
    // patchify + patch embedding (C.1): x = u W_pe^T + b_pe, fp32 (K = 4C)
    launch_k(h->pdl, patchify_kernel, dim3((rows * h->P + 255) / 256), dim3(256), 0, h->stream, h->st.lat, h->u, rows, h->L, h->C, h->T, h->hh,
                                                                       h->ww);
    CKL();
    {
      EpiArgs ep{};
      ep.out = h->st.x; ep.ldo = h->d; ep.bias = h->gw[G_PATCH_B]; ep.L = h->L;
      TRY((gemm_simt<float, float, float>(h, h->u, h->gw[G_PATCH_W], rows, h->d, h->P, h->P, EPI_STORE, ep)));
    }
    launch_k(h->pdl, sinusoid_kernel, dim3(na), dim3(128), 0, h->stream, h->st.sig, h->emb, na, h->md.freq_dim);
    CKL();
    const int d = h->d;
    // time MLP (C.2): e = W_t2 SiLU(W_t1 emb + b) + b; e0 = W_tp SiLU(e) + b
    // the entry count is a template bound (registers): 4 / 8 / 16
    auto gemvs = [&](auto nmax) {
      constexpr int NM = decltype(nmax)::value;
      launch_k(h->pdl, gemv2_kernel<float, NM>, dim3((d + 31) / 32), dim3(256), size_t(na) * h->md.freq_dim * 4, h->stream,
               h->gw[G_T1_W], h->gw[G_T1_B], h->emb, h->t1, na, d, h->md.freq_dim, 0);
      launch_k(h->pdl, gemv2_kernel<float, NM>, dim3((d + 31) / 32), dim3(256), size_t(na) * d * 4, h->stream,
               h->gw[G_T2_W], h->gw[G_T2_B], h->t1, h->st.e, na, d, d, 1);
      launch_k(h->pdl, gemv2_kernel<TA, NM>, dim3((6 * d + 31) / 32), dim3(256), size_t(na) * d * 4, h->stream,
               static_cast<const TA*>(h->tp_w), h->gw[G_TP_B], h->st.e, h->st.e0, na, 6 * d, d, 1);
    };
    if (na <= 4) gemvs(std::integral_constant<int, 4>{});
    else if (na <= 8) gemvs(std::integral_constant<int, 8>{});
    else gemvs(std::integral_constant<int, 16>{});
    h->launches += 2;
    CKL();
  }
  for (int b = h->a0; b < h->a1; ++b) {
    ProfScope ps(h, 4, 0.0, b);
    TRY(run_block<TA>(h, b, rows, na));
  }
  if (last) {
    ProfScope ps(h, 5, 0.0);
    // head (C.7): a = N(x)(1 + mod_h[1] + e) + mod_h[0] + e; y = a W_h^T + b_h (fp32 out);
    // then unpatchify + x0 + output / re-noise (C.8, O5)
    ModArgs m{};
    m.modA = h->gw[G_HEAD_MOD]; m.sc_off = h->d; m.sh_off = 0;
    m.eA = h->st.e; m.estride = h->d; m.esc_off = 0; m.esh_off = 0; m.a0 = 1.f;
    TRY(launch_norm_args<TA>(h, rows, m));
    EpiArgs ep{};
    ep.out = h->yh; ep.ldo = h->P; ep.bias = h->gw[G_HEAD_B]; ep.L = h->L;
    if (h->prec == SDV2_FP32) {
      TRY((gemm_simt<float, float, float>(h, static_cast<const float*>(h->a), h->gw[G_HEAD_W], rows, h->P, h->d,
                                          h->d, EPI_STORE, ep)));
    } else {
      ++h->launches;
      gemm_pdl_flag() = h->pdl;
      const bool ok = tc_gemm(h->stream, h->gplan, h->a, h->head_w_tw, rows, h->P, h->d, EPI_STORE_F32, ep, &h->err);
      gemm_pdl_flag() = false;
      if (!ok) return SDV2_E_CUDA;
    }
    launch_k(h->pdl, flow_kernel, dim3((na * h->CTHW + 255) / 256), dim3(256), 0, h->stream, 
        h->yh, h->st.lat, h->st.sig, h->st.sign, h->out_stage, h->ring[1][par], h->td_dev, na, h->L, h->C, h->T,
        h->hh, h->ww, h->n, h->scfg.seed);
    CKL();
  }
  return SDV2_OK;
}

// kv_mode 1 (clean-context re-run, reading Q5-clean, N4): the previous call's finished
// chunks (its na entries, n = 1) go through the DiT again on their prediction x0 (still
// in out_stage) at sigma = 0, with the descriptor they were admitted with (rebase
// cleared: it was applied then).  qkv_post2 writes their K/V over the step-0 K/V in the
// same slots (window slot or sink fill, plus the sinks the chunk refreshed) and the
// attention reads the same prefix as then.  No head: the pass only rewrites the cache.
template <typename TA>
sdv2_status clean_body(sdv2_handle* h, int na) {
  const int rows = na * h->L;
  launch_k(h->pdl, patchify_kernel, dim3((rows * h->P + 255) / 256), dim3(256), 0, h->stream, h->out_stage, h->u, rows,
           h->L, h->C, h->T, h->hh, h->ww);
  CKL();
  {
    EpiArgs ep{};
    ep.out = h->st.x; ep.ldo = h->d; ep.bias = h->gw[G_PATCH_B]; ep.L = h->L;
    TRY((gemm_simt<float, float, float>(h, h->u, h->gw[G_PATCH_W], rows, h->d, h->P, h->P, EPI_STORE, ep)));
  }
  launch_k(h->pdl, sinusoid_kernel, dim3(na), dim3(128), 0, h->stream, h->sig_zero, h->emb, na, h->md.freq_dim);
  CKL();
  const int d = h->d;
  auto gemvs = [&](auto nmax) {
    constexpr int NM = decltype(nmax)::value;
    launch_k(h->pdl, gemv2_kernel<float, NM>, dim3((d + 31) / 32), dim3(256), size_t(na) * h->md.freq_dim * 4, h->stream,
             h->gw[G_T1_W], h->gw[G_T1_B], h->emb, h->t1, na, d, h->md.freq_dim, 0);
    launch_k(h->pdl, gemv2_kernel<float, NM>, dim3((d + 31) / 32), dim3(256), size_t(na) * d * 4, h->stream,
             h->gw[G_T2_W], h->gw[G_T2_B], h->t1, h->st.e, na, d, d, 1);
    launch_k(h->pdl, gemv2_kernel<TA, NM>, dim3((6 * d + 31) / 32), dim3(256), size_t(na) * d * 4, h->stream,
             static_cast<const TA*>(h->tp_w), h->gw[G_TP_B], h->st.e, h->st.e0, na, 6 * d, d, 1);
  };
  if (na <= 4) gemvs(std::integral_constant<int, 4>{});
  else if (na <= 8) gemvs(std::integral_constant<int, 8>{});
  else gemvs(std::integral_constant<int, 16>{});
  h->launches += 2;
  CKL();
  for (int b = h->a0; b < h->a1; ++b) {
    ProfScope ps(h, 4, 0.0, b);
    TRY(run_block<TA>(h, b, rows, na));
  }
  return SDV2_OK;
}

// Runs clean_body on the previous call's entries (from a graph keyed by their count),
// with the kernels reading the clean descriptor; the block tap stays off.
template <typename TA>
sdv2_status clean_pass(sdv2_handle* h, TickDesc* tdc) {
  const int na = tdc->n_active;
  TickDesc* const td_dev = h->td_dev;
  TickDesc* const td_cur = h->td_host_cur;
  float* const tap = h->tap;
  h->td_dev = h->td_clean_dev;
  h->td_host_cur = tdc;
  h->tap = nullptr;
  sdv2_status st = SDV2_OK;
  const bool use_graph = h->graphs && !h->prof && !tap && !h->debug_sync && h->stream != nullptr;
  if (use_graph) {
    if (!h->clean_graph_exec[na]) {
      const int64_t l0 = h->launches;
      cudaError_t e = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        st = clean_body<TA>(h, na);
        cudaGraph_t g = nullptr;
        e = cudaStreamEndCapture(h->stream, &g);
        if (st == SDV2_OK && e == cudaSuccess) e = cudaGraphInstantiate(&h->clean_graph_exec[na], g, 0);
        if (g) cudaGraphDestroy(g);
      }
      if (st == SDV2_OK && e != cudaSuccess) {
        h->err = std::string("clean-pass graph: ") + cudaGetErrorString(e);
        st = SDV2_E_CUDA;
      }
      h->clean_graph_launches[na] = h->launches - l0;
      h->launches = l0;
    }
    if (st == SDV2_OK) {
      if (cudaGraphLaunch(h->clean_graph_exec[na], h->stream) != cudaSuccess) st = SDV2_E_CUDA;
      h->launches += h->clean_graph_launches[na];
    }
  } else {
    st = clean_body<TA>(h, na);
  }
  h->td_dev = td_dev;
  h->td_host_cur = td_cur;
  h->tap = tap;
  return st;
}

template <typename TA>
sdv2_status tick(sdv2_handle* h, const float* chunk_latent, float* out_latent, int64_t* out_chunk) {
  const int64_t call = h->ctl.calls();
  const int slot = int(call % kTdRing);
  if (h->td_ev_used[slot]) CK(cudaEventSynchronize(h->td_ev[slot]));
  TickDesc* tdh = h->td_host + slot;
  TickDesc* tdc = h->td_host + kTdRing + slot;   // kv_mode 1: the clean pass's descriptor
  const bool clean = h->g.kv_mode == 1 && h->td_prev_valid && h->td_prev.n_active > 0;
  if (clean) {
    *tdc = h->td_prev;
    for (int e = 0; e < kMaxEntries; ++e) tdc->e[e].rebase = 0;   // applied at admission
    CK(cudaMemcpyAsync(h->td_clean_dev, tdc, sizeof(TickDesc), cudaMemcpyHostToDevice, h->stream));
  }
  h->ctl.plan_call(tdh);
  h->td_host_cur = tdh;
  CK(cudaMemcpyAsync(h->td_dev, tdh, sizeof(TickDesc), cudaMemcpyHostToDevice, h->stream));
  CK(cudaEventRecord(h->td_ev[slot], h->stream));
  h->td_ev_used[slot] = true;
  const int na = tdh->n_active;
  const int par = int(call & 1);
  set_packet(h, packet_for(h, par));   // captured graphs are keyed by parity: pointers match
  const bool first = h->rank == 0, last = h->rank == h->K - 1;
  // tick info (host, no sync: the schedule is deterministic)
  h->info.call = call;
  h->info.num_entries = na;
  h->info.steps = h->n;
  for (int j = 0; j < 8; ++j) h->info.chunk[j] = (j < h->n && tdh->e[j * h->B].active) ? tdh->e[j * h->B].X : -1;
  h->info.out_chunk = (last && tdh->out_entry >= 0) ? h->ctl.out_chunk(call) : -1;
  if (out_chunk) *out_chunk = h->info.out_chunk;

  if (first) CK(cudaMemcpyAsync(h->lat_in, chunk_latent, size_t(h->B) * h->CTHW * 4, cudaMemcpyDefault, h->stream));
  // clean re-run of the previous call's chunks, before this call's re-base / writes
  if (clean) TRY(clean_pass<TA>(h, tdc));
  if (h->g.kv_mode == 1) {
    h->td_prev = *tdh;
    h->td_prev_valid = true;
  }
  // RoPE re-base (rare: once every T_reset frames) of every local block's ring slots of
  // the re-basing lanes, before any block of this call writes or attends (R3).
  bool any_rebase = false;
  for (int e = 0; e < h->NE; ++e) any_rebase |= (tdh->e[e].active && tdh->e[e].rebase);
  if (any_rebase) {
    rebase_kernel<TA><<<dim3(512, h->NE), 256, 0, h->stream>>>(
        static_cast<TA*>(h->Kc) + size_t(h->a0) * h->NE * h->S * h->L * h->d, h->td_dev, h->rt, h->a1 - h->a0, h->NE,
                                                                h->S, h->m, h->W, h->L, h->d, h->hd, h->T_reset);
    CKL();
  }
  const bool use_graph = h->graphs && !h->prof && !h->tap && !h->debug_sync && h->stream != nullptr;
  if (use_graph) {
    const int key = na * 2 + par;
    if (!h->graph_exec[key]) {
      const int64_t l0 = h->launches;
      CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
      sdv2_status s = tick_body<TA>(h, na, par);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(h->stream, &g);
      if (s != SDV2_OK) return s;
      if (e != cudaSuccess) {
        h->err = std::string("graph capture: ") + cudaGetErrorString(e);
        return SDV2_E_CUDA;
      }
      CK(cudaGraphInstantiate(&h->graph_exec[key], g, 0));
      cudaGraphDestroy(g);
      h->graph_launches[key] = h->launches - l0;
      h->launches = l0;
    }
    CK(cudaGraphLaunch(h->graph_exec[key], h->stream));
    h->launches += h->graph_launches[key];
  } else {
    TRY(tick_body<TA>(h, na, par));
  }
  if (last && tdh->out_entry >= 0 && out_latent)
    CK(cudaMemcpyAsync(out_latent, h->out_stage, size_t(h->B) * h->CTHW * 4, cudaMemcpyDefault, h->stream));
  h->info.kernel_launches = h->launches;
  return SDV2_OK;
}

}  // namespace

extern "C" {

const char* sdv2_status_string(sdv2_status s) {
  switch (s) {
    case SDV2_OK: return "ok";
    case SDV2_E_INVALID: return "invalid argument";
    case SDV2_E_SHAPE: return "invalid shape";
    case SDV2_E_STATE: return "invalid state";
    case SDV2_E_WORKSPACE: return "workspace too small";
    case SDV2_E_CUDA: return "cuda error";
    case SDV2_E_UNSUPPORTED: return "unsupported shape";
  }
  return "unknown status";
}

const char* sdv2_last_error(const sdv2_handle* h) { return h ? h->err.c_str() : "null handle"; }

size_t sdv2_workspace_bytes(const sdv2_model_desc* md, const sdv2_geometry* g, const sdv2_pipeline_desc* pp,
                            sdv2_precision prec) {
  sdv2_handle tmp;
  std::string why;
  if (fill_dims(&tmp, md, g, pp, prec, &why) != SDV2_OK) return 0;
  return carve(&tmp, nullptr);
}

sdv2_status sdv2_create(const sdv2_model_desc* md, const sdv2_geometry* g, const sdv2_pipeline_desc* pp,
                        sdv2_precision prec, const sdv2_weights* w, void* workspace, size_t workspace_bytes,
                        int device, void* stream, const sdv2_exec_options* opts, sdv2_handle** out) {
  if (!out) return SDV2_E_INVALID;
  *out = nullptr;
  auto* h = new sdv2_handle();
  std::string why;
  sdv2_status s = fill_dims(h, md, g, pp, prec, &why);
  if (s != SDV2_OK) {
    delete h;
    return s;
  }
  const size_t need = carve(h, nullptr);
  if (!workspace || workspace_bytes < need) {
    delete h;
    return SDV2_E_WORKSPACE;
  }
  if (!w || !w->tensors || w->count != kNumGlobal + kNumBlockT * h->nb) {
    delete h;
    return SDV2_E_INVALID;
  }
  h->device = device;
  h->stream = static_cast<cudaStream_t>(stream);
  if (opts) {
    h->tune = opts->tune_gemms != 0;
    h->pdl = opts->pdl != 0;
    h->graphs = opts->graphs != 0;
    h->l2_persist = opts->l2_persist != 0;
    if (opts->gemm_table && opts->gemm_table_len > 0)
      h->gemm_table.assign(opts->gemm_table, opts->gemm_table + size_t(opts->gemm_table_len) * 8);
  }
  h->ws_bytes = workspace_bytes;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete h;
    return SDV2_E_CUDA;
  }
  // align the base to 1 KB
  char* base = static_cast<char*>(workspace);
  const size_t adj = (1024 - (reinterpret_cast<uintptr_t>(base) & 1023)) & 1023;
  if (workspace_bytes < need + adj) {
    delete h;
    return SDV2_E_WORKSPACE;
  }
  carve(h, base + adj);
  auto fail = [&](sdv2_status st) {
    *out = h;   // keep the handle so the caller can read sdv2_last_error, then destroy
    return st;
  };
  if (cudaHostAlloc(reinterpret_cast<void**>(&h->td_host), sizeof(TickDesc) * 2 * kTdRing, cudaHostAllocDefault) != cudaSuccess)
    return fail(SDV2_E_CUDA);
  for (int i = 0; i < kTdRing; ++i) {
    cudaEventCreateWithFlags(&h->td_ev[i], cudaEventDisableTiming);
    h->td_ev_used[i] = false;
  }
  const void* const* T = w->tensors;
  const int d = h->d;
  const size_t sizes[kNumGlobal] = {size_t(d) * h->P, size_t(d), size_t(d) * h->Dt, size_t(d), size_t(d) * d, size_t(d),
                                    size_t(d) * 256, size_t(d), size_t(d) * d, size_t(d), size_t(6) * d * d,
                                    size_t(6) * d, size_t(2) * d, size_t(h->P) * d, size_t(h->P)};
  for (int i = 0; i < kNumGlobal; ++i) {
    if (i == G_TP_W) s = load_tensor(h, T[i], h->tp_w, sizes[i], true);
    else s = load_tensor(h, T[i], h->gw[i], sizes[i], false);
    if (s == SDV2_OK && i == G_HEAD_W) s = load_tensor(h, T[i], h->head_w_tw, sizes[i], true);
    if (s != SDV2_OK) return fail(s);
  }
  for (int b = 0; b < h->nb; ++b) {
    const void* const* Bt = T + kNumGlobal + kNumBlockT * b;
    BlockW& B = h->bw[b];
    const size_t dd = size_t(d) * d, tb = h->ta;
    struct { int id; void* dst; size_t n; bool tw; } list[] = {
        {B_MOD, B.mod, size_t(6) * d, false},
        {B_WQ, B.wqkv, dd, true}, {B_WK, static_cast<char*>(B.wqkv) + dd * tb, dd, true},
        {B_WV, static_cast<char*>(B.wqkv) + 2 * dd * tb, dd, true},
        {B_BQ, B.bqkv, size_t(d), false}, {B_BK, B.bqkv + d, size_t(d), false}, {B_BV, B.bqkv + 2 * d, size_t(d), false},
        {B_WO, B.wo, dd, true}, {B_BO, B.bo, size_t(d), false},
        {B_GQ, B.gq, size_t(d), false}, {B_GK, B.gk, size_t(d), false},
        {B_N3G, B.n3g, size_t(d), false}, {B_N3B, B.n3b, size_t(d), false},
        {B_WCQ, B.wcq, dd, true}, {B_BCQ, B.bcq, size_t(d), false},
        {B_WCK, B.wck, dd, true}, {B_BCK, B.bck, size_t(d), false},
        {B_WCV, B.wcv, dd, true}, {B_BCV, B.bcv, size_t(d), false},
        {B_WCO, B.wco, dd, true}, {B_BCO, B.bco, size_t(d), false},
        {B_GCQ, B.gcq, size_t(d), false}, {B_GCK, B.gck, size_t(d), false},
        {B_W1, B.w1, size_t(h->F) * d, true}, {B_B1, B.b1, size_t(h->F), false},
        {B_W2, B.w2, size_t(d) * h->F, true}, {B_B2, B.b2, size_t(d), false},
    };
    for (auto& it : list) {
      s = load_tensor(h, Bt[it.id], it.dst, it.n, it.tw);
      if (s != SDV2_OK) return fail(s);
    }
  }
  for (int b = 0; b < h->nb; ++b)   // g_ck * g_cq for the fused cross-q RMS
    mul_vec_kernel<<<(d + 255) / 256, 256, 0, h->stream>>>(h->bw[b].gck, h->bw[b].gcq, h->bw[b].gkq, d);
  // both precisions: sigma = 0 of the clean pass, the motion kernel's arrival counters
  if (cudaMemsetAsync(h->sig_zero, 0, kMaxEntries * sizeof(float), h->stream) != cudaSuccess ||
      cudaMemsetAsync(h->motion_arrive, 0, h->B * sizeof(unsigned), h->stream) != cudaSuccess) {
    h->err = "workspace initialisation failed";
    return fail(SDV2_E_CUDA);
  }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) {
    h->err = cudaGetErrorString(cudaGetLastError());
    return fail(SDV2_E_CUDA);
  }
  if (h->prec == SDV2_BF16) {
    if (!tc_gemm_plan(h->gplan, &h->err)) return fail(SDV2_E_CUDA);
    // configurations given by the caller (exec options): valid candidates only
    for (size_t i = 0; i + 8 <= h->gemm_table.size(); i += 8) {
      const int32_t* r = h->gemm_table.data() + i;
      GemmCfg gc{r[4], r[5], r[6]};
      gc.XE = r[7];
      for (const GemmCfg& c : tc_gemm_candidates(h->gplan, r[0], r[1], r[3]))
        if (c.MC == gc.MC && c.BN == gc.BN && c.SK == gc.SK && c.XE == gc.XE) {
          h->gplan.tuned[gemm_key(r[0], r[1], r[2], r[3])] = gc;
          break;
        }
    }
    if (cudaMemsetAsync(h->attn_flags, 0, kMaxSMs * sizeof(int), h->stream) != cudaSuccess ||
        !attn_plan_init(h->aplan, h->gplan.encode, std::min(h->gplan.num_sms, kMaxSMs), h->attn_flags) ||
        !xattn_plan_init()) {
      h->err = "attention plan initialisation failed";
      return fail(SDV2_E_CUDA);
    }
  }
  if (h->l2_persist) {
    // the packet (x [M, d] fp32 first) as a persisting L2 window on the handle's stream;
    // captured call graphs inherit the window as a kernel-node attribute
    int maxp = 0, maxwin = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device);
    cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, device);
    const size_t win = std::min(h->st.bytes, size_t(maxwin));
    if (maxp > 0 && win > 0) {
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(size_t(maxp), win));
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = h->packet_base;
      v.accessPolicyWindow.num_bytes = win;
      v.accessPolicyWindow.hitRatio = std::min(1.0f, float(maxp) / float(win));
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      if (cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
        h->err = "cannot set the L2 access-policy window";
        return fail(SDV2_E_CUDA);
      }
    }
  }
  if (h->prec == SDV2_BF16 && h->tune) {
    // Autotune the projection GEMMs of every tick shape (M = active entries x L) on the
    // real buffers (their contents are scratch until reset_stream).
    const BlockW& B = h->bw[0];
    const int d = h->d;
    for (int na = 1; na <= h->n; ++na) {
      const int M = na * h->B * h->L;
      EpiArgs ep{};
      ep.L = h->L; ep.mod = B.mod; ep.e0 = h->st.e0; ep.gate_row = 2; ep.rowsq = h->rowsq;
      // weights of every local block (the timed launches cycle through them)
      const int nW = h->nb;
      std::vector<const void*> wl[6];
      for (int b = 0; b < nW; ++b) {
        const BlockW& Bb = h->bw[b];
        const void* ws[6] = {Bb.wqkv, Bb.wo, Bb.wcq, Bb.wco, Bb.w1, Bb.w2};
        for (int k = 0; k < 6; ++k) wl[k].push_back(ws[k]);
      }
      const void* head_w[1] = {h->head_w_tw};
      struct Sh { const void* A; const void* const* W; int nW, N, K, epi; void* out; int ldo; const float* bias; } shapes[] = {
          {h->a, wl[0].data(), nW, 3 * d, d, EPI_STORE, h->qkv, 3 * d, B.bqkv},
          {h->o, wl[1].data(), nW, d, d, EPI_RES_GATE, h->st.x, d, B.bo},
          {h->a, wl[2].data(), nW, d, d, fused_cross_rms(h) ? EPI_STORE_RSQ : EPI_STORE, h->q, d, B.bcq},
          {h->o, wl[3].data(), nW, d, d, EPI_RES, h->st.x, d, B.bco},
          {h->a, wl[4].data(), nW, h->F, d, EPI_GELU, h->hbuf, h->F, B.b1},
          {h->hbuf, wl[5].data(), nW, d, h->F, EPI_RES_GATE, h->st.x, d, B.b2},
          {h->a, head_w, 1, h->P, d, EPI_STORE_F32, h->yh, h->P, h->gw[G_HEAD_B]},
      };
      for (auto& sh : shapes) {
        ep.out = sh.out; ep.ldo = sh.ldo; ep.bias = sh.bias;
        if (!tc_gemm_tune(h->stream, h->gplan, sh.A, sh.W, sh.nW, M, sh.N, sh.K, sh.epi, ep, &h->err))
          return fail(SDV2_E_CUDA);
      }
    }
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) return fail(SDV2_E_CUDA);
  }
  cudaFuncSetAttribute(gemv2_kernel<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gemv2_kernel<float, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gemv2_kernel<float, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gemv2_kernel<bf16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gemv2_kernel<bf16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gemv2_kernel<bf16, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  *out = h;
  return SDV2_OK;
}

sdv2_status sdv2_reset_stream(sdv2_handle* h, const sdv2_stream_desc* sd, const float* prompt_host) {
  if (!h || !sd || !prompt_host) return SDV2_E_INVALID;
  if (!sd->timesteps || sd->num_timesteps != h->n) return SDV2_E_INVALID;
  for (int j = 0; j < h->n; ++j) {
    if (!(sd->timesteps[j] > 0.f) || sd->timesteps[j] > 1000.f) return SDV2_E_INVALID;
    if (j > 0 && !(sd->timesteps[j] < sd->timesteps[j - 1])) return SDV2_E_INVALID;
  }
  if (!(sd->s_min <= sd->s_max) || sd->s_min < 0.f || sd->s_max > 1.f) return SDV2_E_INVALID;
  if (!(sd->ema_lambda > 0.f) || sd->ema_lambda > 1.f) return SDV2_E_INVALID;
  if (!(sd->motion_sigma > 0.f) || sd->motion_k < 0 || sd->motion_k >= 63) return SDV2_E_INVALID;
  if (sd->sink_tau < -1.f || sd->sink_tau > 1.f) return SDV2_E_INVALID;
  if (sd->rope_reset_frames < std::max(h->m, h->W) * h->T || sd->rope_reset_frames + h->T > 4096) return SDV2_E_INVALID;
  // captured call graphs bake the stream constants in as kernel arguments: keep them only
  // if this reset leaves those constants unchanged
  const StreamCfg old_cfg = h->scfg;
  const RopeTabs old_rt = h->rt;
  const int old_T_reset = h->T_reset;
  h->T_reset = sd->rope_reset_frames;
  std::memset(&h->scfg, 0, sizeof(h->scfg));
  for (int j = 0; j < kMaxSteps; ++j) h->scfg.t[j] = j < h->n ? sd->timesteps[j] : 0.f;
  h->scfg.n = h->n;
  h->scfg.k = sd->motion_k;
  h->scfg.sigma_m = sd->motion_sigma;
  h->scfg.s_min = sd->s_min;
  h->scfg.s_max = sd->s_max;
  h->scfg.lam = sd->ema_lambda;
  h->scfg.seed = sd->seed;
  CtlParams p;
  p.T = h->T; p.m = h->m; p.W = h->W; p.n = h->n; p.K = h->K; p.rank = h->rank; p.T_reset = h->T_reset;
  p.B = h->B;
  p.tau = sd->sink_tau;
  h->ctl.reset(p);
  // RoPE tables (C.6): temporal positions -t_off..t_off, height 0..hn-1, width 0..wn-1; fp64 -> fp32
  const int t_off = h->T_reset + h->T + 1;
  {
    std::vector<float> tab;
    const int rows_t = 2 * t_off + 1;
    tab.resize(size_t(rows_t) * h->ct * 2 + size_t(h->hn) * h->ch * 2 + size_t(h->wn) * h->cw * 2);
    float* p0 = tab.data();
    auto fill = [&](float* cs, float* sn, int rows, int c, int base) {
      for (int r = 0; r < rows; ++r)
        for (int i = 0; i < c; ++i) {
          const double om = std::pow(10000.0, -double(i) / double(c));
          const double ang = double(r + base) * om;
          cs[size_t(r) * c + i] = float(std::cos(ang));
          sn[size_t(r) * c + i] = float(std::sin(ang));
        }
    };
    float* tcs = p0; float* tsn = tcs + size_t(rows_t) * h->ct;
    float* hcs = tsn + size_t(rows_t) * h->ct; float* hsn = hcs + size_t(h->hn) * h->ch;
    float* wcs = hsn + size_t(h->hn) * h->ch; float* wsn = wcs + size_t(h->wn) * h->cw;
    fill(tcs, tsn, rows_t, h->ct, -t_off);
    fill(hcs, hsn, h->hn, h->ch, 0);
    fill(wcs, wsn, h->wn, h->cw, 0);
    CK(cudaMemcpyAsync(h->rope, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, h->stream));
    const size_t o_tsn = size_t(rows_t) * h->ct, o_hcs = 2 * o_tsn, o_hsn = o_hcs + size_t(h->hn) * h->ch,
                 o_wcs = o_hsn + size_t(h->hn) * h->ch, o_wsn = o_wcs + size_t(h->wn) * h->cw;
    h->rt.ct_cos = h->rope; h->rt.ct_sin = h->rope + o_tsn;
    h->rt.ch_cos = h->rope + o_hcs; h->rt.ch_sin = h->rope + o_hsn;
    h->rt.cw_cos = h->rope + o_wcs; h->rt.cw_sin = h->rope + o_wsn;
    h->rt.ct = h->ct; h->rt.ch = h->ch; h->rt.cw = h->cw; h->rt.t_off = t_off;
    CK(cudaStreamSynchronize(h->stream));   // the host table vector dies here
  }
  if (old_T_reset != h->T_reset || std::memcmp(&old_cfg, &h->scfg, sizeof(StreamCfg)) != 0 ||
      std::memcmp(&old_rt, &h->rt, sizeof(RopeTabs)) != 0)
    drop_graphs(h);
  h->td_prev_valid = false;   // kv_mode 1: nothing finished yet to re-run
  // zero lanes, controller state
  const size_t kv = size_t(h->nb) * h->NE * h->S * h->L * h->d * h->ta;
  CK(cudaMemsetAsync(h->Kc, 0, kv, h->stream));
  CK(cudaMemsetAsync(h->Vc, 0, kv, h->stream));
  // Attention key tiles are 128 rows and may extend past a lane's valid keys into other
  // slots / blocks / prompt versions: those rows get P = 0, but must hold finite values
  // (0 x NaN = NaN in the PV MMA), so every K/V buffer starts zeroed.
  const size_t px = size_t(2) * h->B * h->nb * h->Lt * h->d * h->ta;
  CK(cudaMemsetAsync(h->Kx, 0, px, h->stream));
  CK(cudaMemsetAsync(h->Vx, 0, px, h->stream));
  CK(cudaMemsetAsync(h->packet_base, 0, h->st.bytes, h->stream));
  for (int io = 0; io < 2; ++io)
    for (int par = 0; par < 2; ++par)
      if (h->act_io[io][par]) CK(cudaMemsetAsync(h->act_io[io][par], 0, h->st.bytes, h->stream));
  {
    std::vector<CtrlState> cs(h->B);
    std::memset(cs.data(), 0, sizeof(CtrlState) * h->B);
    for (auto& c : cs) c.s = double(sd->s_max);   // s_{-1} = s_max (Q15)
    CK(cudaMemcpyAsync(h->ctrl, cs.data(), sizeof(CtrlState) * h->B, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  for (int b = 0; b < h->B; ++b) {
    h->pver[b] = 0;
    h->last_switch_call[b] = -1;
    sdv2_status s = set_prompt_common(h, prompt_host + size_t(b) * h->Lt * h->Dt, b, 0);
    if (s != SDV2_OK) return s;
  }
  h->stream_ready = true;
  return SDV2_OK;
}

sdv2_status sdv2_set_prompt(sdv2_handle* h, int32_t stream, const float* prompt_host) {
  if (!h || !prompt_host || stream < 0 || stream >= h->B) return SDV2_E_INVALID;
  if (!h->stream_ready) return SDV2_E_STATE;
  const int b = stream;
  // Versions alternate between two resident slots: the switch to version v overwrites
  // the slot of version v-2, whose last chunk was admitted at call c_{v-1} - 1 and is
  // processed (entry j = n-1) at call c_{v-1} - 1 + (n-1) K.  The overwrite is ordered
  // before call c_v, so it is safe iff c_v - c_{v-1} >= (n-1) K.
  const int64_t now = h->ctl.calls();
  if (h->last_switch_call[b] >= 0 && now - h->last_switch_call[b] < int64_t(h->n - 1) * h->K) {
    h->err = "prompt switch too soon: " + std::to_string(now - h->last_switch_call[b]) + " calls after the previous one, " +
             std::to_string(int64_t(h->n - 1) * h->K) + " needed (two prompt versions are resident)";
    return SDV2_E_STATE;
  }
  sdv2_status s = set_prompt_common(h, prompt_host, b, h->pver[b] + 1);
  if (s == SDV2_OK) {
    h->pver[b] += 1;
    h->last_switch_call[b] = now;
  }
  return s;
}

sdv2_status sdv2_set_chunk_embedding(sdv2_handle* h, int32_t stream, const double* emb, int32_t dim) {
  if (!h || !emb || dim < 1 || stream < 0 || stream >= h->B) return SDV2_E_INVALID;
  double nrm = 0.0;
  for (int i = 0; i < dim; ++i) nrm += emb[i] * emb[i];
  if (!(nrm > 0.0)) {
    h->err = "zero-norm chunk embedding";
    return SDV2_E_INVALID;
  }
  h->ctl.set_chunk_embedding(stream, std::vector<double>(emb, emb + dim));
  return SDV2_OK;
}

sdv2_status sdv2_denoise_chunk(sdv2_handle* h, const float* chunk_latent, float* out_latent, int64_t* out_chunk_index) {
  if (!h) return SDV2_E_INVALID;
  if (!h->stream_ready) return SDV2_E_STATE;
  if (h->rank == 0 && !chunk_latent) return SDV2_E_STATE;
  if (h->rank != 0 && chunk_latent) return SDV2_E_STATE;
  if (h->rank != h->K - 1 && out_latent) return SDV2_E_STATE;
  return h->prec == SDV2_FP32 ? tick<float>(h, chunk_latent, out_latent, out_chunk_index)
                              : tick<bf16>(h, chunk_latent, out_latent, out_chunk_index);
}

sdv2_status sdv2_stage_io_buffers(sdv2_handle* h, int32_t parity, sdv2_stage_io* io) {
  if (!h || !io || parity < 0 || parity > 1) return SDV2_E_INVALID;
  io->act_in = h->act_io[0][parity];
  io->act_out = h->rank == 0 ? h->act_io[1][parity] : h->act_io[0][parity];   // in place (packet_for)
  io->act_bytes = h->K > 1 ? h->st.bytes : 0;
  io->ring_in = h->ring[0][parity];
  io->ring_out = h->ring[1][parity];
  io->ring_bytes = size_t(h->n > 1 ? h->n - 1 : 0) * h->B * h->CTHW * 4;
  return SDV2_OK;
}

sdv2_status sdv2_get_tick_info(const sdv2_handle* h, sdv2_tick_info* info) {
  if (!h || !info) return SDV2_E_INVALID;
  *info = h->info;
  info->kernel_launches = h->launches;
  return SDV2_OK;
}

sdv2_status sdv2_get_cache_state(sdv2_handle* h, int32_t local_block, int32_t lane, sdv2_cache_state* st) {
  if (!h || !st || local_block < 0 || local_block >= h->nb || lane < 0 || lane >= h->NE) return SDV2_E_INVALID;
  const LaneMeta& L = h->ctl.lane(lane);
  std::memset(st, 0, sizeof(*st));
  st->num_slots = h->S;
  st->num_valid = L.nvalid;
  for (int s = 0; s < h->S; ++s) {
    st->tag[s] = L.tag[s];
    st->pos[s] = L.pos[s][0];
  }
  st->resets = L.r;
  st->evictions = L.evictions;
  if (h->rank == 0) {
    CtrlState cs;
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(&cs, h->ctrl + lane % h->B, sizeof(cs), cudaMemcpyDeviceToHost));
    st->noise_rate = cs.s;
    st->d_hat = cs.d_hat;
  }
  return SDV2_OK;
}

sdv2_status sdv2_set_block_tap(sdv2_handle* h, float* per_block_out) {
  if (!h) return SDV2_E_INVALID;
  h->tap = per_block_out;
  return SDV2_OK;
}

sdv2_status sdv2_kv_lane(sdv2_handle* h, int32_t local_block, int32_t lane, int32_t which, void** ptr, size_t* elems) {
  if (!h || !ptr || !elems || local_block < 0 || local_block >= h->nb || lane < 0 || lane >= h->NE) return SDV2_E_INVALID;
  const size_t per_lane = size_t(h->S) * h->L * h->d;
  char* base = static_cast<char*>(which ? h->Vc : h->Kc);
  *ptr = base + ((size_t(local_block) * h->NE + lane) * per_lane) * h->ta;
  *elems = per_lane;
  return SDV2_OK;
}

sdv2_status sdv2_debug_sync(sdv2_handle* h, int32_t enable) {
  if (!h) return SDV2_E_INVALID;
  h->debug_sync = enable != 0;
  return SDV2_OK;
}

sdv2_status sdv2_set_graphs(sdv2_handle* h, int32_t enable) {
  if (!h) return SDV2_E_INVALID;
  h->graphs = enable != 0;
  return SDV2_OK;
}

sdv2_status sdv2_profile_enable(sdv2_handle* h, int32_t enable) {
  if (!h) return SDV2_E_INVALID;
  CK(cudaStreamSynchronize(h->stream));
  h->prof = enable != 0;
  h->prof_recs.clear();
  h->ev_next = 0;
  std::memset(&h->prof_acc, 0, sizeof(h->prof_acc));
  h->prof_blk_ms.assign(h->nb, 0.0);
  h->prof_blk_n.assign(h->nb, 0);
  return SDV2_OK;
}

sdv2_status sdv2_profile_read(sdv2_handle* h, sdv2_profile* out) {
  if (!h || !out) return SDV2_E_INVALID;
  CK(cudaStreamSynchronize(h->stream));
  // SDV2_PROF_DETAIL=1: per (class, work) breakdown on stderr (one line per GEMM shape)
  const bool detail = getenv("SDV2_PROF_DETAIL") != nullptr;
  std::map<std::pair<int, double>, std::pair<int, double>> det;
  if (int(h->prof_blk_ms.size()) != h->nb) {
    h->prof_blk_ms.assign(h->nb, 0.0);
    h->prof_blk_n.assign(h->nb, 0);
  }
  for (auto& r : h->prof_recs) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    if (r.blk >= 0 && r.blk < h->nb) {
      h->prof_blk_ms[r.blk] += ms;
      h->prof_blk_n[r.blk] += 1;
    }
    h->prof_acc.launches[r.cls] += 1;
    h->prof_acc.ms[r.cls] += ms;
    h->prof_acc.flops[r.cls] += r.flops;
    if (detail) {
      auto& d = det[{r.cls, r.flops}];
      d.first += 1;
      d.second += ms;
    }
  }
  for (auto& kv : det)
    fprintf(stderr, "sdv2 prof class %d work %.4g: %d launches, avg %.2f us, %.0f TFLOP/s\n", kv.first.first,
            kv.first.second, kv.second.first, kv.second.second * 1e3 / kv.second.first,
            kv.second.first * kv.first.second / (kv.second.second * 1e-3) / 1e12);
  h->prof_recs.clear();
  h->ev_next = 0;
  *out = h->prof_acc;
  return SDV2_OK;
}

sdv2_status sdv2_profile_block_ms(sdv2_handle* h, double* out, int32_t count) {
  if (!h || !out || count < h->nb) return SDV2_E_INVALID;
  sdv2_profile tmp;
  sdv2_status s = sdv2_profile_read(h, &tmp);   // folds pending event pairs into the accumulators
  if (s != SDV2_OK) return s;
  for (int i = 0; i < h->nb; ++i) out[i] = h->prof_blk_n[i] ? h->prof_blk_ms[i] / double(h->prof_blk_n[i]) : 0.0;
  return SDV2_OK;
}

sdv2_status sdv2_set_block_range(sdv2_handle* h, int32_t block_begin, int32_t block_end) {
  if (!h) return SDV2_E_INVALID;
  if (block_begin < h->r0 || block_end > h->r0 + h->nb || block_begin >= block_end) {
    h->err = "block range outside the resident range";
    return SDV2_E_INVALID;
  }
  if (block_begin == h->b0 && block_end == h->b1) return SDV2_OK;
  CK(cudaStreamSynchronize(h->stream));
  h->b0 = block_begin;
  h->b1 = block_end;
  h->a0 = block_begin - h->r0;
  h->a1 = block_end - h->r0;
  drop_graphs(h);   // the captured call bodies loop over the old range
  return SDV2_OK;
}

sdv2_status sdv2_block_kv(sdv2_handle* h, int32_t block, int32_t which, void** ptr, size_t* bytes) {
  if (!h || !ptr || !bytes || block < h->r0 || block >= h->r0 + h->nb || which < 0 || which > 1) return SDV2_E_INVALID;
  const size_t per_block = size_t(h->NE) * h->S * h->L * h->d;
  char* base = static_cast<char*>(which ? h->Vc : h->Kc);
  *ptr = base + size_t(block - h->r0) * per_block * h->ta;
  *bytes = per_block * h->ta;
  return SDV2_OK;
}

sdv2_status sdv2_gemm_configs(const sdv2_handle* h, int32_t* out, int32_t cap, int32_t* count) {
  if (!h || !count || (cap > 0 && !out)) return SDV2_E_INVALID;
  int32_t n = 0;
  for (const auto& kv : h->gplan.tuned) {
    int M = 0, N = 0, K = 0, epi = 0;
    if (sscanf(kv.first.c_str(), "%d:%d:%d:%d", &M, &N, &K, &epi) != 4) continue;
    if (n < cap) {
      const int32_t rec[8] = {M, N, K, epi, kv.second.MC, kv.second.BN, kv.second.SK, kv.second.XE};
      std::memcpy(out + size_t(n) * 8, rec, sizeof(rec));
    }
    ++n;
  }
  *count = n;
  return SDV2_OK;
}

sdv2_status sdv2_destroy(sdv2_handle* h) {
  if (!h) return SDV2_E_INVALID;
  if (h->stream_ready || h->td_host) cudaStreamSynchronize(h->stream);
  for (int i = 0; i < kTdRing; ++i)
    if (h->td_host) cudaEventDestroy(h->td_ev[i]);
  if (h->td_host) cudaFreeHost(h->td_host);
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  drop_graphs(h);
  delete h;
  return SDV2_OK;
}

}  // extern "C"

namespace {
// Test-hook GEMM plan with a private stream-K partial workspace (the product path never
// runs stream-K; the hook keeps it reachable for kernel tests).
bool debug_gemm_plan(TmaGemmPlan*& out, std::string* err) {
  static TmaGemmPlan plan;
  static bool ready = false;
  if (!ready) {
    if (!tc_gemm_plan(plan, err)) return false;
    if (cudaMalloc(&plan.sk_ws, size_t(plan.num_sms) * kGemmSkSlotFloats * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&plan.sk_flags, size_t(plan.num_sms) * sizeof(int)) != cudaSuccess ||
        cudaMemset(plan.sk_flags, 0, size_t(plan.num_sms) * sizeof(int)) != cudaSuccess) {
      *err = "test-hook stream-K workspace allocation failed";
      return false;
    }
    ready = true;
  }
  out = &plan;
  return true;
}
}  // namespace

extern "C" sdv2_status sdv2_debug_gemm_candidates(int32_t M, int32_t N, int32_t K, int32_t epi, int32_t* cfg4,
                                                  int32_t max_cfgs, int32_t* count) {
  TmaGemmPlan* pl = nullptr;
  std::string err;
  if (!cfg4 || !count || !debug_gemm_plan(pl, &err)) return SDV2_E_INVALID;
  if (!tc_gemm_check(N, K, epi, &err)) return SDV2_E_SHAPE;
  const std::vector<GemmCfg> c = tc_gemm_candidates(*pl, M, N, epi);
  *count = int32_t(c.size());
  for (int i = 0; i < int(c.size()) && i < max_cfgs; ++i) {
    cfg4[4 * i] = c[i].MC; cfg4[4 * i + 1] = c[i].BN; cfg4[4 * i + 2] = c[i].SK; cfg4[4 * i + 3] = c[i].XE;
  }
  return SDV2_OK;
}

extern "C" sdv2_status sdv2_debug_gemm_cfg(const void* A, const void* W, const float* bias, void* out, int32_t M,
                                           int32_t N, int32_t K, int32_t epi, const float* mod, const float* e0,
                                           int32_t gate_row, int32_t L, const int32_t* cfg4, void* stream) {
  TmaGemmPlan* pl = nullptr;
  std::string err;
  if (!cfg4 || !debug_gemm_plan(pl, &err)) return SDV2_E_INVALID;
  EpiArgs ep{};
  ep.out = out;
  ep.ldo = N;
  ep.bias = bias;
  ep.mod = mod;
  ep.e0 = e0;
  ep.gate_row = gate_row;
  ep.L = L > 0 ? L : 1;
  GemmCfg gc{cfg4[0], cfg4[1], cfg4[2]};
  gc.XE = cfg4[3];
  if (!tc_gemm_check(N, K, epi, &err) ||
      !tc_gemm_cfg(static_cast<cudaStream_t>(stream), *pl, A, W, M, N, K, epi, ep, gc, &err)) {
    fprintf(stderr, "sdv2_debug_gemm_cfg: %s\n", err.c_str());
    return SDV2_E_CUDA;
  }
  return SDV2_OK;
}

extern "C" sdv2_status sdv2_debug_gemm(const void* A, const void* W, const float* bias, void* out, int32_t M, int32_t N,
                                       int32_t K, int32_t epi, const float* mod, const float* e0, int32_t gate_row,
                                       int32_t L, void* stream) {
  TmaGemmPlan* pl = nullptr;
  std::string err;
  if (!debug_gemm_plan(pl, &err)) return SDV2_E_CUDA;
  TmaGemmPlan& plan = *pl;
  EpiArgs ep{};
  ep.out = out;
  ep.ldo = N;
  ep.bias = bias;
  ep.mod = mod;
  ep.e0 = e0;
  ep.gate_row = gate_row;
  ep.L = L > 0 ? L : 1;
  // SDV2_GEMM_TRACE=<file>: clock64 stamps of CTAs 0 and 1 (pipeline analysis)
  const char* trace_path = getenv("SDV2_GEMM_TRACE");
  static long long* trace = nullptr;
  const size_t tn = 2 * 4096 + 1024 * 4;
  if (trace_path) {
    if (!trace && cudaMalloc(&trace, tn * sizeof(long long)) != cudaSuccess) return SDV2_E_CUDA;
    cudaMemsetAsync(trace, 0, tn * sizeof(long long), static_cast<cudaStream_t>(stream));
    ep.trace = trace;
  }
  ep.dbg = getenv("SDV2_GEMM_DBG") ? atoi(getenv("SDV2_GEMM_DBG")) : 0;
  // SDV2_GEMM_CFG="MC,BN,SK": explicit configuration (else the default balance model)
  bool ok;
  if (const char* cfg = getenv("SDV2_GEMM_CFG")) {
    GemmCfg gc{1, 128, 0};
    sscanf(cfg, "%d,%d,%d", &gc.MC, &gc.BN, &gc.SK);
    ok = tc_gemm_check(N, K, epi, &err) &&
         tc_gemm_cfg(static_cast<cudaStream_t>(stream), plan, A, W, M, N, K, epi, ep, gc, &err);
  } else {
    ok = tc_gemm(static_cast<cudaStream_t>(stream), plan, A, W, M, N, K, epi, ep, &err);
  }
  if (!ok) {
    fprintf(stderr, "sdv2_debug_gemm: %s\n", err.c_str());
    return SDV2_E_CUDA;
  }
  if (trace_path) {
    std::vector<long long> h(tn);
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    cudaMemcpy(h.data(), trace, tn * sizeof(long long), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_path, "w")) {
      for (size_t i = 0; i < 8192 / 8; ++i) {
        for (int e = 0; e < 8; ++e) fprintf(f, "%lld%c", h[i * 8 + e], e == 7 ? '\n' : ',');
      }
      fclose(f);
    }
    if (FILE* f = fopen((std::string(trace_path) + ".cta").c_str(), "w")) {
      for (int t = 0; t < 1024; ++t)
        for (int e = 0; e < 4; ++e) fprintf(f, "%lld%c", h[8192 + t * 4 + e], e == 3 ? '\n' : ',');
      fclose(f);
    }
  }
  return SDV2_OK;
}

extern "C" sdv2_status sdv2_debug_attention(const void* q, const void* K, const void* V, void* o, int32_t Lq,
                                            int32_t Lk, int32_t H, int32_t hd, void* scratch, void* stream) {
  static TmaGemmPlan gp;
  static AttnPlan ap;
  static bool ready = false;
  static int* flags = nullptr;
  std::string err;
  if (!ready) {
    if (!tc_gemm_plan(gp, &err)) return SDV2_E_CUDA;
    if (cudaMalloc(&flags, kMaxSMs * sizeof(int)) != cudaSuccess ||
        cudaMemset(flags, 0, kMaxSMs * sizeof(int)) != cudaSuccess ||
        !attn_plan_init(ap, gp.encode, std::min(gp.num_sms, kMaxSMs), flags) || !xattn_plan_init())
      return SDV2_E_CUDA;
    ready = true;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // one active entry, written on every call from a pinned host copy (asynchronous: no
  // stream serialisation; a caller's new scratch tensor may reuse a freed address, so
  // "written once per buffer" is not safe)
  static TickDesc* tdh = nullptr;
  if (!tdh) {
    if (cudaMallocHost(&tdh, sizeof(TickDesc)) != cudaSuccess) return SDV2_E_CUDA;
    std::memset(tdh, 0, sizeof(TickDesc));
    tdh->n_active = 1;
    tdh->e[0].active = 1;
  }
  if (cudaMemcpyAsync(scratch, tdh, sizeof(TickDesc), cudaMemcpyHostToDevice, s) != cudaSuccess) return SDV2_E_CUDA;
  static float* part = nullptr;
  if (!part && cudaMalloc(&part, attn_scratch_floats(kMaxSMs, 128) * 4) != cudaSuccess) return SDV2_E_CUDA;
  AttnTcArgs ta{};
  ta.L = Lq;
  ta.cross = 1;
  ta.Lk_cross = Lk;
  ta.H = H;
  ta.QT = (Lq + kAttnBQ - 1) / kAttnBQ;
  ta.n_entries = 1;
  ta.part_o = part;
  ta.part_ml = part + size_t(kMaxSMs) * 2 * kAttnBQ * hd;
  ta.scale_log2 = 1.4426950408889634f / sqrtf(float(hd));
  ta.o = o;
  ta.ldo = H * hd;
  ta.kv_row0 = 0;
  ta.kv_lane_rows = 0;
  const long long tiles = (long long)H * ta.QT * ((Lk + kAttnBKV - 1) / kAttnBKV);
  if (Lk <= kXattnMaxJ * kAttnBKV) {   // the product path's cross-attention kernel for short key sets
    XattnArgs xa{};
    xa.L = Lq;
    xa.H = H;
    xa.QT = (Lq + kAttnBQ - 1) / kAttnBQ;
    xa.n_entries = 1;
    xa.Lk = Lk;
    xa.kv_row0 = 0;
    xa.kv_slot_rows = 0;
    xa.scale_log2 = 1.4426950408889634f / sqrtf(float(hd));
    xa.o = o;
    xa.ldo = H * hd;
    // SDV2_ATTN_TRACE=<file>: CTA wall stamps of the cross kernel to <file>.xcta (test hook)
    const char* xtrace_path = getenv("SDV2_ATTN_TRACE");
    static long long* xtrace = nullptr;
    if (xtrace_path) {
      if (!xtrace && cudaMalloc(&xtrace, (4096 + 1024 * 8) * sizeof(long long)) != cudaSuccess) return SDV2_E_CUDA;
      cudaMemsetAsync(xtrace, 0, (4096 + 1024 * 8) * sizeof(long long), s);
      xa.trace = xtrace;
    }
    if (!tc_cross_attention(s, ap, q, Lq, K, V, Lk, H * hd, hd, xa, static_cast<const TickDesc*>(scratch), &err)) {
      fprintf(stderr, "sdv2_debug_attention: %s\n", err.c_str());
      return SDV2_E_CUDA;
    }
    if (xtrace_path) {
      std::vector<long long> hx(4096 + 1024 * 8);
      cudaStreamSynchronize(s);
      cudaMemcpy(hx.data(), xtrace, hx.size() * sizeof(long long), cudaMemcpyDeviceToHost);
      if (FILE* f = fopen((std::string(xtrace_path) + ".xcta").c_str(), "w")) {
        for (int t = 0; t < 1024; ++t)
          for (int e = 0; e < 8; ++e) fprintf(f, "%lld%c", hx[4096 + t * 8 + e], e == 7 ? '\n' : ',');
        fclose(f);
      }
    }
    return SDV2_OK;
  }
  ta.per_unit = getenv("SDV2_ATTN_PER_UNIT") ? atoi(getenv("SDV2_ATTN_PER_UNIT")) : 0;
  ta.rr = attn_rr();
  ta.dbg = getenv("SDV2_ATTN_DBG") ? atoi(getenv("SDV2_ATTN_DBG")) : 0;
  // SDV2_ATTN_TRACE=<file>: per-tile clock64 stamps of CTA 0 (pipeline analysis)
  const char* trace_path = getenv("SDV2_ATTN_TRACE");
  static long long* trace = nullptr;
  if (trace_path) {
    if (!trace && cudaMalloc(&trace, (256 * 16 + 1024 * 4) * sizeof(long long)) != cudaSuccess) return SDV2_E_CUDA;
    cudaMemsetAsync(trace, 0, (256 * 16 + 1024 * 4) * sizeof(long long), s);
    ta.trace = trace;
  }
  if (!tc_attention(s, ap, q, Lq, K, V, Lk, H * hd, hd, tiles, ta, static_cast<const TickDesc*>(scratch), &err)) {
    fprintf(stderr, "sdv2_debug_attention: %s\n", err.c_str());
    return SDV2_E_CUDA;
  }
  if (trace_path) {
    std::vector<long long> h(256 * 16 + 1024 * 4);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_path, "w")) {
      for (int t = 0; t < 256; ++t) {
        for (int e = 0; e < 16; ++e) fprintf(f, "%lld%c", h[t * 16 + e], e == 15 ? '\n' : ',');
      }
      fclose(f);
    }
    if (FILE* f = fopen((std::string(trace_path) + ".cta").c_str(), "w")) {
      for (int t = 0; t < 1024; ++t)
        for (int e = 0; e < 4; ++e) fprintf(f, "%lld%c", h[4096 + t * 4 + e], e == 3 ? '\n' : ',');
      fclose(f);
    }
  }
  return SDV2_OK;
}
