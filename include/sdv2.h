/*
 * sdv2.h — C ABI of the B200-native StreamDiffusionV2 stream-batched causal-DiT hot path.
 *
 * Citations: "P:n" = line n of the paper's LaTeX (PAPER.md, arXiv 2511.07399);
 * SURVEY.md §8 is the scope contract and DESIGN.md lists every reading taken where
 * the paper is silent.
 *
 * The library denoises a live stream of latent chunks (inputs reformulated as
 * B x T' x H x W with small T') with n = B in-flight (chunk, step) entries per pass
 * (Stream Batch, P:164 / P:227: "treating the n denoising steps as an effective batch
 * multiplier").  Each pass ("stage-tick") runs, for every entry, the causal DiT blocks
 * of this rank: adaLN-modulated norm, QKV/out/FFN projections, 3D RoPE with reset
 * temporal offsets, attention over the entry's [sink || rolling window] KV
 * lane, prompt cross-attention, the ring-buffer cache update and,
 * on the first rank, the motion-aware noise blend.  DiT blocks may be
 * split across ranks (pipeline parallel); the hand-off buffers are
 * exposed so the caller's transport (torch.distributed / NCCL) moves them.
 *
 * Conventions
 *  - Every call returns sdv2_status; nothing throws across the ABI.
 *  - All device work is enqueued on the stream given to sdv2_create; calls return
 *    before completion.  A handle is single-owner and not thread-safe.
 *  - The library never calls cudaMalloc on the product path: all device memory is the
 *    caller-owned workspace (sdv2_workspace_bytes), carved at create (weights, KV lanes,
 *    activations, attention split partials and hand-off flags).  The small pinned host
 *    staging area for per-tick descriptors is allocated with cudaHostAlloc; sdv2_destroy
 *    frees it.  (The kernel-level test hooks at the end own a private scratch.)
 *  - No environment variable changes what the product path computes or how fast:
 *    execution choices are the explicit sdv2_exec_options given to sdv2_create.
 *  - Tensors are row-major, fp32 unless stated.
 */
#ifndef SDV2_H
#define SDV2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SDV2_OK = 0,
  SDV2_E_INVALID = -1,     /* bad controller / schedule / prompt argument            */
  SDV2_E_SHAPE = -2,       /* inconsistent model / geometry shape                     */
  SDV2_E_STATE = -3,       /* call out of order, or wrong pointer role for this rank  */
  SDV2_E_WORKSPACE = -4,   /* workspace missing or too small                          */
  SDV2_E_CUDA = -5,        /* CUDA runtime error (text in sdv2_last_error)            */
  SDV2_E_UNSUPPORTED = -6  /* shape outside what the kernels are built for            */
} sdv2_status;

typedef enum { SDV2_FP32 = 0, SDV2_BF16 = 1 } sdv2_precision;

/* Model card (SURVEY.md §8(c) C.1–C.8; Wan2.1-shaped causal DiT).
 * head_dim = dim / num_heads must be even (RoPE pairs) and is 64 or 128 on the bf16 path. */
typedef struct {
  int32_t num_blocks, dim, num_heads, ffn_dim;
  int32_t latent_channels, patch_t, patch_h, patch_w;  /* patch must be (1,2,2) */
  int32_t text_len, text_dim, freq_dim;                /* freq_dim = 256 */
  float eps;                                           /* 1e-6 */
  int32_t norm_center;                                 /* 0 = RMSNorm, 1 = LayerNorm (affine-free) */
} sdv2_model_desc;

/* Stream geometry ("B x T' x H x W"; P:190 sink set size m; P:472 rolling window).
 * `streams` independent latent streams (the SLO batch B of P:174-185; "different colors
 * denote distinct latent streams", Fig. parallel) are batched into every call, each with
 * its own noise controller, prompt, sink set and KV lanes.  A call holds streams x steps
 * entries (<= 16): entry e = j * streams + b is step j of stream b and uses KV lane e. */
typedef struct {
  int32_t latent_h, latent_w;   /* latent frame; divisible by the patch */
  int32_t chunk_frames;         /* T' latent frames per chunk (<= 16)   */
  int32_t steps;                /* n denoising steps in flight per stream (Stream Batch, <= 8) */
  int32_t sink_chunks;          /* m >= 0 sink chunks (first chunks, refreshed by P:190) */
  int32_t window_chunks;        /* W >= 1 rolling-window chunks, current chunk included */
  int32_t streams;              /* B >= 1 streams per call; streams * steps <= 16 */
  int32_t kv_mode;              /* what the KV lanes cache (SURVEY reading Q5):
                                 *  0 = step-j K/V in lane j, written during the step (R1);
                                 *  1 = clean-context re-run (Q5-clean, CausVid, EXT; N4):
                                 *      each call first re-runs the previous call's finished
                                 *      chunks through the DiT on their prediction x0 at
                                 *      t = 0 and overwrites their cached K/V (sink fill /
                                 *      window slot / refreshed sinks) before admitting the
                                 *      new chunk.  Needs steps == 1 and a single stage
                                 *      (SDV2_E_UNSUPPORTED otherwise); ~2x DiT work per call. */
} sdv2_geometry;

/* Pipeline stage of this handle.  world = K stages; this rank runs DiT
 * blocks [block_begin, block_end).  NULL desc = single stage owning every block.
 * Online re-partitioning ("dynamically reallocates blocks between devices"):
 * the handle keeps weights, prompt K/V and KV lanes for the resident blocks
 * [resident_begin, resident_end) ⊇ [block_begin, block_end) (0, 0 = the block range), so
 * sdv2_set_block_range can move the boundary inside it after the moved blocks' KV lanes
 * were copied in (sdv2_block_kv).  local_block arguments below index the resident range. */
typedef struct {
  int32_t world, rank, block_begin, block_end;
  int32_t resident_begin, resident_end;
} sdv2_pipeline_desc;

/* Weights: fp32 values that are bf16-representable, nn.Linear
 * layout [out, in], host or device pointers (copied with cudaMemcpyDefault and packed
 * into the workspace during sdv2_create; the caller may free them afterwards).
 * Order: the 15 global tensors
 *   patch_w[d,4C] patch_b[d] txt1_w[d,Dt] txt1_b[d] txt2_w[d,d] txt2_b[d]
 *   t1_w[d,256] t1_b[d] t2_w[d,d] t2_b[d] tp_w[6d,d] tp_b[6d] head_mod[2,d] head_w[4C,d] head_b[4C]
 * then, for each RESIDENT block b (sdv2_pipeline_desc), the 27 block tensors
 *   mod[6,d] wq bq wk bk wv bv wo bo gq gk n3_g n3_b wcq bcq wck bck wcv bcv wco bco gcq gck
 *   w1[F,d] b1[F] w2[d,F] b2[d]            ([d,d] / [d] unless stated)            */
typedef struct {
  const void* const* tensors;
  int32_t count;
} sdv2_weights;

/* Per-stream controls (P:190 tau; P:191 T_reset; P:210–219 k, sigma, s_min, s_max, lambda).
 * timesteps: host array of `steps` strictly decreasing values, t_0 in (0, 1000]; the
 * noise level of step j of chunk X is sigma = s_X * t_j / t_0 (reading R5).
 * seed keys the Philox4x32-10 noise (counter layout in DESIGN.md); stream b uses the key
 * (seed_lo32, seed_hi32 + b).  Every stream shares these controls. */
typedef struct {
  const float* timesteps;
  int32_t num_timesteps;
  int32_t rope_reset_frames;    /* T_reset >= max(m, W) * T', T_reset + T' <= 4096 */
  int32_t motion_k;             /* window of k+1 motion values, 0 <= k <= 62 */
  float motion_sigma;           /* > 0 */
  float s_min, s_max;           /* 0 <= s_min <= s_max <= 1 (equal: a constant noise rate) */
  float ema_lambda;             /* in (0, 1] */
  float sink_tau;               /* in [-1, 1] */
  uint64_t seed;
} sdv2_stream_desc;

/* Stage hand-off buffers (device pointers inside the workspace), "transmits the
 * results to the next stage within a ring structure".  For call index c on this rank
 * the library reads act_in/ring_in of parity c%2 and writes act_out/ring_out of parity
 * c%2.  Rank s>0 must receive, before its call c, the act packet rank s-1 produced at
 * its call c; rank 0 (world > 1) must receive, before its call c >= K, the ring packet
 * the last rank produced at its call c-K.  The packet is computed in place: on ranks
 * s > 0 act_out == act_in (the received buffer is updated and sent on), so a send of call
 * c must complete before the receive for call c+2 lands in the same parity buffer (NCCL
 * groups on one communicator are ordered; pipeline.py waits a send one call later).
 * K = 1 needs no transport. */
typedef struct {
  void* act_in;  void* act_out;  size_t act_bytes;
  void* ring_in; void* ring_out; size_t ring_bytes;
} sdv2_stage_io;

/* Per-call schedule introspection (host-only; deterministic R2 schedule). */
typedef struct {
  int64_t call;                  /* call index on this rank                         */
  int32_t num_entries;           /* active entries this call (prefix of e = j B + b) */
  int32_t steps;
  int64_t chunk[8];              /* chunk X of step j, every stream (-1 if inactive) */
  int64_t out_chunk;             /* chunk whose clean latent this call emits, or -1 */
  int64_t kernel_launches;       /* cumulative kernels this handle has launched      */
} sdv2_tick_info;

/* Per-kernel-class device time (CUDA events around each launch on the handle's
 * stream) and algorithmic work, accumulated while profiling is enabled.
 * Classes: 0 projection GEMMs, 1 self-attention, 2 cross-attention, 3 other,
 * 4 whole DiT blocks (one span per local block and call: the per-block stage time the
 * partition balances), 5 stage extras outside the blocks (rank 0: noise
 * controller + patch / time embedding; last rank: head + x0 + output).  Spans of
 * classes 4/5 contain the launches of classes 0-3. */
#define SDV2_PROFILE_CLASSES 6
typedef struct {
  int64_t launches[SDV2_PROFILE_CLASSES];
  double ms[SDV2_PROFILE_CLASSES];
  double flops[SDV2_PROFILE_CLASSES];
} sdv2_profile;

/* Cache metadata of one (local block, lane) after the last call (test introspection). */
typedef struct {
  int32_t num_slots;             /* m + W                                            */
  int32_t num_valid;             /* valid slots (always a prefix)                    */
  int64_t tag[64];               /* chunk held by slot s, -1 = empty                 */
  int32_t pos[64];               /* temporal position of the slot's first frame      */
  int32_t resets;                /* r                                                */
  int64_t evictions;
  double noise_rate;             /* s of the last admitted chunk (rank 0)            */
  double d_hat;                  /* d_hat of the last admitted chunk (rank 0)        */
} sdv2_cache_state;

typedef struct sdv2_handle sdv2_handle;

/* Execution options (NULL = the defaults in brackets).  None changes the numerics:
 * every GEMM configuration the tuner may pick reduces each output element over K in
 * the same order (no split-K), so results are bit-identical across tunings.
 *   tune_gemms   [1] time every candidate tile configuration of each projection GEMM
 *                    shape at create (CUDA-graph replay on the real buffers) and keep
 *                    the fastest; 0 = the tile-balance model's pick, no timing.
 *   pdl          [1] programmatic dependent launch between the call's kernels.
 *   graphs       [1] replay the per-call device work from CUDA graphs.
 *   l2_persist   [1] mark the tick packet (fp32 residual stream x, embeddings) as
 *                    persisting in L2 (stream access-policy window; sets the process's
 *                    persisting-L2 limit) so the residual epilogues and norms re-read it
 *                    from L2 instead of HBM (+0.5-0.8 % fps measured at 1.3B 480p). */
typedef struct {
  int32_t tune_gemms;
  int32_t pdl;
  int32_t graphs;
  int32_t l2_persist;
  /* gemm_table   [NULL] gemm_table_len records of 8 int32 (M, N, K, epi, MC, BN, SK, XE),
   *                    e.g. from sdv2_gemm_configs of an earlier handle: these shapes take
   *                    the given configuration and are not timed (a record that is not one
   *                    of the shape's candidates is ignored).  Makes the tile choice
   *                    independent of the timing environment (profilers, clock state);
   *                    the bits never depend on it (see above). */
  const int32_t* gemm_table;
  int32_t gemm_table_len;
} sdv2_exec_options;

/* The projection-GEMM configurations the handle uses (tuned, or from gemm_table): up to
 * cap records of 8 int32 (M, N, K, epi, MC, BN, SK, XE) into out; *count = records
 * available (may exceed cap).  SDV2_E_INVALID on NULL arguments. */
sdv2_status sdv2_gemm_configs(const sdv2_handle* h, int32_t* out, int32_t cap, int32_t* count);

/* Bytes of device workspace a handle needs (0 on invalid descriptors). */
size_t sdv2_workspace_bytes(const sdv2_model_desc* md, const sdv2_geometry* g,
                            const sdv2_pipeline_desc* pp, sdv2_precision prec);

/* Validate, carve the workspace, pack this rank's weights (fp32 -> bf16 K-major for
 * SDV2_BF16), build TMA descriptors.  `stream` is a cudaStream_t (NULL = legacy);
 * `opts` may be NULL (defaults).  Errors: SDV2_E_SHAPE / SDV2_E_UNSUPPORTED for shapes,
 * SDV2_E_INVALID for a bad pipeline descriptor or (steps - 1) * world + 1 > 128 (the
 * chunk-record ring), SDV2_E_WORKSPACE, SDV2_E_CUDA (text in sdv2_last_error; the handle
 * is then returned in *out so the caller can read the text and destroy it). */
sdv2_status sdv2_create(const sdv2_model_desc* md, const sdv2_geometry* g,
                        const sdv2_pipeline_desc* pp, sdv2_precision prec,
                        const sdv2_weights* w, void* workspace, size_t workspace_bytes,
                        int device, void* stream, const sdv2_exec_options* opts, sdv2_handle** out);

/* Start new streams: zero KV lanes, metadata and controller states; embed the prompts
 * (host [streams][text_len][text_dim] fp32, one per stream) and compute every local
 * block's cross K/V. */
sdv2_status sdv2_reset_stream(sdv2_handle* h, const sdv2_stream_desc* sd, const float* prompt_host);

/* Switch prompt: takes effect from the next chunk admitted (the next
 * call); in-flight entries keep the prompt they were admitted with.  Two prompt versions
 * are resident, so a switch must come at least (steps - 1) * world calls after the
 * previous one (the oldest chunk admitted under the version being overwritten has then
 * left the pipeline); an earlier switch returns SDV2_E_STATE and changes nothing.
 * SDV2_E_INVALID for a zero-norm prompt mean or a stream index out of range.
 * prompt_host: host [text_len, text_dim] fp32 for stream `stream`. */
sdv2_status sdv2_set_prompt(sdv2_handle* h, int32_t stream, const float* prompt_host);

/* Chunk embedding h_t of the sink refresh ("given a new chunk embedding h_t").
 * The default reading (Q8) is the mean-pooled prompt embedding, set by reset_stream /
 * set_prompt.  The visual reading (N4): before each call the caller passes stream b's
 * embedding of the chunk it is about to admit (e.g. sdv2_chunk_embedding of the latent);
 * every rank must receive the same values (the control plane is replicated).  Any
 * dimension >= 1; the sinks compare against embeddings of the same dimension.
 * SDV2_E_INVALID: zero norm, bad stream. */
sdv2_status sdv2_set_chunk_embedding(sdv2_handle* h, int32_t stream, const double* emb, int32_t dim);
/* Host helper: out[c] = mean over T' x h x w of channel c of a host chunk [C, T', h, w]
 * fp32, accumulated in fp64 in index order (the visual chunk embedding of N4). */
sdv2_status sdv2_chunk_embedding(const float* chunk_host, int32_t C, int32_t T, int32_t H, int32_t W, double* out);

/* One stage-tick.  Rank 0: chunk_latent [streams][C, T', h, w] fp32 (host or device
 * pointer): chunk X = call index of every stream is admitted.  Last rank: if this call
 * emits clean chunks, their x0 are written to out_latent (host or device,
 * [streams][C, T', h, w] fp32) and *out_chunk_index = their chunk index, else
 * *out_chunk_index = -1 (known without a device sync: the schedule is deterministic).
 * Other ranks pass NULL. */
sdv2_status sdv2_denoise_chunk(sdv2_handle* h, const float* chunk_latent, float* out_latent,
                               int64_t* out_chunk_index);

sdv2_status sdv2_stage_io_buffers(sdv2_handle* h, int32_t parity, sdv2_stage_io* io);
sdv2_status sdv2_get_tick_info(const sdv2_handle* h, sdv2_tick_info* info);
sdv2_status sdv2_destroy(sdv2_handle* h);
const char* sdv2_status_string(sdv2_status s);
const char* sdv2_last_error(const sdv2_handle* h);

/* ---- test-only introspection (not on the timed path) ---- */
/* Metadata of (local block, lane e = j * streams + b); also copies stream b's controller
 * state (s, d_hat). */
sdv2_status sdv2_get_cache_state(sdv2_handle* h, int32_t local_block, int32_t lane, sdv2_cache_state* out);
/* If per_block_out != NULL (device, [local_blocks, n*L, dim] fp32) every following
 * call copies the residual stream x after each local block into it. */
sdv2_status sdv2_set_block_tap(sdv2_handle* h, float* per_block_out);
/* Device pointer + element count of the K (which=0) or V (which=1) storage of
 * (local block, lane): [m+W slots][L tokens][dim], element type = precision. */
sdv2_status sdv2_kv_lane(sdv2_handle* h, int32_t local_block, int32_t lane, int32_t which,
                         void** ptr, size_t* elems);

/* Test hook: synchronise the stream after every launch and log the call site on stderr
 * (graphs are bypassed while on) — names a kernel that does not complete. */
sdv2_status sdv2_debug_sync(sdv2_handle* h, int32_t enable);
/* CUDA-graph replay of the per-call device work (default on; keyed by the number of
 * active entries and the call parity; not used while profiling or tapping). */
sdv2_status sdv2_set_graphs(sdv2_handle* h, int32_t enable);
/* Mean device time per call of each resident block's span (class 4) since profiling was
 * enabled; out[i] = resident block resident_begin + i (0 if it did not run).  count >=
 * resident blocks.  Feeds the online block scheduler (sdv2_rebalance). */
sdv2_status sdv2_profile_block_ms(sdv2_handle* h, double* out, int32_t count);
/* Change the active block range inside the resident range (between calls; synchronises
 * the stream and drops the captured call graphs).  The caller must first copy into this
 * handle the KV lanes of every block that becomes active here, from its previous owner
 * (the control-plane metadata is replicated on every rank, so only K / V move). */
sdv2_status sdv2_set_block_range(sdv2_handle* h, int32_t block_begin, int32_t block_end);
/* K (which = 0) or V (1) lane storage of resident global block `block`: one contiguous
 * device range [streams * steps lanes][m + W slots][L][dim] of the precision's element
 * type (the unit an online re-partition moves between ranks). */
sdv2_status sdv2_block_kv(sdv2_handle* h, int32_t block, int32_t which, void** ptr, size_t* bytes);
/* Enable (1, resets the accumulators) or disable (0) per-class event timing. */
sdv2_status sdv2_profile_enable(sdv2_handle* h, int32_t enable);
/* Synchronises the stream and returns the accumulated per-class times. */
sdv2_status sdv2_profile_read(sdv2_handle* h, sdv2_profile* out);

/* Kernel-level test hook: one tensor-core GEMM C = A W^T + b on device pointers
 * (A [M,K] bf16, W [N,K] bf16, bias [N] fp32), epilogue epi = 0 store bf16 to out
 * [M,N], 1 GELU-tanh store bf16, 2 out (fp32 [M,N]) += (mod[gate_row] + e0[r/L][gate_row]) *
 * (AW^T + b), 3 out += AW^T + b.  Enqueued on `stream`. */
sdv2_status sdv2_debug_gemm(const void* A, const void* W, const float* bias, void* out, int32_t M, int32_t N,
                            int32_t K, int32_t epi, const float* mod, const float* e0, int32_t gate_row, int32_t L,
                            void* stream);

/* Kernel-level test hooks: the configurations the create-time GEMM tuner chooses from
 * for shape (M, N, K, epi) as (cluster size MC, tile width BN, stream-K SK, early residual
 * fetch XE) quadruples, and one GEMM launched with an explicit configuration. */
sdv2_status sdv2_debug_gemm_candidates(int32_t M, int32_t N, int32_t K, int32_t epi, int32_t* cfg4,
                                       int32_t max_cfgs, int32_t* count);
sdv2_status sdv2_debug_gemm_cfg(const void* A, const void* W, const float* bias, void* out, int32_t M, int32_t N,
                                int32_t K, int32_t epi, const float* mod, const float* e0, int32_t gate_row,
                                int32_t L, const int32_t* cfg4, void* stream);

/* Kernel-level test hook: tensor-core attention softmax(q K^T / sqrt(hd)) V for one
 * query block q [Lq, H*hd] over keys K/V [Lk, H*hd] (bf16, device) -> o [Lq, H*hd]
 * bf16.  `scratch` is >= 1 KB of device memory; enqueued on `stream`. */
sdv2_status sdv2_debug_attention(const void* q, const void* K, const void* V, void* o, int32_t Lq, int32_t Lk,
                                 int32_t H, int32_t hd, void* scratch, void* stream);

/* ---- host control plane (no GPU needed; also exported by libsdv2_ctl.so) ---- */
/* Exact min-max contiguous partition of per-block costs over K stages, with extra
 * cost on the first / last stage (P:231–233 DiT block scheduler).  Ties: earlier
 * stages take as many blocks as the optimum allows.  bounds_out has K+1 entries. */
sdv2_status sdv2_partition(const double* block_costs, int32_t num_blocks, int32_t stages,
                           double extra_first, double extra_last, int32_t* bounds_out,
                           double* max_stage_out);

/* Online DiT-block scheduler: ema[b] <- alpha * measured[b] +
 * (1 - alpha) * ema[b] (ema[b] == 0: first sample), then the exact min-max partition of
 * the smoothed times with the first / last stage extras; the new bounds (K+1 entries) are
 * adopted (changed = 1) only if they lower the predicted max stage time by more than
 * (hysteresis + 1e-9) x the current partition's, else new_bounds = cur_bounds.  Never increases the
 * predicted max stage time.  pred_cur / pred_new may be NULL. */
sdv2_status sdv2_rebalance(const double* measured_block_ms, int32_t num_blocks, int32_t stages,
                           double extra_first, double extra_last, double alpha, double hysteresis,
                           double* ema, const int32_t* cur_bounds, int32_t* new_bounds, int32_t* changed,
                           double* pred_cur, double* pred_new);

/* ---- Stream-VAE stand-in ("processes short video chunks
 * (e.g., 4 frames) and caches intermediate features within each 3D convolution") ----
 * Wan2.1-VAE-shaped causal 3D-conv encoder / decoder: 4 video frames [3][4][H][W] <-> one
 * latent frame [latent_channels][1][H/8][W/8] (fp32, host or device pointers), every 3x3x3
 * conv causal in time with a two-frame feature cache carried across chunks (so a streamed
 * run equals the full-sequence causal VAE).  Layer list in DESIGN.md / oracle/vae.py.
 * Weights: fp32, in layer order: conv (w [co][3][3][3][ci], b [co]); residual block (n1 [c],
 * c1.w, c1.b, n2 [c], c2.w, c2.b); norm (g [c]) — synthgen.vae_tensor_specs order.
 * The workspace is caller-owned (sdv2_vae_workspace_bytes), zeroed and carved at create. */
typedef struct {
  int32_t video_h, video_w;      /* multiples of 8 */
  int32_t dims[3];               /* stage channels (96, 192, 384); each <= 384 */
  int32_t latent_channels;       /* 16; <= 384 */
  float eps;                     /* RMS epsilon */
} sdv2_vae_desc;
typedef struct sdv2_vae sdv2_vae;
size_t sdv2_vae_workspace_bytes(const sdv2_vae_desc* d);
sdv2_status sdv2_vae_create(const sdv2_vae_desc* d, const sdv2_weights* w, void* workspace, size_t workspace_bytes,
                            int device, void* stream, sdv2_vae** out);
/* New video stream: zero every convolution's feature cache. */
sdv2_status sdv2_vae_reset(sdv2_vae* v);
sdv2_status sdv2_vae_encode_chunk(sdv2_vae* v, const float* video, float* latent);
sdv2_status sdv2_vae_decode_chunk(sdv2_vae* v, const float* latent, float* video);
int64_t sdv2_vae_launches(const sdv2_vae* v);
const char* sdv2_vae_last_error(const sdv2_vae* v);
sdv2_status sdv2_vae_destroy(sdv2_vae* v);

/* ---- SLO-aware batching scheduler (host only) ----
 * A latency point is one MEASURED call latency L(T', B): chunk_frames = T' latent frames
 * per chunk, streams = B streams batched per call (sdv2_geometry.streams).  Every stream
 * emits one clean chunk per call in steady state, so its output rate is
 * px_per_latent * T' / L frames/s (px_per_latent = 4: Wan VAE temporal factor, Q23). */
typedef struct {
  int32_t chunk_frames;
  int32_t streams;
  double latency_s;
} sdv2_latency_point;

typedef struct {
  double target_fps;            /* f_SLO per stream, output frames/s                    */
  double frame_deadline_s;      /* per-frame deadline; chunk deadline = it x px T'       */
  int32_t px_per_latent;        /* output frames per latent frame (4)                    */
} sdv2_slo;

typedef struct {
  int32_t chunk_frames;
  int32_t streams;
  double latency_s;
  double fps;                   /* aggregate px B T' / L                                 */
  int32_t feasible;             /* 0: no point meets the SLO (reported, never relaxed)   */
} sdv2_batch_decision;

/* Exhaustive search of the table: the (T', B) with B <= b_max and B T' <= buffered_frames
 * ("B.T must not exceed the number of frames already collected") that keeps every
 * stream at >= target_fps and within the chunk deadline, maximising aggregate fps; ties:
 * smaller B, then smaller T'.  None feasible: B = 1 at the lowest latency, feasible = 0.
 * SDV2_E_INVALID: empty table, buffered_frames < min T' (not enough input), bad args. */
sdv2_status sdv2_slo_select(const sdv2_latency_point* table, int32_t n, const sdv2_slo* slo,
                            int32_t buffered_frames, int32_t b_max, sdv2_batch_decision* out);

/* Online adaptation ("continuously adapts B to the observed end-to-end latency"):
 * AIMD on the caller-owned state; a violation halves streams (floor 1, infeasible = 1 if
 * it was already 1), `streak` compliant calls add one (cap b_max). */
typedef struct {
  int32_t streams, chunk_frames, b_max, streak;
  int32_t ok_run, infeasible;
} sdv2_aimd_state;
sdv2_status sdv2_slo_adapt(sdv2_aimd_state* st, double observed_latency_s, const sdv2_slo* slo);

/* P:178-180 memory-bound latency model L = a + b (B T') fitted to the table (least squares). */
sdv2_status sdv2_slo_fit(const sdv2_latency_point* table, int32_t n, double* a, double* b);

#ifdef __cplusplus
}
#endif
#endif /* SDV2_H */
