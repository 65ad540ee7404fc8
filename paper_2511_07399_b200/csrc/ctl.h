// Host control plane of the stream: chunk admission (RoPE reset, sink fill /
// refresh, ring slot), per-lane KV metadata, the stream-batch / pipeline tick
// schedule and the DiT-block partition.  Plain C++17, no CUDA: it is compiled
// into libsdv2.so and, alone, into libsdv2_ctl.so for CPU tests.
//
// Paper passages (PAPER.md line numbers):
//   P:190  sink set S_t, alpha_i = cos(h_t, s_i), keep if alpha >= tau else s_i <- h_t
//   P:191  RoPE phase reset theta_t = theta_{t - T_reset} for t > T_reset
//   P:472  rolling KV cache with sink tokens (caption of Fig. kv_cache)
//   P:164, P:224–227  pipeline-parallel stream batch, ring of stages
//   P:231–233  DiT block scheduler (min-max partition of measured block times)
// Readings R1–R4 / Q5–Q11 / Q26 are listed in DESIGN.md.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace sdv2 {

constexpr int kMaxSteps = 8;      // n
constexpr int kMaxEntries = 16;   // entries per call = streams B x steps n (Stream Batch x SLO batch)
constexpr int kMaxFrames = 16;    // T'
constexpr int kMaxSlots = 64;     // m + W
constexpr int kRecRing = 128;     // chunk records kept (>= (n-1)K + 1)

// Per-entry device descriptor (uploaded every call; POD, identical on host/device).
// Entry e = j * B + b is step j of stream b (step-major, so the active entries of a
// call are always a prefix); its KV lane is e.
struct EntryDesc {
  int32_t X;            // chunk index (Philox counter word 0, s-table index)
  int32_t j;            // step
  int32_t stream;       // b: the latent stream (controller, prompt, noise key of its own)
  int32_t xslot;        // prompt K/V slot of the cross-attention: 2 b + (pver & 1)
  int32_t active;
  int32_t write_slot;   // physical slot the chunk's K/V go to (sink slot or m + ring slot)
  int32_t nvalid;       // valid slots of the lane after the write (a prefix)
  int32_t refresh_mask; // sink slots that get this chunk at their anchor positions
  int32_t rebase;       // rotate ring slots of the lane by R(-T_reset) before writing
  int32_t pver;         // prompt version (cross-attention K/V) in effect for chunk X
  int32_t pos[kMaxFrames];  // temporal RoPE position of each frame of the chunk
};

struct TickDesc {
  int32_t n_active;     // active entries (a prefix; a multiple of B)
  int32_t call_lo;
  int32_t out_entry;    // first of the B entries that emit a clean chunk this call (-1 none)
  int32_t pad;
  EntryDesc e[kMaxEntries];
};

struct ChunkRecord {
  int64_t X = -1;
  int32_t r = 0;
  bool rebase = false;
  int32_t sink_fill = -1;
  uint32_t refresh_mask = 0;
  int32_t ring_slot = -1;
  int32_t pver = 0;
  int32_t pos[kMaxFrames] = {};
};

struct LaneMeta {
  int64_t tag[kMaxSlots];
  int32_t pos[kMaxSlots][kMaxFrames];
  int32_t nvalid = 0;
  int64_t evictions = 0;
  int64_t last_X = -1;
  int32_t r = 0;
};

struct CtlParams {
  int T = 1, m = 1, W = 1, n = 1, K = 1, rank = 0, T_reset = 1;
  double tau = 0.95;
  int B = 1;            // streams batched per call (all admitted in lockstep: chunk X = call)
};

class Control {
 public:
  void reset(const CtlParams& p);
  // Prompt of stream b in effect from its next admitted chunk: h = mean-pooled prompt
  // (fp64, reading Q8).
  void set_prompt_mean(int b, const std::vector<double>& h, int32_t pver);
  // Visual reading of the chunk embedding h_t (N4): the embedding stream b's next
  // admitted chunk is compared against its sinks with (the prompt version is unchanged).
  void set_chunk_embedding(int b, const std::vector<double>& h) { st_[b].h = h; }
  // One call (stage-tick) on this rank: admits chunk X = call index of every stream (R2),
  // applies the chunk records of every active entry to its lane and fills the device
  // descriptor.
  void plan_call(TickDesc* td);
  int64_t calls() const { return calls_; }
  const LaneMeta& lane(int e) const { return lanes_[e]; }
  const ChunkRecord& record(int b, int64_t X) const { return st_[b].recs[X % kRecRing]; }
  int32_t resets() const { return r_; }
  const CtlParams& params() const { return p_; }
  // Entry chunk of step j at call c under R2: X = c - j K (valid if >= 0).
  int64_t entry_chunk(int64_t c, int j) const { return c - int64_t(j) * p_.K; }
  // Chunk whose clean latent the last stage emits at call c (-1 while filling).
  int64_t out_chunk(int64_t c) const { return c - int64_t(p_.n - 1) * p_.K; }

 private:
  ChunkRecord admit(int b, int64_t X, int32_t r, bool rebase);
  void apply(LaneMeta& L, const ChunkRecord& rec);

  // per-stream admission state
  struct StreamState {
    std::vector<std::vector<double>> sink_emb;
    std::vector<double> h;
    int32_t pver = 0;
    std::vector<ChunkRecord> recs;
  };
  CtlParams p_;
  int32_t r_ = 0;
  int64_t calls_ = 0;
  std::vector<StreamState> st_;
  std::vector<LaneMeta> lanes_;   // [n * B], lane e = j * B + b
};

// Exact min-max contiguous partition (DP over prefix sums), earliest-heavy tie-break.
bool partition(const double* costs, int B, int K, double e_first, double e_last,
               int32_t* bounds, double* best);

}  // namespace sdv2
