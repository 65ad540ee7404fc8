// C entry points of the host control plane.  sdv2_partition is part of the public
// ABI (sdv2.h); the sdv2ctl_* functions drive the control plane without a GPU and
// exist for the CPU tests (they are exported by both libsdv2.so and libsdv2_ctl.so).
#include <cstring>
#include <vector>

#include "../../include/sdv2.h"
#include "ctl.h"

using namespace sdv2;

extern "C" {

sdv2_status sdv2_partition(const double* block_costs, int32_t num_blocks, int32_t stages,
                           double extra_first, double extra_last, int32_t* bounds_out,
                           double* max_stage_out) {
  if (!block_costs || !bounds_out || stages < 1) return SDV2_E_INVALID;
  if (stages > num_blocks) return SDV2_E_INVALID;  // K > blocks is infeasible
  return partition(block_costs, num_blocks, stages, extra_first, extra_last, bounds_out, max_stage_out)
             ? SDV2_OK
             : SDV2_E_INVALID;
}

void* sdv2ctl_new(int32_t T, int32_t m, int32_t W, int32_t n, int32_t K, int32_t rank,
                  int32_t T_reset, double tau, int32_t B) {
  if (T < 1 || T > kMaxFrames || m < 0 || W < 1 || m + W > kMaxSlots || n < 1 || n > kMaxSteps ||
      K < 1 || T_reset < 1 || B < 1 || B * n > kMaxEntries || int64_t(n - 1) * K + 1 > kRecRing)
    return nullptr;
  auto* c = new Control();
  CtlParams p;
  p.T = T; p.m = m; p.W = W; p.n = n; p.K = K; p.rank = rank; p.T_reset = T_reset; p.tau = tau; p.B = B;
  c->reset(p);
  return c;
}

void sdv2ctl_free(void* c) { delete static_cast<Control*>(c); }

int32_t sdv2ctl_set_prompt_mean(void* c, int32_t stream, const double* h, int32_t dim, int32_t pver) {
  auto* ctl = static_cast<Control*>(c);
  if (stream < 0 || stream >= ctl->params().B) return -1;
  ctl->set_prompt_mean(stream, std::vector<double>(h, h + dim), pver);
  return 0;
}

// One call; writes the device descriptor fields of every entry e = j B + b into
// out[B n][10 + kMaxFrames]: X, j, active, write_slot, nvalid, refresh_mask, rebase, pver,
// stream, xslot, pos[0..kMaxFrames).
int32_t sdv2ctl_call(void* c, int32_t* out, int64_t* out_chunk) {
  auto* ctl = static_cast<Control*>(c);
  TickDesc td;
  const int64_t call = ctl->calls();
  ctl->plan_call(&td);
  const int ne = ctl->params().n * ctl->params().B;
  for (int i = 0; i < ne; ++i) {
    const EntryDesc& e = td.e[i];
    int32_t* o = out + i * (10 + kMaxFrames);
    o[0] = e.X; o[1] = e.j; o[2] = e.active; o[3] = e.write_slot; o[4] = e.nvalid;
    o[5] = e.refresh_mask; o[6] = e.rebase; o[7] = e.pver; o[8] = e.stream; o[9] = e.xslot;
    for (int f = 0; f < kMaxFrames; ++f) o[10 + f] = e.pos[f];
  }
  if (out_chunk) *out_chunk = td.out_entry >= 0 ? ctl->out_chunk(call) : -1;
  return td.n_active;
}

int32_t sdv2ctl_lane_state(void* c, int32_t lane, sdv2_cache_state* st) {
  auto* ctl = static_cast<Control*>(c);
  const LaneMeta& L = ctl->lane(lane);
  std::memset(st, 0, sizeof(*st));
  st->num_slots = ctl->params().m + ctl->params().W;
  st->num_valid = L.nvalid;
  for (int s = 0; s < st->num_slots; ++s) {
    st->tag[s] = L.tag[s];
    st->pos[s] = L.pos[s][0];
  }
  st->resets = L.r;
  st->evictions = L.evictions;
  return 0;
}

int32_t sdv2ctl_max_frames(void) { return kMaxFrames; }

int32_t sdv2ctl_set_chunk_embedding(void* c, int32_t stream, const double* h, int32_t dim) {
  auto* ctl = static_cast<Control*>(c);
  if (stream < 0 || stream >= ctl->params().B || !h || dim < 1) return -1;
  ctl->set_chunk_embedding(stream, std::vector<double>(h, h + dim));
  return 0;
}

// Visual chunk embedding (N4, reading Q8-visual in DESIGN.md): h_c = mean over the chunk's
// T' frames and h x w pixels of latent channel c, accumulated in fp64 in index order.
sdv2_status sdv2_chunk_embedding(const float* chunk_host, int32_t C, int32_t T, int32_t H, int32_t W, double* out) {
  if (!chunk_host || !out || C < 1 || T < 1 || H < 1 || W < 1) return SDV2_E_INVALID;
  const size_t per = size_t(T) * H * W;
  for (int c = 0; c < C; ++c) {
    double acc = 0.0;
    const float* p = chunk_host + size_t(c) * per;
    for (size_t i = 0; i < per; ++i) acc += double(p[i]);
    out[c] = acc / double(per);
  }
  return SDV2_OK;
}

}  // extern "C"
