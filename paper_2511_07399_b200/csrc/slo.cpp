// SLO-aware batching scheduler: pick the
// number of streams B batched per call and the chunk length T' from a MEASURED latency
// table L(T', B) so that every stream keeps f_SLO, maximising aggregate throughput, and
// adapt B online to the observed latency (AIMD).  Host-only, fp64.
#include <cmath>
#include <vector>

#include "../../include/sdv2.h"

extern "C" {

// Exhaustive search (the table is small: a handful of T' x B points).
//   feasible: B <= b_max, B T' <= buffered_frames, per-stream rate px T' / L >=
//   target_fps, chunk latency L <= frame_deadline_s * px T'
//   objective: throughput px B T' / L; ties -> smaller B, then smaller T'.
//   none feasible: B = 1 (else the smallest B) at the lowest latency that fits the
//   buffer, flagged infeasible.
sdv2_status sdv2_slo_select(const sdv2_latency_point* table, int32_t n, const sdv2_slo* slo,
                            int32_t buffered_frames, int32_t b_max, sdv2_batch_decision* out) {
  if (!table || n < 1 || !slo || !out || b_max < 1 || slo->px_per_latent < 1) return SDV2_E_INVALID;
  int32_t min_t = table[0].chunk_frames;
  for (int i = 0; i < n; ++i) {
    if (table[i].chunk_frames < 1 || table[i].streams < 1) return SDV2_E_INVALID;
    if (table[i].chunk_frames < min_t) min_t = table[i].chunk_frames;
  }
  if (buffered_frames < min_t) return SDV2_E_INVALID;   // not enough input
  const double px = slo->px_per_latent;
  int best = -1;
  double best_thr = 0.0;
  for (int i = 0; i < n; ++i) {
    const sdv2_latency_point& p = table[i];
    if (p.streams > b_max || int64_t(p.streams) * p.chunk_frames > buffered_frames || !(p.latency_s > 0.0)) continue;
    const double rate = px * p.chunk_frames / p.latency_s;
    if (rate < slo->target_fps || p.latency_s > slo->frame_deadline_s * px * p.chunk_frames) continue;
    const double thr = p.streams * rate;
    bool take = best < 0 || thr > best_thr;
    if (!take && thr == best_thr) {
      const sdv2_latency_point& q = table[best];
      take = p.streams < q.streams || (p.streams == q.streams && p.chunk_frames < q.chunk_frames);
    }
    if (take) {
      best = i;
      best_thr = thr;
    }
  }
  int feasible = best >= 0;
  if (!feasible) {
    // fallback: prefer B = 1, then the lowest latency (ties: smaller T', then B)
    for (int pass = 0; pass < 2 && best < 0; ++pass) {
      for (int i = 0; i < n; ++i) {
        const sdv2_latency_point& p = table[i];
        if (p.streams > b_max || int64_t(p.streams) * p.chunk_frames > buffered_frames) continue;
        if (pass == 0 && p.streams != 1) continue;
        if (best < 0) {
          best = i;
          continue;
        }
        const sdv2_latency_point& q = table[best];
        if (p.latency_s < q.latency_s ||
            (p.latency_s == q.latency_s &&
             (p.chunk_frames < q.chunk_frames || (p.chunk_frames == q.chunk_frames && p.streams < q.streams))))
          best = i;
      }
    }
    if (best < 0) return SDV2_E_INVALID;
  }
  const sdv2_latency_point& p = table[best];
  out->chunk_frames = p.chunk_frames;
  out->streams = p.streams;
  out->latency_s = p.latency_s;
  out->fps = px * p.streams * p.chunk_frames / p.latency_s;
  out->feasible = feasible;
  return SDV2_OK;
}

// AIMD: an SLO violation (per-stream rate < target or chunk latency > deadline) halves B
// (floor 1; B = 1 violating is flagged infeasible); `streak` compliant calls in a row
// add one stream (cap b_max).  Deterministic given the history.
sdv2_status sdv2_slo_adapt(sdv2_aimd_state* st, double observed_latency_s, const sdv2_slo* slo) {
  if (!st || !slo || !(observed_latency_s > 0.0) || st->streams < 1 || st->b_max < 1 || st->streak < 1 ||
      st->chunk_frames < 1)
    return SDV2_E_INVALID;
  const double px = slo->px_per_latent;
  const double rate = px * st->chunk_frames / observed_latency_s;
  const bool violated = rate < slo->target_fps || observed_latency_s > slo->frame_deadline_s * px * st->chunk_frames;
  if (violated) {
    st->infeasible = st->streams == 1;
    st->streams = st->streams / 2 > 1 ? st->streams / 2 : 1;
    st->ok_run = 0;
  } else {
    st->infeasible = 0;
    if (++st->ok_run >= st->streak) {
      st->streams = st->streams + 1 < st->b_max ? st->streams + 1 : st->b_max;
      st->ok_run = 0;
    }
  }
  return SDV2_OK;
}

// P:178-180 memory-bound latency model L(T', B) = a + b (B T'), least squares.
sdv2_status sdv2_slo_fit(const sdv2_latency_point* table, int32_t n, double* a, double* b) {
  if (!table || n < 2 || !a || !b) return SDV2_E_INVALID;
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (int i = 0; i < n; ++i) {
    const double x = double(table[i].streams) * table[i].chunk_frames, y = table[i].latency_s;
    sx += x; sy += y; sxx += x * x; sxy += x * y;
  }
  const double den = n * sxx - sx * sx;
  if (den == 0.0) return SDV2_E_INVALID;
  *b = (n * sxy - sx * sy) / den;
  *a = (sy - *b * sx) / n;
  return SDV2_OK;
}

}  // extern "C"
