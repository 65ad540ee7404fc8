// Online DiT-block scheduler ("a lightweight
// inference-time DiT block scheduler that dynamically reallocates blocks between devices
// based on measured execution time"; SPEC S:201-209 rebalance_online): EMA-smoothed
// measured block times, the exact min-max partition (ctl.cpp), adopted only when the
// predicted max-stage improvement exceeds a hysteresis fraction.  Host-only, fp64.
#include "../../include/sdv2.h"
#include "ctl.h"

#include <vector>

namespace {
double max_stage(const double* t, int nb, int K, const int32_t* bounds, double ef, double el) {
  double mx = 0.0;
  for (int s = 0; s < K; ++s) {
    double v = 0.0;
    for (int b = bounds[s]; b < bounds[s + 1]; ++b) v += t[b];
    if (s == 0) v += ef;
    if (s == K - 1) v += el;
    if (v > mx) mx = v;
  }
  (void)nb;
  return mx;
}
}  // namespace

extern "C" sdv2_status sdv2_rebalance(const double* measured_block_ms, int32_t num_blocks, int32_t stages,
                                      double extra_first, double extra_last, double alpha, double hysteresis,
                                      double* ema, const int32_t* cur_bounds, int32_t* new_bounds,
                                      int32_t* changed, double* pred_cur, double* pred_new) {
  if (!measured_block_ms || !ema || !cur_bounds || !new_bounds || !changed || num_blocks < 1 || stages < 1 ||
      stages > num_blocks || !(alpha > 0.0 && alpha <= 1.0) || hysteresis < 0.0)
    return SDV2_E_INVALID;
  if (cur_bounds[0] != 0 || cur_bounds[stages] != num_blocks) return SDV2_E_INVALID;
  for (int s = 0; s < stages; ++s)
    if (cur_bounds[s] >= cur_bounds[s + 1]) return SDV2_E_INVALID;
  // EMA of the measured block times (an element never measured before takes the sample)
  for (int b = 0; b < num_blocks; ++b) {
    if (measured_block_ms[b] < 0.0) return SDV2_E_INVALID;
    ema[b] = ema[b] > 0.0 ? alpha * measured_block_ms[b] + (1.0 - alpha) * ema[b] : measured_block_ms[b];
  }
  const double cur = max_stage(ema, num_blocks, stages, cur_bounds, extra_first, extra_last);
  std::vector<int32_t> best(stages + 1);
  double opt = 0.0;
  if (!sdv2::partition(ema, num_blocks, stages, extra_first, extra_last, best.data(), &opt)) return SDV2_E_INVALID;
  opt = max_stage(ema, num_blocks, stages, best.data(), extra_first, extra_last);   // same summation as cur
  // a relative 1e-9 margin keeps rounding-level "improvements" from moving blocks
  const bool adopt = cur - opt > (hysteresis + 1e-9) * cur;
  for (int s = 0; s <= stages; ++s) new_bounds[s] = adopt ? best[s] : cur_bounds[s];
  *changed = adopt ? 1 : 0;
  if (pred_cur) *pred_cur = cur;
  if (pred_new) *pred_new = adopt ? opt : cur;
  return SDV2_OK;
}
