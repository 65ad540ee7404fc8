// Host control plane (see ctl.h).  Integer / fp64 only.
#include "ctl.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

namespace sdv2 {

void Control::reset(const CtlParams& p) {
  p_ = p;
  r_ = 0;
  calls_ = 0;
  st_.assign(p.B, StreamState{});
  for (auto& S : st_) {
    S.sink_emb.assign(p.m, {});
    S.recs.assign(kRecRing, ChunkRecord{});
  }
  lanes_.assign(size_t(p.n) * p.B, LaneMeta{});
  for (auto& L : lanes_) {
    for (int s = 0; s < kMaxSlots; ++s) L.tag[s] = -1;
    std::memset(L.pos, 0, sizeof(L.pos));
  }
}

void Control::set_prompt_mean(int b, const std::vector<double>& h, int32_t pver) {
  st_[b].h = h;
  st_[b].pver = pver;
}

static double cosine(const std::vector<double>& a, const std::vector<double>& b) {
  double ab = 0, aa = 0, bb = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    ab += a[i] * b[i];
    aa += a[i] * a[i];
    bb += b[i] * b[i];
  }
  return ab / (std::sqrt(aa) * std::sqrt(bb));
}

// Chunk admission of stream b; r / rebase are the call's (every
// stream admits chunk X = call, so the RoPE reset count is common):
//   positions p_f = X T' + f - r T_reset
//   X < m: sink slot X (anchor X T' + f), s_X <- h_X
//   X >= m: refresh every sink with cos(h_X, s_i) < tau (ties keep), ring slot (X-m) mod W
ChunkRecord Control::admit(int b, int64_t X, int32_t r, bool rebase) {
  StreamState& S = st_[b];
  ChunkRecord rec;
  rec.X = X;
  rec.rebase = rebase;
  rec.r = r;
  for (int f = 0; f < p_.T; ++f) rec.pos[f] = int32_t(X * p_.T + f - int64_t(r) * p_.T_reset);
  rec.pver = S.pver;
  if (X < p_.m) {
    rec.sink_fill = int32_t(X);
    S.sink_emb[X] = S.h;
  } else {
    for (int i = 0; i < p_.m; ++i) {
      if (cosine(S.h, S.sink_emb[i]) < p_.tau) {
        rec.refresh_mask |= (1u << i);
        S.sink_emb[i] = S.h;
      }
    }
    rec.ring_slot = int32_t((X - p_.m) % p_.W);
  }
  return rec;
}

// Per-lane application (O3): 1. re-base ring slots, 2. write / refresh, then attend.
void Control::apply(LaneMeta& L, const ChunkRecord& rec) {
  const int m = p_.m, T = p_.T;
  if (rec.rebase) {
    for (int s = m; s < m + p_.W; ++s)
      if (L.tag[s] >= 0)
        for (int f = 0; f < T; ++f) L.pos[s][f] -= p_.T_reset;
  }
  if (rec.sink_fill >= 0) {
    L.tag[rec.sink_fill] = rec.X;
    for (int f = 0; f < T; ++f) L.pos[rec.sink_fill][f] = rec.pos[f];
  } else {
    for (int i = 0; i < m; ++i)
      if (rec.refresh_mask & (1u << i)) {
        L.tag[i] = rec.X;
        for (int f = 0; f < T; ++f) L.pos[i][f] = i * T + f;
      }
    const int s = m + rec.ring_slot;
    if (L.tag[s] >= 0) ++L.evictions;
    L.tag[s] = rec.X;
    for (int f = 0; f < T; ++f) L.pos[s][f] = rec.pos[f];
  }
  int nv = 0;
  while (nv < m + p_.W && L.tag[nv] >= 0) ++nv;
  L.nvalid = nv;
  L.last_X = rec.X;
  L.r = rec.r;
}

// Call c on this rank (reading R2): micro-batch mu = c holds entries (c - jK, j) for
// j = 0..n-1 with c - jK >= 0, for each of the B streams (entry e = j B + b); the active
// entries are always the prefix e < B n_active_steps.
void Control::plan_call(TickDesc* td) {
  const int64_t c = calls_;
  // reset: while X T' - r T_reset > T_reset: r += 1 (repeated wrap of P:191), X = c
  bool rebase = false;
  while (c * p_.T - int64_t(r_) * p_.T_reset > p_.T_reset) {
    ++r_;
    rebase = true;
  }
  for (int b = 0; b < p_.B; ++b) st_[b].recs[c % kRecRing] = admit(b, c, r_, rebase);
  std::memset(td, 0, sizeof(*td));
  td->call_lo = int32_t(c);
  td->out_entry = -1;
  int na = 0;
  for (int j = 0; j < p_.n; ++j) {
    const int64_t X = entry_chunk(c, j);
    for (int b = 0; b < p_.B; ++b) {
      const int ei = j * p_.B + b;
      EntryDesc& e = td->e[ei];
      e.j = j;
      e.stream = b;
      if (X < 0) {
        e.active = 0;
        e.X = -1;
        continue;
      }
      const ChunkRecord& rec = st_[b].recs[X % kRecRing];
      LaneMeta& L = lanes_[ei];
      apply(L, rec);
      e.X = int32_t(X);
      e.active = 1;
      e.write_slot = rec.sink_fill >= 0 ? rec.sink_fill : p_.m + rec.ring_slot;
      e.nvalid = L.nvalid;
      e.refresh_mask = int32_t(rec.refresh_mask);
      e.rebase = rec.rebase ? 1 : 0;
      e.pver = rec.pver;
      e.xslot = 2 * b + (rec.pver & 1);
      for (int f = 0; f < p_.T; ++f) e.pos[f] = rec.pos[f];
      ++na;
    }
    if (X >= 0 && j == p_.n - 1) td->out_entry = j * p_.B;
  }
  td->n_active = na;
  ++calls_;
}

// Exact min-max contiguous partition: DP over (stage, prefix) for the optimum value,
// then a front-greedy reconstruction (each stage takes as many blocks as the optimum
// allows, leaving at least one block per remaining stage).
bool partition(const double* c, int B, int K, double e_first, double e_last, int32_t* bounds,
               double* best) {
  if (K < 1 || B < K) return false;
  std::vector<double> pre(B + 1, 0.0);
  for (int i = 0; i < B; ++i) pre[i + 1] = pre[i] + c[i];
  auto cost = [&](int s, int a, int b) {
    double t = pre[b] - pre[a];
    if (s == 0) t += e_first;
    if (s == K - 1) t += e_last;
    return t;
  };
  const double INF = std::numeric_limits<double>::infinity();
  // f[s][b] = best max over the first s+1 stages covering blocks [0, b)
  std::vector<std::vector<double>> f(K, std::vector<double>(B + 1, INF));
  for (int b = 1; b <= B; ++b) f[0][b] = cost(0, 0, b);
  for (int s = 1; s < K; ++s)
    for (int b = s + 1; b <= B; ++b)
      for (int a = s; a < b; ++a) f[s][b] = std::min(f[s][b], std::max(f[s - 1][a], cost(s, a, b)));
  const double opt = f[K - 1][B];
  // Tie-break among optimal partitions: the most even one (minimum sum of squared stage
  // times, every stage <= opt), then earlier stages heavier.  g[s][a] = min sum of
  // squares of stages s..K-1 covering [a, B) with each stage <= opt.
  const double tol = 1e-12 * std::max(1.0, std::fabs(opt));
  std::vector<std::vector<double>> g(K + 1, std::vector<double>(B + 1, INF));
  g[K][B] = 0.0;
  for (int s = K - 1; s >= 0; --s)
    for (int a = s; a <= B; ++a)
      for (int b = a + 1; b <= B; ++b) {
        const double cs = cost(s, a, b);
        if (cs <= opt + tol && g[s + 1][b] < INF) g[s][a] = std::min(g[s][a], cs * cs + g[s + 1][b]);
      }
  bounds[0] = 0;
  int a = 0;
  for (int s = 0; s < K; ++s) {
    int pick = -1;
    const double target = g[s][a];
    const double stol = 1e-9 * std::max(1.0, std::fabs(target));
    for (int b = B; b > a; --b) {
      const double cs = cost(s, a, b);
      if (cs <= opt + tol && g[s + 1][b] < INF && std::fabs(cs * cs + g[s + 1][b] - target) <= stol) {
        pick = b;
        break;
      }
    }
    if (pick < 0) return false;
    bounds[s + 1] = pick;
    a = pick;
  }
  if (best) *best = opt;
  return true;
}

}  // namespace sdv2
