// Host placement planner of the FSSDP path, native C++.
//
// Decision-for-decision (and bit-for-bit in its float64 arithmetic) the reference
// moesim planner: placement.py, costmodel.py, dispatch.py, planner.py and the per-layer
// part of engine.py FssdpState.run_iteration.  Each function cites the reference
// lines it restates.  Placements are dense chunk-major masks mask[c*D + d].
//
// Float-order contract (SURVEY.md §8a "float-order hazards"): every float64 reduction
// below reproduces numpy's order for the corresponding reference expression —
// sequential for axis-0 reductions and Python loops, numpy's 8-lane pairwise
// summation (pairwise_sum, PW_BLOCKSIZE 128) for 1-D ndarray.sum().
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "fssdp.h"

namespace fssdp {
void set_error(const char* msg);
}

namespace {

using fssdp::set_error;

struct Err {
  int code;
  std::string msg;
};

struct Topo {
  int nodes, dpn;
  double intra, inter, alpha;
  int devices() const { return nodes * dpn; }
  int node_of(int d) const { return d / dpn; }
};

Topo to_topo(const fssdp_topology* t) {
  return Topo{t->nodes, t->devices_per_node, t->intra_bw, t->inter_bw, t->alpha};
}

int check_topo(const fssdp_topology* t) {
  // ClusterTopology.__post_init__ (topology.py:29-39) raises ConfigError; callers build
  // the topology in Python first, so here it is an internal invariant.
  if (!t || t->nodes <= 0 || t->devices_per_node <= 0 || !(t->intra_bw > 0) ||
      !(t->inter_bw > 0) || t->alpha < 0) {
    set_error("invalid topology");
    return FSSDP_ERR_INTERNAL;
  }
  return FSSDP_OK;
}

// ------------------------------------------------------------------ placement
struct Placement {
  int C, D;
  std::vector<uint8_t> m;  // [C*D]
  Placement(int c, int d) : C(c), D(d), m(static_cast<size_t>(c) * d, 0) {}
  Placement(int c, int d, const uint8_t* src) : C(c), D(d), m(src, src + static_cast<size_t>(c) * d) {
    for (auto& v : m) v = v ? 1 : 0;
  }
  bool has(int c, int d) const { return m[static_cast<size_t>(c) * D + d] != 0; }
  void set(int c, int d) { m[static_cast<size_t>(c) * D + d] = 1; }
  int holders_count(int c) const {
    int n = 0;
    for (int d = 0; d < D; ++d) n += has(c, d);
    return n;
  }
  std::vector<int> holders(int c) const {  // ascending
    std::vector<int> h;
    for (int d = 0; d < D; ++d)
      if (has(c, d)) h.push_back(d);
    return h;
  }
  int chunks_on(int d) const {
    int n = 0;
    for (int c = 0; c < C; ++c) n += has(c, d);
    return n;
  }
  bool is_partition() const {
    for (int c = 0; c < C; ++c)
      if (holders_count(c) != 1) return false;
    return true;
  }
  int owner(int c) const {
    for (int d = 0; d < D; ++d)
      if (has(c, d)) return d;
    return -1;
  }
  bool operator==(const Placement& o) const { return C == o.C && D == o.D && m == o.m; }
};

// Verdict (placement.py:31-48)
struct Verdict {
  int reason = FSSDP_VERDICT_OK;
  int chunk = -1, device = -1;
  bool ok() const { return reason == FSSDP_VERDICT_OK; }
  std::string describe() const {
    static const char* names[] = {"valid", "missing_chunk", "duplicate_owner", "dropped_entry"};
    if (ok()) return "valid";
    std::string s = names[reason];
    if (chunk >= 0) s += " chunk=" + std::to_string(chunk);
    if (device >= 0) s += " device=" + std::to_string(device);
    return s;
  }
};

// _check_partition (placement.py:181-190): first chunk with no holder, or the
// second-lowest holder of the first multiply-held chunk.
bool check_partition(const Placement& p, Verdict* v) {
  for (int c = 0; c < p.C; ++c) {
    std::vector<int> h = p.holders(c);
    if (h.empty()) {
      v->reason = FSSDP_VERDICT_MISSING_CHUNK;
      v->chunk = c;
      return false;
    }
    if (h.size() > 1) {
      v->reason = FSSDP_VERDICT_DUPLICATE_OWNER;
      v->chunk = c;
      v->device = h[1];
      return false;
    }
  }
  return true;
}

// _check_subset (placement.py:193-197): first entry of `small` (sorted order) missing in `big`.
bool check_subset(const Placement& small, const Placement& big, Verdict* v) {
  for (int c = 0; c < small.C; ++c)
    for (int d = 0; d < small.D; ++d)
      if (small.has(c, d) && !big.has(c, d)) {
        v->reason = FSSDP_VERDICT_DROPPED_ENTRY;
        v->chunk = c;
        v->device = d;
        return false;
      }
  return true;
}

Verdict validate_spag(const Placement& pre, const Placement& post) {  // placement.py:200-204
  Verdict v;
  if (check_partition(pre, &v)) check_subset(pre, post, &v);
  return v;
}

Verdict validate_sprs(const Placement& pre, const Placement& post) {  // placement.py:207-211
  Verdict v;
  if (check_partition(post, &v)) check_subset(post, pre, &v);
  return v;
}

// ------------------------------------------------------------------ numpy reductions
// numpy pairwise_sum (8 accumulators, PW_BLOCKSIZE = 128) for a contiguous float64 run.
double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// ------------------------------------------------------------------ traffic (costmodel.py)
struct Report {
  double sparsity, total, bottleneck_device, bottleneck_bytes;
};

// _report (costmodel.py:75-84).  Entries are whole multiples of chunk_bytes, so the
// sums below are exact in any order; total mirrors ndarray.sum() regardless.
Report make_report(const std::vector<double>& mat, int D, int touched, int C) {
  std::vector<double> in(D, 0.0), out(D, 0.0);
  for (int s = 0; s < D; ++s)
    for (int r = 0; r < D; ++r) {
      out[s] += mat[s * D + r];
      in[r] += mat[s * D + r];
    }
  int best = 0;
  double best_v = 0.0;
  for (int d = 0; d < D; ++d) {
    double v = std::max(in[d], out[d]);
    if (d == 0 || v > best_v) {  // np.argmax: first maximum
      best_v = v;
      best = d;
    }
  }
  Report rep;
  rep.sparsity = C ? static_cast<double>(touched) / C : 0.0;
  rep.total = np_pairwise_sum(mat.data(), static_cast<int64_t>(mat.size()));
  rep.bottleneck_device = best;
  rep.bottleneck_bytes = best_v;
  return rep;
}

// spag_traffic (costmodel.py:87-108)
bool spag_traffic(const Placement& pre, const Placement& post, double bytes,
                  std::vector<double>* mat, Report* rep, Err* err) {
  Verdict v = validate_spag(pre, post);
  if (!v.ok()) {
    err->code = FSSDP_ERR_INVALID_PAIR;
    err->msg = "invalid all-gather pair: " + v.describe();
    return false;
  }
  const int D = pre.D;
  mat->assign(static_cast<size_t>(D) * D, 0.0);
  int touched = 0;
  for (int c = 0; c < pre.C; ++c) {
    int owner = pre.owner(c);
    bool any = false;
    for (int d = 0; d < D; ++d)
      if (post.has(c, d) && !pre.has(c, d)) {
        (*mat)[owner * D + d] += bytes;
        any = true;
      }
    touched += any;
  }
  if (rep) *rep = make_report(*mat, D, touched, pre.C);
  return true;
}

// sprs_traffic (costmodel.py:111-132)
bool sprs_traffic(const Placement& pre, const Placement& post, double bytes,
                  std::vector<double>* mat, Report* rep, Err* err) {
  Verdict v = validate_sprs(pre, post);
  if (!v.ok()) {
    err->code = FSSDP_ERR_INVALID_PAIR;
    err->msg = "invalid reduce-scatter pair: " + v.describe();
    return false;
  }
  const int D = pre.D;
  mat->assign(static_cast<size_t>(D) * D, 0.0);
  int touched = 0;
  for (int c = 0; c < pre.C; ++c) {
    int final_owner = post.owner(c);
    bool any = false;
    for (int d = 0; d < D; ++d)
      if (pre.has(c, d) && d != final_owner) {
        (*mat)[d * D + final_owner] += bytes;
        any = true;
      }
    touched += any;
  }
  if (rep) *rep = make_report(*mat, D, touched, pre.C);
  return true;
}

// collective_latency (costmodel.py:149-182): volumes accumulate in np.nonzero order.
double collective_latency(const std::vector<double>& mat, int D, const Topo& t) {
  bool zero = true;
  for (double v : mat)
    if (v != 0.0) {
      zero = false;
      break;
    }
  if (zero) return 0.0;
  std::vector<double> dev_in(D, 0.0), dev_out(D, 0.0), node_in(t.nodes, 0.0),
      node_out(t.nodes, 0.0);
  for (int s = 0; s < D; ++s)
    for (int r = 0; r < D; ++r) {
      double vol = mat[s * D + r];
      if (vol == 0.0) continue;
      int ns = t.node_of(s), nr = t.node_of(r);
      if (ns == nr) {
        dev_out[s] += vol;
        dev_in[r] += vol;
      } else {
        node_out[ns] += vol;
        node_in[nr] += vol;
      }
    }
  double dmax = std::max(*std::max_element(dev_in.begin(), dev_in.end()),
                         *std::max_element(dev_out.begin(), dev_out.end()));
  double nmax = std::max(*std::max_element(node_in.begin(), node_in.end()),
                         *std::max_element(node_out.begin(), node_out.end()));
  double worst = std::max(dmax / t.intra, nmax / t.inter);
  return t.alpha + worst;
}

// overlap_degree (costmodel.py:185-194)
int64_t overlap_degree(double t_nonmoe, const Topo& t, double expert_bytes) {
  if (t_nonmoe <= 0 || expert_bytes <= 0) return 0;
  double bw = t.inter < t.intra ? t.inter : t.intra;
  return static_cast<int64_t>(floor(t_nonmoe * bw / expert_bytes));
}

// ------------------------------------------------------------------ dispatch (dispatch.py)
struct Route {
  int D, E;
  std::vector<int64_t> r;  // [D*E*D]
  int64_t& at(int s, int e, int d) { return r[(static_cast<size_t>(s) * E + e) * D + d]; }
};

// build_dispatch (dispatch.py:49-97); counts validated non-negative by the caller.
bool build_dispatch(const int64_t* counts, const Placement& p, const Topo& t, Route* out,
                    Err* err) {
  const int D = p.D, E = p.C;
  out->D = D;
  out->E = E;
  out->r.assign(static_cast<size_t>(D) * E * D, 0);
  // scratch reused across (source, expert) cells: this runs several times per plan on the
  // planning critical path
  std::vector<int64_t> assigned(D, 0), share(D);
  std::vector<int> targets(D), order(D);
  for (int src = 0; src < D; ++src) {
    const int node = t.node_of(src);
    for (int e = 0; e < E; ++e) {
      const int64_t n = counts[static_cast<size_t>(src) * E + e];
      if (n == 0) continue;
      if (p.has(e, src)) {
        out->at(src, e, src) += n;
        assigned[src] += n;
        continue;
      }
      int k = 0;
      for (int d = 0; d < D; ++d)
        if (p.has(e, d) && t.node_of(d) == node) targets[k++] = d;
      if (k == 0)
        for (int d = 0; d < D; ++d)
          if (p.has(e, d)) targets[k++] = d;
      if (k == 0) {
        err->code = FSSDP_ERR_ORPHAN_EXPERT;
        err->msg = "expert " + std::to_string(e) + " has tokens but is materialized nowhere";
        return false;
      }
      const int64_t base = n / k, rem = n % k;
      for (int i = 0; i < k; ++i) share[i] = base;
      if (rem) {
        for (int i = 0; i < k; ++i) order[i] = i;
        std::sort(order.begin(), order.begin() + k, [&](int a, int b) {
          const int da = targets[a], db = targets[b];
          if (assigned[da] != assigned[db]) return assigned[da] < assigned[db];
          return da < db;
        });
        for (int64_t i = 0; i < rem; ++i) share[order[i]] += 1;
      }
      for (int i = 0; i < k; ++i) {
        out->at(src, e, targets[i]) += share[i];
        assigned[targets[i]] += share[i];
      }
    }
  }
  return true;
}

// dispatch_traffic (dispatch.py:100-104)
std::vector<double> dispatch_traffic(Route& route, double token_bytes) {
  const int D = route.D, E = route.E;
  std::vector<double> mat(static_cast<size_t>(D) * D, 0.0);
  for (int s = 0; s < D; ++s)
    for (int d = 0; d < D; ++d) {
      if (s == d) continue;
      int64_t sum = 0;
      for (int e = 0; e < E; ++e) sum += route.at(s, e, d);
      mat[s * D + d] = static_cast<double>(sum) * token_bytes;
    }
  return mat;
}

int64_t max_device_tokens(Route& route) {
  const int D = route.D, E = route.E;
  int64_t best = 0;
  for (int d = 0; d < D; ++d) {
    int64_t tot = 0;
    for (int s = 0; s < D; ++s)
      for (int e = 0; e < E; ++e) tot += route.at(s, e, d);
    if (d == 0 || tot > best) best = tot;
  }
  return best;
}

// estimate_moe_latency (planner.py:205-216)
bool estimate_moe_latency(const Placement& p, const int64_t* tokens, const Topo& t,
                          double token_bytes, double ptt, double* out, Err* err) {
  Route route;
  if (!build_dispatch(tokens, p, t, &route, err)) return false;
  double compute = static_cast<double>(max_device_tokens(route)) * ptt;
  double a2a = collective_latency(dispatch_traffic(route, token_bytes), p.D, t);
  *out = compute + a2a;
  return true;
}

// ------------------------------------------------------------------ planner (planner.py)
// _descending (planner.py:74-76): value descending, lowest index first on ties.
std::vector<int> descending(const double* v, int n) {
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    if (v[a] != v[b]) return v[a] > v[b];
    return a < b;
  });
  return idx;
}

// Column sums of a D x E float64 matrix, numpy axis-0 order (sequential over rows).
std::vector<double> column_sums(const double* a, int rows, int cols) {
  std::vector<double> out(a, a + cols);
  for (int r = 1; r < rows; ++r)
    for (int c = 0; c < cols; ++c) out[c] += a[static_cast<size_t>(r) * cols + c];
  return out;
}

// _extend_placement (planner.py:79-168)
Placement extend_placement(const Placement& base, const std::vector<double>& per_expert,
                           int64_t t, int64_t m, const Topo& topo) {
  const int E = base.C, D = base.D;
  t = std::min<int64_t>(t, E);
  m = std::min<int64_t>(m, t);
  if (t <= 0 || m <= 0) return base;
  std::vector<int> order = descending(per_expert.data(), E);
  std::vector<int> top(order.begin(), order.begin() + t);
  Placement out = base;
  if (t <= m) {
    for (int e : top)
      for (int d = 0; d < D; ++d)
        if (!base.has(e, d)) out.set(e, d);
    return out;
  }
  const int64_t total_slots = static_cast<int64_t>(D) * m;
  std::vector<int64_t> avail(D, m);
  // holders[e] tracked in `out` (base + placed replicas of the top experts)

  auto place_one = [&](int expert) -> bool {
    // node key (node_has_expert, -node_free, node); device key (-avail, d)
    bool have = false;
    int best_node_has = 0;
    int64_t best_neg_free = 0;
    int best_node = -1, best_dev = -1;
    for (int node = 0; node < topo.nodes; ++node) {
      const int d0 = node * topo.dpn, d1 = d0 + topo.dpn;
      int cand = -1;
      int64_t node_free = 0;
      int node_has = 0;
      for (int d = d0; d < d1; ++d) {
        node_free += avail[d];
        if (out.has(expert, d)) node_has = 1;
        if (avail[d] > 0 && !out.has(expert, d)) {
          if (cand < 0 || avail[d] > avail[cand]) cand = d;  // (-avail, d): ties keep lower d
        }
      }
      if (cand < 0) continue;
      const int64_t neg_free = -node_free;
      bool better = !have || node_has < best_node_has ||
                    (node_has == best_node_has &&
                     (neg_free < best_neg_free || (neg_free == best_neg_free && node < best_node)));
      if (better) {
        have = true;
        best_node_has = node_has;
        best_neg_free = neg_free;
        best_node = node;
        best_dev = cand;
      }
    }
    if (best_dev < 0) return false;
    out.set(expert, best_dev);
    avail[best_dev] -= 1;
    return true;
  };

  // top_sum = float(sum(per_expert[e] for e in top)) — Python sum from int 0, in top order
  double top_sum = 0.0;
  for (int e : top) top_sum += per_expert[e];
  int64_t remaining = total_slots;
  for (int e : top) {
    int64_t share;
    if (top_sum > 0) {
      share = static_cast<int64_t>(floor(static_cast<double>(total_slots) * per_expert[e] / top_sum));
      if (share < 1) share = 1;
    } else {
      share = std::max<int64_t>(1, total_slots / t);
    }
    const int64_t cap = D - out.holders_count(e);
    const int64_t want = std::min(std::min(share, cap), remaining);
    int64_t placed = 0;
    while (placed < want && place_one(e)) ++placed;
    remaining -= placed;
  }
  bool progress = true;
  while (remaining > 0 && progress) {
    progress = false;
    for (int e : top) {
      if (remaining == 0) break;
      if (out.holders_count(e) < D && place_one(e)) {
        remaining -= 1;
        progress = true;
      }
    }
  }
  return out;
}

std::vector<int32_t> added_per_device(const Placement& source, const Placement& target) {
  std::vector<int32_t> a(source.D);
  for (int d = 0; d < source.D; ++d) a[d] = target.chunks_on(d) - source.chunks_on(d);
  return a;
}

struct CalOutcome {
  bool accepted = false;
  Placement target{0, 1};
  double extra = 0, before = 0, after = 0;
};

// calibrate (planner.py:228-276)
bool calibrate(const Placement& source, const Placement& target, const double* actual,
               int64_t remaining_m, double t_remaining, const Topo& topo, double chunk_bytes,
               double token_bytes, double ptt, CalOutcome* out, Err* err) {
  const int E = source.C, D = source.D;
  // build_dispatch(np.asarray(actual, float64)): must be integral and non-negative
  std::vector<int64_t> tokens(static_cast<size_t>(D) * E);
  for (size_t i = 0; i < tokens.size(); ++i) {
    if (actual[i] < 0 || actual[i] != floor(actual[i])) {
      err->code = FSSDP_ERR_DIMENSION;
      err->msg = "token counts must be non-negative integers";
      return false;
    }
    tokens[i] = static_cast<int64_t>(actual[i]);
  }
  double base_est;
  if (!estimate_moe_latency(target, tokens.data(), topo, token_bytes, ptt, &base_est, err))
    return false;
  out->target = target;
  out->before = out->after = base_est;
  out->extra = 0.0;
  out->accepted = false;
  const int64_t t_cal = overlap_degree(t_remaining, topo, chunk_bytes);
  if (remaining_m <= 0 || t_cal <= 0) return true;
  Placement extended =
      extend_placement(target, column_sums(actual, D, E), t_cal, remaining_m, topo);
  if (extended == target) return true;
  std::vector<double> tr, orig;
  if (!spag_traffic(source, extended, chunk_bytes, &tr, nullptr, err)) return false;
  if (!spag_traffic(source, target, chunk_bytes, &orig, nullptr, err)) return false;
  for (size_t i = 0; i < tr.size(); ++i) tr[i] -= orig[i];
  const double extra = collective_latency(tr, D, topo);
  double ext_est;
  if (!estimate_moe_latency(extended, tokens.data(), topo, token_bytes, ptt, &ext_est, err))
    return false;
  out->after = ext_est;
  if (ext_est + extra < base_est) {
    out->accepted = true;
    out->target = extended;
    out->extra = extra;
  }
  return true;
}

// heterogeneous_sharding (planner.py:302-385)
bool heterogeneous_sharding(int L, int E, const double* profile, int64_t t, const Topo& topo,
                            std::vector<int32_t>* owner, Err* err) {
  const int D = topo.devices();
  const int64_t total = static_cast<int64_t>(L) * E;
  const int64_t base = total / D, extra = total % D;
  std::vector<int64_t> avail(D);
  for (int d = 0; d < D; ++d) avail[d] = base + (d < extra ? 1 : 0);
  t = std::max<int64_t>(0, std::min<int64_t>(t, E));
  std::vector<std::vector<int>> reserved(L), rest(L);
  for (int l = 0; l < L; ++l) {
    std::vector<int> order = descending(profile + static_cast<size_t>(l) * E, E);
    reserved[l].assign(order.begin(), order.begin() + t);
    std::sort(reserved[l].begin(), reserved[l].end());
    rest[l].assign(order.begin() + t, order.end());
  }
  std::vector<double> node_load(topo.nodes, 0.0), dev_load(D, 0.0);
  owner->assign(static_cast<size_t>(L) * E, -1);

  auto pick_device = [&](double load, int* dev_out) -> bool {
    int best_node = -1;
    double bl = 0;
    int64_t bf = 0;
    for (int node = 0; node < topo.nodes; ++node) {
      const int d0 = node * topo.dpn, d1 = d0 + topo.dpn;
      bool any_free = false;
      int64_t node_free = 0;
      for (int d = d0; d < d1; ++d) {
        node_free += avail[d];
        if (avail[d] > 0) any_free = true;
      }
      if (!any_free) continue;
      // key (node_load, node_free, node)
      bool better = best_node < 0 || node_load[node] < bl ||
                    (node_load[node] == bl && (node_free < bf || (node_free == bf && node < best_node)));
      if (better) {
        best_node = node;
        bl = node_load[node];
        bf = node_free;
      }
    }
    if (best_node < 0) {
      err->code = FSSDP_ERR_INFEASIBLE;
      err->msg = "no device slot left while placing experts";
      return false;
    }
    int dev = -1;
    for (int d = best_node * topo.dpn; d < (best_node + 1) * topo.dpn; ++d) {
      if (avail[d] <= 0) continue;
      // key (dev_load, avail, d)
      if (dev < 0 || dev_load[d] < dev_load[dev] ||
          (dev_load[d] == dev_load[dev] && avail[d] < avail[dev]))
        dev = d;
    }
    avail[dev] -= 1;
    dev_load[dev] += load;
    node_load[best_node] += load;
    *dev_out = dev;
    return true;
  };

  std::vector<double> heaviest(L, -INFINITY);
  for (int l = 0; l < L; ++l)
    for (int e : rest[l]) {
      double v = profile[static_cast<size_t>(l) * E + e];
      if (v > heaviest[l]) heaviest[l] = v;
    }
  std::vector<int> layer_order(L);
  for (int l = 0; l < L; ++l) layer_order[l] = l;
  std::stable_sort(layer_order.begin(), layer_order.end(), [&](int a, int b) {
    if (heaviest[a] != heaviest[b]) return heaviest[a] > heaviest[b];
    return a < b;
  });
  for (int l : layer_order)
    for (int e : rest[l]) {
      int dev;
      if (!pick_device(profile[static_cast<size_t>(l) * E + e], &dev)) return false;
      (*owner)[static_cast<size_t>(l) * E + e] = dev;
    }
  int cursor = 0;
  for (int l = 0; l < L; ++l)
    for (int e : reserved[l]) {
      int scanned = 0;
      while (avail[cursor] == 0) {
        cursor = (cursor + 1) % D;
        if (++scanned > D) {
          err->code = FSSDP_ERR_INFEASIBLE;
          err->msg = "slot accounting exhausted during fill";
          return false;
        }
      }
      (*owner)[static_cast<size_t>(l) * E + e] = cursor;
      avail[cursor] -= 1;
      cursor = (cursor + 1) % D;
    }
  return true;
}

int fail(const Err& e) {
  set_error(e.msg.c_str());
  return e.code;
}

// Estimate-based candidate + adoption gate (engine.py:497-501, _adopt_materialization
// engine.py:406-429).  Depends only on the load history, so it is known before the gate.
bool adopted_candidate_uncached(const Placement& base, const double* est, const Topo& t,
                       const fssdp_layer_knobs* knobs, Placement* target, int* adopted, Err* err) {
  const int D = base.D, E = base.C;
  *target = base;
  *adopted = 0;
  Placement cand = extend_placement(base, column_sums(est, D, E), knobs->t, knobs->m, t);
  if (cand == base) return true;
  std::vector<int64_t> tokens(static_cast<size_t>(D) * E);
  for (size_t i = 0; i < tokens.size(); ++i) {
    double r = nearbyint(est[i]);  // np.rint: half to even
    tokens[i] = r > 0 ? static_cast<int64_t>(r) : 0;
  }
  double before, after;
  if (!estimate_moe_latency(base, tokens.data(), t, knobs->token_bytes,
                            knobs->per_token_expert_time, &before, err) ||
      !estimate_moe_latency(cand, tokens.data(), t, knobs->token_bytes,
                            knobs->per_token_expert_time, &after, err))
    return false;
  std::vector<double> mat;
  if (!spag_traffic(base, cand, knobs->expert_bytes, &mat, nullptr, err)) return false;
  const double s_lat = collective_latency(mat, D, t);
  if (!sprs_traffic(cand, base, knobs->expert_bytes, &mat, nullptr, err)) return false;
  const double r_lat = collective_latency(mat, D, t);
  const double remat = knobs->rematerialize ? s_lat : 0.0;
  if (after + s_lat + r_lat + remat < before) {
    *target = cand;
    *adopted = 1;
  }
  return true;
}

// The candidate is computed twice per layer-iteration with identical inputs (early SpAG
// before the gate, then fssdp_plan_layer after it): memoize the last few by exact inputs.
struct CandidateMemo {
  std::vector<uint8_t> key;
  Placement target{0, 1};
  int adopted = 0;
};

bool adopted_candidate(const Placement& base, const double* est, const Topo& t,
                       const fssdp_layer_knobs* knobs, Placement* target, int* adopted, Err* err) {
  static thread_local std::vector<CandidateMemo> memo;
  static thread_local size_t next = 0;
  // key: every input, as exact bytes
  std::vector<uint8_t> key;
  auto put = [&key](const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    key.insert(key.end(), b, b + n);
  };
  const size_t est_bytes = static_cast<size_t>(base.C) * base.D * sizeof(double);
  key.reserve(6 * 8 + 7 * 8 + 8 + base.m.size() + est_bytes);
  const int64_t ints[6] = {base.C, base.D, t.nodes, t.dpn, knobs->t, knobs->m};
  const double dbls[7] = {t.intra, t.inter, t.alpha, knobs->expert_bytes, knobs->token_bytes,
                          knobs->attn_fwd_time, knobs->per_token_expert_time};
  const int32_t flags[2] = {knobs->calibration, knobs->rematerialize};
  put(ints, sizeof(ints));
  put(dbls, sizeof(dbls));
  put(flags, sizeof(flags));
  put(base.m.data(), base.m.size());
  put(est, est_bytes);
  for (const CandidateMemo& c : memo)
    if (c.key == key) {
      *target = c.target;
      *adopted = c.adopted;
      return true;
    }
  if (!adopted_candidate_uncached(base, est, t, knobs, target, adopted, err)) return false;
  if (memo.size() < 16) memo.emplace_back();
  CandidateMemo& slot = memo[next++ % memo.size()];
  slot.key = std::move(key);
  slot.target = *target;
  slot.adopted = *adopted;
  return true;
}

void copy_mask(const Placement& p, uint8_t* out) { memcpy(out, p.m.data(), p.m.size()); }

}  // namespace

extern "C" {

int fssdp_make_even_partition(int32_t num_chunks, int32_t num_devices, int32_t* owner_out) {
  if (num_chunks < 0 || num_devices <= 0) {
    set_error("placement needs num_chunks >= 0 and num_devices > 0");
    return FSSDP_ERR_DIMENSION;
  }
  const int base = num_chunks / num_devices, extra = num_chunks % num_devices;
  int chunk = 0;
  for (int d = 0; d < num_devices; ++d)
    for (int i = 0; i < base + (d < extra ? 1 : 0); ++i) owner_out[chunk++] = d;
  return FSSDP_OK;
}

int fssdp_shard_plan_even(int32_t layers, int32_t experts, int32_t devices, int32_t* owner_out) {
  if (layers <= 0 || experts < 0 || devices <= 0) {
    set_error("shard plan needs at least one layer");
    return FSSDP_ERR_DIMENSION;
  }
  const int base = experts / devices, extra = experts % devices;
  int cursor = 0;
  std::vector<int> counts(devices);
  for (int l = 0; l < layers; ++l) {
    std::fill(counts.begin(), counts.end(), base);
    for (int j = 0; j < extra; ++j) counts[(cursor + j) % devices] += 1;
    cursor = (cursor + extra) % devices;
    int chunk = 0;
    for (int d = 0; d < devices; ++d)
      for (int i = 0; i < counts[d]; ++i) owner_out[static_cast<size_t>(l) * experts + chunk++] = d;
  }
  return FSSDP_OK;
}

int fssdp_validate_pair(int32_t kind, int32_t num_chunks, int32_t num_devices,
                        const uint8_t* pre_mask, const uint8_t* post_mask, int32_t* verdict_out) {
  Placement pre(num_chunks, num_devices, pre_mask), post(num_chunks, num_devices, post_mask);
  Verdict v = kind == 0 ? validate_spag(pre, post) : validate_sprs(pre, post);
  verdict_out[0] = v.reason;
  verdict_out[1] = v.chunk;
  verdict_out[2] = v.device;
  return FSSDP_OK;
}

static int traffic_common(bool spag, int32_t C, int32_t D, const uint8_t* pre_mask,
                          const uint8_t* post_mask, double bytes, double* matrix_out,
                          double* report_out) {
  Placement pre(C, D, pre_mask), post(C, D, post_mask);
  std::vector<double> mat;
  Report rep;
  Err err;
  bool ok = spag ? spag_traffic(pre, post, bytes, &mat, &rep, &err)
                 : sprs_traffic(pre, post, bytes, &mat, &rep, &err);
  if (!ok) return fail(err);
  memcpy(matrix_out, mat.data(), mat.size() * sizeof(double));
  report_out[0] = rep.sparsity;
  report_out[1] = rep.total;
  report_out[2] = rep.bottleneck_device;
  report_out[3] = rep.bottleneck_bytes;
  return FSSDP_OK;
}

int fssdp_spag_traffic(int32_t C, int32_t D, const uint8_t* pre, const uint8_t* post, double bytes,
                       double* matrix_out, double* report_out) {
  return traffic_common(true, C, D, pre, post, bytes, matrix_out, report_out);
}

int fssdp_sprs_traffic(int32_t C, int32_t D, const uint8_t* pre, const uint8_t* post, double bytes,
                       double* matrix_out, double* report_out) {
  return traffic_common(false, C, D, pre, post, bytes, matrix_out, report_out);
}

int fssdp_collective_latency(int32_t num_devices, const double* matrix, const fssdp_topology* topo,
                             double* seconds_out) {
  if (int rc = check_topo(topo)) return rc;
  Topo t = to_topo(topo);
  if (num_devices != t.devices()) {
    char buf[96];
    snprintf(buf, sizeof(buf), "traffic is %d devices, topology has %d", num_devices, t.devices());
    set_error(buf);
    return FSSDP_ERR_DIM_MISMATCH;
  }
  std::vector<double> mat(matrix, matrix + static_cast<size_t>(num_devices) * num_devices);
  *seconds_out = collective_latency(mat, num_devices, t);
  return FSSDP_OK;
}

int fssdp_overlap_degree(double t_nonmoe, const fssdp_topology* topo, double expert_bytes,
                         int64_t* t_out) {
  if (int rc = check_topo(topo)) return rc;
  *t_out = overlap_degree(t_nonmoe, to_topo(topo), expert_bytes);
  return FSSDP_OK;
}

int fssdp_build_dispatch(int32_t D, int32_t E, const int64_t* counts, const uint8_t* placement_mask,
                         const fssdp_topology* topo, int64_t* route_out) {
  if (int rc = check_topo(topo)) return rc;
  Topo t = to_topo(topo);
  if (D != t.devices()) {
    set_error("token matrix and topology disagree on device count");
    return FSSDP_ERR_DIMENSION;
  }
  for (int64_t i = 0; i < static_cast<int64_t>(D) * E; ++i)
    if (counts[i] < 0) {
      set_error("token counts must be non-negative");
      return FSSDP_ERR_DIMENSION;
    }
  Placement p(E, D, placement_mask);
  Route route;
  Err err;
  if (!build_dispatch(counts, p, t, &route, &err)) return fail(err);
  memcpy(route_out, route.r.data(), route.r.size() * sizeof(int64_t));
  return FSSDP_OK;
}

int fssdp_estimate_moe_latency(int32_t D, int32_t E, const uint8_t* placement_mask,
                               const int64_t* tokens, const fssdp_topology* topo, double token_bytes,
                               double per_token_expert_time, double* seconds_out) {
  if (int rc = check_topo(topo)) return rc;
  Placement p(E, D, placement_mask);
  Err err;
  if (!estimate_moe_latency(p, tokens, to_topo(topo), token_bytes, per_token_expert_time,
                            seconds_out, &err))
    return fail(err);
  return FSSDP_OK;
}

int fssdp_sparse_materialization(int32_t E, int32_t D, const uint8_t* base_mask,
                                 const double* per_expert_loads, int64_t t, int64_t m,
                                 const fssdp_topology* topo, uint8_t* target_out,
                                 int32_t* added_out) {
  if (int rc = check_topo(topo)) return rc;
  Placement base(E, D, base_mask);
  if (!base.is_partition()) {
    set_error("materialization must start from a partition");
    return FSSDP_ERR_INTERNAL;
  }
  std::vector<double> per(per_expert_loads, per_expert_loads + E);
  Placement target = extend_placement(base, per, t, m, to_topo(topo));
  copy_mask(target, target_out);
  std::vector<int32_t> added = added_per_device(base, target);
  memcpy(added_out, added.data(), added.size() * sizeof(int32_t));
  return FSSDP_OK;
}

int fssdp_calibrate(int32_t E, int32_t D, const uint8_t* source_mask, const uint8_t* target_mask,
                    const double* actual, int64_t remaining_m, double t_remaining,
                    const fssdp_topology* topo, double chunk_bytes, double token_bytes,
                    double per_token_expert_time, int32_t* accepted_out, uint8_t* target_out,
                    int32_t* added_out, double* doubles_out) {
  if (int rc = check_topo(topo)) return rc;
  Placement source(E, D, source_mask), target(E, D, target_mask);
  CalOutcome out;
  Err err;
  if (!calibrate(source, target, actual, remaining_m, t_remaining, to_topo(topo), chunk_bytes,
                 token_bytes, per_token_expert_time, &out, &err))
    return fail(err);
  *accepted_out = out.accepted ? 1 : 0;
  copy_mask(out.target, target_out);
  std::vector<int32_t> added = added_per_device(source, out.target);
  memcpy(added_out, added.data(), added.size() * sizeof(int32_t));
  doubles_out[0] = out.extra;
  doubles_out[1] = out.before;
  doubles_out[2] = out.after;
  return FSSDP_OK;
}

int fssdp_heterogeneous_sharding(int32_t layers, int32_t experts, const double* profile, int64_t t,
                                 const fssdp_topology* topo, int32_t* owner_out) {
  if (int rc = check_topo(topo)) return rc;
  std::vector<int32_t> owner;
  Err err;
  if (!heterogeneous_sharding(layers, experts, profile, t, to_topo(topo), &owner, &err))
    return fail(err);
  memcpy(owner_out, owner.data(), owner.size() * sizeof(int32_t));
  return FSSDP_OK;
}

int fssdp_estimate_loads(int32_t n, int32_t rows, int32_t cols, const double* history,
                         int32_t window, double* mean_out) {
  if (n <= 0) {
    set_error("cannot estimate loads from an empty history");
    return FSSDP_ERR_EMPTY_HISTORY;
  }
  if (window <= 0) {
    char buf[64];
    snprintf(buf, sizeof(buf), "window must be positive, got %d", window);
    set_error(buf);
    return FSSDP_ERR_EMPTY_HISTORY;
  }
  const int w = std::min(n, window);
  const size_t cells = static_cast<size_t>(rows) * cols;
  const double* first = history + (n - w) * cells;
  for (size_t i = 0; i < cells; ++i) mean_out[i] = first[i];
  for (int k = 1; k < w; ++k)
    for (size_t i = 0; i < cells; ++i) mean_out[i] += first[k * cells + i];
  for (size_t i = 0; i < cells; ++i) mean_out[i] /= static_cast<double>(w);
  return FSSDP_OK;
}

int fssdp_plan_candidate(int32_t E, const int32_t* base_owner, const double* est,
                         const fssdp_topology* topo, const fssdp_layer_knobs* knobs,
                         uint8_t* target_out, int32_t* adopted_out) {
  if (int rc = check_topo(topo)) return rc;
  const Topo t = to_topo(topo);
  const int D = t.devices();
  Placement base(E, D);
  for (int e = 0; e < E; ++e) base.set(e, base_owner[e]);
  Placement target = base;
  int adopted = 0;
  Err err;
  if (est != nullptr && knobs->t > 0 && knobs->m > 0 &&
      !adopted_candidate(base, est, t, knobs, &target, &adopted, &err))
    return fail(err);
  copy_mask(target, target_out);
  *adopted_out = adopted;
  return FSSDP_OK;
}

int fssdp_plan_layer(int32_t E, const int32_t* base_owner, const double* est,
                     const int64_t* actual, const fssdp_topology* topo,
                     const fssdp_layer_knobs* knobs, uint8_t* target_out, int32_t* added_out,
                     int64_t* route_out, double* doubles_out, int32_t* flags_out) {
  if (int rc = check_topo(topo)) return rc;
  const Topo t = to_topo(topo);
  const int D = t.devices();
  Placement base(E, D);
  for (int e = 0; e < E; ++e) base.set(e, base_owner[e]);
  Err err;
  Placement target = base;
  double spag_lat = 0, sprs_lat = 0, remat_lat = 0, calib_time = 0;
  int adopted = 0, accepted = 0;
  std::vector<double> mat;

  for (int64_t i = 0; i < static_cast<int64_t>(D) * E; ++i)
    if (actual[i] < 0) {
      set_error("token counts must be non-negative");
      return FSSDP_ERR_DIMENSION;
    }

  // engine.py:459-468 — nothing fits in the overlap window: plain expert parallelism
  const bool degenerate = knobs->t <= 0 || knobs->m <= 0;
  if (!degenerate) {
    if (est != nullptr) {  // engine.py:497-501
      if (!adopted_candidate(base, est, t, knobs, &target, &adopted, &err)) return fail(err);
    }
    if (!(target == base)) {  // engine.py:502-506
      if (!spag_traffic(base, target, knobs->expert_bytes, &mat, nullptr, &err)) return fail(err);
      spag_lat = collective_latency(mat, D, t);
    }
    if (knobs->calibration) {  // engine.py:507-532
      std::vector<int32_t> added = added_per_device(base, target);
      int32_t added_max = added.empty() ? 0 : *std::max_element(added.begin(), added.end());
      std::vector<double> actual_f(static_cast<size_t>(D) * E);
      for (size_t i = 0; i < actual_f.size(); ++i) actual_f[i] = static_cast<double>(actual[i]);
      CalOutcome out;
      double t_rem = knobs->attn_fwd_time - spag_lat;
      if (!(t_rem > 0.0)) t_rem = 0.0;  // max(0.0, attn - spag_lat)
      if (!calibrate(base, target, actual_f.data(), knobs->m - added_max, t_rem, t,
                     knobs->expert_bytes, knobs->token_bytes, knobs->per_token_expert_time, &out,
                     &err))
        return fail(err);
      if (out.accepted) {
        target = out.target;
        calib_time = out.extra;
        accepted = 1;
      }
      if (!(target == base)) {
        // kept = estimate_moe_latency(target, actual): calibrate already priced exactly
        // this placement on these counts (after if accepted, before otherwise)
        double kept = out.accepted ? out.after : out.before, bare;
        if (!estimate_moe_latency(base, actual, t, knobs->token_bytes,
                                  knobs->per_token_expert_time, &bare, &err))
          return fail(err);
        kept += calib_time;
        if (kept >= bare) {
          target = base;
          calib_time = 0.0;
        }
      }
    }
    if (!(target == base)) {  // engine.py:533-542
      if (!sprs_traffic(target, base, knobs->expert_bytes, &mat, nullptr, &err)) return fail(err);
      sprs_lat = collective_latency(mat, D, t);
      if (knobs->rematerialize) {
        if (!spag_traffic(base, target, knobs->expert_bytes, &mat, nullptr, &err)) return fail(err);
        remat_lat = collective_latency(mat, D, t);
      }
    }
  }
  Route route;
  if (!build_dispatch(actual, target, t, &route, &err)) return fail(err);
  copy_mask(target, target_out);
  std::vector<int32_t> added = added_per_device(base, target);
  memcpy(added_out, added.data(), added.size() * sizeof(int32_t));
  memcpy(route_out, route.r.data(), route.r.size() * sizeof(int64_t));
  doubles_out[0] = spag_lat;
  doubles_out[1] = sprs_lat;
  doubles_out[2] = remat_lat;
  doubles_out[3] = calib_time;
  flags_out[0] = adopted;
  flags_out[1] = accepted;
  return FSSDP_OK;
}

int fssdp_shard_score(int32_t layers, int32_t experts, const int32_t* owner, const double* profile,
                      const fssdp_topology* topo, double* score_out) {
  if (int rc = check_topo(topo)) return rc;
  const Topo t = to_topo(topo);
  const int D = t.devices();
  std::vector<double> dev_load(D, 0.0);
  for (int l = 0; l < layers; ++l)
    for (int e = 0; e < experts; ++e)
      dev_load[owner[static_cast<size_t>(l) * experts + e]] +=
          profile[static_cast<size_t>(l) * experts + e];
  double node_max = 0.0, dev_max = 0.0;
  for (int n = 0; n < t.nodes; ++n) {
    double s = np_pairwise_sum(dev_load.data() + n * t.dpn, t.dpn);  // fancy-index copy .sum()
    if (n == 0 || s > node_max) node_max = s;
  }
  for (int d = 0; d < D; ++d)
    if (d == 0 || dev_load[d] > dev_max) dev_max = dev_load[d];
  score_out[0] = node_max;
  score_out[1] = dev_max;
  return FSSDP_OK;
}

// ------------------------------------------------------------------ device plan tables
// Native twin of plan_tables.build_rank_tables (the Python version is the test oracle of
// this one): one rank's kernel tables for one layer-iteration, packed for a single H2D.
int fssdp_tables_layout(int32_t num_experts, int32_t num_devices, int64_t* offsets_out,
                        int64_t* total_bytes_out) {
  const int64_t E = num_experts, D = num_devices;
  const int64_t G = E * static_cast<int64_t>(sizeof(fssdp_gemm_group));
  const int64_t sizes[FSSDP_TAB_NSECTIONS] = {
      E * (D + 1) * 4, E * D * 4, E * 2 * 4, E * 3 * 4, E * 3 * 4, E * D * 2 * 4,
      G, G, G, G, G, G,
      E * 4, E * 4, E * 4, E * 4, E * D * 2 * 4};
  int64_t off = 0;
  for (int i = 0; i < FSSDP_TAB_NSECTIONS; ++i) {
    offsets_out[i] = off;
    off += (sizes[i] + 15) / 16 * 16;
  }
  *total_bytes_out = off;
  return FSSDP_OK;
}

int fssdp_build_rank_tables(int32_t rank, int32_t D, int32_t E, const int32_t* base_owner,
                            const uint8_t* target_mask, const uint8_t* pre_mask,
                            const int64_t* route, int32_t d_model, int32_t d_ff, int32_t n_mats,
                            const int64_t* slot_layout, uint8_t* blob, int64_t blob_bytes,
                            int32_t* header_out) {
  // pre_mask (nullable): replicas already fetched by the early, estimate-based SpAG.  They
  // take the first replica slots (ascending expert id) and get no SpAG copy here.
  auto pre = [&](int e, int d) {
    return pre_mask != nullptr && pre_mask[static_cast<int64_t>(e) * D + d] != 0;
  };
  int64_t off[FSSDP_TAB_NSECTIONS], total;
  fssdp_tables_layout(E, D, off, &total);
  if (blob_bytes < total || rank < 0 || rank >= D || d_model % 256 || d_ff % 128 ||
      (n_mats != 2 && n_mats != 3)) {
    set_error("build_rank_tables: bad arguments");
    return FSSDP_ERR_DIMENSION;
  }
  memset(blob, 0, static_cast<size_t>(total));
  auto R = [&](int s, int e, int d) { return route[(static_cast<int64_t>(s) * E + e) * D + d]; };
  // slot maps of every device: owned experts (ascending) then replicas (ascending)
  std::vector<std::vector<int>> slot_of(D, std::vector<int>(E, -1));
  std::vector<std::vector<int>> slot_expert(D);
  for (int d = 0; d < D; ++d) {
    for (int e = 0; e < E; ++e)
      if (base_owner[e] == d) slot_expert[d].push_back(e);
    for (int pass = 0; pass < 2; ++pass)  // prefetched replicas first, then the rest
      for (int e = 0; e < E; ++e)
        if (target_mask[static_cast<int64_t>(e) * D + d] && base_owner[e] != d &&
            pre(e, d) == (pass == 0))
          slot_expert[d].push_back(e);
    for (size_t s = 0; s < slot_expert[d].size(); ++s) slot_of[d][slot_expert[d][s]] = static_cast<int>(s);
  }
  // segments (padded to 256 rows) of every device
  std::vector<std::vector<int64_t>> seg_start(D), seg_rows(D), seg_pad(D);
  for (int d = 0; d < D; ++d) {
    int64_t st = 0;
    for (int e : slot_expert[d]) {
      int64_t rows = 0;
      for (int s = 0; s < D; ++s) rows += R(s, e, d);
      const int64_t padded = (rows + 255) / 256 * 256;  // CTA-pair GEMM M tile
      seg_start[d].push_back(st);
      seg_rows[d].push_back(rows);
      seg_pad[d].push_back(padded);
      st += padded;
    }
  }
  int32_t* route_cum = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_ROUTE_CUM]);
  int32_t* recv_base = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_RECV_BASE]);
  for (int e = 0; e < E; ++e) {
    int64_t run = 0;
    route_cum[e * (D + 1)] = 0;
    for (int d = 0; d < D; ++d) {
      run += R(rank, e, d);
      route_cum[e * (D + 1) + d + 1] = static_cast<int32_t>(run);
      const int s = slot_of[d][e];
      if (s >= 0) {
        int64_t before = 0;
        for (int src = 0; src < rank; ++src) before += R(src, e, d);
        recv_base[e * D + d] = static_cast<int32_t>(seg_start[d][s] + before);
      }
    }
  }
  const int n_slots = static_cast<int>(slot_expert[rank].size());
  int32_t* zero = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_ZERO_ROWS]);
  int n_zero = 0;
  for (int s = 0; s < n_slots; ++s)
    if (seg_pad[rank][s] > seg_rows[rank][s]) {
      zero[2 * n_zero] = static_cast<int32_t>(seg_start[rank][s] + seg_rows[rank][s]);
      zero[2 * n_zero + 1] = static_cast<int32_t>(seg_pad[rank][s] - seg_rows[rank][s]);
      ++n_zero;
    }
  // parameter slot of local slot s (owned slots first, then replicas): the layer's own
  // contiguous region (slot_layout null) or, in a model-level parameter region, owned slot i
  // at owned_base + i and replica j at replica_base + j — replicas of every layer may share
  // one region (re-materialization keeps only one layer's replicas resident)
  int n_owned = 0;
  for (int s = 0; s < n_slots; ++s) n_owned += base_owner[slot_expert[rank][s]] == rank;
  auto pslot = [&](int s, int owned) -> int32_t {
    if (slot_layout == nullptr) return s;
    return static_cast<int32_t>(s < owned ? slot_layout[0] + s : slot_layout[1] + (s - owned));
  };
  int32_t* spag = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SPAG]);
  int n_spag = 0;
  for (int s = 0; s < n_slots; ++s) {
    const int e = slot_expert[rank][s];
    const int o = base_owner[e];
    if (o == rank) continue;
    if (pre(e, rank)) continue;  // fetched early
    spag[3 * n_spag] = o;
    spag[3 * n_spag + 1] = pslot(slot_of[o][e], E);  // an owned slot on the owner
    spag[3 * n_spag + 2] = pslot(s, n_owned);
    ++n_spag;
  }
  // SpRS by push: a holder's wgrad epilogue writes its partial of a replica straight into
  // the owner's staging slot (NVLink); the owner then sums locally, ascending rank.
  // Staging index on owner o: its owned experts with other holders in slot order, each
  // followed by its non-owner holders ascending.  Every rank derives the same indices.
  auto holds = [&](int e, int dd) { return target_mask[static_cast<int64_t>(e) * D + dd] != 0; };
  std::vector<int> stage_idx(static_cast<size_t>(E) * D, -1);  // [e][holder]
  int n_stage = 0;
  for (int o = 0; o < D; ++o) {
    int j = 0;
    for (int e : slot_expert[o]) {
      if (base_owner[e] != o) continue;
      for (int h = 0; h < D; ++h)
        if (h != o && holds(e, h)) stage_idx[static_cast<size_t>(e) * D + h] = j++;
    }
    if (o == rank) n_stage = j;
  }
  int32_t* jobs = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SPRS_JOBS]);
  int32_t* srcs = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SPRS_SRCS]);
  int32_t* pull = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SPRS_PULL]);
  int n_jobs = 0, n_srcs = 0;
  for (int s = 0; s < n_slots; ++s) {
    const int e = slot_expert[rank][s];
    if (base_owner[e] != rank) continue;
    int holders = 0;
    for (int dd = 0; dd < D; ++dd) holders += holds(e, dd);
    if (holders <= 1) continue;
    jobs[3 * n_jobs] = s;
    jobs[3 * n_jobs + 1] = n_srcs;
    jobs[3 * n_jobs + 2] = holders;
    ++n_jobs;
    for (int dd = 0; dd < D; ++dd)
      if (holds(e, dd)) {  // {rank, own grads slot | staging slot}
        srcs[2 * n_srcs] = dd;
        srcs[2 * n_srcs + 1] = dd == rank ? s : stage_idx[static_cast<size_t>(e) * D + dd];
        pull[2 * n_srcs] = dd;  // the standalone pull transport: the holder's grads slot
        pull[2 * n_srcs + 1] = slot_of[dd][e];
        ++n_srcs;
      }
  }
  // the six grouped-GEMM descriptor arrays (see plan_tables.gemm_groups); the wgrads list
  // the slots shared with other holders first (their SpRS can start before the rest runs)
  auto shared = [&](int s) {
    const int e = slot_expert[rank][s];
    int holders = 0;
    for (int dd = 0; dd < D; ++dd) holders += holds(e, dd);
    return holders > 1;
  };
  // each part longest-first (K = segment rows): the GEMM's snake tile order then deals
  // the tiles out close to LPT
  std::vector<int> wg_order;
  for (int s = 0; s < n_slots; ++s)
    if (shared(s)) wg_order.push_back(s);
  const int n_shared = static_cast<int>(wg_order.size());
  for (int s = 0; s < n_slots; ++s)
    if (!shared(s)) wg_order.push_back(s);
  auto longer = [&](int a, int b) { return seg_pad[rank][a] > seg_pad[rank][b]; };
  std::stable_sort(wg_order.begin(), wg_order.begin() + n_shared, longer);
  std::stable_sort(wg_order.begin() + n_shared, wg_order.end(), longer);
  // slot = [W1 (f x d) | W2 (d x f)] (GeLU, n_mats 2) or [W13 (2f x d) | W2] (SwiGLU, 3);
  // n1 = fwd1's N.  N tiles of width f use 128 columns when f % 256 != 0; SwiGLU's fwd1
  // always uses 256 (an a1|a3 block pair per tile)
  const int64_t d = d_model, f = d_ff, nm = n_mats, n1 = (nm - 1) * f;
  // dgrad2 / wgrad2 (N = f, B read N-contiguous): 256-wide tiles, the last one ragged (TMA
  // zero-fills B past f and clips the stores) — plan_tables.n_tile_widths
  const int64_t bnf = f % 256 == 0 ? 256 : 128, bn1 = nm == 3 ? 256 : bnf;
  const int64_t nf = (f + 255) / 256;
  const int n_tiles[6] = {static_cast<int>(n1 / bn1), static_cast<int>(d / 256),
                          static_cast<int>(nf), static_cast<int>(d / 256),
                          static_cast<int>(d / 256), static_cast<int>(nf)};
  int ints = 7;
  int32_t shared_tiles[2] = {0, 0};
  for (int gi = 0; gi < 6; ++gi) {
    fssdp_gemm_group* g = reinterpret_cast<fssdp_gemm_group*>(blob + off[FSSDP_TAB_GEMM0 + gi]);
    const bool wgrad = gi >= 4;
    int32_t tile = 0, total = 0;
    for (int i = 0; i < n_slots; ++i) {
      const int s = wgrad ? wg_order[i] : i;
      if (wgrad && i == n_shared) {  // the rest restarts at tile 0
        shared_tiles[gi - 4] = tile;
        tile = 0;
      }
      const int32_t st = static_cast<int32_t>(seg_start[rank][s]);
      const int32_t mt = static_cast<int32_t>(seg_pad[rank][s] / 128);
      // wgrad K = the segment's rows rounded up to one 64-row K block: the zero padding
      // beyond it would only add exact zeros
      const int32_t kt = static_cast<int32_t>((seg_rows[rank][s] + 63) / 64);
      fssdp_gemm_group& x = g[i];
      const int64_t ps = pslot(s, n_owned);
      const int32_t w1r = static_cast<int32_t>(ps * nm * f), w2r = static_cast<int32_t>(ps * nm * d);
      switch (gi) {
        case 0: x = {mt, 0, st, 0, w1r, 0, static_cast<int32_t>(d / 64), 0, st * n1}; break;
        case 1: x = {mt, 0, st, 0, w2r, 0, static_cast<int32_t>(f / 64), 0, st * d}; break;
        case 2: x = {mt, 0, st, 0, 0, w2r, static_cast<int32_t>(d / 64), 0, st * n1}; break;
        case 3: x = {mt, 0, st, 0, 0, w1r, static_cast<int32_t>(n1 / 64), 0, st * d}; break;
        case 4: x = {static_cast<int32_t>(n1 / 128), 0, 0, st, 0, st, kt, 0, s * nm * f * d}; break;
        default: x = {static_cast<int32_t>(d / 128), 0, 0, st, 0, st, kt, 0, s * nm * f * d + n1 * d}; break;
      }
      if (!wgrad) x.rows = static_cast<int32_t>(seg_rows[rank][s]);  // the real rows
      if (wgrad) {  // a replica's partial goes to its owner's staging slot
        const int e = slot_expert[rank][s];
        const int o = base_owner[e];
        if (o != rank) {
          x.c_dest = o + 1;
          x.c_off = static_cast<int64_t>(stage_idx[static_cast<size_t>(e) * D + rank]) * nm * f * d +
                    (gi == 5 ? n1 * d : 0);
        }
      }
      x.tile_start = tile;
      tile += x.m_tiles * n_tiles[gi];
      total += x.m_tiles * n_tiles[gi];
    }
    if (wgrad && n_shared == n_slots) shared_tiles[gi - 4] = tile;
    header_out[ints++] = n_slots;
    header_out[ints++] = n_tiles[gi];
    header_out[ints++] = total;
  }
  header_out[25] = n_shared;
  header_out[26] = shared_tiles[0];
  header_out[27] = shared_tiles[1];
  header_out[28] = n_stage;
  int32_t* se = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SLOT_EXPERT]);
  int32_t* ss = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SEG_START]);
  int32_t* sr = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SEG_ROWS]);
  int32_t* sp = reinterpret_cast<int32_t*>(blob + off[FSSDP_TAB_SEG_PADDED]);
  int64_t recv_rows = 0;
  for (int s = 0; s < n_slots; ++s) {
    se[s] = slot_expert[rank][s];
    ss[s] = static_cast<int32_t>(seg_start[rank][s]);
    sr[s] = static_cast<int32_t>(seg_rows[rank][s]);
    sp[s] = static_cast<int32_t>(seg_pad[rank][s]);
    recv_rows += seg_pad[rank][s];
  }
  header_out[0] = n_slots;
  header_out[1] = n_owned;
  header_out[2] = static_cast<int32_t>(recv_rows);
  header_out[3] = n_zero;
  header_out[4] = n_spag;
  header_out[5] = n_jobs;
  header_out[6] = n_srcs;
  return FSSDP_OK;
}

}  // extern "C"
