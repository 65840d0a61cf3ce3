// Host program builder. See program.hpp. Reference anchors are cited inline.
#include "program.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <unordered_map>

#include "jsonlite.hpp"

namespace qcg {

namespace {

std::string fmt_double_fixed(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", v);  // std::to_string(double)
  return buf;
}

}  // namespace

RankGuard::RankGuard(int r, int m)
    : std::runtime_error("contraction would produce a rank-" + std::to_string(r) + " tensor (" +
                         fmt_double_fixed(16.0 * std::pow(4.0, r)) +
                         " bytes), exceeding max rank " + std::to_string(m)),
      rank(r),
      max_rank(m) {}

uint64_t Program::jobs_density() const { return uint64_t{1} << (2 * M); }
uint64_t Program::jobs_ket() const { return uint64_t{1} << M; }

// ---------------------------------------------------------------------------
// decode_payload (serialize.cpp:156-167, plan_from_json :106-128,
// load_network_json tensor_network.cpp:179-196)
// ---------------------------------------------------------------------------
Payload decode_payload(const char* text, size_t len) {
  JValue j = json_parse(text, len);
  if (j.at("v").as_int() != 1) throw std::invalid_argument("unsupported payload version");
  Payload p;
  const JValue& net = j.at("network");
  if (net.has("v") && net.at("v").as_int() != 1)
    throw std::invalid_argument("unsupported network dump version");
  std::map<int, Vertex> verts;
  for (const JValue& jv : net.at("vertices").arr) {
    Vertex v;
    v.id = jv.at("id").as_int();
    v.rank = jv.at("rank").as_int();
    if (v.rank < 0 || v.rank > 16) throw std::invalid_argument("vertex rank out of range");
    const JValue& data = jv.at("data");
    size_t want = size_t{1} << (2 * v.rank);
    if (data.size() != want) throw std::invalid_argument("tensor data length mismatch");
    v.data.resize(want);
    for (size_t i = 0; i < want; ++i)
      v.data[i] = cxd{data[i][0].as_double(), data[i][1].as_double()};
    verts[v.id] = std::move(v);
  }
  for (auto& kv : verts) p.vertices.push_back(std::move(kv.second));
  for (const JValue& je : net.at("edges").arr) {
    const JValue& ep = je.at("endpoints");
    p.edges.push_back(NetEdge{je.at("id").as_int(), ep[0][0].as_int(), ep[0][1].as_int(),
                              ep[1][0].as_int(), ep[1][1].as_int()});
  }
  p.cut = j.at("cut").as_int_vec();
  const JValue& plan = j.at("plan");
  for (const JValue& s : plan.at("steps").arr) {
    PlanStep st;
    st.a = s.at("a").as_int();
    st.b = s.at("b").as_int();
    st.out = s.at("out").as_int();
    st.edges = s.at("edges").as_int_vec();
    st.legs_a = s.at("legs_a").as_int_vec();
    st.legs_b = s.at("legs_b").as_int_vec();
    st.rank_a = s.at("rank_a").as_int();
    st.rank_b = s.at("rank_b").as_int();
    st.result_rank = s.at("result_rank").as_int();
    st.work_rank = s.at("work_rank").as_int();
    p.steps.push_back(std::move(st));
  }
  p.scalars = plan.at("scalars").as_int_vec();
  p.peak_rank = plan.at("peak_rank").as_int();
  p.cost_estimate = plan.at("cost_estimate").as_double();
  p.max_rank = j.at("max_rank").as_int();
  check_closed(p);
  return p;
}

// check_closed (tensor_network.cpp:128-153)
void check_closed(const Payload& p) {
  std::map<std::pair<int, int>, int> uses;
  for (const NetEdge& e : p.edges) {
    ++uses[{e.u, e.leg_u}];
    ++uses[{e.v, e.leg_v}];
  }
  std::map<int, int> rank;
  for (const Vertex& v : p.vertices) rank[v.id] = v.rank;
  for (const Vertex& v : p.vertices) {
    for (int leg = 0; leg < v.rank; ++leg) {
      auto it = uses.find({v.id, leg});
      int count = it == uses.end() ? 0 : it->second;
      if (count != 1)
        throw std::invalid_argument("network not closed: vertex " + std::to_string(v.id) + " leg " +
                                    std::to_string(leg) + " used " + std::to_string(count) +
                                    " times");
    }
  }
  for (const auto& kv : uses) {
    auto it = rank.find(kv.first.first);
    if (it == rank.end())
      throw std::invalid_argument("edge references unknown vertex " + std::to_string(kv.first.first));
    if (kv.first.second < 0 || kv.first.second >= it->second)
      throw std::invalid_argument("edge references leg out of range on vertex " +
                                  std::to_string(kv.first.first));
  }
}

// apply_cut argument checks (cutting.cpp:67-92) and subnetwork_count (:33-39).
void check_cut(const Payload& p) {
  const int m = static_cast<int>(p.cut.size());
  if (m > 31) throw std::invalid_argument("cut size " + std::to_string(m) + " outside [0, 31]");
  std::vector<int> sorted = p.cut;
  std::sort(sorted.begin(), sorted.end());
  if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
    throw std::invalid_argument("cut set repeats an edge id");
  if (sorted != p.cut) throw std::invalid_argument("cut set must be sorted ascending");
  std::set<int> ids;
  for (const NetEdge& e : p.edges) ids.insert(e.id);
  for (int c : p.cut)
    if (!ids.count(c)) throw std::invalid_argument("cut references unknown edge " + std::to_string(c));
}

// check_rank_guard (contraction.cpp:280-286)
void check_rank_guard(const Payload& p) {
  for (const PlanStep& s : p.steps)
    if (s.result_rank > p.max_rank) throw RankGuard(s.result_rank, p.max_rank);
}

// ---------------------------------------------------------------------------
// Ket factorisation. Density index bit layout per leg i of a rank-r tensor:
// ket bit at position 2(r-1-i)+1, bra bit at 2(r-1-i) (digit a = 2*ket + bra,
// tensor_network.cpp:25-32).
// ---------------------------------------------------------------------------
std::vector<cxd> ket_factor(const std::vector<cxd>& t, int rank) {
  const size_t n = size_t{1} << rank;
  if (rank == 0) return t;
  auto didx = [rank](size_t k, size_t b) {
    size_t idx = 0;
    for (int i = 0; i < rank; ++i) {
      size_t kb = (k >> (rank - 1 - i)) & 1, bb = (b >> (rank - 1 - i)) & 1;
      idx |= ((kb << 1) | bb) << (2 * (rank - 1 - i));
    }
    return idx;
  };
  size_t jstar = 0;
  double best = -1;
  double vmax = 0;
  for (size_t j = 0; j < n; ++j) {
    const cxd& d = t[didx(j, j)];
    double mag = std::hypot(d.re, d.im);
    if (mag > best) {
      best = mag;
      jstar = j;
    }
  }
  for (const cxd& v : t) vmax = std::max(vmax, std::hypot(v.re, v.im));
  std::vector<cxd> K(n, cxd{0, 0});
  if (best <= 0) {
    if (vmax > 0) throw std::invalid_argument("tensor does not factorise as K (x) conj(K)");
    return K;
  }
  const cxd pivot = t[didx(jstar, jstar)];
  const double norm = std::sqrt(pivot.re);
  if (!(pivot.re > 0)) throw std::invalid_argument("tensor does not factorise as K (x) conj(K)");
  for (size_t i = 0; i < n; ++i) {
    const cxd v = t[didx(i, jstar)];  // K[i] conj(K[j*]) with K[j*] = norm real
    K[i] = cxd{v.re / norm, v.im / norm};
  }
  double err = 0;
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j) {
      const cxd v = t[didx(i, j)];
      const double re = K[i].re * K[j].re + K[i].im * K[j].im;
      const double im = K[i].im * K[j].re - K[i].re * K[j].im;
      err = std::max(err, std::hypot(v.re - re, v.im - im));
    }
  if (err > 1e-12 * std::max(1.0, vmax))
    throw std::invalid_argument("tensor does not factorise as K (x) conj(K) (pure inputs, unitary "
                                "gates and projector measurements are required for the ket view)");
  return K;
}

// ---------------------------------------------------------------------------
// Program builder
// ---------------------------------------------------------------------------
namespace {

struct TensorInfo {
  std::vector<int> bits;  // storage order, MSB first
  int64_t off = -1;       // element offset once placed
  int64_t start = 0, end = 0;  // lifetime (step indices, inclusive) for arena tensors
  bool is_static = false;
  bool per_pass = false;  // depends on the pass's fixed (unbatched) slice bits
  int64_t size() const { return int64_t{1} << bits.size(); }
  int pos(int bit) const {
    for (size_t i = 0; i < bits.size(); ++i)
      if (bits[i] == bit) return static_cast<int>(bits.size() - 1 - i);
    return -1;
  }
};

// Smallest big operand (log2 elements) that gets its own gate launch; smaller gate-shaped
// steps run as tiles inside the dataflow groups (latency over bandwidth). Override with
// QCG_GATE_MIN_BITS for experiments.
// Planner tuning knobs (measurement only; defaults are the shipped values).
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

int gate_min_bits() {
  static const int v = [] {
    const char* e = std::getenv("QCG_GATE_MIN_BITS");
    return e ? std::atoi(e) : 14;
  }();
  return v;
}

// Threads (log2) a gate pair with few columns is spread to through R_hi (QCG_PAIR_RHI_TARGET).
int qcg_pair_rhi_target() {
  static const int v = [] {
    const char* e = std::getenv("QCG_PAIR_RHI_TARGET");
    return e ? std::atoi(e) : 16;
  }();
  return v;
}

// Expanding steps (small inputs) qualify for a gate launch by their output from 2^this
// elements (QCG_GATE_OUT_BITS; default = the gate threshold itself).
int qcg_gate_out_bits() {
  static const int v = [] {
    const char* e = std::getenv("QCG_GATE_OUT_BITS");
    return e ? std::atoi(e) : 14;
  }();
  return v;
}

Runs make_runs(std::vector<std::pair<int, int>> pairs) {
  std::sort(pairs.begin(), pairs.end());
  Runs r{};
  r.n = 0;
  for (const auto& pr : pairs) {
    if (r.n > 0) {
      int i = r.n - 1;
      if (r.src[i] + r.len[i] == pr.first && r.dst[i] + r.len[i] == pr.second) {
        ++r.len[i];
        continue;
      }
    }
    if (r.n >= kMaxRuns) throw std::runtime_error("bit map needs too many runs");
    r.src[r.n] = static_cast<uint8_t>(pr.first);
    r.dst[r.n] = static_cast<uint8_t>(pr.second);
    r.len[r.n] = 1;
    ++r.n;
  }
  return r;
}

constexpr int64_t kAlign = 32;  // elements (512 B)

// Largest value a bit-scatter map can produce (all source bits set).
uint64_t runs_max(const Runs& r) {
  uint64_t y = 0;
  for (int i = 0; i < r.n; ++i) y |= ((uint64_t{1} << r.len[i]) - 1) << r.dst[i];
  return y;
}

// Memory-safety validation of every descriptor (compute-sanitizer is not available on
// the GPU pool): each index map, at its largest value, must stay inside its tensor.
void check_extent(uint64_t max_index, int64_t size, const char* what) {
  if (max_index >= static_cast<uint64_t>(size))
    throw std::logic_error(std::string("descriptor out of bounds: ") + what);
}

uint64_t eval_runs(const Runs& r, uint64_t x) {
  uint64_t y = 0;
  for (int i = 0; i < r.n; ++i) y |= ((x >> r.src[i]) & ((uint64_t{1} << r.len[i]) - 1)) << r.dst[i];
  return y;
}

int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Greedy offset assignment, largest first. Two tensors may share memory only when
// the last reader of one is ordered before the producer of the other (`before`, over
// launch groups: -1 = k_prep, groups in between, max+1 = the final stage) -- with
// concurrent launches a lower group index alone does not order them.
template <class Before>
int64_t place(std::vector<TensorInfo*>& ts, int64_t base, const Before& before) {
  std::vector<TensorInfo*> order = ts;
  std::stable_sort(order.begin(), order.end(),
                   [](const TensorInfo* a, const TensorInfo* b) { return a->size() > b->size(); });
  std::vector<TensorInfo*> placed;
  int64_t top = base;
  for (TensorInfo* t : order) {
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (TensorInfo* q : placed)
      if (!(before(q->end, t->start) || before(t->end, q->start)))
        busy.emplace_back(q->off, q->off + align_up(q->size()));
    std::sort(busy.begin(), busy.end());
    int64_t at = base;
    for (const auto& iv : busy) {
      if (at + t->size() <= iv.first) break;
      at = std::max(at, iv.second);
    }
    t->off = at;
    top = std::max(top, at + align_up(t->size()));
    placed.push_back(t);
  }
  return top;
}

}  // namespace

// Payloads batched as amplitudes of one program (bitstrings, angle sets, ...) must be the same
// network, cut and plan; only tensor values may differ.
void check_same_structure(const Payload& a, const Payload& b) {
  auto bad = [](const std::string& what) {
    throw std::invalid_argument("batched payloads differ in " + what + " (only tensor values may differ)");
  };
  if (a.vertices.size() != b.vertices.size()) bad("vertices");
  for (size_t i = 0; i < a.vertices.size(); ++i)
    if (a.vertices[i].id != b.vertices[i].id || a.vertices[i].rank != b.vertices[i].rank) bad("vertices");
  if (a.edges.size() != b.edges.size()) bad("edges");
  for (size_t i = 0; i < a.edges.size(); ++i) {
    const NetEdge &x = a.edges[i], &y = b.edges[i];
    if (x.id != y.id || x.u != y.u || x.leg_u != y.leg_u || x.v != y.v || x.leg_v != y.leg_v) bad("edges");
  }
  if (a.cut != b.cut) bad("cut");
  if (a.steps.size() != b.steps.size() || a.scalars != b.scalars || a.max_rank != b.max_rank) bad("plan");
  for (size_t i = 0; i < a.steps.size(); ++i) {
    const PlanStep &x = a.steps[i], &y = b.steps[i];
    if (x.a != y.a || x.b != y.b || x.out != y.out || x.edges != y.edges || x.legs_a != y.legs_a ||
        x.legs_b != y.legs_b)
      bad("plan");
  }
}

Program build_program(const Payload& p, Mode mode, int batch_bits) {
  return build_program(std::vector<const Payload*>{&p}, mode, batch_bits);
}

Program build_program(const std::vector<const Payload*>& amps, Mode mode, int batch_bits) {
  if (amps.empty()) throw std::invalid_argument("no payload");
  const Payload& p = *amps[0];
  for (size_t i = 1; i < amps.size(); ++i) check_same_structure(p, *amps[i]);
  Program prog;
  prog.mode = mode;
  // amplitude bits: the batch index of the payloads, extra batch bits of every tensor that
  // descends from a vertex whose values differ between payloads (bit ids -1 - i, i < nA)
  prog.n_amps = static_cast<int>(amps.size());
  while ((1 << prog.amp_bits) < prog.n_amps) ++prog.amp_bits;
  const int nA = prog.amp_bits;
  prog.M = static_cast<int>(p.cut.size());
  prog.bpc = mode == kKet ? 1 : 2;
  prog.id_bits = prog.M * prog.bpc;
  if (batch_bits < 0 || batch_bits > prog.id_bits) throw std::invalid_argument("bad batch bits");
  prog.b = batch_bits;
  prog.passes = uint64_t{1} << (prog.id_bits - prog.b);
  const int M = prog.M;
  const int D = mode == kKet ? 2 : 4;

  std::unordered_map<int, const NetEdge*> edge_by_id;
  for (const NetEdge& e : p.edges) edge_by_id[e.id] = &e;
  std::unordered_map<int, int> cut_index;  // edge id -> i
  for (int i = 0; i < M; ++i) cut_index[p.cut[i]] = i;

  // Bit ids: ket bit of edge e = 2e, bra bit = 2e+1 (density only).
  // Slice-id position of a cut bit (cutting.cpp:41-52: digit i is the MSB-first
  // i-th digit; digit = 2*ket + bra in the density view).
  auto slice_pos = [&](int bit) -> int {
    if (bit < 0) return -1;  // amplitude bit
    int e = bit >> 1;
    auto it = cut_index.find(e);
    if (it == cut_index.end()) return -1;
    int i = it->second;
    if (mode == kKet) return M - 1 - i;
    return 2 * (M - 1 - i) + ((bit & 1) ? 0 : 1);
  };
  auto edge_bits = [&](int e) {
    std::vector<int> v{2 * e};
    if (mode == kDensity) v.push_back(2 * e + 1);
    return v;
  };

  // Per-vertex leg lists (edge ids) of the uncut network.
  std::map<int, const Vertex*> vert;
  for (const Vertex& v : p.vertices) vert[v.id] = &v;
  std::map<int, std::vector<int>> legs;
  for (const Vertex& v : p.vertices) legs[v.id].assign(v.rank, -1);
  for (const NetEdge& e : p.edges) {
    legs[e.u][e.leg_u] = e.id;
    legs[e.v][e.leg_v] = e.id;
  }

  std::vector<std::unique_ptr<TensorInfo>> pool;
  auto make = [&]() {
    pool.push_back(std::make_unique<TensorInfo>());
    return pool.back().get();
  };

  // ---- initial tensors (static region) and per-pass slicing (prep) ----
  std::map<int, TensorInfo*> tens;             // live root -> tensor
  std::map<int, std::vector<int>> ref_legs;    // live root -> reference leg list (cut network)
  std::vector<TensorInfo*> statics, arena_ts;
  struct PrepPlan {
    TensorInfo* src;
    TensorInfo* dst;
  };
  std::vector<PrepPlan> preps;
  std::vector<char> differs(p.vertices.size(), 0);
  for (size_t i = 0; i < p.vertices.size(); ++i)
    for (size_t a = 1; a < amps.size(); ++a) {
      const std::vector<cxd>& x = p.vertices[i].data;
      const std::vector<cxd>& y = amps[a]->vertices[i].data;
      for (size_t k = 0; k < x.size() && !differs[i]; ++k) differs[i] = x[k].re != y[k].re || x[k].im != y[k].im;
    }
  for (size_t vi = 0; vi < p.vertices.size(); ++vi) {
    const Vertex& v = p.vertices[vi];
    TensorInfo* full = make();
    full->is_static = true;
    if (differs[vi])
      for (int i = nA - 1; i >= 0; --i) full->bits.push_back(-1 - i);  // amplitude index, most significant
    std::vector<int> rl;
    bool fixed_any = false;
    for (int e : legs[v.id]) {
      for (int bit : edge_bits(e)) {
        full->bits.push_back(bit);
        int sp = slice_pos(bit);
        if (sp >= prog.b) fixed_any = true;
      }
      if (!cut_index.count(e)) rl.push_back(e);
    }
    statics.push_back(full);
    ref_legs[v.id] = rl;
    if (fixed_any) {
      TensorInfo* dst = make();
      for (int bit : full->bits) {
        int sp = slice_pos(bit);
        if (sp < 0 || sp < prog.b) dst->bits.push_back(bit);
      }
      dst->start = 0;
      dst->end = 0;
      dst->per_pass = true;
      arena_ts.push_back(dst);
      preps.push_back({full, dst});
      tens[v.id] = dst;
    } else {
      tens[v.id] = full;
    }
  }
  // static region layout + data
  {
    int64_t at = 0;
    for (size_t i = 0; i < statics.size(); ++i) {
      statics[i]->off = at;
      at += align_up(statics[i]->size());
    }
    prog.static_elems = at;
    prog.static_data.assign(static_cast<size_t>(at), cxd{0, 0});
    for (size_t i = 0; i < p.vertices.size(); ++i) {
      const int na = differs[i] ? (1 << nA) : 1;
      for (int a = 0; a < na; ++a) {  // amplitude-major; padded amplitudes repeat the last payload
        const Vertex& v = amps[std::min<size_t>(static_cast<size_t>(a), amps.size() - 1)]->vertices[i];
        std::vector<cxd> d = mode == kKet ? ket_factor(v.data, v.rank) : v.data;
        std::copy(d.begin(), d.end(), prog.static_data.begin() + statics[i]->off + static_cast<int64_t>(a) * static_cast<int64_t>(d.size()));
      }
    }
  }

  // slice dependence (for §8(d) accounting): does a root carry any cut variable?
  std::map<int, bool> dep;
  for (const Vertex& v : p.vertices) {
    bool d = false;
    for (int e : legs[v.id]) d = d || cut_index.count(e);
    dep[v.id] = d;
  }

  // ---- plan steps (execute_plan, contraction.cpp:288-319) ----
  struct KPlan {
    TensorInfo *A, *B, *C;
    std::vector<int> S, T;  // summed bits; C-tile bits (tile kind)
    TensorInfo *G, *X;      // gate kind: small (staged) and big (streamed) operand
    int plan_step;
    int kind;
    bool dep;
  };
  std::vector<KPlan> kplans;
  std::vector<TensorInfo*> factor_ts;
  const int nsteps = static_cast<int>(p.steps.size());
  // Dense contraction (contraction.cpp:104-115 with all three extents large): >= 8 summed
  // index values, both free sides >= 8 wide, >= 2^20 complex MACs per pass -- everything
  // else is gate-shaped or small and stays on the streaming / dataflow kernels.
  auto gemm_shaped = [&](TensorInfo* A, TensorInfo* B, const std::set<int>& sbits) {
    const bool dense_off = env_int("QCG_NO_GEMM", 0) != 0;  // A/B knob: dense steps stay dataflow tiles
    std::set<int> ab(A->bits.begin(), A->bits.end()), bb(B->bits.begin(), B->bits.end());
    int fa = 0, fb = 0, g = 0;
    for (int x : A->bits)
      if (!sbits.count(x)) ++(bb.count(x) ? g : fa);
    for (int x : B->bits)
      if (!sbits.count(x) && !ab.count(x)) ++fb;
    const int k = static_cast<int>(sbits.size());
    // index tables of <= 2^20 entries each, <= 2^30 result tiles (64 x 64) per launch
    if (fa > 20 || fb > 20 || k > 20 || g > 20 || g + std::max(0, fa - 6) + std::max(0, fb - 6) > 30) return false;
    // (a sum over >= 2^9 index values does not fit the dataflow kernel's shared-memory tiles
    // either way: the GEMM's k loop takes it whatever the free sides are)
    return (!dense_off && k >= 3 && fa >= 3 && fb >= 3 && fa + fb + k + g >= env_int("QCG_GEMM_MIN_BITS", 20)) ||
           k >= 9;
  };
  for (int t = 0; t < nsteps; ++t) {
    const PlanStep& st = p.steps[t];
    auto ia = tens.find(st.a), ib = tens.find(st.b);
    if (ia == tens.end() || ib == tens.end() || st.a == st.b)
      throw std::invalid_argument("plan references a missing vertex");
    std::vector<int>& la = ref_legs[st.a];
    std::vector<int>& lb = ref_legs[st.b];
    // contract_pair's leg-list validation (contraction.cpp:40-56, 74-84)
    if (st.legs_a.empty() || st.legs_b.empty())
      throw std::invalid_argument("contract_pair needs at least one shared leg");
    if (st.legs_a.size() != st.legs_b.size())
      throw std::invalid_argument("shared leg lists differ in length: " + std::to_string(st.legs_a.size()) +
                                  " vs " + std::to_string(st.legs_b.size()));
    auto check = [](const std::vector<int>& ls, size_t rank, const char* side) {
      std::vector<char> seen(rank, 0);
      for (int l : ls) {
        if (l < 0 || static_cast<size_t>(l) >= rank)
          throw std::invalid_argument("leg " + std::to_string(l) + " out of range for rank-" +
                                      std::to_string(rank) + " tensor (" + side + ")");
        if (seen[l]) throw std::invalid_argument("leg " + std::to_string(l) + " repeated (" + side + ")");
        seen[l] = 1;
      }
    };
    check(st.legs_a, la.size(), "left");
    check(st.legs_b, lb.size(), "right");
    const int k = static_cast<int>(st.legs_a.size());
    std::vector<int> shared_edges;
    for (int i = 0; i < k; ++i) {
      int ea = la[st.legs_a[i]], eb = lb[st.legs_b[i]];
      if (ea != eb)
        throw std::invalid_argument("plan step " + std::to_string(t) + " pairs different edges " +
                                    std::to_string(ea) + " and " + std::to_string(eb));
      shared_edges.push_back(ea);
    }
    const int ra = static_cast<int>(la.size()), rbk = static_cast<int>(lb.size());
    if (st.rank_a != ra || st.rank_b != rbk || st.result_rank != ra + rbk - 2 * k ||
        st.work_rank != ra + rbk - k)
      throw std::invalid_argument("plan step " + std::to_string(t) + " ranks disagree with the network");
    prog.ra.push_back(ra);
    prog.rb.push_back(rbk);
    prog.rk.push_back(k);
    prog.rr.push_back(ra + rbk - 2 * k);
    // reference result legs: free(a) in order ++ free(b) in order
    std::set<int> sh(shared_edges.begin(), shared_edges.end());
    std::vector<int> lc;
    for (int e : la)
      if (!sh.count(e)) lc.push_back(e);
    for (int e : lb)
      if (!sh.count(e)) lc.push_back(e);

    TensorInfo* A = ia->second;
    TensorInfo* B = ib->second;
    std::set<int> sbits;
    for (int e : shared_edges)
      for (int bit : edge_bits(e)) sbits.insert(bit);
    std::set<int> abits(A->bits.begin(), A->bits.end()), bbits(B->bits.begin(), B->bits.end());
    std::vector<int> cset;  // H ∪ Fa ∪ Fb
    for (int bit : A->bits)
      if (!sbits.count(bit)) cset.push_back(bit);
    for (int bit : B->bits)
      if (!sbits.count(bit) && !abits.count(bit)) cset.push_back(bit);
    for (int bit : sbits)
      if (!abits.count(bit) || !bbits.count(bit)) throw std::logic_error("shared bit missing");
    for (int bit : A->bits)
      if (bbits.count(bit) && !sbits.count(bit) && slice_pos(bit) < 0 && bit >= 0)
        throw std::logic_error("non-cut bit shared but not summed");

    const int nS = static_cast<int>(sbits.size());
    TensorInfo* big = A->size() >= B->size() ? A : B;
    TensorInfo* small = big == A ? B : A;
    TensorInfo* C = make();
    C->per_pass = A->per_pass || B->per_pass;
    KPlan kp{};
    kp.A = A;
    kp.B = B;
    kp.C = C;
    kp.plan_step = t;
    // S enumerated in the small operand's storage order (low to high)
    for (int i = static_cast<int>(small->bits.size()) - 1; i >= 0; --i)
      if (sbits.count(small->bits[i])) kp.S.push_back(small->bits[i]);

    // gate kind: the small operand is staged in shared memory (split along its
    // highest free bits when larger than 2^12 elements, then the big operand is
    // re-read once per split and must be L2-resident)
    // (batch bits it shares with the big operand go to the grid first: each value owns
    // a disjoint column subset, nothing is re-read)
    int small_free = 0, small_h = 0;
    for (int x : small->bits)
      if (!sbits.count(x)) ++((small == A ? bbits : abits).count(x) ? small_h : small_free);
    const int split = std::max(0, static_cast<int>(small->bits.size()) - 12);
    const int fhi = split - std::min(split, small_h);
    // expanding steps (small inputs, large output) are gate-shaped too: the output size
    // counts toward the threshold (one thread per column writes all 2^nF outputs)
    int c_bits = 0;
    {
      std::set<int> u(A->bits.begin(), A->bits.end());
      u.insert(B->bits.begin(), B->bits.end());
      c_bits = static_cast<int>(u.size()) - nS;
    }
    const int gate_bits = std::max(static_cast<int>(big->bits.size()), c_bits >= qcg_gate_out_bits() ? c_bits : 0);
    const bool gate = nS <= 4 && gate_bits >= gate_min_bits() && fhi <= small_free &&
                      split <= 15 &&
                      (fhi == 0 || big->size() * 16 <= (int64_t{64} << 20));
    if (gate) {
      // ---- gate kind: C = [G free bits, G order] ++ [X non-summed bits, X order] ----
      kp.kind = kGate;
      kp.G = small;
      kp.X = big;
      // free bits of G: neither summed nor shared with X
      std::set<int> xbits(big->bits.begin(), big->bits.end());
      for (int x : small->bits)
        if (!sbits.count(x) && !xbits.count(x)) C->bits.push_back(x);
      for (int x : big->bits)
        if (!sbits.count(x)) C->bits.push_back(x);
    } else if (gemm_shaped(A, B, sbits)) {
      // ---- dense step: batched complex GEMM on the FP64 tensor pipe ----
      // C = [batch bits (A order)] ++ [A free bits, A order] ++ [B free bits, B order]
      kp.kind = kGemm;
      for (int x : A->bits)
        if (!sbits.count(x) && bbits.count(x)) C->bits.push_back(x);
      for (int x : A->bits)
        if (!sbits.count(x) && !bbits.count(x)) C->bits.push_back(x);
      for (int x : B->bits)
        if (!sbits.count(x) && !abits.count(x)) C->bits.push_back(x);
    } else {
      // ---- tile kind ----
      kp.kind = kTile;
      const int LIM = std::max(10, nS + 3);
      const int TCMAX = 8;
      std::set<int> T;
      auto tile_counts = [&](int extra) {
        int na = nS, nb = nS;
        for (int x : T) {
          na += abits.count(x) ? 1 : 0;
          nb += bbits.count(x) ? 1 : 0;
        }
        na += abits.count(extra) ? 1 : 0;
        nb += bbits.count(extra) ? 1 : 0;
        return std::make_pair(na, nb);
      };
      auto try_add = [&](int x, int tcmax) {
        if (T.count(x) || sbits.count(x)) return;
        if (static_cast<int>(T.size()) + 1 > tcmax) return;
        auto c = tile_counts(x);
        if (c.first > LIM || c.second > LIM) return;
        T.insert(x);
      };
      // must: the lowest 3 storage bits of each operand (coalescing)
      for (TensorInfo* X : {big, small}) {
        int n = static_cast<int>(X->bits.size());
        for (int q = 0; q < std::min(3, n); ++q) try_add(X->bits[n - 1 - q], TCMAX + 2);
      }
      // then the small operand's free bits (the big operand is then read once),
      // then low bits of the big operand
      for (int i = static_cast<int>(small->bits.size()) - 1; i >= 0; --i)
        if (!(small == A ? bbits : abits).count(small->bits[i])) try_add(small->bits[i], TCMAX);
      for (int i = static_cast<int>(big->bits.size()) - 1; i >= 0; --i) try_add(big->bits[i], TCMAX);
      for (int i = static_cast<int>(small->bits.size()) - 1; i >= 0; --i) try_add(small->bits[i], TCMAX);
      // C layout: grid bits on top, tile bits at the bottom
      auto key = [&](int x) {
        int pb = big->pos(x);
        if (pb >= 0) return pb;
        return 64 + small->pos(x);
      };
      std::vector<int> grid, tile;
      for (int x : cset) (T.count(x) ? tile : grid).push_back(x);
      std::sort(grid.begin(), grid.end(), [&](int a, int b) { return key(a) > key(b); });
      std::sort(tile.begin(), tile.end(), [&](int a, int b) { return key(a) > key(b); });
      C->bits = grid;
      C->bits.insert(C->bits.end(), tile.begin(), tile.end());
      kp.T = tile;
    }
    if (C->bits.size() != cset.size()) throw std::logic_error("result layout lost a bit");
    // element counts past 2^56 would overflow the int64 arena offsets (no device holds them)
    if (C->bits.size() > 56) throw WorkspaceTooLarge(static_cast<int>(C->bits.size()));
    arena_ts.push_back(C);
    kp.dep = dep[st.a] || dep[st.b];
    kplans.push_back(kp);
    dep[st.a] = kp.dep;

    tens.erase(st.b);
    ref_legs.erase(st.b);
    if (lc.empty()) {
      // rank-0 result: acc *= value (contraction.cpp:304-306)
      for (int x : C->bits)
        if (x >= 0 && (slice_pos(x) < 0 || slice_pos(x) >= prog.b))
          throw std::logic_error("scalar carries a non-batched bit");
      factor_ts.push_back(C);
      tens.erase(st.a);
      ref_legs.erase(st.a);
    } else {
      tens[st.a] = C;
      ref_legs[st.a] = lc;
    }
  }
  // leftovers (contraction.cpp:311-317), ascending vertex id
  for (auto& kv : tens) {
    if (!ref_legs[kv.first].empty())
      throw std::invalid_argument("plan does not reduce vertex " + std::to_string(kv.first) + " to a scalar");
    TensorInfo* X = kv.second;
    for (int x : X->bits)
      if (x >= 0 && (slice_pos(x) < 0 || slice_pos(x) >= prog.b))
        throw std::logic_error("scalar carries a non-batched bit");
    factor_ts.push_back(X);
  }
  // ---- pass 2: fuse chains of gate steps (state-vector gate fusion) ----
  std::map<TensorInfo*, int> producer;  // tensor -> kplan index
  for (size_t i = 0; i < kplans.size(); ++i) producer[kplans[i].C] = static_cast<int>(i);
  struct PairPlan {
    std::vector<int> P, Q, R, cols, F2, S1, S2;  // bit lists, ascending positions
    int nRlo = 0, nRmid = 0, nRhi = 0, nHhi = 0;
    std::vector<int> H;  // H_hi bits (cols' bits G1 carries, on the grid), hhi index order
  };
  struct Seg {
    std::vector<int> steps;
    bool pair = false;  // exactly two steps fused at register level (k_pair)
    PairPlan pp;
    // stage tiles (bit lists in tile-index order, low to high)
    std::vector<std::vector<int>> tiles;  // tiles[0] = T0, tiles[j] = T_j
    std::vector<int> outer;               // O bits, C0 position ascending
  };
#ifndef QCG_CHAIN_LIM
#define QCG_CHAIN_LIM 11
#endif
  const int kChainLim = QCG_CHAIN_LIM;  // max tile bits (32 KB buffer)
  const int kChainMinOut = 8;        // every stage emits >= 256 outputs per tile
  const int64_t kChainGElems = 2048;  // all G_j staged in shared memory
  // Tile bit lists for a candidate chain; empty result = infeasible.
  auto plan_chain = [&](const std::vector<int>& steps, Seg& out) -> bool {
    if (steps.size() > static_cast<size_t>(kMaxChain)) return false;
    TensorInfo* C0 = kplans[steps.front()].X;
    TensorInfo* Cm = kplans[steps.back()].C;
    std::set<int> c0(C0->bits.begin(), C0->bits.end());
    std::set<int> need;
    int64_t gel = 0;
    for (int i : steps) {
      for (int x : kplans[i].S)
        if (c0.count(x)) need.insert(x);
      gel += kplans[i].G->size();
      if (kplans[i].S.size() > 4) return false;
    }
    if (gel > kChainGElems) return false;
    const int n0 = static_cast<int>(C0->bits.size());
    for (int q = 0; q < std::min(3, n0); ++q) need.insert(C0->bits[n0 - 1 - q]);
    const int nm = static_cast<int>(Cm->bits.size());
    for (int q = 0; q < std::min(3, nm); ++q)
      if (c0.count(Cm->bits[nm - 1 - q])) need.insert(Cm->bits[nm - 1 - q]);
    // stage tile sizes for a given T0: |T_j| = |T0| - sum_{i<=j} |S_i ∩ C0| ... computed exactly below
    int tmin = 0;  // smallest stage output of the last simulation
    auto simulate = [&](const std::set<int>& t0set, std::vector<std::vector<int>>& tiles_out,
                        std::vector<int>& outer_out) -> int {
      tiles_out.clear();
      outer_out.clear();
      std::vector<int> t0;
      for (int q = 0; q < n0; ++q) {  // C0 position ascending
        const int x = C0->bits[n0 - 1 - q];
        (t0set.count(x) ? t0 : outer_out).push_back(x);
      }
      tiles_out.push_back(t0);
      int tmax = static_cast<int>(t0.size());
      tmin = 1 << 30;
      std::vector<int> cur = t0;
      for (size_t j = 0; j < steps.size(); ++j) {
        const KPlan& kp = kplans[steps[j]];
        std::set<int> sj(kp.S.begin(), kp.S.end());
        std::set<int> curset(cur.begin(), cur.end());
        for (int x : kp.S)
          if (!curset.count(x)) return 1 << 30;
        std::vector<int> nxt;
        for (int x : cur)
          if (!sj.count(x)) nxt.push_back(x);
        std::set<int> state(kp.X->bits.begin(), kp.X->bits.end());
        for (int q = 0; q < static_cast<int>(kp.G->bits.size()); ++q) {
          const int x = kp.G->bits[kp.G->bits.size() - 1 - q];
          if (!sj.count(x) && !state.count(x)) nxt.push_back(x);
        }
        if (j + 1 == steps.size())
          for (int x : nxt)
            if (Cm->pos(x) < 0) return 1 << 30;
        tmax = std::max(tmax, static_cast<int>(nxt.size()));
        tmin = std::min(tmin, static_cast<int>(nxt.size()));
        tiles_out.push_back(nxt);
        cur = nxt;
      }
      return tmax;
    };
    if (simulate(need, out.tiles, out.outer) > kChainLim) return false;
    // grow the tile with C0's lowest outer bits while every stage fits: bigger
    // contiguous loads, more columns per stage, fewer CTA iterations
    for (int q = 0; q < n0; ++q) {
      const int x = C0->bits[n0 - 1 - q];
      if (need.count(x)) continue;
      std::set<int> trial = need;
      trial.insert(x);
      std::vector<std::vector<int>> tt;
      std::vector<int> oo;
      if (simulate(trial, tt, oo) > kChainLim) break;
      need = trial;
      out.tiles = tt;
      out.outer = oo;
    }
    simulate(need, out.tiles, out.outer);
    // a stage with fewer outputs than a CTA has threads leaves warps idle at its
    // barrier; such chains are slower than the unfused gate kernels
    if (tmin < kChainMinOut) return false;
    out.steps = steps;
    return true;
  };
  // Register-level fusion of two gate steps (see PairDesc); worthwhile when the
  // intermediate is large (it never touches HBM) and the register tiles are small.
  auto plan_pair = [&](int p1, int i2, PairPlan& pp) -> bool {
    const KPlan& a = kplans[p1];
    const KPlan& b = kplans[i2];
    TensorInfo *G1 = a.G, *X1 = a.X, *C1 = a.C, *G2 = b.G, *C2 = b.C;
    if (C1->size() < (int64_t{1} << env_int("QCG_PAIR_MIN_C1_BITS", 19))) return false;
    if (a.S.size() > 4 || b.S.size() > 4 || G2->size() > 4096) return false;
    std::set<int> s1(a.S.begin(), a.S.end()), s2(b.S.begin(), b.S.end());
    pp = PairPlan{};
    pp.S1 = a.S;
    pp.S2 = b.S;
    std::set<int> g1set(G1->bits.begin(), G1->bits.end());
    for (int q = 0; q < static_cast<int>(X1->bits.size()); ++q) {
      const int x = X1->bits[X1->bits.size() - 1 - q];
      if (s1.count(x)) continue;
      (s2.count(x) ? pp.P : pp.cols).push_back(x);
    }
    const int nCol1 = static_cast<int>(X1->bits.size() - a.S.size());
    const int nF1 = static_cast<int>(C1->bits.size()) - nCol1;
    for (int q = 0; q < nF1; ++q) {  // F1, ascending position in C1 (= G1 order)
      const int x = C1->bits[nF1 - 1 - q];
      (s2.count(x) ? pp.Q : pp.R).push_back(x);
    }
    const int nCol = static_cast<int>(pp.cols.size()), nR = static_cast<int>(pp.R.size());
    for (int q = 0; q < nCol; ++q)
      if (C2->pos(pp.cols[q]) != q) return false;
    for (int q = 0; q < nR; ++q)
      if (C2->pos(pp.R[q]) != nCol + q) return false;
    const int nF2 = static_cast<int>(C2->bits.size()) - nCol - nR;
    for (int q = 0; q < nF2; ++q) pp.F2.push_back(C2->bits[nF2 - 1 - q]);
    const int xregs = (1 << pp.P.size()) * (1 << a.S.size());  // X values a thread holds (<= 16)
    const int acc_bits = xregs >= 16 ? 2 : 3;                   // accumulators: 4 or 8 (mirrors k_pair's NA)
    if (xregs > 16 || nF2 > acc_bits) return false;
    pp.nRlo = std::min(nR, acc_bits - nF2);
    // the expanded G1 tile (k_pair's shared layout) also spans the P bits G1 lacks;
    // R's top bits move to blockIdx.y until it fits with G2 (2 CTAs per SM)
    int hp = 0;
    for (int x : pp.P) hp += g1set.count(x) ? 1 : 0;
    int g1x_full = static_cast<int>(G1->bits.size() + pp.P.size()) - hp;
    // first cols' bits that G1 carries onto the grid (highest column positions first, never
    // the lowest 6: a warp's columns stay contiguous) -- free: disjoint column subsets,
    // each CTA stages its G1x sub-block only
    pp.H.clear();
    for (int q = nCol - 1; q >= 6; --q)
      if (g1set.count(pp.cols[q])) pp.H.push_back(pp.cols[q]);
    pp.nHhi = 0;
    while (pp.nHhi < static_cast<int>(pp.H.size()) && nCol - pp.nHhi > 11 &&
           (g1x_full - pp.nHhi > 12 || ((int64_t{1} << (g1x_full - pp.nHhi)) + G2->size()) * 16 > 96 * 1024))
      ++pp.nHhi;
    pp.H.resize(pp.nHhi);
    g1x_full -= pp.nHhi;
    pp.nRhi = std::max(0, g1x_full - 12);
    while (pp.nRhi < nR - pp.nRlo && ((int64_t{1} << (g1x_full - pp.nRhi)) + G2->size()) * 16 > 96 * 1024)
      ++pp.nRhi;
    if (pp.nRhi > nR - pp.nRlo || pp.nRhi + pp.nHhi > 15) return false;
    if (((int64_t{1} << (g1x_full - pp.nRhi)) + G2->size()) * 16 > 96 * 1024) return false;
    // few columns (an expanding first step): more R bits onto the grid until the pair
    // has enough threads to cover the GPU (X, re-read per R_hi value, is small then)
    while (nCol + pp.nRhi < qcg_pair_rhi_target() && pp.nRhi < nR - pp.nRlo && pp.nRhi + pp.nHhi < 15 &&
           X1->size() * 16 <= (int64_t{16} << 20))
      ++pp.nRhi;
    pp.nRmid = nR - pp.nRlo - pp.nRhi;
    if (pp.nRmid + pp.nRlo > 12) return false;
    if (pp.nRhi > 0 && X1->size() * 16 > (int64_t{64} << 20)) return false;
    return true;
  };
  auto est_gate = [&](int i) {
    const KPlan& k = kplans[i];
    return std::max(16.0 * static_cast<double>(k.X->size() + k.G->size() + k.C->size()) / 6.0e12,
                    1e-6 * env_int("QCG_EST_GATE_FLOOR_US", 3));
  };
  auto est_chain = [&](const std::vector<int>& st) {
    double b = 16.0 * static_cast<double>(kplans[st.front()].X->size() + kplans[st.back()].C->size());
    for (int i : st) b += 16.0 * static_cast<double>(kplans[i].G->size());
    return std::max(b / 1.7e12, 1e-6 * env_int("QCG_EST_CHAIN_FLOOR_US", 4));
  };
  std::vector<int> seg_of(kplans.size(), -1);
  std::vector<Seg> segs;
  for (size_t i = 0; i < kplans.size(); ++i) {
    if (kplans[i].kind != kGate) continue;
    auto pit = producer.find(kplans[i].X);
    const int p = pit == producer.end() ? -1 : pit->second;
    if (p >= 0 && kplans[p].kind == kGate && seg_of[p] >= 0 && segs[seg_of[p]].steps.size() == 1 &&
        segs[seg_of[p]].steps.back() == p) {
      PairPlan pp;
      if (plan_pair(p, static_cast<int>(i), pp)) {
        Seg& sg = segs[seg_of[p]];
        sg.steps.push_back(static_cast<int>(i));
        sg.pair = true;
        sg.pp = pp;
        seg_of[i] = seg_of[p];
        continue;
      }
    }
    if (p >= 0 && kplans[p].kind == kGate && seg_of[p] >= 0 && !segs[seg_of[p]].pair &&
        segs[seg_of[p]].steps.back() == p) {
      std::vector<int> cand = segs[seg_of[p]].steps;
      cand.push_back(static_cast<int>(i));
      Seg trial;
      // fuse only when the estimated chain time beats the segment so far plus a separate
      // gate launch (measured rates: gate kernels ~6.0 TB/s of their own traffic, the
      // shared-memory chain ~1.7 TB/s of its input + output; launch floors 3 / 4 us)
      const double prev_t = cand.size() == 2 ? est_gate(cand[0]) : est_chain(segs[seg_of[p]].steps);
      if (plan_chain(cand, trial) && est_chain(cand) <= prev_t + est_gate(static_cast<int>(i))) {
        segs[seg_of[p]] = trial;
        seg_of[i] = seg_of[p];
        continue;
      }
    }
    Seg one;
    one.steps = {static_cast<int>(i)};
    seg_of[i] = static_cast<int>(segs.size());
    segs.push_back(one);
  }
  std::set<TensorInfo*> fused_away;  // intermediates that live only in shared memory
  for (const Seg& sg : segs)
    for (size_t j = 0; j + 1 < sg.steps.size(); ++j) fused_away.insert(kplans[sg.steps[j]].C);

  // ---- pass 3: ops, dependency levels, lifetimes ----
  struct Op {
    int kind;                 // kTile, kGate, kChain
    int kplan = -1;           // kTile / kGate
    int seg = -1;             // kChain
    std::vector<TensorInfo*> in;
    TensorInfo* out = nullptr;
    int level = 0;
  };
  std::vector<Op> ops;
  std::vector<int> op_of_step(kplans.size(), -1);
  for (size_t i = 0; i < kplans.size(); ++i) {
    const KPlan& kp = kplans[i];
    if (kp.kind == kTile) {
      Op o;
      o.kind = kTile;
      o.kplan = static_cast<int>(i);
      o.in = {kp.A, kp.B};
      o.out = kp.C;
      op_of_step[i] = static_cast<int>(ops.size());
      ops.push_back(o);
      continue;
    }
    if (kp.kind == kGemm) {
      Op o;
      o.kind = kGemm;
      o.kplan = static_cast<int>(i);
      o.in = {kp.A, kp.B};
      o.out = kp.C;
      op_of_step[i] = static_cast<int>(ops.size());
      ops.push_back(o);
      continue;
    }
    const Seg& sg = segs[seg_of[i]];
    if (sg.steps.back() != static_cast<int>(i)) continue;  // emitted at the chain's last step
    Op o;
    if (sg.steps.size() == 1) {
      o.kind = kGate;
      o.kplan = static_cast<int>(i);
      o.in = {kp.G, kp.X};
    } else {
      o.kind = sg.pair ? kPair : kChain;
      o.seg = seg_of[i];
      o.in.push_back(kplans[sg.steps.front()].X);
      for (int st : sg.steps) o.in.push_back(kplans[st].G);
    }
    o.out = kp.C;
    for (int st : sg.steps) op_of_step[st] = static_cast<int>(ops.size());
    ops.push_back(o);
  }
  // Launch schedule: a topological order that packs every ready tile-kind op into
  // the current dataflow group (one persistent k_flow launch resolves their
  // dependencies on the device) and gives each gate / chain / pair op its own
  // launch. o.level = launch group; lifetimes are measured in groups.
  std::map<TensorInfo*, int> producer_op;
  for (size_t i = 0; i < ops.size(); ++i) producer_op[ops[i].out] = static_cast<int>(i);
  std::vector<std::vector<int>> op_deps(ops.size()), op_users(ops.size());
  for (size_t i = 0; i < ops.size(); ++i)
    for (TensorInfo* X : ops[i].in) {
      auto it = producer_op.find(X);
      if (it != producer_op.end()) {
        op_deps[i].push_back(it->second);
        op_users[it->second].push_back(static_cast<int>(i));
      }
    }
  std::vector<int> pending(ops.size());
  for (size_t i = 0; i < ops.size(); ++i) pending[i] = static_cast<int>(op_deps[i].size());
  std::vector<char> done_op(ops.size(), 0);
  std::set<int> ready;
  for (size_t i = 0; i < ops.size(); ++i)
    if (pending[i] == 0) ready.insert(static_cast<int>(i));
  std::vector<std::vector<int>> groups;  // launch groups in execution order
  auto finish = [&](int i) {
    done_op[i] = 1;
    for (int u : op_users[i])
      if (--pending[u] == 0) ready.insert(u);
  };
  // A dataflow group is a forest of independent subtrees (plans are trees) whose roots feed
  // different later launches. One launch for all of them makes every consumer wait for the
  // slowest subtree (measured on config 5: subtrees of 2-23 us in one k_forest launch, the
  // first big op on the critical path needs a 10 us one), so the group is split into up to
  // three launches by estimated subtree time; they run concurrently on the pass's streams.
  auto split_tile_group = [&](const std::vector<int>& grp) -> std::vector<std::vector<int>> {
    const char* env = std::getenv("QCG_FOREST_SPLIT");
    const bool enabled = env == nullptr || std::atoi(env) != 0;
    std::vector<std::vector<int>> out;
    if (!enabled || grp.size() < 8) {
      out.push_back(grp);
      return out;
    }
    std::set<int> mset(grp.begin(), grp.end());
    std::map<int, int> cons;
    for (int oi : grp)
      for (int u : op_users[oi])
        if (mset.count(u)) cons[oi] = u;
    // root, depth and MACs of every member's subtree (members listed producers first)
    std::map<int, int> root_of, depth;
    std::map<int, double> macs, depth_max;
    for (auto it = grp.rbegin(); it != grp.rend(); ++it) {
      const int oi = *it;
      auto c = cons.find(oi);
      root_of[oi] = c == cons.end() ? oi : root_of.at(c->second);
      depth[oi] = c == cons.end() ? 1 : depth.at(c->second) + 1;
      const KPlan& kp = kplans[ops[oi].kplan];
      macs[root_of[oi]] += std::ldexp(1.0, static_cast<int>(kp.C->bits.size() + kp.S.size()));
      depth_max[root_of[oi]] = std::max(depth_max[root_of[oi]], static_cast<double>(depth[oi]));
    }
    auto cls = [&](int root) {  // microseconds: operand staging + a barrier per level + the arithmetic
      const double est = 1.5 + 0.45 * depth_max.at(root) + macs.at(root) / 8000.0;
      return est <= 0.1 * env_int("QCG_FOREST_CLASS_A", 80) ? 0 : (est <= 0.1 * env_int("QCG_FOREST_CLASS_B", 110) ? 1 : 2);
    };
    std::vector<std::vector<int>> bins(3);
    for (int oi : grp) bins[static_cast<size_t>(cls(root_of.at(oi)))].push_back(oi);
    for (std::vector<int>& b : bins)
      if (!b.empty()) out.push_back(std::move(b));
    return out;
  };
  while (!ready.empty()) {
    std::vector<int> grp;
    for (bool grew = true; grew;) {
      grew = false;
      for (auto it = ready.begin(); it != ready.end();) {
        if (ops[*it].kind == kTile) {
          const int i = *it;
          it = ready.erase(it);
          grp.push_back(i);
          finish(i);
          grew = true;
        } else {
          ++it;
        }
      }
    }
    if (!grp.empty()) {
      for (std::vector<int>& g : split_tile_group(grp)) groups.push_back(std::move(g));
      continue;
    }
    const int i = *ready.begin();  // smallest plan position among ready fused/gate ops
    ready.erase(ready.begin());
    groups.push_back({i});
    finish(i);
  }
  for (size_t i = 0; i < ops.size(); ++i)
    if (!done_op[i]) throw std::logic_error("op schedule left an op behind");
  for (size_t g = 0; g < groups.size(); ++g)
    for (int i : groups[g]) ops[i].level = static_cast<int>(g);
  std::map<TensorInfo*, int> prod_level;  // producing launch group; initial tensors -1
  for (const Op& o : ops) prod_level[o.out] = o.level;
  const int max_level = static_cast<int>(groups.size()) - 1;
  for (TensorInfo* X : arena_ts) {
    auto it = prod_level.find(X);
    X->start = X->end = it == prod_level.end() ? -1 : it->second;  // prep outputs: -1
  }
  for (const Op& o : ops)
    for (TensorInfo* X : o.in)
      if (!X->is_static) X->end = std::max<int64_t>(X->end, o.level);
  for (TensorInfo* X : factor_ts)
    if (!X->is_static) X->end = max_level + 1;  // read by the final stage

  // ---- launch DAG: one launch per group; its dependencies are the groups producing
  // its inputs. The captured pass runs independent launches concurrently. ----
  const int n_groups = max_level + 1;
  prog.launch_deps.assign(n_groups, {});
  for (const Op& o : ops)
    for (TensorInfo* X : o.in) {
      auto it = prod_level.find(X);
      if (it == prod_level.end() || it->second == o.level) continue;
      auto& dv = prog.launch_deps[o.level];
      if (std::find(dv.begin(), dv.end(), it->second) == dv.end()) dv.push_back(it->second);
    }
  for (auto& dv : prog.launch_deps) std::sort(dv.begin(), dv.end());
  // reach[a][b]: launch b depends (transitively) on launch a
  std::vector<std::vector<char>> reach(n_groups, std::vector<char>(n_groups, 0));
  for (int b = 0; b < n_groups; ++b)
    for (int a : prog.launch_deps[b]) {
      reach[a][b] = 1;
      for (int z = 0; z < a; ++z)
        if (reach[z][a]) reach[z][b] = 1;
    }
  auto before = [&](int64_t a, int64_t b) {  // a's launch completes before b's starts
    if (a < 0) return b >= 0;
    if (a > max_level) return false;
    if (b > max_level) return true;
    return b >= 0 && reach[a][b] != 0;
  };
  // ---- memory plan ----
  {
    std::vector<TensorInfo*> live_ts;
    for (TensorInfo* X : arena_ts)
      if (!fused_away.count(X)) live_ts.push_back(X);
    prog.arena_elems = place(live_ts, prog.static_elems, before);
  }

  // ---- descriptors ----
  for (const PrepPlan& pp : preps) {
    PrepDesc d{};
    d.src = pp.src->off;
    d.dst = pp.dst->off;
    d.nbits = static_cast<int32_t>(pp.dst->bits.size());
    d.nfix = 0;
    std::vector<std::pair<int, int>> m;
    const int nd = static_cast<int>(pp.dst->bits.size());
    for (int i = 0; i < nd; ++i) m.emplace_back(nd - 1 - i, pp.src->pos(pp.dst->bits[i]));
    d.map = make_runs(m);
    for (int bit : pp.src->bits) {
      int sp = slice_pos(bit);
      if (sp >= prog.b) {
        if (d.nfix >= 16) throw std::runtime_error("too many fixed bits on one vertex");
        d.fix_pos[d.nfix] = static_cast<uint8_t>(sp);
        d.fix_stride[d.nfix] = int64_t{1} << pp.src->pos(bit);
        ++d.nfix;
      }
    }
    {
      uint64_t fixed_max = 0;
      for (int q = 0; q < d.nfix; ++q) fixed_max += static_cast<uint64_t>(d.fix_stride[q]);
      check_extent(runs_max(d.map) + fixed_max, pp.src->size(), "prep source");
    }
    prog.prep.push_back(d);
  }
  const double all_slices = std::ldexp(1.0, prog.id_bits);
  std::vector<StepDesc> tile_desc(kplans.size());
  std::vector<GateDesc> gate_desc(kplans.size());
  std::vector<Program::GemmOp> gemm_desc(kplans.size());
  prog.step_kind.resize(kplans.size());
  prog.step_level.resize(kplans.size());
  prog.step_fused.resize(kplans.size());
  for (size_t i = 0; i < kplans.size(); ++i) {
    const KPlan& kp = kplans[i];
    TensorInfo *A = kp.A, *B = kp.B, *C = kp.C;
    const bool fused = kp.kind == kGate && segs[seg_of[i]].steps.size() > 1;
    prog.step_kind[i] = fused ? (segs[seg_of[i]].pair ? kPair : kChain) : kp.kind;
    prog.step_level[i] = ops[op_of_step[i]].level;
    prog.step_fused[i] = fused ? 1 : 0;
    if (kp.kind == kGate && !fused) {
      GateDesc g{};
      TensorInfo *G = kp.G, *X = kp.X;
      g.offG = G->off;
      g.offX = X->off;
      g.offC = C->off;
      g.nS = static_cast<int32_t>(kp.S.size());
      g.nCol = static_cast<int32_t>(X->bits.size()) - g.nS;
      const int nFall = static_cast<int>(C->bits.size()) - g.nCol;
      // grid split of G: H_hi (batch bits shared with X, highest X positions first), then F_hi
      std::vector<int> hbits;
      for (int x : X->bits)  // X position descending
        if (G->pos(x) >= 0 && std::find(kp.S.begin(), kp.S.end(), x) == kp.S.end()) hbits.push_back(x);
      const int nGall = static_cast<int>(G->bits.size());
      const int split = std::max(0, nGall - 12);
      g.nHhi = std::min(split, static_cast<int>(hbits.size()));
      g.nFhi = split - g.nHhi;
      // More H bits onto grid rows while the G tile exceeds 2^8 elements: free (each row
      // owns a disjoint column subset of X and C), and a small tile means a short per-CTA
      // prologue and no shared-memory occupancy limit. Rows keep >= 2^11 columns.
      // Only H bits above the lowest 6 column bits: a warp's 32 columns stay contiguous
      // in X and C (a split low bit would halve every access's sector efficiency).
      auto col_pos = [&](int x) {  // position of X bit x among X's non-summed bits
        int c = 0;
        for (int y : X->bits)
          if (X->pos(y) < X->pos(x) && std::find(kp.S.begin(), kp.S.end(), y) == kp.S.end()) ++c;
        return c;
      };
      while (g.nHhi < static_cast<int>(hbits.size()) && nGall - g.nHhi - g.nFhi > 8 &&
             g.nCol - g.nHhi - 1 >= 11 && g.nHhi + g.nFhi < 14 && col_pos(hbits[g.nHhi]) >= 6)
        ++g.nHhi;
      // Expanding steps with few columns: F bits onto grid rows until the grid covers the
      // SMs (X, re-read once per F row, must be small enough to stay in L2).
      {
        const double x_bytes = 16.0 * std::ldexp(1.0, static_cast<int>(X->bits.size()));
        auto ctas = [&](int nfhi) {
          return std::ldexp(1.0, std::max(0, g.nCol - g.nHhi - 8)) * std::ldexp(1.0, g.nHhi + nfhi);
        };
        while (x_bytes <= 16e6 && nFall - g.nFhi >= 4 && ctas(g.nFhi) < 2 * 148 && g.nHhi + g.nFhi < 14) ++g.nFhi;
      }
      g.nF = nFall - g.nFhi;
      g.nG = static_cast<int32_t>(nGall - g.nHhi - g.nFhi);
      // F index bit i <-> the i-th lowest F bit of G (C = [F in G order] ++ [X columns])
      std::set<int> hi_bits;
      for (int q = 0; q < g.nFhi; ++q) hi_bits.insert(C->bits[g.nFhi - 1 - q]);
      for (int q = 0; q < g.nHhi; ++q) hi_bits.insert(hbits[q]);
      // G-tile layout: G's bits minus F_hi and H_hi, G order, compacted
      std::map<int, int> tpos;
      std::vector<std::pair<int, int>> gtile, gfhi, ghhi, xhhi, chhi;
      {
        int t = 0;
        for (int q = 0; q < static_cast<int>(G->bits.size()); ++q) {  // G position ascending
          const int x = G->bits[G->bits.size() - 1 - q];
          if (hi_bits.count(x)) continue;
          tpos[x] = t;
          gtile.emplace_back(t, q);
          ++t;
        }
        for (int q = 0; q < g.nFhi; ++q) gfhi.emplace_back(q, G->pos(C->bits[g.nFhi - 1 - q]));
      }
      std::vector<std::pair<int, int>> xcol, xs, gcol, gs, gf, ccol;
      int p2 = 0, pt = 0;  // column index position; thread column index position
      for (int q = 0; q < static_cast<int>(X->bits.size()); ++q) {  // X position ascending
        int x = X->bits[X->bits.size() - 1 - q];
        if (std::find(kp.S.begin(), kp.S.end(), x) != kp.S.end()) continue;
        const auto h = std::find(hbits.begin(), hbits.begin() + g.nHhi, x);
        if (h != hbits.begin() + g.nHhi) {
          const int hq = static_cast<int>(h - hbits.begin());
          ghhi.emplace_back(hq, G->pos(x));
          xhhi.emplace_back(hq, q);
          chhi.emplace_back(hq, p2);
        } else {
          xcol.emplace_back(pt, q);
          ccol.emplace_back(pt, p2);
          if (tpos.count(x)) gcol.emplace_back(pt, tpos.at(x));
          ++pt;
        }
        ++p2;
      }
      for (int j = 0; j < g.nS; ++j) {
        xs.emplace_back(j, X->pos(kp.S[j]));
        gs.emplace_back(j, tpos.at(kp.S[j]));
      }
      for (int f = 0; f < g.nF; ++f) gf.emplace_back(f, tpos.at(C->bits[nFall - 1 - f]));
      g.xcol = make_runs(xcol);
      g.xs = make_runs(xs);
      g.gcol = make_runs(gcol);
      g.gs = make_runs(gs);
      g.gf = make_runs(gf);
      g.gtile = make_runs(gtile);
      g.gfhi = make_runs(gfhi);
      g.ghhi = make_runs(ghhi);
      g.xhhi = make_runs(xhhi);
      g.chhi = make_runs(chhi);
      g.ccol = make_runs(ccol);
      // two adjacent columns per thread when column bit 0 is X's lowest bit and C's
      // (always C's when no H split) and enough columns remain
      // (measured: a win for large column counts and for expanding steps with a small G;
      // a loss for mid-size reducing steps and for a G that fills shared memory)
      g.pair2 = (!xcol.empty() && xcol[0] == std::make_pair(0, 0) && !ccol.empty() && ccol[0].second == 0 &&
                 g.nS <= 3 && (g.nCol - g.nHhi >= 22 || (g.nF >= 3 && g.nG < 12 && g.nCol - g.nHhi >= 9)))
                    ? 1
                    : 0;
      for (int q = 0; q < (1 << g.nS); ++q) {
        g.xs_tab[q] = static_cast<int64_t>(eval_runs(g.xs, q));
        g.gs_tab[q] = static_cast<int32_t>(eval_runs(g.gs, q));
      }
      check_extent(runs_max(g.xcol) + runs_max(g.xs) + runs_max(g.xhhi), X->size(), "gate X");
      check_extent(runs_max(g.gfhi) + runs_max(g.ghhi) + runs_max(g.gtile), G->size(), "gate G");
      if (runs_max(g.ccol) + runs_max(g.chhi) >= (uint64_t{1} << g.nCol))
        throw std::logic_error("descriptor out of bounds: gate C column");
      check_extent(((uint64_t{1} << (g.nFhi + g.nF)) << g.nCol) - 1, C->size(), "gate C");
      if (runs_max(g.gcol) + runs_max(g.gs) + runs_max(g.gf) >= (uint64_t{1} << g.nG))
        throw std::logic_error("descriptor out of bounds: gate G tile index");
      gate_desc[i] = g;
    } else if (kp.kind == kGemm) {
      Program::GemmOp g{};
      g.offA = A->off;
      g.offB = B->off;
      g.offC = C->off;
      std::set<int> sset(kp.S.begin(), kp.S.end());
      // index bit lists, low to high
      std::vector<int> kb = kp.S, mb, nb, gb;
      for (auto it = A->bits.rbegin(); it != A->bits.rend(); ++it)
        if (!sset.count(*it)) (B->pos(*it) >= 0 ? gb : mb).push_back(*it);
      for (auto it = B->bits.rbegin(); it != B->bits.rend(); ++it)
        if (!sset.count(*it) && A->pos(*it) < 0) nb.push_back(*it);
      g.nK = static_cast<int32_t>(kb.size());
      g.nM = static_cast<int32_t>(mb.size());
      g.nN = static_cast<int32_t>(nb.size());
      g.nG = static_cast<int32_t>(gb.size());
      g.tab = static_cast<int64_t>(prog.gemm_image.size());
      auto table = [&](const std::vector<int>& idx, TensorInfo* T) {
        const int64_t n = int64_t{1} << idx.size();
        for (int64_t x = 0; x < n; ++x) {
          int64_t off = 0;
          for (size_t j = 0; j < idx.size(); ++j)
            if ((x >> j) & 1) off |= int64_t{1} << T->pos(idx[j]);
          prog.gemm_image.push_back(off);
        }
      };
      table(kb, A);
      table(kb, B);
      table(mb, A);
      table(nb, B);
      table(mb, C);
      table(nb, C);
      table(gb, A);
      table(gb, B);
      table(gb, C);
      g.a_kfast = sset.count(A->bits.back()) ? 1 : 0;
      g.b_kfast = sset.count(B->bits.back()) ? 1 : 0;
      g.c_pair = (!nb.empty() && C->pos(nb[0]) == 0) ? 1 : 0;  // adjacent n are adjacent in C
      if (C->bits.size() != kb.size() * 0 + mb.size() + nb.size() + gb.size())
        throw std::logic_error("descriptor out of bounds: gemm result bits");
      gemm_desc[i] = g;
    } else {
      StepDesc d{};
      d.offA = A->off;
      d.offB = B->off;
      d.offC = C->off;
      d.nS = static_cast<int32_t>(kp.S.size());
      d.nTC = static_cast<int32_t>(kp.T.size());
      d.nG = static_cast<int32_t>(C->bits.size()) - d.nTC;
      std::set<int> tileset(kp.T.begin(), kp.T.end());
      std::set<int> sset(kp.S.begin(), kp.S.end());
      auto tile_of = [&](TensorInfo* X) {
        std::vector<std::pair<int, int>> v;  // (pos, bit)
        for (int x : X->bits)
          if (tileset.count(x) || sset.count(x)) v.emplace_back(X->pos(x), x);
        std::sort(v.begin(), v.end());
        std::map<int, int> tpos;
        std::vector<std::pair<int, int>> load;
        for (size_t q = 0; q < v.size(); ++q) {
          tpos[v[q].second] = static_cast<int>(q);
          load.emplace_back(static_cast<int>(q), v[q].first);
        }
        return std::make_pair(tpos, load);
      };
      auto ta = tile_of(A), tb = tile_of(B);
      d.nTA = static_cast<int32_t>(ta.first.size());
      d.nTB = static_cast<int32_t>(tb.first.size());
      d.lA = make_runs(ta.second);
      d.lB = make_runs(tb.second);
      std::vector<std::pair<int, int>> ga, gb, ca, cb, sa, sb;
      const int nC = static_cast<int>(C->bits.size());
      for (int j = 0; j < d.nG; ++j) {
        int x = C->bits[d.nG - 1 - j];
        if (A->pos(x) >= 0) ga.emplace_back(j, A->pos(x));
        if (B->pos(x) >= 0) gb.emplace_back(j, B->pos(x));
      }
      for (int j = 0; j < d.nTC; ++j) {
        int x = C->bits[nC - 1 - j];
        if (ta.first.count(x)) ca.emplace_back(j, ta.first[x]);
        if (tb.first.count(x)) cb.emplace_back(j, tb.first[x]);
      }
      for (int j = 0; j < d.nS; ++j) {
        sa.emplace_back(j, ta.first.at(kp.S[j]));
        sb.emplace_back(j, tb.first.at(kp.S[j]));
      }
      d.gA = make_runs(ga);
      d.gB = make_runs(gb);
      d.cA = make_runs(ca);
      d.cB = make_runs(cb);
      d.sA = make_runs(sa);
      d.sB = make_runs(sb);
      check_extent(runs_max(d.gA) + runs_max(d.lA), A->size(), "tile A");
      check_extent(runs_max(d.gB) + runs_max(d.lB), B->size(), "tile B");
      check_extent((((uint64_t{1} << d.nG) - 1) << d.nTC) + (uint64_t{1} << d.nTC) - 1, C->size(), "tile C");
      if (runs_max(d.cA) + runs_max(d.sA) >= (uint64_t{1} << d.nTA) ||
          runs_max(d.cB) + runs_max(d.sB) >= (uint64_t{1} << d.nTB))
        throw std::logic_error("descriptor out of bounds: tile smem index");
      tile_desc[i] = d;
    }
    const double bytes = 16.0 * static_cast<double>(A->size() + B->size() + C->size());
    prog.kernel_bytes.push_back(bytes);
    prog.kernel_flops.push_back(8.0 * std::ldexp(1.0, static_cast<int>(C->bits.size()) + static_cast<int>(kp.S.size())));
    prog.kernel_dep.push_back(kp.dep ? 1 : 0);
    const PlanStep& st = p.steps[kp.plan_step];
    const double per_slice = 16.0 * (std::pow(D, st.rank_a) + std::pow(D, st.rank_b) + std::pow(D, st.result_rank));
    const double fl = 8.0 * std::pow(D, st.work_rank);
    if (kp.dep) {
      prog.essential_bytes += per_slice * all_slices;
      prog.flops += fl * all_slices;
    } else {
      prog.essential_bytes += per_slice;
      prog.flops += fl;
      ++prog.n_invariant;
    }
    if (!fused) prog.moved_bytes += bytes * static_cast<double>(prog.passes);
    prog.algo_flops += prog.kernel_flops.back() * static_cast<double>(prog.passes);
  }
  // ---- fused chains ----
  std::vector<ChainDesc> chain_desc(segs.size());
  std::vector<double> chain_bytes(segs.size(), 0.0);
  std::vector<uint64_t> chain_ctas(segs.size(), 1);
  for (size_t si = 0; si < segs.size(); ++si) {
    const Seg& sg = segs[si];
    if (sg.steps.size() < 2 || sg.pair) continue;
    ChainDesc& c = chain_desc[si];
    c = ChainDesc{};
    TensorInfo* C0 = kplans[sg.steps.front()].X;
    TensorInfo* Cm = kplans[sg.steps.back()].C;
    c.offIn = C0->off;
    c.offOut = Cm->off;
    c.nStages = static_cast<int32_t>(sg.steps.size());
    c.nT0 = static_cast<int32_t>(sg.tiles[0].size());
    c.nGrid = static_cast<int32_t>(sg.outer.size());
    c.nTmax = 0;  // stage outputs 1, 3, 5, ... (work buffer 0)
    c.nW1 = 0;    // stage outputs 2, 4, ...    (work buffer 1)
    for (size_t j = 1; j < sg.tiles.size(); ++j) {
      int32_t& w = (j % 2) ? c.nTmax : c.nW1;
      w = std::max<int32_t>(w, static_cast<int32_t>(sg.tiles[j].size()));
    }
    std::vector<std::pair<int, int>> load, g2in, g2out;
    for (size_t q = 0; q < sg.tiles[0].size(); ++q) load.emplace_back(static_cast<int>(q), C0->pos(sg.tiles[0][q]));
    for (size_t q = 0; q < sg.outer.size(); ++q) {
      g2in.emplace_back(static_cast<int>(q), C0->pos(sg.outer[q]));
      if (Cm->pos(sg.outer[q]) < 0) throw std::logic_error("chain outer bit missing from its output");
      g2out.emplace_back(static_cast<int>(q), Cm->pos(sg.outer[q]));
    }
    c.load = make_runs(load);
    c.grid2in = make_runs(g2in);
    c.grid2out = make_runs(g2out);
    int gsm = 0, tab = 0;
    double bytes = 16.0 * static_cast<double>(C0->size() + Cm->size());
    for (size_t j = 0; j < sg.steps.size(); ++j) {
      const KPlan& kp = kplans[sg.steps[j]];
      TensorInfo* G = kp.G;
      ChainStage& stg = c.st[j];
      stg.offG = G->off;
      stg.gsm = gsm;
      stg.nG = static_cast<int32_t>(G->bits.size());
      gsm += static_cast<int>(G->size());
      bytes += 16.0 * static_cast<double>(G->size());
      const bool last = j + 1 == sg.steps.size();
      const std::vector<int>& tin = sg.tiles[j];
      const std::vector<int>& tout = sg.tiles[j + 1];
      std::set<int> sj(kp.S.begin(), kp.S.end());
      std::map<int, int> inpos;
      for (size_t q = 0; q < tin.size(); ++q) inpos[tin[q]] = static_cast<int>(q);
      std::vector<int> kept;
      for (int x : tin)
        if (!sj.count(x)) kept.push_back(x);
      if (!std::equal(kept.begin(), kept.end(), tout.begin())) throw std::logic_error("chain tile order");
      stg.nS = static_cast<int32_t>(kp.S.size());
      stg.nKp = static_cast<int32_t>(kept.size());
      stg.nF = static_cast<int32_t>(tout.size() - kept.size());
      stg.tab = tab;
      // mirrors chain_tab_ints() in kernels.cuh (+1 for int64 alignment slack, kept even)
      tab += 2 * (1 << stg.nS) + (1 << stg.nF) + 2 * (256 + 8) + 1 + 2 * ((1 << stg.nF) + 256 + 8);
      tab += tab & 1;
      std::vector<std::pair<int, int>> col, gh, g2g, ccol, sin, gs, gf, cf;
      for (size_t q = 0; q < kept.size(); ++q) {
        col.emplace_back(static_cast<int>(q), inpos.at(kept[q]));
        if (G->pos(kept[q]) >= 0) gh.emplace_back(static_cast<int>(q), G->pos(kept[q]));
        if (last) ccol.emplace_back(static_cast<int>(q), Cm->pos(kept[q]));
      }
      for (size_t q = 0; q < sg.outer.size(); ++q)
        if (G->pos(sg.outer[q]) >= 0) g2g.emplace_back(static_cast<int>(q), G->pos(sg.outer[q]));
      for (size_t q = 0; q < kp.S.size(); ++q) {
        sin.emplace_back(static_cast<int>(q), inpos.at(kp.S[q]));
        gs.emplace_back(static_cast<int>(q), G->pos(kp.S[q]));
      }
      for (int q = 0; q < stg.nF; ++q) {
        const int x = tout[kept.size() + q];
        gf.emplace_back(q, G->pos(x));
        if (last) cf.emplace_back(q, Cm->pos(x));
      }
      stg.col = make_runs(col);
      stg.gH = make_runs(gh);
      stg.grid2g = make_runs(g2g);
      stg.ccol = make_runs(ccol);
      stg.sin = make_runs(sin);
      stg.gS = make_runs(gs);
      stg.gF = make_runs(gf);
      stg.cF = make_runs(cf);
      if (static_cast<int>(gh.size() + g2g.size() + gs.size() + gf.size()) != stg.nG)
        throw std::logic_error("chain stage does not address every bit of its small operand");
    }
    c.tabInts = tab;
    c.gElems = gsm;
    check_extent(runs_max(c.grid2in) + runs_max(c.load), C0->size(), "chain input");
    {
      const ChainStage& lst = c.st[c.nStages - 1];
      check_extent(runs_max(c.grid2out) + runs_max(lst.ccol) + runs_max(lst.cF), Cm->size(), "chain output");
    }
    // ---- shared-memory table image, laid out exactly as k_chain reads it ----
    {
      const int extra = (tab + 1) & ~1;  // 8-byte aligned start of the int64 tables
      const int nlo = 1 << std::min(7, c.nGrid);
      std::vector<int32_t> img(static_cast<size_t>(extra) + 2 * (256 + 8 + 128 + 128) + kMaxChain * 128, 0);
      auto put64 = [&](int at, int64_t v) {
        std::memcpy(&img[static_cast<size_t>(at)], &v, sizeof v);
      };
      for (int j = 0; j < c.nStages; ++j) {
        const ChainStage& st = c.st[j];
        const int K = 1 << st.nS, nf = 1 << st.nF, b = st.tab;
        for (int q = 0; q < K; ++q) {
          img[b + q] = static_cast<int32_t>(eval_runs(st.sin, q));
          img[b + K + q] = static_cast<int32_t>(eval_runs(st.gS, q));
        }
        for (int f = 0; f < nf; ++f) img[b + 2 * K + f] = static_cast<int32_t>(eval_runs(st.gF, f)) + st.gsm;
        const int colLo = b + 2 * K + nf, colHi = colLo + 256, gHLo = colHi + 8, gHHi = gHLo + 256;
        for (int i = 0; i < 256; ++i) {
          const bool in = i < (1 << std::min(st.nKp, 8));
          img[colLo + i] = in ? static_cast<int32_t>(eval_runs(st.col, i)) : 0;
          img[gHLo + i] = in ? static_cast<int32_t>(eval_runs(st.gH, i)) : 0;
        }
        for (int i = 0; i < 8; ++i) {
          img[colHi + i] = static_cast<int32_t>(eval_runs(st.col, static_cast<uint64_t>(i) << 8));
          img[gHHi + i] = static_cast<int32_t>(eval_runs(st.gH, static_cast<uint64_t>(i) << 8));
        }
        int e = gHHi + 8;
        e += e & 1;  // 8-byte alignment (the image base is 16-byte aligned)
        for (int f = 0; f < nf; ++f) put64(e + 2 * f, static_cast<int64_t>(eval_runs(st.cF, f)));
        const int ccLo = e + 2 * nf, ccHi = ccLo + 512;
        for (int i = 0; i < 256; ++i)
          put64(ccLo + 2 * i, i < (1 << std::min(st.nKp, 8)) ? static_cast<int64_t>(eval_runs(st.ccol, i)) : 0);
        for (int i = 0; i < 8; ++i)
          put64(ccHi + 2 * i, static_cast<int64_t>(eval_runs(st.ccol, static_cast<uint64_t>(i) << 8)));
      }
      const int loadLo = extra, loadHi = loadLo + 512, itIn = loadHi + 16, itOut = itIn + 256, itG = itOut + 256;
      for (int i = 0; i < 256; ++i)
        put64(loadLo + 2 * i, i < (1 << std::min(c.nT0, 8)) ? static_cast<int64_t>(eval_runs(c.load, i)) : 0);
      for (int i = 0; i < 8; ++i) put64(loadHi + 2 * i, static_cast<int64_t>(eval_runs(c.load, static_cast<uint64_t>(i) << 8)));
      for (int i = 0; i < nlo; ++i) {
        put64(itIn + 2 * i, static_cast<int64_t>(eval_runs(c.grid2in, i)));
        put64(itOut + 2 * i, static_cast<int64_t>(eval_runs(c.grid2out, i)));
        for (int j = 0; j < c.nStages; ++j) img[itG + j * 128 + i] = static_cast<int32_t>(eval_runs(c.st[j].grid2g, i));
      }
      img.resize((img.size() + 3) & ~size_t{3});  // whole int4s
      c.extraOff = extra;
      c.imgInts = static_cast<int32_t>(img.size());
      c.img = static_cast<int64_t>(prog.chain_image.size());
      prog.chain_image.insert(prog.chain_image.end(), img.begin(), img.end());
    }
    // grid index = (hi << nIter) | lo with lo tabulated per CTA (<= 128 entries)
    c.nIter = std::min(7, c.nGrid);
    {
      const int smem = (2 * (1 << c.nT0) + (1 << c.nTmax) + (1 << c.nW1) + c.gElems) * 16 + c.tabInts * 4 + 16 * 1024;
      int smax = 0;
      for (int j = 0; j < c.nStages; ++j) smax = std::max(smax, c.st[j].nS);
      const int occ = std::max(1, std::min(smax <= 3 ? 3 : 2, (227 * 1024) / (smem + 10 * 1024)));
      chain_ctas[si] = std::min<uint64_t>(uint64_t{1} << c.nGrid, 148ull * occ);  // one resident wave
    }
    chain_bytes[si] = bytes;
    prog.moved_bytes += bytes * static_cast<double>(prog.passes);
  }
  // ---- register-fused gate pairs ----
  std::vector<PairDesc> pair_desc(segs.size());
  std::vector<double> pair_bytes(segs.size(), 0.0);
  for (size_t si = 0; si < segs.size(); ++si) {
    const Seg& sg = segs[si];
    if (!sg.pair) continue;
    const KPlan& a = kplans[sg.steps[0]];
    const KPlan& b = kplans[sg.steps[1]];
    const PairPlan& pp = sg.pp;
    TensorInfo *G1 = a.G, *X1 = a.X, *G2 = b.G, *C2 = b.C;
    PairDesc d{};
    d.offG1 = G1->off;
    d.offG2 = G2->off;
    d.offX = X1->off;
    d.offC = C2->off;
    d.nS1 = static_cast<int32_t>(pp.S1.size());
    d.nS2 = static_cast<int32_t>(pp.S2.size());
    d.nP = static_cast<int32_t>(pp.P.size());
    d.nQ = static_cast<int32_t>(pp.Q.size());
    d.nRlo = pp.nRlo;
    d.nRmid = pp.nRmid;
    d.nRhi = pp.nRhi;
    d.nF2 = static_cast<int32_t>(pp.F2.size());
    d.nCol = static_cast<int32_t>(pp.cols.size());
    d.nR = static_cast<int32_t>(pp.R.size());
    d.nG2 = static_cast<int32_t>(G2->bits.size());
    const int nRt = pp.nRlo + pp.nRmid;
    std::vector<std::pair<int, int>> xcol, xp, xs1, g1stage, g1hi, g1hc, g2stage, g2hc, g2r, g1hcx, g2hcx;
    // expanded G1 tile, low to high: s1, p, q, (r_lo, r_mid), hc1 (cols' bits G1 carries)
    {
      int k = 0;
      auto put = [&](int bit) {
        if (G1->pos(bit) >= 0) g1stage.emplace_back(k, G1->pos(bit));
        ++k;
      };
      for (int x : pp.S1) put(x);
      for (int x : pp.P) put(x);
      for (int x : pp.Q) put(x);
      for (int q = 0; q < nRt; ++q) put(pp.R[q]);
      // hc1 bits: the non-H_hi ones (cols' order), then the H_hi ones (hhi order) on top
      const std::set<int> hset(pp.H.begin(), pp.H.end());
      std::vector<int> hc_order;
      for (size_t q = 0; q < pp.cols.size(); ++q)
        if (G1->pos(pp.cols[q]) >= 0 && !hset.count(pp.cols[q])) hc_order.push_back(static_cast<int>(q));
      for (int x : pp.H)
        hc_order.push_back(static_cast<int>(std::find(pp.cols.begin(), pp.cols.end(), x) - pp.cols.begin()));
      for (int q : hc_order) {
        g1hcx.emplace_back(q, static_cast<int>(g1hc.size()));
        g1hc.emplace_back(q, k);
        put(pp.cols[static_cast<size_t>(q)]);
      }
      d.nG1x = k;
      d.sh1 = k - static_cast<int32_t>(g1hc.size());
      d.nG1h = static_cast<int32_t>(g1hc.size());
      d.nHhi = pp.nHhi;
      // thread column index <-> cols' index with the H_hi bits on the grid
      std::vector<std::pair<int, int>> jc, jh;
      int t = 0;
      for (size_t q = 0; q < pp.cols.size(); ++q)
        if (!hset.count(pp.cols[q])) jc.emplace_back(t++, static_cast<int>(q));
      for (int h = 0; h < d.nHhi; ++h)
        jh.emplace_back(h, static_cast<int>(std::find(pp.cols.begin(), pp.cols.end(), pp.H[h]) - pp.cols.begin()));
      d.jcol = make_runs(jc);
      d.jhhi = make_runs(jh);
    }
    for (int q = 0; q < pp.nRhi; ++q) g1hi.emplace_back(q, G1->pos(pp.R[nRt + q]));
    // G2, low to high: p, q, f2, r bits G2 carries, hc2 (cols' bits G2 carries)
    {
      int k = 0;
      auto put = [&](int bit) {
        g2stage.emplace_back(k, G2->pos(bit));
        ++k;
      };
      for (int x : pp.P) put(x);
      for (int x : pp.Q) put(x);
      for (int x : pp.F2) put(x);
      for (size_t q = 0; q < pp.R.size(); ++q)
        if (G2->pos(pp.R[q]) >= 0) {
          g2r.emplace_back(static_cast<int>(q), k);
          put(pp.R[q]);
        }
      for (size_t q = 0; q < pp.cols.size(); ++q)
        if (G2->pos(pp.cols[q]) >= 0) {
          g2hcx.emplace_back(static_cast<int>(q), static_cast<int>(g2hc.size()));
          g2hc.emplace_back(static_cast<int>(q), k);
          put(pp.cols[q]);
        }
      if (k != d.nG2) throw std::logic_error("gate pair does not address its operands");
      d.sh2 = k - static_cast<int32_t>(g2hc.size());
    }
    for (size_t q = 0; q < pp.cols.size(); ++q) xcol.emplace_back(static_cast<int>(q), X1->pos(pp.cols[q]));
    for (size_t q = 0; q < pp.P.size(); ++q) xp.emplace_back(static_cast<int>(q), X1->pos(pp.P[q]));
    for (size_t q = 0; q < pp.S1.size(); ++q) xs1.emplace_back(static_cast<int>(q), X1->pos(pp.S1[q]));
    if (static_cast<int>(g1stage.size()) + pp.nRhi != static_cast<int>(G1->bits.size()))
      throw std::logic_error("gate pair does not address its operands");
    d.xcol = make_runs(xcol);
    d.g1stage = make_runs(g1stage);
    d.g1hi = make_runs(g1hi);
    d.g1hc = make_runs(g1hc);
    d.g2stage = make_runs(g2stage);
    d.g2hc = make_runs(g2hc);
    d.g1hcx = make_runs(g1hcx);
    d.g2hcx = make_runs(g2hcx);
    d.g2r = make_runs(g2r);
    const Runs rxp = make_runs(xp), rxs1 = make_runs(xs1);
    for (int p2 = 0; p2 < (1 << d.nP); ++p2)
      for (int q = 0; q < (1 << d.nS1); ++q)
        d.xoff_tab[(p2 << d.nS1) + q] = static_cast<int64_t>(eval_runs(rxp, p2) + eval_runs(rxs1, q));
    check_extent(runs_max(d.xcol) + runs_max(rxp) + runs_max(rxs1), X1->size(), "pair X");
    check_extent(runs_max(d.g1hi) + runs_max(d.g1stage), G1->size(), "pair G1");
    check_extent(runs_max(d.g2stage), G2->size(), "pair G2");
    check_extent(((uint64_t{1} << (d.nF2 + d.nR)) << d.nCol) - 1, C2->size(), "pair C");
    if (runs_max(d.g1hc) + (uint64_t{1} << (d.nS1 + d.nP + d.nQ + nRt)) - 1 >= (uint64_t{1} << d.nG1x) ||
        runs_max(d.g2hc) + runs_max(d.g2r) + (uint64_t{1} << (d.nP + d.nQ + d.nF2)) - 1 >= (uint64_t{1} << d.nG2))
      throw std::logic_error("descriptor out of bounds: pair shared-memory index");
    pair_desc[si] = d;
    pair_bytes[si] = 16.0 * static_cast<double>(X1->size() + C2->size() + G1->size() + G2->size());
    prog.moved_bytes += pair_bytes[si] * static_cast<double>(prog.passes);
  }
  // ---- k_forest: a dataflow group whose steps are all small runs as independent subtrees,
  // one (or a pack of small ones) per CTA, in phases inside shared memory (desc.hpp) ----
  auto fmap_of = [](const std::vector<std::pair<int, int>>& pairs) -> FMap {
    const Runs r = make_runs(pairs);
    FMap m{};
    if (r.n > kFMapRuns) throw std::runtime_error("forest map needs too many runs");
    m.n = static_cast<uint16_t>(r.n);
    for (int i = 0; i < r.n; ++i) {
      if (r.src[i] > 31 || r.len[i] > 31 || r.dst[i] > 31) throw std::runtime_error("forest map out of range");
      m.r[i] = static_cast<uint16_t>(r.src[i] | (r.len[i] << 5) | (r.dst[i] << 10));
    }
    return m;
  };
  auto forest_ok = [&](int oi) {
    const KPlan& kp = kplans[ops[oi].kplan];
    return kp.C->bits.size() <= 14 && kp.A->bits.size() <= 16 && kp.B->bits.size() <= 16 && kp.S.size() <= 4;
  };
  // Forest units of group L (a k_forest launch): every step of the group must be small, else
  // the group stays a k_flow launch.
  auto build_forest = [&](int L) -> bool {
    const std::vector<int>& grp = groups[L];
    if (std::getenv("QCG_NO_FOREST")) return false;
    std::vector<int> members;
    for (int oi : grp) {
      if (ops[oi].kind != kTile || !forest_ok(oi)) return false;
      members.push_back(oi);
    }
    std::set<int> mset(members.begin(), members.end());
    // in-group consumer among the small steps (plans are trees: every tensor has at most one consumer)
    std::map<int, int> cons;  // op -> in-unit consumer op
    for (int oi : members)
      for (int u : op_users[oi])
        if (mset.count(u)) cons[oi] = u;
    std::map<int, std::vector<int>> prods;  // op -> in-unit producer ops
    for (int oi : members)
      for (int q : op_deps[oi])
        if (mset.count(q)) prods[oi].push_back(q);
    std::vector<int> roots;
    for (int oi : members)
      if (!cons.count(oi)) roots.push_back(oi);
    // subtree of each root: members, depth (longest producer chain), output elements
    std::map<int, int> depth;
    std::function<int(int)> dep_of = [&](int oi) -> int {
      auto it = depth.find(oi);
      if (it != depth.end()) return it->second;
      int d = 1;
      for (int q : prods[oi]) d = std::max(d, 1 + dep_of(q));
      return depth[oi] = d;
    };
    struct Sub {
      std::vector<int> members;  // producers before consumers
      int depth = 0;
      int64_t elems = 0;
    };
    std::vector<Sub> subs;
    for (int r : roots) {
      Sub sb;
      sb.depth = dep_of(r);
      std::function<void(int)> walk = [&](int oi) {
        for (int q : prods[oi]) walk(q);
        sb.members.push_back(oi);
        sb.elems += kplans[ops[oi].kplan].C->size();
      };
      walk(r);
      subs.push_back(sb);
    }
    // units: one subtree each, packed (largest first onto the least-loaded unit) when a
    // group has more subtrees than two CTAs per SM
    const int nunits = std::min<int>(static_cast<int>(subs.size()), 296);
    std::vector<int> order(subs.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return subs[a].elems > subs[b].elems; });
    std::vector<std::vector<int>> unit_subs(nunits);
    std::vector<int64_t> load(nunits, 0);
    for (int si : order) {
      const int u = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
      unit_subs[u].push_back(si);
      load[u] += subs[si].elems + 64;
    }
    if (roots.empty()) return false;
    Program::Launch fl{};
    fl.kind = kForest;
    fl.first = static_cast<int>(prog.forest_units.size());
    fl.prefix_off = -1;
    fl.plan_step = -1;
    int smem_max = 0;
    for (int u = 0; u < nunits; ++u) {
      // phases: ALAP inside each subtree (root at its depth, a producer one phase before its
      // consumer) -- a producer's output is live for one phase boundary only
      std::map<int, int> phase;
      std::vector<int> steps;  // unit-local step order: by phase, then subtree order
      int nph = 0;
      for (int si : unit_subs[u]) {
        const Sub& sb = subs[si];
        for (auto it = sb.members.rbegin(); it != sb.members.rend(); ++it) {
          const int oi = *it;
          phase[oi] = cons.count(oi) ? phase.at(cons.at(oi)) - 1 : sb.depth;
        }
        nph = std::max(nph, sb.depth);
        steps.insert(steps.end(), sb.members.begin(), sb.members.end());
      }
      std::stable_sort(steps.begin(), steps.end(), [&](int a, int b) { return phase.at(a) < phase.at(b); });
      std::map<int, int> local;
      for (size_t i = 0; i < steps.size(); ++i) local[steps[i]] = static_cast<int>(i);
      // tensors: leaves (produced outside the unit) and intermediates (consumed in the unit)
      struct FT {
        TensorInfo* t;
        int birth, death;
        bool leaf;
        int64_t soff = -1;
      };
      std::vector<FT> fts;
      std::map<TensorInfo*, int> ft_of;
      for (int oi : steps) {
        const KPlan& kp = kplans[ops[oi].kplan];
        for (TensorInfo* X : {kp.A, kp.B}) {
          auto pit = producer_op.find(X);
          const bool inner = pit != producer_op.end() && local.count(pit->second);
          if (inner) {
            fts.push_back({X, phase.at(pit->second), phase.at(oi), false});
          } else if (X->size() <= 8192) {  // staged (bulk copy) when it fits the data region
            fts.push_back({X, 0, phase.at(oi), true});
          } else {
            continue;  // a large leaf is read in place
          }
          ft_of[X] = static_cast<int>(fts.size()) - 1;
        }
      }
      // data region: what the unit's image leaves of the shared memory (image size bound: every
      // leaf listed, every step's 32-column items)
      int64_t img_bound = 16 + 16 * (nph + 8) + 16 * static_cast<int64_t>(fts.size()) +
                          static_cast<int64_t>(steps.size()) * static_cast<int64_t>(sizeof(FStep));
      for (int oi : steps) {  // 32-column items (see the item list below)
        const KPlan& kq = kplans[ops[oi].kplan];
        int nx = 0, na = 0, nb = 0;
        for (int x : kq.C->bits) {
          na += kq.A->pos(x) >= 0;
          nb += kq.B->pos(x) >= 0;
        }
        const bool ax = kq.A->size() > kq.B->size() || (kq.A->size() == kq.B->size() && na >= nb);
        nx = ax ? na : nb;
        const int ngo = static_cast<int>(kq.C->bits.size()) - nx;
        img_bound += 4 * (((int64_t{1} << (nx + ngo - std::min(2, ngo))) + 31) / 32 + 1);
      }
      const int64_t kForestDataElems = (kForestSmemMax - img_bound) / 16;
      {  // placement in the data region: largest first, lifetimes (phases, inclusive) disjoint
        std::vector<int> ord(fts.size());
        for (size_t i = 0; i < ord.size(); ++i) ord[i] = static_cast<int>(i);
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return fts[a].t->size() > fts[b].t->size(); });
        std::vector<int> placed;
        for (int i : ord) {
          FT& f = fts[i];
          std::vector<std::pair<int64_t, int64_t>> busy;
          for (int j : placed)
            if (!(fts[j].death < f.birth || f.death < fts[j].birth))
              busy.emplace_back(fts[j].soff, fts[j].soff + fts[j].t->size());
          std::sort(busy.begin(), busy.end());
          int64_t at = 0;
          for (const auto& iv : busy) {
            if (at + f.t->size() <= iv.first) break;
            at = std::max(at, iv.second);
          }
          if (at + f.t->size() > kForestDataElems) continue;  // stays in the arena
          f.soff = at;
          placed.push_back(i);
        }
      }
      int64_t data_elems = 0;
      for (const FT& f : fts)
        if (f.soff >= 0) data_elems = std::max(data_elems, f.soff + f.t->size());
      if (std::getenv("QCG_FOREST_DEBUG")) {
        int64_t gl = 0, gi = 0, big_in_place = 0, work = 0;
        for (const FT& f : fts)
          if (f.soff < 0) (f.leaf ? gl : gi) += f.t->size();
        for (int oi : steps) {
          const KPlan& kp = kplans[ops[oi].kplan];
          for (TensorInfo* X : {kp.A, kp.B})
            if (!ft_of.count(X)) big_in_place += X->size();
          work += int64_t{1} << (kp.C->bits.size() + kp.S.size());
        }
        for (int ph = 1; ph <= nph; ++ph) {
          std::string d;
          for (int oi : steps)
            if (phase.at(oi) == ph) {
              const KPlan& kp = kplans[ops[oi].kplan];
              d += " (" + std::to_string(kp.C->bits.size()) + "," + std::to_string(kp.S.size()) + "," +
                   std::to_string(kp.A->bits.size()) + "," + std::to_string(kp.B->bits.size()) + ")";
            }
          std::fprintf(stderr, "  L%d u%d phase %d: (C,S,A,B)%s\n", L, u, ph, d.c_str());
        }
        {
          std::string cl;
          for (int si : unit_subs[u]) {
            const int r = subs[si].members.back();
            int lv = 1 << 30;
            for (int c : op_users[r]) lv = std::min(lv, ops[c].level);
            cl += " " + (lv == (1 << 30) ? std::string("final") : std::to_string(lv));
          }
          std::fprintf(stderr, "  L%d u%d root consumers (launch):%s\n", L, u, cl.c_str());
        }
        std::fprintf(stderr, "forest L%d unit %d: steps %zu phases %d data %lld elems, global leaves %lld, global "
                     "intermediates %lld, in-place leaves %lld, MACs %lld\n",
                     L, u, steps.size(), nph, static_cast<long long>(data_elems), static_cast<long long>(gl),
                     static_cast<long long>(gi), static_cast<long long>(big_in_place), static_cast<long long>(work));
      }
      auto soff = [&](TensorInfo* X) -> int32_t {
        auto it = ft_of.find(X);
        return it == ft_of.end() || fts[it->second].soff < 0 ? -1 : static_cast<int32_t>(fts[it->second].soff);
      };
      // image
      std::vector<int32_t> img;
      const int nsteps_u = static_cast<int>(steps.size());
      std::vector<int32_t> phase_off(nph + 1, 0);
      std::vector<uint32_t> items;
      for (int ph = 1; ph <= nph; ++ph) {
        phase_off[ph - 1] = static_cast<int32_t>(items.size());
        for (int oi : steps) {
          if (phase.at(oi) != ph) continue;
          const KPlan& kq = kplans[ops[oi].kplan];
          // columns: the C bits of the streamed operand (see FStep)
          TensorInfo* Xq = kq.A->size() > kq.B->size() || (kq.A->size() == kq.B->size() && [&] {
            int na = 0, nb = 0;
            for (int x : kq.C->bits) {
              na += kq.A->pos(x) >= 0;
              nb += kq.B->pos(x) >= 0;
            }
            return na >= nb;
          }()) ? kq.A : kq.B;
          int ncb = 0, ngo = 0;
          for (int x : kq.C->bits) (Xq->pos(x) >= 0 ? ncb : ngo) += 1;
          const int64_t nc = int64_t{1} << (ncb + ngo - std::min(2, ngo));
          for (int64_t ch = 0; ch < (nc + 31) / 32; ++ch)
            items.push_back(static_cast<uint32_t>(local.at(oi)) << 16 | static_cast<uint32_t>(ch));
        }
      }
      phase_off[nph] = static_cast<int32_t>(items.size());
      std::vector<const FT*> leaves;
      for (const FT& f : fts)
        if (f.leaf && f.soff >= 0) leaves.push_back(&f);
      auto pad4 = [&]() {
        while (img.size() % 4) img.push_back(0);
      };
      img.push_back(nph);
      img.push_back(nsteps_u);
      img.push_back(static_cast<int32_t>(items.size()));
      img.push_back(static_cast<int32_t>(leaves.size()));
      img.insert(img.end(), phase_off.begin(), phase_off.end());
      pad4();
      for (uint32_t it : items) img.push_back(static_cast<int32_t>(it));
      pad4();
      const int leaf_off = static_cast<int>(img.size());
      int64_t leaf_bytes = 0;
      for (const FT* f : leaves) {
        int32_t w[4];
        std::memcpy(w, &f->t->off, 8);
        w[2] = static_cast<int32_t>(f->soff);
        w[3] = static_cast<int32_t>(f->t->size() * 16);
        img.insert(img.end(), w, w + 4);
        leaf_bytes += f->t->size() * 16;
      }
      for (int oi : steps) {
        const KPlan& kp = kplans[ops[oi].kplan];
        TensorInfo *A = kp.A, *B = kp.B, *C = kp.C;
        // X = the operand streamed through registers (the larger; ties: the one with more C
        // bits), G = the other; column bits = C bits of X, loop bits = C bits only G carries
        const bool a_is_x = A->size() > B->size() || (A->size() == B->size() && [&] {
          int na = 0, nb = 0;
          for (int x : C->bits) {
            na += A->pos(x) >= 0;
            nb += B->pos(x) >= 0;
          }
          return na >= nb;
        }());
        TensorInfo* X = a_is_x ? A : B;
        TensorInfo* G = a_is_x ? B : A;
        FStep d{};
        d.gG = G->off;
        d.gX = X->off;
        d.gC = C->off;
        d.sG = soff(G);
        d.sX = soff(X);
        d.sC = soff(C);
        d.nS = static_cast<int32_t>(kp.S.size());
        if (d.nS > 4) throw std::logic_error("forest step with more than 4 summed bits");
        std::vector<std::pair<int, int>> colC, colG, colX, loopC, loopG;
        const int nC = static_cast<int>(C->bits.size());
        // loop bits: the two highest G-only C bits (the rest stay columns: lanes in parallel)
        std::vector<int> gonly;
        for (int j = 0; j < nC; ++j)
          if (X->pos(C->bits[nC - 1 - j]) < 0) gonly.push_back(j);
        std::set<int> loopset(gonly.end() - std::min<size_t>(2, gonly.size()), gonly.end());
        for (int j = 0; j < nC; ++j) {  // C position ascending
          const int x = C->bits[nC - 1 - j];
          if (!loopset.count(j)) {
            const int q = static_cast<int>(colC.size());
            colC.emplace_back(q, j);
            if (X->pos(x) >= 0) colX.emplace_back(q, X->pos(x));
            if (G->pos(x) >= 0) colG.emplace_back(q, G->pos(x));
          } else {
            const int q = static_cast<int>(loopC.size());
            loopC.emplace_back(q, j);
            loopG.emplace_back(q, G->pos(x));
          }
        }
        d.nCol = static_cast<int32_t>(colC.size());
        d.nLoop = static_cast<int32_t>(loopC.size());
        {
          const Runs rlg = make_runs(loopG), rlc = make_runs(loopC);
          for (int l = 0; l < 4; ++l) {
            d.loopG[l] = l < (1 << d.nLoop) ? static_cast<uint16_t>(eval_runs(rlg, static_cast<uint64_t>(l))) : 0;
            d.loopC[l] = l < (1 << d.nLoop) ? static_cast<uint16_t>(eval_runs(rlc, static_cast<uint64_t>(l))) : 0;
          }
          const Runs rcc = make_runs(colC), rcg = make_runs(colG), rcx = make_runs(colX);
          const uint64_t cmask = (uint64_t{1} << d.nCol) - 1;
          for (int l = 0; l < 32; ++l) {
            const uint64_t lo = static_cast<uint64_t>(l) & cmask, mid = (static_cast<uint64_t>(l) << 5) & cmask;
            d.laneC[l] = static_cast<uint16_t>(eval_runs(rcc, lo));
            d.laneG[l] = static_cast<uint16_t>(eval_runs(rcg, lo));
            d.laneX[l] = static_cast<uint16_t>(eval_runs(rcx, lo));
            d.midC[l] = static_cast<uint16_t>(eval_runs(rcc, mid));
            d.midG[l] = static_cast<uint16_t>(eval_runs(rcg, mid));
            d.midX[l] = static_cast<uint16_t>(eval_runs(rcx, mid));
            if (l < 16) {
              const uint64_t hi = (static_cast<uint64_t>(l) << 10) & cmask;
              d.highC[l] = static_cast<uint16_t>(eval_runs(rcc, hi));
              d.highG[l] = static_cast<uint16_t>(eval_runs(rcg, hi));
              d.highX[l] = static_cast<uint16_t>(eval_runs(rcx, hi));
            }
          }
          if (d.nCol > 14) throw std::logic_error("forest step with more than 2^14 columns");
        }
        int64_t tg_max = 0, tx_max = 0;
        for (int q = 0; q < 16; ++q) {
          int64_t og = 0, ox = 0;
          for (int j = 0; j < d.nS; ++j)
            if ((q >> j) & 1) {
              if (A->pos(kp.S[j]) < 0 || B->pos(kp.S[j]) < 0) throw std::logic_error("forest: summed bit missing");
              og += int64_t{1} << G->pos(kp.S[j]);
              ox += int64_t{1} << X->pos(kp.S[j]);
            }
          d.tg[q] = q < (1 << d.nS) ? static_cast<uint16_t>(og) : 0;
          d.tx[q] = q < (1 << d.nS) ? static_cast<uint16_t>(ox) : 0;
          tg_max = std::max<int64_t>(tg_max, d.tg[q]);
          tx_max = std::max<int64_t>(tx_max, d.tx[q]);
        }
        // memory safety: every index stays inside its tensor
        check_extent(runs_max(make_runs(colG)) + runs_max(make_runs(loopG)) + static_cast<uint64_t>(tg_max), G->size(),
                     "forest G");
        check_extent(runs_max(make_runs(colX)) + static_cast<uint64_t>(tx_max), X->size(), "forest X");
        check_extent(runs_max(make_runs(colC)) + runs_max(make_runs(loopC)), C->size(), "forest C");
        if (C->bits.size() > 14) throw std::logic_error("forest step output too large");
        const int32_t* w = reinterpret_cast<const int32_t*>(&d);
        img.insert(img.end(), w, w + sizeof(FStep) / 4);
      }
      pad4();
      ForestUnit fu{};
      fu.img = static_cast<int64_t>(prog.forest_image.size());
      fu.img_words = static_cast<int32_t>(img.size());
      fu.leaf_off = leaf_off;
      fu.nleaves = static_cast<int32_t>(leaves.size());
      fu.leaf_bytes = static_cast<int32_t>(leaf_bytes);
      fu.data_off = 16 + static_cast<int32_t>(img.size()) * 4;  // after the mbarrier and the image
      const int smem = fu.data_off + static_cast<int>(data_elems) * 16;
      if (smem > kForestSmemMax) return false;
      fu.smem = smem;
      smem_max = std::max(smem_max, smem);
      prog.forest_image.insert(prog.forest_image.end(), img.begin(), img.end());
      prog.forest_units.push_back(fu);
    }
    for (int oi : grp) {
      fl.bytes += prog.kernel_bytes[static_cast<size_t>(ops[oi].kplan)];
      fl.flops += prog.kernel_flops[static_cast<size_t>(ops[oi].kplan)];
    }
    fl.count = nunits;
    fl.items = static_cast<uint64_t>(nunits);
    fl.smem = smem_max;
    prog.launches.push_back(fl);
    return true;
  };
  // ---- launches: one per schedule group (a dataflow group of tile steps, or one fused/gate op) ----
  for (int L = 0; L <= max_level; ++L) {
    {
      // a failed attempt may have appended units of this group: drop them
      const size_t nu = prog.forest_units.size(), ni = prog.forest_image.size();
      if (build_forest(L)) continue;
      prog.forest_units.resize(nu);
      prog.forest_image.resize(ni);
    }
    Program::Launch tl{};
    tl.kind = kTile;
    tl.first = static_cast<int>(prog.tiles.size());
    tl.prefix_off = static_cast<int>(prog.tile_prefix.size());
    tl.plan_step = -1;
    uint64_t items = 0;
    int smem = 0;
    prog.tile_prefix.push_back(0);
    std::map<int, int> local;  // op index -> step index within this launch
    for (int oi : groups[L]) {
      const Op& o = ops[oi];
      if (o.kind != kTile) continue;
      const size_t i = static_cast<size_t>(o.kplan);
      const StepDesc& d = tile_desc[i];
      local[oi] = static_cast<int>(prog.tiles.size()) - tl.first;
      prog.tiles.push_back(d);
      std::vector<int> deps;  // producers inside this group (earlier groups are complete)
      for (int q : op_deps[oi])
        if (ops[q].level == L) deps.push_back(local.at(q));
      prog.flow_dep_off.push_back(static_cast<int>(prog.flow_deps.size()));
      if (deps.size() > 32) throw std::logic_error("dataflow step with more than 32 in-group producers");
      prog.flow_deps.insert(prog.flow_deps.end(), deps.begin(), deps.end());
      tl.bytes += prog.kernel_bytes[i];
      tl.flops += prog.kernel_flops[i];
      items += uint64_t{1} << d.nG;
      prog.tile_prefix.push_back(items);
      smem = std::max(smem, static_cast<int>(((1 << d.nTA) + (1 << d.nTB)) * 16 + 2 * (1 << d.nS) * 4));
    }
    tl.count = static_cast<int>(prog.tiles.size()) - tl.first;
    tl.items = items;
    tl.smem = smem + kFlowCs * 16;  // + the shared-memory hand-off tile (k_flow's Cs)
    // continuation: a single-tile step c whose in-group producers all have c as their
    // only consumer is continuation-only -- the CTA that completes the last of its
    // producers runs it next (k_flow); every such producer points at c
    {
      std::map<int, int> conly;  // op index -> 1 if continuation-only
      for (int oi : groups[L]) {
        const Op& o = ops[oi];
        if (o.kind != kTile || tile_desc[o.kplan].nG != 0) continue;
        int n_in = 0;
        bool ok = true;
        for (int q : op_deps[oi]) {
          if (ops[q].level != L) continue;
          ++n_in;
          ok = ok && ops[q].kind == kTile && op_users[q].size() == 1 && op_users[q][0] == oi;
        }
        if (ok && n_in > 0) conly[oi] = 1;
      }
      // k_flow prefetches a continuation's operand from outside the group while the
      // producer computes: two buffers of the largest operand tile of a continuation-only step
      // (only continuations with a single in-group producer take that private path)
      int npre = 0;
      for (const auto& kv : conly) {
        if (!QCG_FLOW_PREFETCH) break;
        int n_in = 0;
        for (int q : op_deps[kv.first]) n_in += ops[q].level == L ? 1 : 0;
        if (n_in != 1) continue;
        const StepDesc& dc = tile_desc[ops[kv.first].kplan];
        npre = std::max(npre, std::max(1 << dc.nTA, 1 << dc.nTB));
      }
      tl.npre = npre;
      tl.smem += 2 * npre * 16;
      for (int oi : groups[L]) {
        const Op& o = ops[oi];
        if (o.kind != kTile) continue;
        int cont = -1;
        if (op_users[oi].size() == 1 && conly.count(op_users[oi][0])) cont = local.at(op_users[oi][0]);
        prog.flow_cont.push_back(cont);
        prog.flow_conly.push_back(conly.count(oi) ? 1 : 0);
      }
    }
    if (tl.smem > kFlowSmemMax) throw std::logic_error("k_flow launch needs more shared memory than its attribute");
    if (tl.count > 0) {
      tl.dep_off = static_cast<int>(prog.flow_dep_off.size()) - tl.count;
      prog.flow_dep_off.push_back(static_cast<int>(prog.flow_deps.size()));  // sentinel
      prog.launches.push_back(tl);
    } else {
      prog.tile_prefix.pop_back();
    }
    for (int oi : groups[L]) {
      const Op& o = ops[oi];
      if (o.kind == kPair) {
        const PairDesc& d = pair_desc[o.seg];
        Program::Launch pl{};
        pl.kind = kPair;
        pl.first = static_cast<int>(prog.pairs.size());
        pl.count = 1;
        pl.prefix_off = -1;
        pl.plan_step = kplans[segs[o.seg].steps.back()].plan_step;
        pl.bytes = pair_bytes[o.seg];
        pl.flops = prog.kernel_flops[segs[o.seg].steps[0]] + prog.kernel_flops[segs[o.seg].steps[1]];
        pl.items = uint64_t{1} << (d.nCol - d.nHhi);  // columns per grid row (grid.y = 2^(nRhi + nHhi))
        const int rt = 1 << (d.nRmid + d.nRlo);
        const int nmask = (1 << d.nRmid) * (1 << d.nQ);
        const int g1t = d.nG1x - d.nHhi;  // staged G1x sub-block
        pl.smem = ((1 << g1t) + (1 << (g1t - d.sh1)) + (1 << d.nG2) + (1 << (d.nG2 - d.sh2))) * 16 + rt * 4 +
                  (d.g2hc.n == 0 && nmask <= 1024 ? nmask * 4 : 0);
        prog.pairs.push_back(d);
        prog.launches.push_back(pl);
        continue;
      }
      if (o.kind == kChain) {
        const ChainDesc& c = chain_desc[o.seg];
        Program::Launch cl{};
        cl.kind = kChain;
        cl.first = static_cast<int>(prog.chains.size());
        cl.count = 1;
        cl.prefix_off = -1;
        cl.plan_step = kplans[segs[o.seg].steps.back()].plan_step;
        cl.bytes = chain_bytes[o.seg];
        cl.flops = 0;
        for (int st : segs[o.seg].steps) cl.flops += prog.kernel_flops[st];
        cl.items = chain_ctas[o.seg];  // CTAs (contiguous tile ranges)
        cl.smem = (2 * (1 << c.nT0) + (1 << c.nTmax) + (1 << c.nW1) + c.gElems) * 16 + c.imgInts * 4;
        prog.chains.push_back(c);
        prog.launches.push_back(cl);
        continue;
      }
      if (o.kind == kGemm) {
        const size_t i = static_cast<size_t>(o.kplan);
        const Program::GemmOp& g = gemm_desc[i];
        Program::Launch ml{};
        ml.kind = kGemm;
        ml.first = static_cast<int>(prog.gemms.size());
        ml.count = 1;
        ml.prefix_off = -1;
        ml.plan_step = kplans[i].plan_step;
        ml.bytes = prog.kernel_bytes[i];
        ml.flops = prog.kernel_flops[i];
        // CTAs: 64 x 64 result tiles x batch
        ml.items = (uint64_t{1} << g.nG) * (((uint64_t{1} << g.nM) + 63) / 64) * (((uint64_t{1} << g.nN) + 63) / 64);
        ml.smem = 0;  // fixed by the kernel (kGemmSmemBytes)
        if (ml.items > 0x7fffffffull) throw std::logic_error("gemm step with too many result tiles");
        prog.gemms.push_back(g);
        prog.launches.push_back(ml);
        continue;
      }
      if (o.kind != kGate) continue;
      const size_t i = static_cast<size_t>(o.kplan);
      Program::Launch gl{};
      gl.kind = kGate;
      gl.first = static_cast<int>(prog.gates.size());
      gl.count = 1;
      gl.prefix_off = -1;
      gl.plan_step = kplans[i].plan_step;
      gl.bytes = prog.kernel_bytes[i];
      gl.flops = prog.kernel_flops[i];
      const GateDesc& g = gate_desc[i];
      gl.items = uint64_t{1} << (g.nCol - g.nHhi - g.pair2);  // threads per grid row (grid.y = 2^(nFhi + nHhi))
      gl.smem = (1 << g.nG) * 16 + (1 << g.nF) * 4;
      prog.gates.push_back(g);
      prog.launches.push_back(gl);
    }
  }
  for (TensorInfo* X : factor_ts) {
    FactorDesc f{};
    f.off = X->off;
    std::vector<std::pair<int, int>> m;
    // pass-local index: the batched slice bits, then the amplitude bits above them
    for (int x : X->bits) m.emplace_back(x < 0 ? prog.b + (-1 - x) : slice_pos(x), X->pos(x));
    f.map = make_runs(m);
    check_extent(runs_max(f.map), X->size(), "final factor");
    prog.factors.push_back(f);
  }
  // lookup tables only pay when walking the maps costs more than the table copy each CTA makes
  int max_runs = 0;
  for (const FactorDesc& f : prog.factors) max_runs = std::max(max_runs, f.map.n);
  if (!prog.factors.empty() && static_cast<int>(prog.factors.size()) <= kFinalTabFactors && prog.b + nA <= 20 &&
      max_runs > 3) {
    for (const FactorDesc& f : prog.factors)
      for (int h = 0; h < 2; ++h)
        for (uint64_t e = 0; e < 1024; ++e)
          prog.final_tab.push_back(static_cast<uint32_t>(eval_runs(f.map, e << (10 * h))));
    // lead factor: one that carries every batched slice bit (a bijection between the
    // pass-local slice index and its storage offset). k_final then walks ITS storage order
    // (coalesced loads of the one large operand) and recovers the slice index through the
    // inverse map, appended as one more table pair.
    if (nA == 0 && !env_int("QCG_FINAL_NO_LEAD", 0))
      for (size_t j = 0; j < factor_ts.size() && prog.final_lead < 0; ++j)
        if (static_cast<int>(factor_ts[j]->bits.size()) == prog.b && prog.b >= 12) {
          std::vector<std::pair<int, int>> inv;
          for (int x : factor_ts[j]->bits) inv.emplace_back(factor_ts[j]->pos(x), slice_pos(x));
          const Runs r = make_runs(inv);
          for (int h = 0; h < 2; ++h)
            for (uint64_t e = 0; e < 1024; ++e)
              prog.final_tab.push_back(static_cast<uint32_t>(eval_runs(r, e << (10 * h))));
          prog.final_lead = static_cast<int>(j);
        }
    // the lead factor's producer, when it is a plain gate launch, does the final product and
    // sum in its epilogue (k_gate_reduce): its result tensor is neither written nor re-read
    if (prog.final_lead >= 0 && !env_int("QCG_FINAL_NO_FUSE", 0)) {
      auto it = producer_op.find(factor_ts[static_cast<size_t>(prog.final_lead)]);
      if (it != producer_op.end() && ops[static_cast<size_t>(it->second)].kind == kGate) {
        const int li = ops[static_cast<size_t>(it->second)].level;
        Program::Launch& L = prog.launches[static_cast<size_t>(li)];
        GateDesc& g = prog.gates[static_cast<size_t>(L.first)];
        if (L.kind == kGate && !g.pair2 && g.nS <= 2) {
          g.reduce = 1;
          prog.final_fused = li;
          const double cbytes = 16.0 * std::ldexp(1.0, prog.b);
          L.bytes -= cbytes;  // the result tensor is not written
          prog.moved_bytes -= cbytes * static_cast<double>(prog.passes);
        }
      }
    }
  }
  if (prog.launches.size() != prog.launch_deps.size()) throw std::logic_error("launch groups and launches differ");
  for (Program::Launch& L : prog.launches) L.per_pass = 0;
  for (const Op& o : ops)
    if (o.out->per_pass) prog.launches[o.level].per_pass = 1;
  // ---- memory-plan validation: in the arena, and disjoint while simultaneously live ----
  {
    std::vector<TensorInfo*> live_ts;
    for (TensorInfo* X : arena_ts)
      if (!fused_away.count(X)) live_ts.push_back(X);
    for (TensorInfo* X : live_ts)
      if (X->off < prog.static_elems || X->off + X->size() > prog.arena_elems)
        throw std::logic_error("tensor placed outside the workspace");
    for (TensorInfo* X : statics)
      if (X->off < 0 || X->off + X->size() > prog.static_elems)
        throw std::logic_error("initial tensor placed outside the static region");
    for (size_t i = 0; i < live_ts.size(); ++i)
      for (size_t j = i + 1; j < live_ts.size(); ++j) {
        const TensorInfo *a = live_ts[i], *b = live_ts[j];
        const bool live_together = !(before(a->end, b->start) || before(b->end, a->start));
        const bool overlap = a->off < b->off + b->size() && b->off < a->off + a->size();
        if (live_together && overlap) throw std::logic_error("memory plan aliases two live tensors");
      }
  }
  return prog;
}

std::string describe_program(const Program& prog) {
  std::string out;
  char buf[512];
  std::snprintf(buf, sizeof buf, "mode=%s M=%d b=%d passes=%llu arena=%.3f GB launches=%zu\n",
                prog.mode == kKet ? "ket" : "density", prog.M, prog.b,
                static_cast<unsigned long long>(prog.passes), prog.arena_elems * 16e-9, prog.launches.size());
  out += buf;
  const bool tiles_detail = std::getenv("QCG_DESCRIBE_TILES") != nullptr;
  if (tiles_detail) {
    std::string fb = "  factors:";
    for (const FactorDesc& f : prog.factors) {
      int bits = 0;
      for (int r = 0; r < f.map.n; ++r) bits += f.map.len[r];
      fb += " " + std::to_string(bits);
    }
    out += fb + "\n";
  }
  for (size_t i = 0; i < prog.launches.size(); ++i) {
    const Program::Launch& L = prog.launches[i];
    const char* kind = L.kind == kTile     ? "tiles"
                       : L.kind == kForest ? "forest"
                       : L.kind == kGate   ? "gate"
                       : L.kind == kChain  ? "chain"
                       : L.kind == kGemm   ? "gemm"
                                           : "pair";
    if (tiles_detail && L.kind == kTile) {
      for (int k = 0; k < L.count; ++k) {
        const StepDesc& d = prog.tiles[L.first + k];
        std::string dl;
        for (int q = prog.flow_dep_off[L.dep_off + k]; q < prog.flow_dep_off[L.dep_off + k + 1]; ++q)
          dl += std::to_string(prog.flow_deps[q]) + ",";
        std::snprintf(buf, sizeof buf,
                      "    tile %d: A@%lld B@%lld C@%lld nS=%d nTA=%d nTB=%d nTC=%d nG=%d deps=%s cont=%d conly=%d\n", k,
                      static_cast<long long>(d.offA), static_cast<long long>(d.offB), static_cast<long long>(d.offC),
                      d.nS, d.nTA, d.nTB, d.nTC, d.nG, dl.c_str(), prog.flow_cont[L.first + k],
                      prog.flow_conly[L.first + k]);
        out += buf;
      }
    }
    std::snprintf(buf, sizeof buf, "  [%zu] %-5s steps=%d items=%llu smem=%d bytes=%.4g", i, kind, L.count,
                  static_cast<unsigned long long>(L.items), L.smem, L.bytes);
    out += buf;
    if (L.kind == kTile && L.npre > 0) out += " prefetch=" + std::to_string(L.npre);
    if (!L.per_pass) out += " invariant";
    if (i < prog.launch_deps.size() && !prog.launch_deps[i].empty()) {
      out += " deps=";
      for (size_t q = 0; q < prog.launch_deps[i].size(); ++q)
        out += (q ? "," : "") + std::to_string(prog.launch_deps[i][q]);
    }
    if (L.kind == kForest) {
      int steps = 0, phases = 0, leaves = 0;
      for (int u = L.first; u < L.first + L.count; ++u) {
        const ForestUnit& fu = prog.forest_units[u];
        phases = std::max(phases, prog.forest_image[fu.img]);
        steps += prog.forest_image[fu.img + 1];
        leaves += fu.nleaves;
      }
      std::snprintf(buf, sizeof buf, " units=%d steps=%d max_phases=%d staged_leaves=%d", L.count, steps, phases, leaves);
      out += buf;
    } else if (L.kind == kGate) {
      const GateDesc& g = prog.gates[L.first];
      std::snprintf(buf, sizeof buf, " plan_step=%d nG=%d nS=%d nF=%d nFhi=%d nHhi=%d nCol=%d", L.plan_step, g.nG,
                    g.nS, g.nF, g.nFhi, g.nHhi, g.nCol);
      out += buf;
      if (g.reduce) out += " +final (product with the other rank-0 factors and slice sum in the epilogue)";
    } else if (L.kind == kGemm) {
      const Program::GemmOp& g = prog.gemms[L.first];
      std::snprintf(buf, sizeof buf, " plan_step=%d M=2^%d N=2^%d K=2^%d batch=2^%d (DMMA)", L.plan_step, g.nM, g.nN,
                    g.nK, g.nG);
      out += buf;
    } else if (L.kind == kPair) {
      const PairDesc& d = prog.pairs[L.first];
      std::snprintf(buf, sizeof buf,
                    " last_step=%d S1=%d S2=%d P=%d Q=%d R=%d(lo%d mid%d hi%d) F2=%d cols=%d Hhi=%d G1x=%d G2=%d",
                    L.plan_step, d.nS1, d.nS2, d.nP, d.nQ, d.nR, d.nRlo, d.nRmid, d.nRhi, d.nF2, d.nCol, d.nHhi,
                    d.nG1x, d.nG2);
      out += buf;
    } else if (L.kind == kChain) {
      const ChainDesc& c = prog.chains[L.first];
      std::snprintf(buf, sizeof buf, " last_step=%d stages=%d nT0=%d nGrid=%d nTmax=%d gElems=%d img=%d nIter=%d |", L.plan_step,
                    c.nStages, c.nT0, c.nGrid, c.nTmax, c.gElems, c.imgInts, c.nIter);
      out += buf;
      for (int j = 0; j < c.nStages; ++j) {
        std::snprintf(buf, sizeof buf, " (S%d Kp%d F%d G%d)", c.st[j].nS, c.st[j].nKp, c.st[j].nF, c.st[j].nG);
        out += buf;
      }
    }
    out += "\n";
  }
  return out;
}

WorkspaceTooLarge::WorkspaceTooLarge(int b)
    : std::runtime_error("a batched intermediate of 2^" + std::to_string(b) + " elements"), bits(b) {}

Program plan_program(const Payload& p, Mode mode, uint64_t budget_bytes, int max_batch_bits) {
  return plan_program(std::vector<const Payload*>{&p}, mode, budget_bytes, max_batch_bits);
}

Program plan_program(const std::vector<const Payload*>& amps, Mode mode, uint64_t budget_bytes, int max_batch_bits) {
  const Payload& p = *amps.at(0);
  const int id_bits = static_cast<int>(p.cut.size()) * (mode == kKet ? 1 : 2);
  // Keep pass-local slice counts bounded so per-pass bookkeeping stays small.
  int b0 = std::min(id_bits, 26);
  if (max_batch_bits >= 0) b0 = std::min(b0, max_batch_bits);
  std::string why;
  for (int b = b0; b >= 0; --b) {
    try {
      Program prog = build_program(amps, mode, b);
      if (static_cast<uint64_t>(prog.arena_elems) * 16ull <= budget_bytes) return prog;
      why = "device workspace of " + std::to_string(prog.arena_elems * 16) + " bytes";
    } catch (const WorkspaceTooLarge& e) {
      why = std::string("device workspace with ") + e.what();
    }
  }
  throw std::runtime_error(why + " for one slice exceeds the memory budget of " + std::to_string(budget_bytes) +
                           " bytes");
}

}  // namespace qcg
