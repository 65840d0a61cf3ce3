// cut_search — SURVEY §8(f)-1 extended to the cut: a joint search over the M cut edges and
// the elimination order, scored by the planned peak rank of the reference's OWN
// plan_from_order (proj/core/src/contraction.cpp:118-262) on the cut network.
//
// Why: the reference's GA (cutting.cpp:158-270) scores a cut by the vertex-graph width
// of the remaining network (cutting.cpp:131-135), and best_plan compares only two orders
// (contraction.cpp:264-278). On BASELINE config 3 (QAOA p=2, N=50, k=14) the GA cut has
// width 18 but every plan over it peaks at >= 35 legs (2^35 x 16 B per ket tensor), so
// config 3 cannot run in any view. Choosing the cut edges *for* the planned peak (slice
// the legs that the largest intermediates of a good order share, then anneal cut and order
// together) is the standard slicing move of sliced tensor-network simulators and keeps
// everything else the reference's: same network, same number of cut edges M (2^M ket
// slices), same apply_cut / plan_from_order / payload.
//
// Search, per thread (independent seeds, best kept):
//   1. order for the uncut network: reference min-degree / min-fill restarts and a
//      leg-aware greedy, then simulated annealing over the order;
//   2. greedy slicing with that order: M times, cut the edge (among the legs of the
//      current peak-rank intermediates) whose removal gives the best (peak, cost);
//   3. joint annealing: order moves (swap / move one vertex) and cut moves (replace one
//      cut edge by a leg of a large intermediate).
// Candidates are scored by `FastPlan`, an integer restatement of plan_from_order's
// structure (fill-graph parents, parking, smallest-merge absorption, peak and cost); it is
// cross-checked against the reference's plan_from_order on sampled orders at start-up and
// on the final answer, and the emitted plan is the reference's own.
//
//   cut_search --payload in.json --out out.json [--M m] [--evals N] [--seed S]
//              [--threads T] [--split-2q 1] [--objective peak|batched] [--bound R] [--cap C]
//
// --objective peak (default): lexicographic (planned peak rank, reference cost estimate
//   sum 4^work_rank), the reference's own plan metrics.
// --objective batched: the B200 engine's cost model. The engine keeps every cut variable
//   as a tensor bit ("batch bit") on the tensors that depend on it and runs all 2^M slices
//   in one pass, so a step costs 16 B x (2^(ra+ca) + 2^(rb+cb) + 2^(rr+cr)), c = number of
//   cut edges with an endpoint inside the tensor's subtree; slice-invariant steps (c = 0)
//   run once. Minimises that total traffic subject to the per-slice peak <= --bound
//   (BASELINE's rank bound) and the largest batched tensor <= 2^--cap elements;
//   --depth-weight W adds W bytes per level of the step DAG's depth (the engine's
//   latency per dependent level, ~3.5 us x HBM bandwidth ~ 2.3e7 B).
//
// Built by oracle/Makefile against the reference library (maintainer tool, like the
// reference CLI; not part of the GPU engine).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "qcut/contraction.hpp"
#include "qcut/cutting.hpp"
#include "qcut/ordering.hpp"
#include "qcut/serialize.hpp"

#include "search_common.hpp"
#include "../paper_2010_14962_b200/csrc/program.hpp"

namespace {

using qsearch::Score;

// Structural skeleton of a network: vertex ids in map order, each vertex's legs as edge
// ids in leg order, and each edge's endpoints. Cutting an edge drops it from both endpoint
// leg lists in place, order kept (apply_cut's slice_leg_map, tensor.cpp:64-77).
struct Skeleton {
  std::vector<int> vid;                    // index -> vertex id (ascending)
  std::unordered_map<int, int> index;      // vertex id -> index
  std::vector<std::vector<int>> legs;      // index -> edge ids by leg position
  std::vector<std::pair<int, int>> ends;   // edge id -> (u index, v index), -1 if absent
  int n_edges = 0;

  explicit Skeleton(const qcut::TensorNetwork& tn) {
    for (const auto& [id, t] : tn.vertices) {
      index[id] = static_cast<int>(vid.size());
      vid.push_back(id);
      legs.emplace_back(static_cast<size_t>(t.rank), -1);
    }
    for (const auto& e : tn.edges) n_edges = std::max(n_edges, e.id + 1);
    ends.assign(static_cast<size_t>(n_edges), {-1, -1});
    for (const auto& e : tn.edges) {
      const int u = index.at(e.u), v = index.at(e.v);
      legs[u][e.leg_u] = e.id;
      legs[v][e.leg_v] = e.id;
      ends[e.id] = {u, v};
    }
  }
};

struct Objective {
  bool batched = false;
  int bound = 26;  // per-slice peak rank allowed (batched)
  int cap = 31;    // largest batched tensor, log2 elements (batched)
  double depth_w = 0;  // batched: bytes-equivalent cost per level of the step DAG's depth
                       // (the engine's dependent-launch / dataflow-level latency)
};

// plan_from_order restated on integers (contraction.cpp:118-262): same fill-graph parent
// rule, same parking, same absorption order (smallest merged rank, ties to the smallest
// root id), same peak and cost. `cut` marks removed edges; `order` holds vertex indices.
class FastPlan {
 public:
  explicit FastPlan(const Skeleton& sk, Objective obj = {})
      : sk_(sk), n_(static_cast<int>(sk.vid.size())), w_((n_ + 63) / 64), obj_(obj) {
    nb_.assign(static_cast<size_t>(n_) * w_, 0);
    mark_.assign(static_cast<size_t>(sk.n_edges), 0);
  }

  // The active objective's score: eval()'s (peak, sum 4^work), or, batched, (bound + cap
  // violation, batched bytes).
  Score score(const std::vector<int>& order, const std::vector<char>& cut, std::vector<double>* heat = nullptr) {
    const Score r = eval(order, cut, heat);
    if (!obj_.batched || r.peak >= (1 << 29)) return r;
    return Score{std::max(0, r.peak - obj_.bound) + std::max(0, bpeak_ - obj_.cap), bbytes_ + obj_.depth_w * depth_};
  }
  double batched_bytes() const { return bbytes_; }
  int batched_peak() const { return bpeak_; }
  int depth() const { return depth_; }

  // Returns the score; when `heat` is given, adds 2^(r - peak) to heat[e] for every edge e
  // on a result tensor of rank r >= peak - 1 (the legs worth slicing).
  Score eval(const std::vector<int>& order, const std::vector<char>& cut, std::vector<double>* heat = nullptr) {
    const int n = n_;
    pos_.assign(static_cast<size_t>(n), 0);
    for (int i = 0; i < n; ++i) pos_[order[i]] = i;
    std::fill(nb_.begin(), nb_.end(), 0);
    for (int e = 0; e < sk_.n_edges; ++e) {
      const auto [u, v] = sk_.ends[e];
      if (u < 0 || cut[e] || u == v) continue;
      set(u, v);
      set(v, u);
    }
    parent_.assign(static_cast<size_t>(n), -1);
    std::vector<uint64_t> later(static_cast<size_t>(w_));
    for (int i = 0; i < n; ++i) {
      const int v = order[i];
      // later = neighbours eliminated after v
      int best = -1;
      lat_.clear();
      for (int k = 0; k < w_; ++k) {
        uint64_t b = nb_[static_cast<size_t>(v) * w_ + k];
        later[k] = 0;
        while (b) {
          const int u = k * 64 + __builtin_ctzll(b);
          b &= b - 1;
          if (pos_[u] > i) {
            later[k] |= 1ull << (u & 63);
            lat_.push_back(u);
            if (best < 0 || pos_[u] < pos_[best]) best = u;
          }
        }
      }
      for (int u : lat_) {
        uint64_t* row = &nb_[static_cast<size_t>(u) * w_];
        for (int k = 0; k < w_; ++k) row[k] |= later[k];
        row[u >> 6] &= ~(1ull << (u & 63));
      }
      parent_[v] = best;
    }
    // merge simulation
    cur_.assign(static_cast<size_t>(n), {});
    cm_.assign(static_cast<size_t>(n), 0);
    int ci = 0;
    for (int e = 0; e < sk_.n_edges; ++e)
      if (cut[e]) {
        const auto [u, v] = sk_.ends[e];
        cm_[u] |= 1ull << (ci & 63);
        cm_[v] |= 1ull << (ci & 63);
        ++ci;
      }
    bbytes_ = 0;
    depth_ = 0;
    dep_.assign(static_cast<size_t>(n), 0);
    bpeak_ = 0;
    for (int v = 0; v < n; ++v) {
      cur_[v].clear();
      for (int e : sk_.legs[v])
        if (!cut[e]) cur_[v].push_back(e);
      bpeak_ = std::max(bpeak_, static_cast<int>(cur_[v].size()) + __builtin_popcountll(cm_[v]));
    }
    parked_.assign(static_cast<size_t>(n), {});
    Score s{0, 0.0};
    steps_r_.clear();
    for (int i = 0; i < n; ++i) {
      const int v = order[i];
      std::vector<int>& pending = parked_[v];
      std::sort(pending.begin(), pending.end());  // vertex index order == vertex id order
      while (!pending.empty()) {
        std::vector<int>& la = cur_[v];
        ++stamp_;
        for (int e : la) mark_[e] = stamp_;
        size_t pick = pending.size();
        int pick_r = 0, pick_c = 0;
        for (size_t j = 0; j < pending.size(); ++j) {
          const std::vector<int>& lb = cur_[pending[j]];
          int c = 0;
          for (int e : lb) c += mark_[e] == stamp_;
          if (c == 0) continue;
          const int r = static_cast<int>(la.size() + lb.size()) - 2 * c;
          if (pick == pending.size() || r < pick_r) pick = j, pick_r = r, pick_c = c;
        }
        if (pick == pending.size()) return Score{};  // plan_from_order would throw
        const int sidx = pending[pick];
        pending.erase(pending.begin() + static_cast<long>(pick));
        std::vector<int>& lb = cur_[sidx];
        ++stamp_;
        for (int e : lb) mark_[e] = stamp_;
        merged_.clear();
        for (int e : la)
          if (mark_[e] != stamp_) merged_.push_back(e);
        ++stamp_;
        for (int e : la) mark_[e] = stamp_;
        for (int e : lb)
          if (mark_[e] != stamp_) merged_.push_back(e);
        const int work = static_cast<int>(la.size() + lb.size()) - pick_c;
        {
          const int ca = __builtin_popcountll(cm_[v]), cb = __builtin_popcountll(cm_[sidx]);
          const uint64_t cr = cm_[v] | cm_[sidx];
          const int rr = static_cast<int>(merged_.size()) + __builtin_popcountll(cr);
          bbytes_ += 16.0 * (std::ldexp(1.0, static_cast<int>(la.size()) + ca) +
                             std::ldexp(1.0, static_cast<int>(lb.size()) + cb) + std::ldexp(1.0, rr));
          bpeak_ = std::max(bpeak_, rr);
          cm_[v] = cr;
          dep_[v] = std::max(dep_[v], dep_[sidx]) + 1;  // the step waits for both operands
          depth_ = std::max(depth_, dep_[v]);
        }
        la.swap(merged_);
        lb.clear();
        s.peak = std::max(s.peak, pick_r);
        s.cost += std::pow(4.0, work);
        if (heat) steps_r_.push_back({pick_r, v, la});
      }
      if (!cur_[v].empty()) {
        if (parent_[v] < 0) return Score{};
        parked_[parent_[v]].push_back(v);
      }
    }
    if (heat) {
      for (const auto& st : steps_r_)
        if (st.r >= s.peak - 1)
          for (int e : st.legs) (*heat)[e] += std::ldexp(1.0, st.r - s.peak);
    }
    return s;
  }

 private:
  struct StepLegs {
    int r, v;
    std::vector<int> legs;
  };
  void set(int a, int b) { nb_[static_cast<size_t>(a) * w_ + (b >> 6)] |= 1ull << (b & 63); }
  const Skeleton& sk_;
  int n_, w_;
  Objective obj_;
  std::vector<uint64_t> cm_;  // per vertex: cut edges with an endpoint in its merged subtree
  double bbytes_ = 0;
  int bpeak_ = 0;
  int depth_ = 0;
  std::vector<int> dep_;  // per vertex: dependency depth of its merged tensor
  std::vector<uint64_t> nb_;
  std::vector<int> pos_, parent_, lat_, merged_;
  std::vector<std::vector<int>> cur_, parked_;
  std::vector<int> mark_;
  int stamp_ = 0;
  std::vector<StepLegs> steps_r_;
};

qcut::CutSet cut_list(const std::vector<char>& cut) {
  qcut::CutSet c;
  for (size_t e = 0; e < cut.size(); ++e)
    if (cut[e]) c.push_back(static_cast<int>(e));
  return c;
}

Score reference_score(const qcut::TensorNetwork& tn, const std::vector<char>& cut, const std::vector<int>& order,
                      const Skeleton& sk, qcut::ContractionPlan* out = nullptr) {
  const qcut::CutSet c = cut_list(cut);
  const qcut::TensorNetwork sub = qcut::apply_cut(tn, c, qcut::Assignment(c.size(), 0));
  qcut::EliminationOrder ord;
  for (int i : order) ord.push_back(sk.vid[i]);
  qcut::ContractionPlan p = qcut::plan_from_order(sub, ord);
  if (out) *out = p;
  return Score{p.peak_rank, p.cost_estimate};
}

// The B200 engine's own host planner (paper_2010_14962_b200/csrc/program.cpp) on a
// candidate: bytes its kernels move per amplitude after its fusions (the criterion that
// tracks measured time; the FastPlan byte model counts every intermediate).
double engine_moved(const qcut::TensorNetwork& tn, const std::vector<char>& cut, const std::vector<int>& order,
                    const Skeleton& sk, int max_rank) {
  qcut::ContractionPlan plan;
  reference_score(tn, cut, order, sk, &plan);
  const qcut::Payload p{tn, cut_list(cut), plan, std::max(max_rank, plan.peak_rank)};
  const std::string js = qcut::encode_payload(p);
  try {
    const qcg::Payload ep = qcg::decode_payload(js.data(), js.size());
    const qcg::Program prog = qcg::plan_program(ep, qcg::kKet, uint64_t{100} << 30);
    return prog.moved_bytes;
  } catch (const std::exception&) {
    return 1e300;
  }
}

double energy(const Score& s, const Objective& obj) {
  return obj.batched ? 4.0 * s.peak + std::log2(s.cost) : s.peak + 0.05 * std::log2(s.cost);
}

struct Result {
  Score s;
  std::vector<int> order;
  std::vector<char> cut;
  double engine = 1e300;  // engine-moved bytes of the engine-best state (engine_every > 0)
};

// One independent search chain (steps 1-3 of the header).
Result chain(const qcut::TensorNetwork& tn, const Skeleton& sk, const std::vector<int>& valid_edges, int M,
             long evals, uint64_t seed, const Objective& obj, long engine_every, int max_rank) {
  std::mt19937_64 rng(seed);
  FastPlan fp(sk, obj);
  const int n = static_cast<int>(sk.vid.size());
  std::vector<char> cut(static_cast<size_t>(sk.n_edges), 0);
  auto to_idx = [&](const qcut::EliminationOrder& o) {
    std::vector<int> r;
    r.reserve(o.size());
    for (int v : o) r.push_back(sk.index.at(v));
    return r;
  };
  auto mutate = [&](std::vector<int>& o) {
    const size_t i = rng() % n, j = rng() % n;
    if (rng() & 1) {
      std::swap(o[i], o[j]);
    } else {
      const int v = o[i];
      o.erase(o.begin() + static_cast<long>(i));
      o.insert(o.begin() + static_cast<long>(j), v);
    }
  };
  // 1. order for the uncut network
  const qcut::Graph g = qcut::network_graph(tn);
  std::vector<int> ord;
  Score best_s;
  auto take = [&](std::vector<int> o) {
    const Score s = fp.score(o, cut);
    if (s < best_s) best_s = s, ord = std::move(o);
  };
  for (int r = 0; r < 16; ++r) {
    take(to_idx(qcut::min_degree_order(g, rng())));
    take(to_idx(qcut::min_fill_order(g, rng())));
    take(to_idx(qsearch::leg_greedy(tn, rng)));
  }
  auto anneal_order = [&](long iters, double t0) {
    std::vector<int> cur = ord;
    Score cs = best_s;
    for (long it = 0; it < iters; ++it) {
      const double temp = t0 * (1.0 - static_cast<double>(it) / std::max(1L, iters)) + 0.05;
      std::vector<int> cand = cur;
      mutate(cand);
      const Score s = fp.score(cand, cut);
      if (s < best_s) best_s = s, ord = cand;
      const double d = energy(s, obj) - energy(cs, obj);
      if (d <= 0 || std::uniform_real_distribution<double>(0, 1)(rng) < std::exp(-d / temp)) cur.swap(cand), cs = s;
    }
  };
  anneal_order(evals / 4, 2.0);
  // 2. greedy slicing with the current order
  std::vector<double> heat(static_cast<size_t>(sk.n_edges));
  for (int m = 0; m < M; ++m) {
    std::fill(heat.begin(), heat.end(), 0.0);
    fp.score(ord, cut, &heat);
    std::vector<int> cand;
    for (int e : valid_edges)
      if (!cut[e] && (heat[e] > 0 || obj.batched)) cand.push_back(e);
    int pick = -1;
    Score ps;
    for (int e : cand) {
      cut[e] = 1;
      const Score s = fp.score(ord, cut);
      cut[e] = 0;
      if (s < ps) ps = s, pick = e;
    }
    if (pick < 0) {  // nothing large left: any valid edge
      for (int e : valid_edges)
        if (!cut[e]) { pick = e; break; }
    }
    cut[pick] = 1;
    best_s = fp.score(ord, cut);
    anneal_order(evals / (8 * M), 0.5);
  }
  // 3. joint annealing over (cut, order)
  std::vector<int> cur_o = ord;
  std::vector<char> cur_c = cut;
  Score cs = best_s;
  std::vector<char> best_c = cut;
  std::vector<int> cut_ids = cut_list(cut);
  const long iters = evals / 2;
  double eng_best = 1e300;
  std::vector<int> eng_o;
  std::vector<char> eng_c;
  if (engine_every > 0 && best_s.peak == 0) {
    eng_best = engine_moved(tn, cut, ord, sk, max_rank);
    eng_o = ord;
    eng_c = cut;
  }
  for (long it = 0; it < iters; ++it) {
    const double temp = 1.0 * (1.0 - static_cast<double>(it) / std::max(1L, iters)) + 0.03;
    std::vector<int> co = cur_o;
    std::vector<char> cc = cur_c;
    if (rng() % 4 == 0) {
      // cut move: drop one cut edge, add a leg of a large intermediate (or any edge)
      std::vector<int> ids = cut_list(cc);
      const int drop = ids[rng() % ids.size()];
      std::fill(heat.begin(), heat.end(), 0.0);
      fp.score(co, cc, &heat);
      std::vector<int> cand;
      for (int e : valid_edges)
        if (!cc[e] && (heat[e] > 0 || rng() % (obj.batched ? 2 : 64) == 0)) cand.push_back(e);
      if (cand.empty()) continue;
      cc[drop] = 0;
      cc[cand[rng() % cand.size()]] = 1;
    } else {
      mutate(co);
    }
    const Score s = fp.score(co, cc);
    if (s < best_s) best_s = s, ord = co, best_c = cc;
    if (engine_every > 0 && it % engine_every == 0 && cs.peak == 0) {  // feasible states only
      // engine-in-the-loop: re-score the chain's current state with the engine's planner
      const double em = engine_moved(tn, cur_c, cur_o, sk, max_rank);
      if (em < eng_best) eng_best = em, eng_o = cur_o, eng_c = cur_c;
    }
    const double d = energy(s, obj) - energy(cs, obj);
    if (d <= 0 || std::uniform_real_distribution<double>(0, 1)(rng) < std::exp(-d / temp))
      cur_o.swap(co), cur_c.swap(cc), cs = s;
  }
  if (engine_every > 0) {
    // the FastPlan-best too (the engine-best is only taken among feasible states)
    const double em = best_s.peak == 0 ? engine_moved(tn, best_c, ord, sk, max_rank) : 1e300;
    if (em <= eng_best || eng_o.empty()) return Result{best_s, ord, best_c, em};
    FastPlan fe(sk, obj);
    return Result{fe.score(eng_o, eng_c), eng_o, eng_c, eng_best};
  }
  return Result{best_s, ord, best_c};
}

}  // namespace

int main(int argc, char** argv) {
  std::string in, out;
  long evals = 200000;
  uint64_t seed = 1;
  int M = -1, threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  bool split = false;
  Objective obj;
  bool emit_all = false;
  long engine_every = 0;  // > 0: every that many joint-annealing moves, score the chain's state with
                          // the engine's host planner; the answer is the engine-best state  // also write every chain's best as <out>.t<k>.json (re-ranking by the engine)
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--payload") in = v;
    else if (k == "--out") out = v;
    else if (k == "--evals") evals = std::stol(v);
    else if (k == "--seed") seed = std::stoull(v);
    else if (k == "--M") M = std::stoi(v);
    else if (k == "--threads") threads = std::stoi(v);
    else if (k == "--split-2q") split = v == "1";
    else if (k == "--objective") obj.batched = v == "batched";
    else if (k == "--bound") obj.bound = std::stoi(v);
    else if (k == "--cap") obj.cap = std::stoi(v);
    else if (k == "--depth-weight") obj.depth_w = std::stod(v);
    else if (k == "--emit-all") emit_all = v == "1";
    else if (k == "--engine-every") engine_every = std::stol(v);
  }
  std::ifstream f(in);
  std::stringstream ss;
  ss << f.rdbuf();
  qcut::Payload p = qcut::decode_payload(ss.str());
  if (M < 0) M = static_cast<int>(p.cut.size());
  const Score start{p.plan.peak_rank, p.plan.cost_estimate};
  int n_split = 0;
  if (split) n_split = qsearch::split_2q(p.tn);
  const auto t0 = std::chrono::steady_clock::now();
  const Skeleton sk(p.tn);
  std::vector<int> valid_edges;
  for (int e = 0; e < sk.n_edges; ++e)
    if (sk.ends[e].first >= 0 && sk.ends[e].first != sk.ends[e].second) valid_edges.push_back(e);

  // cross-check FastPlan against the reference's plan_from_order on sampled (cut, order)
  {
    std::mt19937_64 rng(seed ^ 0x5eedULL);
    FastPlan fp(sk);
    const qcut::Graph g = qcut::network_graph(p.tn);
    for (int t = 0; t < 6; ++t) {
      std::vector<char> cut(static_cast<size_t>(sk.n_edges), 0);
      if (t % 2) {
        for (int e : p.cut) cut[e] = 1;
      } else {
        for (int m = 0; m < M; ++m) cut[valid_edges[rng() % valid_edges.size()]] = 1;
      }
      qcut::EliminationOrder o = t < 2 ? qcut::min_fill_order(g, rng()) : qcut::min_degree_order(g, rng());
      std::vector<int> oi;
      for (int v : o) oi.push_back(sk.index.at(v));
      if (t >= 4) std::shuffle(oi.begin(), oi.end(), rng);
      const Score a = fp.eval(oi, cut);
      Score b;
      try {
        b = reference_score(p.tn, cut, oi, sk);
      } catch (const std::exception&) {
        b = Score{};
      }
      if (a.peak != b.peak || std::abs(a.cost - b.cost) > 1e-9 * b.cost) {
        std::fprintf(stderr, "FastPlan mismatch: fast (%d, %g) reference (%d, %g)\n", a.peak, a.cost, b.peak, b.cost);
        return 3;
      }
    }
  }

  std::vector<Result> res(static_cast<size_t>(threads));
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { res[t] = chain(p.tn, sk, valid_edges, M, evals, seed * 1000003ULL + t, obj, engine_every, p.max_rank); });
  for (auto& th : pool) th.join();
  size_t bi = 0;
  for (size_t t = 1; t < res.size(); ++t)
    if (engine_every > 0 ? res[t].engine < res[bi].engine : res[t].s < res[bi].s) bi = t;
  const Result& best = res[bi];

  if (emit_all)
    for (size_t t = 0; t < res.size(); ++t) {
      qcut::ContractionPlan pt;
      reference_score(p.tn, res[t].cut, res[t].order, sk, &pt);
      const qcut::CutSet ct = cut_list(res[t].cut);
      std::ofstream ot(out + ".t" + std::to_string(t) + ".json");
      ot << qcut::encode_payload(qcut::Payload{p.tn, ct, pt, std::max(p.max_rank, pt.peak_rank)});
    }
  qcut::ContractionPlan plan;
  const Score chk = reference_score(p.tn, best.cut, best.order, sk, &plan);
  FastPlan fin(sk, obj);
  const Score fast = fin.eval(best.order, best.cut);
  if (chk.peak != fast.peak || std::abs(chk.cost - fast.cost) > 1e-9 * chk.cost) {
    std::fprintf(stderr, "final FastPlan mismatch: %d vs reference %d\n", fast.peak, chk.peak);
    return 3;
  }
  const qcut::CutSet cut = cut_list(best.cut);
  qcut::Payload outp{p.tn, cut, plan, std::max(p.max_rank, plan.peak_rank)};
  std::ofstream o(out);
  o << qcut::encode_payload(outp);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::string cs;
  for (size_t i = 0; i < cut.size(); ++i) cs += (i ? "," : "") + std::to_string(cut[i]);
  std::string per;
  for (size_t t = 0; t < res.size(); ++t) {
    char buf[64];
    if (obj.batched) std::snprintf(buf, sizeof buf, "%.4g", res[t].s.cost);
    else std::snprintf(buf, sizeof buf, "%d", res[t].s.peak);
    per += (t ? "," : "") + std::string(buf);
  }
  std::printf("{\"reference_peak\":%d,\"reference_cost\":%.6g,\"peak\":%d,\"cost\":%.6g,\"M\":%d,\"cut\":[%s],"
              "\"steps\":%zu,\"evals_per_thread\":%ld,\"threads\":%d,\"thread_peaks\":[%s],\"secs\":%.3f,"
              "\"split_2q\":%d,\"objective\":\"%s\",\"batched_bytes\":%.6g,\"batched_peak\":%d,\"depth\":%d,\"depth_weight\":%.4g,\"engine_every\":%ld,\"engine_moved\":%.6g}\n",
              start.peak, start.cost, plan.peak_rank, plan.cost_estimate, M, cs.c_str(), plan.steps.size(), evals,
              threads, per.c_str(), secs, n_split, obj.batched ? "batched" : "peak", fin.batched_bytes(),
              fin.batched_peak(), fin.depth(), obj.depth_w, engine_every, best.engine);
  return 0;
}
