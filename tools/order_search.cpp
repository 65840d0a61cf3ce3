// order_search — SURVEY §8(f)-1: a better host elimination order, fed through the
// reference's OWN plan_from_order (proj/core/src/contraction.cpp:118-262).
//
// The reference picks the lower-peak plan of (best_order's min-degree/min-fill
// winner, creation order) (contraction.cpp:264-278); the GA fitness is the vertex-graph
// width (cutting.cpp:131-135), not the leg peak the executor pays for. This tool keeps
// the network and the cut unchanged and searches elimination orders for the lowest
// planned peak rank (ties: lowest cost estimate), evaluating every candidate with the
// unmodified plan_from_order, then emits a standard payload (encode_payload) whose plan
// any reference backend or the B200 engine can run.
//
// Search: restarts of the reference heuristics (min-degree / min-fill with many
// seeds), a leg-aware greedy, then simulated annealing over the order with
// swap / move moves.
//
//   order_search --payload in.json --out out.json [--evals N] [--seed S]
// Built by oracle/Makefile against the reference library (a maintainer tool, like the
// reference CLI; not part of the GPU engine).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "qcut/contraction.hpp"
#include "qcut/cutting.hpp"
#include "qcut/ordering.hpp"
#include "qcut/serialize.hpp"

namespace {

struct Score {
  int peak = 1 << 30;
  double cost = 1e300;
  bool operator<(const Score& o) const { return peak != o.peak ? peak < o.peak : cost < o.cost; }
};

Score score(const qcut::TensorNetwork& tn, const qcut::EliminationOrder& ord) {
  qcut::ContractionPlan p = qcut::plan_from_order(tn, ord);
  return Score{p.peak_rank, p.cost_estimate};
}

// Leg-aware greedy: repeatedly eliminate the vertex whose neighbourhood (counted in
// legs of the current merged multigraph) is smallest.
qcut::EliminationOrder leg_greedy(const qcut::TensorNetwork& tn, std::mt19937_64& rng) {
  std::map<int, std::map<int, int>> adj;  // v -> (u -> multiplicity)
  for (const auto& [id, t] : tn.vertices) adj[id];
  for (const auto& e : tn.edges) {
    if (e.u == e.v) continue;
    ++adj[e.u][e.v];
    ++adj[e.v][e.u];
  }
  qcut::EliminationOrder ord;
  while (!adj.empty()) {
    int best = -1;
    long long best_key = 0;
    for (const auto& [v, nb] : adj) {
      long long legs = 0;
      for (const auto& kv : nb) legs += kv.second;
      const long long key = legs * 1024 + static_cast<long long>(rng() % 1024);
      if (best < 0 || key < best_key) {
        best = v;
        best_key = key;
      }
    }
    ord.push_back(best);
    // merge best into its neighbours pairwise (clique of its neighbourhood, legs summed)
    std::vector<std::pair<int, int>> nb(adj[best].begin(), adj[best].end());
    for (const auto& [u, m] : nb) adj[u].erase(best);
    for (size_t i = 0; i < nb.size(); ++i)
      for (size_t j = i + 1; j < nb.size(); ++j) {
        const int w = std::min(nb[i].second, nb[j].second);
        adj[nb[i].first][nb[j].first] += w;
        adj[nb[j].first][nb[i].first] += w;
      }
    adj.erase(best);
  }
  return ord;
}

}  // namespace

int main(int argc, char** argv) {
  std::string in, out;
  long evals = 20000;
  uint64_t seed = 1;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--payload") in = v;
    else if (k == "--out") out = v;
    else if (k == "--evals") evals = std::stol(v);
    else if (k == "--seed") seed = std::stoull(v);
  }
  std::ifstream f(in);
  std::stringstream ss;
  ss << f.rdbuf();
  qcut::Payload p = qcut::decode_payload(ss.str());
  // the plan is made on the cut network with all-zero digits (executor.cpp:33-43)
  qcut::TensorNetwork sub = qcut::apply_cut(p.tn, p.cut, qcut::Assignment(p.cut.size(), 0));
  const qcut::Graph g = qcut::network_graph(sub);
  const auto t0 = std::chrono::steady_clock::now();
  std::mt19937_64 rng(seed);

  qcut::EliminationOrder best_ord;
  Score best;
  auto consider = [&](const qcut::EliminationOrder& o) {
    Score s = score(sub, o);
    if (s < best) {
      best = s;
      best_ord = o;
    }
    return s;
  };
  const Score start{p.plan.peak_rank, p.plan.cost_estimate};
  qcut::EliminationOrder creation;
  for (const auto& [id, t] : sub.vertices) creation.push_back(id);
  consider(creation);
  for (int r = 0; r < 64; ++r) {
    consider(qcut::min_degree_order(g, rng()));
    consider(qcut::min_fill_order(g, rng()));
    consider(leg_greedy(sub, rng));
  }
  // simulated annealing over the order (moves: swap two, move one)
  qcut::EliminationOrder cur = best_ord;
  Score cur_s = best;
  const long sa = std::max(0L, evals - 192);
  for (long it = 0; it < sa; ++it) {
    const double temp = 2.0 * (1.0 - static_cast<double>(it) / std::max(1L, sa)) + 0.05;
    qcut::EliminationOrder cand = cur;
    const size_t n = cand.size();
    const size_t i = rng() % n, j = rng() % n;
    if (rng() & 1) {
      std::swap(cand[i], cand[j]);
    } else {
      const int v = cand[i];
      cand.erase(cand.begin() + static_cast<long>(i));
      cand.insert(cand.begin() + static_cast<long>(j), v);
    }
    const Score s = consider(cand);
    const double delta = (s.peak - cur_s.peak) + 0.05 * (std::log2(s.cost) - std::log2(cur_s.cost));
    if (delta <= 0 || std::uniform_real_distribution<double>(0, 1)(rng) < std::exp(-delta / temp)) {
      cur = std::move(cand);
      cur_s = s;
    }
  }
  qcut::ContractionPlan plan = qcut::plan_from_order(sub, best_ord);
  qcut::Payload outp{p.tn, p.cut, plan, std::max(p.max_rank, plan.peak_rank)};
  std::ofstream o(out);
  o << qcut::encode_payload(outp);
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"reference_peak\":%d,\"reference_cost\":%.6g,\"peak\":%d,\"cost\":%.6g,\"steps\":%zu,"
              "\"evals\":%ld,\"secs\":%.3f}\n",
              start.peak, start.cost, plan.peak_rank, plan.cost_estimate, plan.steps.size(), evals, secs);
  return 0;
}
