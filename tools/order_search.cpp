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
//   order_search --payload in.json --out out.json [--evals N] [--seed S] [--split-2q 1]
//
// --split-2q 1 (opt-in rank reduction as a network transform; the
// reference keeps every 2-qubit gate rank 4 on purpose, SPEC.md "Diagonal-gate rank
// reduction"): every rank-4 gate tensor whose ket operator K(s1,s2,t1,t2) has operator
// Schmidt rank <= 2 across (s1,t1)|(s2,t2) -- ZZ phases, CNOT/CZ-type gates -- becomes two
// rank-3 tensors U(in1,out1,bond), V(in2,out2,bond) joined by one new dim-4 edge, with
// U = a (x) conj(a), V = b (x) conj(b) for K = sum_k a_k b_k, so the density tensor is
// reproduced exactly (up to rounding) and every tensor still factorises for the ket view.
// Original vertex and edge ids (and so the cut) are kept; new ids follow the largest.
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

#include "search_common.hpp"

using qsearch::Score;
using qsearch::score;
using qsearch::leg_greedy;
using qsearch::split_2q;

int main(int argc, char** argv) {
  std::string in, out;
  long evals = 20000;
  uint64_t seed = 1;
  bool split = false;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--payload") in = v;
    else if (k == "--out") out = v;
    else if (k == "--evals") evals = std::stol(v);
    else if (k == "--seed") seed = std::stoull(v);
    else if (k == "--split-2q") split = v == "1";
  }
  std::ifstream f(in);
  std::stringstream ss;
  ss << f.rdbuf();
  qcut::Payload p = qcut::decode_payload(ss.str());
  int n_split = 0;
  if (split) {
    n_split = split_2q(p.tn);
    // the reference's own planner on the transformed network, for comparison
    qcut::TensorNetwork sub0 = qcut::apply_cut(p.tn, p.cut, qcut::Assignment(p.cut.size(), 0));
    p.plan = qcut::best_plan(sub0, 4, 1);
  }
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
              "\"evals\":%ld,\"secs\":%.3f,\"split_2q\":%d}\n",
              start.peak, start.cost, plan.peak_rank, plan.cost_estimate, plan.steps.size(), evals, secs, n_split);
  return 0;
}
