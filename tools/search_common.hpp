// search_common.hpp — helpers shared by the host search tools (order_search, cut_search):
// the (peak, cost) score, a leg-aware greedy elimination order, and the opt-in 2-qubit
// operator-Schmidt split. Maintainer tooling built against the
// reference library by oracle/Makefile; not part of the GPU engine.
#pragma once
#include <algorithm>
#include <cmath>
#include <map>
#include <random>
#include <vector>

#include "qcut/contraction.hpp"
#include "qcut/cutting.hpp"
#include "qcut/ordering.hpp"

namespace qsearch {

struct Score {
  int peak = 1 << 30;
  double cost = 1e300;
  bool operator<(const Score& o) const { return peak != o.peak ? peak < o.peak : cost < o.cost; }
};

inline Score score(const qcut::TensorNetwork& tn, const qcut::EliminationOrder& ord) {
  qcut::ContractionPlan p = qcut::plan_from_order(tn, ord);
  return Score{p.peak_rank, p.cost_estimate};
}

// Leg-aware greedy: repeatedly eliminate the vertex whose neighbourhood (counted in
// legs of the current merged multigraph) is smallest.
inline qcut::EliminationOrder leg_greedy(const qcut::TensorNetwork& tn, std::mt19937_64& rng) {
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

// Ket operator of a density tensor T = K (x) conj(K) (digit d = 2*ket + bra, tensor.hpp
// leg 0 most significant); K up to one global phase. Empty when T does not factorise.
inline std::vector<qcut::cx> ket_of(const qcut::Tensor& t) {
  const int r = t.rank;
  const int nk = 1 << r;
  auto dens_index = [&](int k, int b) {
    int idx = 0;
    for (int l = r - 1, sh = 0; l >= 0; --l, ++sh) idx += (2 * ((k >> sh) & 1) + ((b >> sh) & 1)) << (2 * sh);
    return idx;
  };
  int kbest = 0;
  double vbest = -1;
  for (int k = 0; k < nk; ++k) {
    const double v = std::abs(t.data[dens_index(k, k)]);
    if (v > vbest) vbest = v, kbest = k;
  }
  std::vector<qcut::cx> K(nk);
  if (vbest <= 0) return {};
  const double n0 = std::sqrt(vbest);
  for (int k = 0; k < nk; ++k) K[k] = t.data[dens_index(k, kbest)] / n0;
  double scale = 0, err = 0;
  for (int k = 0; k < nk; ++k)
    for (int b = 0; b < nk; ++b) {
      scale = std::max(scale, std::abs(t.data[dens_index(k, b)]));
      err = std::max(err, std::abs(t.data[dens_index(k, b)] - K[k] * std::conj(K[b])));
    }
  return err <= 1e-13 * scale ? K : std::vector<qcut::cx>{};
}

// Operator-Schmidt split of 2-qubit gate tensors (see --split-2q). Returns the count.
inline int split_2q(qcut::TensorNetwork& tn) {
  int next_v = tn.vertices.rbegin()->first + 1, next_e = 0;
  for (const auto& e : tn.edges) next_e = std::max(next_e, e.id + 1);
  std::vector<int> ids;
  for (const auto& [id, t] : tn.vertices)
    if (t.rank == 4) ids.push_back(id);
  int n = 0;
  for (int id : ids) {
    const std::vector<qcut::cx> K = ket_of(tn.vertices.at(id));
    if (K.empty()) continue;
    // ket legs (in1, in2, out1, out2) = bits 3..0 of K's index; M[(in1,out1)][(in2,out2)]
    qcut::cx M[4][4];
    for (int i = 0; i < 16; ++i) M[((i >> 3) & 1) * 2 + ((i >> 1) & 1)][((i >> 2) & 1) * 2 + (i & 1)] = K[i];
    // rank-revealing Gram-Schmidt over M's columns with pivoting: M = A B, A 4x2, B 2x4
    qcut::cx A[4][2] = {}, B[2][4] = {};
    qcut::cx W[4][4];
    std::copy(&M[0][0], &M[0][0] + 16, &W[0][0]);
    double mmax = 0;
    for (auto& row : M)
      for (auto& v : row) mmax = std::max(mmax, std::abs(v));
    int rk = 0;
    for (; rk < 2; ++rk) {
      int jb = -1;
      double nb = 0;
      for (int j = 0; j < 4; ++j) {
        double nn = 0;
        for (int i = 0; i < 4; ++i) nn += std::norm(W[i][j]);
        if (nn > nb) nb = nn, jb = j;
      }
      if (jb < 0 || std::sqrt(nb) <= 1e-14 * mmax) break;
      const double nrm = std::sqrt(nb);
      for (int i = 0; i < 4; ++i) A[i][rk] = W[i][jb] / nrm;
      for (int j = 0; j < 4; ++j) {
        qcut::cx c = 0;
        for (int i = 0; i < 4; ++i) c += std::conj(A[i][rk]) * W[i][j];
        B[rk][j] = c;
        for (int i = 0; i < 4; ++i) W[i][j] -= A[i][rk] * c;
      }
    }
    double err = 0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) err = std::max(err, std::abs(M[i][j] - (A[i][0] * B[0][j] + A[i][1] * B[1][j])));
    if (rk == 0 || err > 1e-13 * mmax) continue;
    // density tensors: U(in1, out1, bond) = a (x) conj(a), V(in2, out2, bond) = b (x) conj(b)
    qcut::Tensor U = qcut::Tensor::zeros(3), V = qcut::Tensor::zeros(3);
    for (int k0 = 0; k0 < 2; ++k0)
      for (int k2 = 0; k2 < 2; ++k2)
        for (int kb = 0; kb < 2; ++kb)
          for (int b0 = 0; b0 < 2; ++b0)
            for (int b2 = 0; b2 < 2; ++b2)
              for (int bb = 0; bb < 2; ++bb) {
                const int d0 = 2 * k0 + b0, d1 = 2 * k2 + b2, d2 = 2 * kb + bb;
                U.data[d0 * 16 + d1 * 4 + d2] = A[k0 * 2 + k2][kb] * std::conj(A[b0 * 2 + b2][bb]);
                V.data[d0 * 16 + d1 * 4 + d2] = B[kb][k0 * 2 + k2] * std::conj(B[bb][b0 * 2 + b2]);
              }
    const int vid = next_v++;
    tn.vertices[id] = U;
    tn.vertices[vid] = V;
    // legs of the old tensor: 0 in1 -> U0, 2 out1 -> U1, 1 in2 -> V0, 3 out2 -> V1
    for (auto& e : tn.edges)
      for (int side = 0; side < 2; ++side) {
        int& vv = side ? e.v : e.u;
        int& ll = side ? e.leg_v : e.leg_u;
        if (vv != id) continue;
        if (ll == 0) ll = 0;
        else if (ll == 2) ll = 1;
        else if (ll == 1) vv = vid, ll = 0;
        else vv = vid, ll = 1;
      }
    tn.edges.push_back(qcut::NetEdge{next_e++, id, 2, vid, 2});
    ++n;
  }
  qcut::check_closed(tn);
  return n;
}

}  // namespace qsearch
