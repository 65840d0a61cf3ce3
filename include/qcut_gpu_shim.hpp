// qcut_gpu_shim.hpp — the reference-side binding (header-only C++).
//
// A maintainer of the reference (`qcut`, proj/core) adds this header to route the
// hot path through the B200 engine without touching callers:
//
//   qcut::gpu::Engine eng(job, /*device=*/0);        // once per JobSpec / payload
//   qcut::cx v = eng.sum_range(lo, hi);               // == qcut::sum_range(job, lo, hi)
//
// It converts the JobSpec into the reference's own lossless payload
// (qcut::encode_payload, proj/core/src/serialize.cpp:147-154), owns one C-ABI engine
// (include/qcut_gpu.h) and rethrows the C-ABI status codes as the reference's
// exception classes (proj/core/src/executor.cpp:48-64):
//   QC_EINVAL -> std::invalid_argument, QC_ERANK -> qcut::RankGuardError,
//   QC_EINTERNAL -> std::runtime_error.
// Calls on one Engine are serialised by the engine; use one Engine per device.
#pragma once

#include <cstdint>
#include <fstream>
#include <regex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "qcut/circuit.hpp"
#include "qcut/contraction.hpp"
#include "qcut/cutting.hpp"
#include "qcut/executor.hpp"
#include "qcut/graph.hpp"
#include "qcut/serialize.hpp"
#include "qcut/tensor_network.hpp"
#include "qcut_gpu.h"

namespace qcut::gpu {

inline void rethrow(int rc) {
  if (rc == QC_OK) return;
  const std::string msg = qc_last_error();
  if (rc == QC_EINVAL) throw std::invalid_argument(msg);
  if (rc == QC_ERANK) {
    std::smatch m;
    static const std::regex re("rank-(\\d+) tensor.*max rank (\\d+)");
    if (std::regex_search(msg, m, re)) throw RankGuardError(std::stoi(m[1]), std::stoi(m[2]));
    throw std::runtime_error(msg);
  }
  throw std::runtime_error(msg);
}

inline std::string read_text(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot read " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// the reference's on-disk formats as engine inputs. A circuit file
// (parse_circuit, circuit.hpp:93) and an optional cut file (parse_cut_json,
// cutting.hpp:86) checked against the network's graph hash exactly as the CLI's
// load_cut does (tools/qcut.cpp:69-78), planned by make_job as `qcut run` does
// (tools/qcut.cpp:280-287). Throws the CLI's std::runtime_error on a hash mismatch.
inline JobSpec job_from_files(const std::string& circuit_path, const std::string& cut_path = "",
                              int restarts = 4, std::uint64_t seed = 1, int max_rank = kDefaultMaxRank) {
  const TensorNetwork tn = build_network(parse_circuit(read_text(circuit_path)));
  CutSet cut;
  if (!cut_path.empty()) {
    const CutFile f = parse_cut_json(read_text(cut_path));
    const std::string want = graph_hash(network_graph(tn));
    if (f.source_graph_hash != want)
      throw std::runtime_error("cut file " + cut_path + " was built for a different network (hash " +
                               f.source_graph_hash + ", expected " + want + ")");
    cut = f.edges;
  }
  return make_job(tn, cut, restarts, seed, max_rank);
}

class Engine {
 public:
  // mode: QC_MODE_DENSITY (the reference's own view) or QC_MODE_KET (binary view;
  // answers density-id queries exactly from ket slice values).
  Engine(const JobSpec& job, int device, int mode = QC_MODE_KET, std::uint64_t mem_budget = 0) {
    const std::string payload = encode_payload(Payload{job.tn, job.cut, job.plan, job.max_rank});
    rethrow(qc_engine_create(payload.data(), payload.size(), device, mode, mem_budget, &e_));
  }
  explicit Engine(const std::string& encoded_payload, int device, int mode = QC_MODE_KET) {
    rethrow(qc_engine_create(encoded_payload.data(), encoded_payload.size(), device, mode, 0, &e_));
  }
  // a payload file as written by encode_payload / shipped by the master (serialize.cpp:147-171)
  static Engine from_payload_file(const std::string& path, int device, int mode = QC_MODE_KET) {
    return Engine(read_text(path), device, mode);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  ~Engine() { qc_engine_destroy(e_); }

  // qcut::sum_range(job, lo, hi) (executor.hpp:46)
  cx sum_range(std::uint64_t lo, std::uint64_t hi) {
    double out[2];
    rethrow(qc_engine_sum_range(e_, lo, hi, out));
    return {out[0], out[1]};
  }
  // qcut::run_serial(job) (executor.hpp:49)
  cx run_serial() {
    qc_plan_stats st;
    rethrow(qc_engine_plan_stats(e_, &st));
    return sum_range(0, st.jobs);
  }
  std::vector<cx> slice_values(std::uint64_t lo, std::uint64_t hi) {
    std::vector<double> raw(2 * (hi > lo ? hi - lo : 0));
    rethrow(qc_engine_slice_values(e_, lo, hi, raw.data()));
    std::vector<cx> v(raw.size() / 2);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = {raw[2 * i], raw[2 * i + 1]};
    return v;
  }
  qc_engine* handle() { return e_; }

 private:
  qc_engine* e_ = nullptr;
};

// qcut::contract_pair (contraction.hpp:46-53) on the device: same arguments, result legs,
// exceptions (std::invalid_argument with the reference's messages, RankGuardError) -- dense
// shapes run as a complex GEMM on the FP64 tensor pipe (qc_contract_pair). The length check
// of the two leg lists lives here because the C-ABI carries one shared-leg count.
inline Tensor contract_pair(const Tensor& e, const std::vector<int>& legs_e, const Tensor& f,
                            const std::vector<int>& legs_f, int max_rank = kDefaultMaxRank, int device = 0) {
  if (legs_e.empty() || legs_f.empty()) throw std::invalid_argument("contract_pair needs at least one shared leg");
  if (legs_e.size() != legs_f.size())
    throw std::invalid_argument("shared leg lists differ in length: " + std::to_string(legs_e.size()) + " vs " +
                                std::to_string(legs_f.size()));
  const int k = static_cast<int>(legs_e.size());
  std::vector<std::int32_t> le(legs_e.begin(), legs_e.end()), lf(legs_f.begin(), legs_f.end());
  const int out_rank = e.rank + f.rank - 2 * k;
  Tensor g;
  g.rank = out_rank > 0 ? out_rank : 0;
  g.data.resize(out_rank >= 0 && out_rank <= 16 ? pow4(out_rank) : 1);
  static_assert(sizeof(cx) == 2 * sizeof(double), "std::complex<double> is two doubles");
  rethrow(qc_contract_pair(device, 4, e.rank, reinterpret_cast<const double*>(e.data.data()), le.data(), f.rank,
                           reinterpret_cast<const double*>(f.data.data()), lf.data(), k, max_rank, QC_PAIR_AUTO,
                           reinterpret_cast<double*>(g.data.data())));
  return g;
}

}  // namespace qcut::gpu
