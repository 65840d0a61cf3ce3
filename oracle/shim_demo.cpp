// shim_demo — proves the reference-side binding (include/qcut_gpu_shim.hpp) is a
// drop-in: a JobSpec decoded by the UNMODIFIED reference library is answered by
// the reference's own sum_range (CPU) and by qcut::gpu::Engine (B200), and a
// run_pool-style thread pool swaps sum_range for the engine unchanged.
// Built by oracle/Makefile against oracle/_ref/libqcut_ref.a + the engine .so;
// run by tests/test_gpu_parity.py::test_reference_side_shim (needs a GPU).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <mutex>
#include <string>
#include <sstream>
#include <random>
#include <thread>
#include <vector>

#include "qcut/executor.hpp"
#include "qcut/serialize.hpp"
#include "qcut_gpu_shim.hpp"

// --files circuit cut.json [other_circuit] [mode]: the reference's on-disk inputs of
// `qcut run` through qcut::gpu::job_from_files; the engine's value vs
// the reference run_serial on the same JobSpec, and the graph-hash check of the cut file
// against a different network (expects the CLI's runtime_error).
// (--check-files: the same without a GPU -- the engine is created host-only, device -1,
// and its plan statistics are compared with the JobSpec's)
int files_mode(int argc, char** argv) {
  const bool gpu_run = std::string(argv[1]) == "--files";
  const std::string circuit = argv[2], cut = argv[3];
  const int mode = argc > 5 ? std::atoi(argv[5]) : QC_MODE_KET;
  const qcut::JobSpec job = qcut::gpu::job_from_files(circuit, cut);
  qcut::cx cpu{}, gpu{};
  if (gpu_run) {
    cpu = qcut::run_serial(job);
    qcut::gpu::Engine eng(job, 0, mode);
    gpu = eng.run_serial();
  } else {
    qcut::gpu::Engine eng(job, -1, mode);
    qc_plan_stats st;
    qcut::gpu::rethrow(qc_engine_plan_stats(eng.handle(), &st));
    if (st.jobs != job.jobs() || st.peak_rank != job.plan.peak_rank) return 1;
  }
  bool hash_ok = argc <= 4;
  if (argc > 4) {
    try {
      qcut::gpu::job_from_files(argv[4], cut);
    } catch (const std::runtime_error& e) {
      hash_ok = std::string(e.what()).find("different network") != std::string::npos;
    }
  }
  const double rel = std::abs(gpu - cpu) / std::max(1e-300, std::abs(cpu));
  std::printf("{\"jobs\":%llu,\"cut\":%zu,\"peak\":%d,\"cpu\":[%.17g,%.17g],\"gpu\":[%.17g,%.17g],"
              "\"rel\":%.3g,\"hash_check\":%s}\n",
              static_cast<unsigned long long>(job.jobs()), job.cut.size(), job.plan.peak_rank, cpu.real(),
              cpu.imag(), gpu.real(), gpu.imag(), rel, hash_ok ? "true" : "false");
  return ((!gpu_run || rel <= 1e-10) && hash_ok) ? 0 : 1;
}

// shim_demo --pair: qcut::contract_pair (CPU, unmodified reference) against
// qcut::gpu::contract_pair on BM_ContractPair's shapes (bench_main.cpp:42-65) and a mixed
// leg order, plus the exception mapping (invalid_argument texts, RankGuardError).
int pair_mode() {
  std::mt19937_64 rng(17);
  std::uniform_real_distribution<double> u(-1, 1);
  auto random_tensor = [&](int rank) {
    qcut::Tensor t;
    t.rank = rank;
    t.data.resize(qcut::pow4(rank));
    for (auto& v : t.data) v = qcut::cx(u(rng), u(rng));
    return t;
  };
  struct Case {
    int ra, rb;
    std::vector<int> la, lb;
  };
  const std::vector<Case> cases = {{4, 4, {2, 3}, {0, 1}}, {6, 6, {3, 4, 5}, {0, 1, 2}}, {7, 6, {6, 0, 3}, {1, 5, 2}},
                                   {2, 2, {1}, {0}}, {8, 8, {4, 5, 6, 7}, {0, 1, 2, 3}}};
  double worst = 0;
  for (const Case& c : cases) {
    const qcut::Tensor a = random_tensor(c.ra), b = random_tensor(c.rb);
    const qcut::Tensor want = qcut::contract_pair(a, c.la, b, c.lb, 30);
    const qcut::Tensor got = qcut::gpu::contract_pair(a, c.la, b, c.lb, 30);
    if (got.rank != want.rank || got.data.size() != want.data.size()) return 1;
    double scale = 0, diff = 0;
    for (std::size_t i = 0; i < want.data.size(); ++i) {
      scale = std::max(scale, std::abs(want.data[i]));
      diff = std::max(diff, std::abs(want.data[i] - got.data[i]));
    }
    worst = std::max(worst, diff / scale);
  }
  bool inval = false, guard = false;
  const qcut::Tensor a = random_tensor(3), b = random_tensor(3);
  try {
    qcut::gpu::contract_pair(a, {5}, b, {0});
  } catch (const std::invalid_argument& e) {
    inval = std::string(e.what()) == "leg 5 out of range for rank-3 tensor (left)";
  }
  try {
    qcut::gpu::contract_pair(a, {2}, b, {0}, 3);
  } catch (const qcut::RankGuardError& e) {
    guard = e.rank() == 4 && e.max_rank() == 3;
  }
  std::printf("{\"worst_rel\":%.3g,\"invalid_argument\":%s,\"rank_guard\":%s}\n", worst, inval ? "true" : "false",
              guard ? "true" : "false");
  return (worst <= 1e-12 && inval && guard) ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "--pair") return pair_mode();
  if (argc >= 4 && (std::string(argv[1]) == "--files" || std::string(argv[1]) == "--check-files"))
    return files_mode(argc, argv);
  if (argc < 2) {
    std::fprintf(stderr, "usage: shim_demo payload.json [mode] | shim_demo --files circuit cut [other] [mode]\n");
    return 2;
  }
  std::ifstream f(argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  const int mode = argc > 2 ? std::atoi(argv[2]) : QC_MODE_KET;
  qcut::Payload p = qcut::decode_payload(ss.str());
  qcut::JobSpec job{p.tn, p.cut, p.plan, p.max_rank};
  const qcut::cx cpu = qcut::run_serial(job);
  qcut::gpu::Engine eng(job, 0, mode);
  const qcut::cx gpu = eng.run_serial();
  // run_pool's grid (executor.cpp:113-136) with the engine as the batch kernel
  const std::uint64_t total = job.jobs();
  const int workers = 3;
  const std::uint64_t batch = qcut::round_count(total, workers);
  std::vector<qcut::WorkerResult> parts;
  std::mutex mu;
  std::vector<std::thread> th;
  for (int w = 0; w < workers; ++w)
    th.emplace_back([&, w] {
      const std::uint64_t lo = std::min<std::uint64_t>(total, w * batch);
      const std::uint64_t hi = std::min<std::uint64_t>(total, lo + batch);
      const qcut::cx v = eng.sum_range(lo, hi);
      std::lock_guard<std::mutex> lk(mu);
      parts.push_back({lo, hi, v, 0.0});
    });
  for (auto& t : th) t.join();
  const qcut::cx pooled = qcut::aggregate(parts, total);
  bool guard_ok = false;
  try {
    qcut::JobSpec small = job;
    small.max_rank = 1;
    qcut::gpu::Engine g2(small, 0, mode);
    g2.run_serial();
  } catch (const qcut::RankGuardError& e) {
    guard_ok = e.max_rank() == 1;
  }
  const double rel = std::abs(gpu - cpu) / std::max(1e-300, std::abs(cpu));
  const double relp = std::abs(pooled - cpu) / std::max(1e-300, std::abs(cpu));
  std::printf("{\"cpu\":[%.17g,%.17g],\"gpu\":[%.17g,%.17g],\"pooled\":[%.17g,%.17g],\"rel\":%.3g,"
              "\"rel_pooled\":%.3g,\"rank_guard\":%s}\n",
              cpu.real(), cpu.imag(), gpu.real(), gpu.imag(), pooled.real(), pooled.imag(), rel, relp,
              guard_ok ? "true" : "false");
  return (rel <= 1e-10 && relp <= 1e-10 && guard_ok) ? 0 : 1;
}
