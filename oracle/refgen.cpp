// refgen — test-infrastructure driver over the UNMODIFIED reference library.
//
// This file is ours; it only calls the reference's public API
// (proj/core/include/qcut/*.hpp) and is linked against the reference core
// compiled from /root/reference (see oracle/Makefile). It never ships in the
// product. It is the one source of instances, payloads and reference values:
//
//   gen     seeded QAOA instance (SURVEY.md §8(d) derivation) -> payload JSON per
//           bitstring + info JSON (cut, plan stats, angles, bitstrings)
//   random  reference-test-style random circuit (proj/tests/helpers.hpp
//           random_circuit) + random cut -> payload + dm_simulate value
//   run     decode_payload -> run_serial (or sum_range over [lo,hi)), optional
//           per-slice values sum_range(s, s+1)
//   mixed   random circuit with mixed inputs and non-projector POVMs (density view only)
//   slices  per-slice values sum_range(s, s+1) for an explicit id list (--ids), threaded
//   pair    the reference's contract_pair on two tensors read from a binary file (doubles:
//           a then b), result appended to --out; --reps > 0 also times it (BM_ContractPair,
//           proj/benchmarks/bench_main.cpp:42-65)
//   bench   CPU timing: sum_range over a bounded slice sample, split over W
//           threads on run_pool's contiguous batch grid (executor.cpp:113-136)
//
// Output is JSON on stdout (doubles printed with 17 significant digits).
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "qcut/circuit.hpp"
#include "qcut/distributed.hpp"
#include "qcut/contraction.hpp"
#include "qcut/cutting.hpp"
#include "qcut/executor.hpp"
#include "qcut/graph.hpp"
#include "qcut/oracle.hpp"
#include "qcut/qaoa.hpp"
#include "qcut/serialize.hpp"
#include "qcut/tensor_network.hpp"
#include "qcut/types.hpp"

#include "helpers.hpp"  // proj/tests/helpers.hpp, included in place (random_circuit)

using qcut::cx;

namespace {

std::map<std::string, std::string> parse_args(int argc, char** argv, int from) {
  std::map<std::string, std::string> a;
  for (int i = from; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) continue;
    std::string v = (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0)
                        ? argv[++i]
                        : "1";
    a[k.substr(2)] = v;
  }
  return a;
}

std::string get(const std::map<std::string, std::string>& a, const std::string& k,
                const std::string& def) {
  auto it = a.find(k);
  return it == a.end() ? def : it->second;
}

std::string d17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string cx_json(cx v) { return "[" + d17(v.real()) + "," + d17(v.imag()) + "]"; }

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

double u01(std::uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void write_file(const std::string& path, const std::string& s) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot write " + path);
  f << s;
}

std::string plan_stats_json(const qcut::ContractionPlan& plan) {
  std::string s = "{\"n_steps\":" + std::to_string(plan.steps.size()) +
                  ",\"peak_rank\":" + std::to_string(plan.peak_rank) +
                  ",\"cost_estimate\":" + d17(plan.cost_estimate) + ",\"scalars\":[";
  for (std::size_t i = 0; i < plan.scalars.size(); ++i)
    s += (i ? "," : "") + std::to_string(plan.scalars[i]);
  s += "]}";
  return s;
}

// gamma_l, beta_l and bitstring b derived from `seed` with the
// reference's own splitmix step (types.cpp:101-106).
qcut::Circuit seeded_qaoa(const qcut::RegularGraph& g, int layers, std::uint64_t seed,
                          int b, std::vector<double>& gammas, std::vector<double>& betas,
                          std::string& z) {
  gammas.clear();
  betas.clear();
  for (int l = 0; l < layers; ++l) {
    gammas.push_back(M_PI * u01(qcut::mix_seed(seed, 0x6A11u + 2u * l)));
    betas.push_back(M_PI * u01(qcut::mix_seed(seed, 0x6A11u + 2u * l + 1u)));
  }
  z.assign(static_cast<std::size_t>(g.n), '0');
  std::uint64_t zs = qcut::mix_seed(seed, 0xB175u + static_cast<std::uint64_t>(b));
  for (int i = 0; i < g.n; ++i)
    z[static_cast<std::size_t>(i)] = (qcut::mix_seed(zs, static_cast<std::uint64_t>(i)) >> 63) ? '1' : '0';
  // Same construction order as qaoa_circuit (qaoa.cpp:35-43), per-layer angles.
  qcut::Circuit c = qcut::Circuit::make(g.n);
  for (int q = 0; q < g.n; ++q) c.add(qcut::standard_gate("h"), {q});
  for (int l = 0; l < layers; ++l) {
    for (const auto& [u, v] : g.edges) c.add(qcut::standard_gate("zz", {gammas[l]}), {u, v});
    for (int q = 0; q < g.n; ++q) c.add(qcut::standard_gate("rx", {2.0 * betas[l]}), {q});
  }
  for (int q = 0; q < g.n; ++q) c.set_measurement(q, z[q] == '0' ? qcut::kProj0 : qcut::kProj1);
  return c;
}

int cmd_gen(const std::map<std::string, std::string>& a) {
  const int n = std::stoi(get(a, "n", "20"));
  const int p = std::stoi(get(a, "p", "1"));
  const std::uint64_t seed = std::stoull(get(a, "seed", "1"));
  const int M = std::stoi(get(a, "M", "4"));
  const int nb = std::stoi(get(a, "bitstrings", "1"));
  const std::string prefix = get(a, "out", "inst");
  qcut::GaParams ga;
  ga.M = M;
  ga.N = std::stoi(get(a, "ga-n", "11"));
  ga.T = std::stoi(get(a, "ga-t", "4"));
  ga.seed = std::stoull(get(a, "ga-seed", std::to_string(seed)));
  ga.fitness_restarts = std::stoi(get(a, "fitness-restarts", "2"));
  const int plan_restarts = std::stoi(get(a, "plan-restarts", "4"));
  const std::uint64_t plan_seed = std::stoull(get(a, "plan-seed", "1"));

  qcut::RegularGraph g = qcut::random_regular_graph(n, 3, seed);
  std::vector<double> gammas, betas;
  std::string z;
  qcut::Circuit c0 = seeded_qaoa(g, p, seed, 0, gammas, betas, z);
  // Explicit overrides (e.g. the README example: --gamma 0.6 --beta 0.4 --zeros).
  const bool explicit_angles = a.count("gamma") > 0;
  auto override = [&](qcut::Circuit& c, int b) {
    if (explicit_angles) {
      for (int l = 0; l < p; ++l) {
        gammas[l] = std::stod(a.at("gamma"));
        betas[l] = std::stod(get(a, "beta", "0.4"));
      }
    }
    if (a.count("zeros")) z.assign(static_cast<std::size_t>(n), '0');
    if (explicit_angles || a.count("zeros")) {
      c = qcut::Circuit::make(g.n);
      for (int q = 0; q < g.n; ++q) c.add(qcut::standard_gate("h"), {q});
      for (int l = 0; l < p; ++l) {
        for (const auto& [u, v] : g.edges) c.add(qcut::standard_gate("zz", {gammas[l]}), {u, v});
        for (int q = 0; q < g.n; ++q) c.add(qcut::standard_gate("rx", {2.0 * betas[l]}), {q});
      }
      for (int q = 0; q < g.n; ++q) c.set_measurement(q, z[q] == '0' ? qcut::kProj0 : qcut::kProj1);
    }
    (void)b;
  };
  override(c0, 0);
  if (p == 1 && get(a, "check-qaoa", "1") == "1") {
    // for p=1 the hand-built circuit must equal qaoa_circuit().
    qcut::Circuit ref = qcut::qaoa_circuit(g, gammas[0], betas[0], 1, z);
    if (!(ref == c0)) throw std::runtime_error("seeded circuit != qaoa_circuit");
  }
  qcut::TensorNetwork tn0 = qcut::build_network(c0);
  double t0 = now_s();
  qcut::GaResult r;
  if (a.count("cut-from")) {
    // the cut of an existing payload of this network (more bitstrings of an instance without
    // repeating its GA search; the network structure must match)
    qcut::Payload src = qcut::decode_payload(read_file(a.at("cut-from")));
    if (qcut::network_graph(src.tn).edges != qcut::network_graph(tn0).edges)
      throw std::runtime_error("--cut-from payload is another network");
    r.cut = src.cut;
    r.width = -1;
  } else {
    r = qcut::ga_search(qcut::network_graph(tn0), ga);
  }
  double t_ga = now_s() - t0;
  t0 = now_s();
  qcut::JobSpec job0 = qcut::make_job(tn0, r.cut, plan_restarts, plan_seed);
  double t_plan = now_s() - t0;
  int max_rank = std::max(qcut::kDefaultMaxRank, job0.plan.peak_rank);
  if (a.count("max-rank")) max_rank = std::stoi(a.at("max-rank"));

  std::string info = "{\"n\":" + std::to_string(n) + ",\"p\":" + std::to_string(p) +
                     ",\"seed\":" + std::to_string(seed) + ",\"M\":" + std::to_string(M) +
                     ",\"ga\":{\"N\":" + std::to_string(ga.N) + ",\"T\":" + std::to_string(ga.T) +
                     ",\"seed\":" + std::to_string(ga.seed) +
                     ",\"fitness_restarts\":" + std::to_string(ga.fitness_restarts) +
                     ",\"width\":" + std::to_string(r.width) + "}" +
                     ",\"plan_restarts\":" + std::to_string(plan_restarts) +
                     ",\"plan_seed\":" + std::to_string(plan_seed) +
                     ",\"max_rank\":" + std::to_string(max_rank) + ",\"gammas\":[";
  for (int l = 0; l < p; ++l) info += (l ? "," : "") + d17(gammas[l]);
  info += "],\"betas\":[";
  for (int l = 0; l < p; ++l) info += (l ? "," : "") + d17(betas[l]);
  info += "],\"cut\":[";
  for (std::size_t i = 0; i < r.cut.size(); ++i) info += (i ? "," : "") + std::to_string(r.cut[i]);
  info += "],\"graph\":[";
  for (std::size_t i = 0; i < g.edges.size(); ++i)
    info += (i ? "," : "") + std::string("[") + std::to_string(g.edges[i].first) + "," +
            std::to_string(g.edges[i].second) + "]";
  info += "],\"plan\":" + plan_stats_json(job0.plan) + ",\"t_ga_s\":" + d17(t_ga) +
          ",\"t_plan_s\":" + d17(t_plan) + ",\"bitstrings\":[";
  for (int b = 0; b < nb; ++b) {
    qcut::Circuit cb = seeded_qaoa(g, p, seed, b, gammas, betas, z);
    override(cb, b);
    qcut::TensorNetwork tn = qcut::build_network(cb);
    // cut and plan depend only on structure; re-plan anyway and
    // check identity so a mismatch can never slip through.
    qcut::JobSpec job = qcut::make_job(tn, r.cut, plan_restarts, plan_seed, max_rank);
    if (job.plan.peak_rank != job0.plan.peak_rank ||
        job.plan.steps.size() != job0.plan.steps.size())
      throw std::runtime_error("plan differs across bitstrings");
    qcut::Payload pl{job.tn, job.cut, job.plan, job.max_rank};
    std::string path = prefix + ".b" + std::to_string(b) + ".payload.json";
    write_file(path, qcut::encode_payload(pl));
    // the reference's on-disk inputs of `qcut run`: circuit file
    // (emit_circuit) and, once, the cut file with the network's graph hash (dump_cut_json)
    write_file(prefix + ".b" + std::to_string(b) + ".circuit", qcut::emit_circuit(cb));
    if (b == 0)
      write_file(prefix + ".cut.json",
                 qcut::dump_cut_json(r.cut, qcut::graph_hash(qcut::network_graph(tn)), r.width, ga, r.history));
    info += (b ? "," : "") + std::string("\"") + z + "\"";
  }
  info += "]}";
  write_file(prefix + ".info.json", info + "\n");
  std::cout << info << "\n";
  return 0;
}

int cmd_random(const std::map<std::string, std::string>& a) {
  const int n = std::stoi(get(a, "n", "3"));
  const int depth = std::stoi(get(a, "depth", "8"));
  const std::uint64_t seed = std::stoull(get(a, "seed", "1"));
  const int M = std::stoi(get(a, "M", "2"));
  const std::string out = get(a, "out", "rand.payload.json");
  std::mt19937_64 rng(seed);
  qcut::Circuit c = qcut_test::random_circuit(n, depth, rng);
  qcut::TensorNetwork tn = qcut::build_network(c);
  std::vector<int> ids;
  for (const auto& e : tn.edges) ids.push_back(e.id);
  std::shuffle(ids.begin(), ids.end(), rng);
  if (M > static_cast<int>(ids.size())) throw std::runtime_error("M too large");
  qcut::CutSet cut(ids.begin(), ids.begin() + M);
  std::sort(cut.begin(), cut.end());
  qcut::JobSpec job = qcut::make_job(tn, cut, 2, seed);
  job.max_rank = std::max(qcut::kDefaultMaxRank, job.plan.peak_rank);
  qcut::Payload pl{job.tn, job.cut, job.plan, job.max_rank};
  write_file(out, qcut::encode_payload(pl));
  cx serial = qcut::run_serial(job);
  std::string s = "{\"serial\":" + cx_json(serial);
  if (n <= 10) s += ",\"dm_simulate\":" + cx_json(qcut::dm_simulate(c));
  s += ",\"plan\":" + plan_stats_json(job.plan) + "}";
  std::cout << s << "\n";
  return 0;
}

// General density mode: the reference test generator's random circuit
// (helpers.hpp random_circuit) with MIXED inputs rho = w|a><a| + (1-w)|b><b| on every second
// qubit and NON-PROJECTOR POVM elements E = u|0><0| + v|psi><psi| (0 < u + v <= 1) on every
// third (circuit.hpp:62-79 set_input / set_measurement): tensors that do not factorise as
// K (x) conj(K), so only the density view can run them. Random cut, make_job, run_serial,
// per-slice values, and dm_simulate for n <= 10.
int cmd_mixed(const std::map<std::string, std::string>& a) {
  const int n = std::stoi(get(a, "n", "3"));
  const int depth = std::stoi(get(a, "depth", "8"));
  const std::uint64_t seed = std::stoull(get(a, "seed", "1"));
  const int M = std::stoi(get(a, "M", "2"));
  const std::string out = get(a, "out", "mixed.payload.json");
  std::mt19937_64 rng(seed);
  qcut::Circuit c = qcut_test::random_circuit(n, depth, rng);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  auto outer = [](cx x0, cx x1) {  // |x><x| for the unit vector (x0, x1)
    return qcut::Mat2{x0 * std::conj(x0), x0 * std::conj(x1), x1 * std::conj(x0), x1 * std::conj(x1)};
  };
  auto unit = [&]() {
    const double th = 3.14159265358979 * u01(rng), ph = 6.28318530717959 * u01(rng);
    return std::make_pair(cx(std::cos(th / 2), 0.0), std::polar(std::sin(th / 2), ph));
  };
  for (int q = 0; q < n; ++q) {
    if (q % 2 == 0) {
      const auto [a0, a1] = unit();
      const auto [b0, b1] = unit();
      const double w = 0.2 + 0.6 * u01(rng);
      const qcut::Mat2 ra = outer(a0, a1), rb = outer(b0, b1);
      qcut::Mat2 rho;
      for (int i = 0; i < 4; ++i) rho[static_cast<std::size_t>(i)] = w * ra[static_cast<std::size_t>(i)] + (1 - w) * rb[static_cast<std::size_t>(i)];
      c.set_input(q, rho);
    }
    if (q % 3 == 0) {
      const auto [p0, p1] = unit();
      const double uu = 0.5 * u01(rng), vv = (1.0 - uu) * (0.3 + 0.6 * u01(rng));
      const qcut::Mat2 e0 = outer(cx(1, 0), cx(0, 0)), ep = outer(p0, p1);
      qcut::Mat2 E;
      for (int i = 0; i < 4; ++i) E[static_cast<std::size_t>(i)] = uu * e0[static_cast<std::size_t>(i)] + vv * ep[static_cast<std::size_t>(i)];
      c.set_measurement(q, E);
    }
  }
  qcut::validate_circuit(c);
  qcut::TensorNetwork tn = qcut::build_network(c);
  std::vector<int> ids;
  for (const auto& e : tn.edges) ids.push_back(e.id);
  std::shuffle(ids.begin(), ids.end(), rng);
  if (M > static_cast<int>(ids.size())) throw std::runtime_error("M too large");
  qcut::CutSet cut(ids.begin(), ids.begin() + M);
  std::sort(cut.begin(), cut.end());
  qcut::JobSpec job = qcut::make_job(tn, cut, 2, seed);
  job.max_rank = std::max(qcut::kDefaultMaxRank, job.plan.peak_rank);
  qcut::Payload pl{job.tn, job.cut, job.plan, job.max_rank};
  write_file(out, qcut::encode_payload(pl));
  std::string s = "{\"serial\":" + cx_json(qcut::run_serial(job));
  if (n <= 10) s += ",\"dm_simulate\":" + cx_json(qcut::dm_simulate(c));
  s += ",\"slices\":[";
  for (std::uint64_t i = 0; i < job.jobs(); ++i)
    s += (i ? "," : "") + cx_json(qcut::sum_range(job, i, i + 1));
  s += "],\"plan\":" + plan_stats_json(job.plan) + "}";
  std::cout << s << "\n";
  return 0;
}

// test_executor.cpp:67-80: cnot on |00>, cut the wire from the gate to qubit 0's
// measurement; --flip adds x on qubit 0 first (test_contraction.cpp:158-168).
int cmd_cnot(const std::map<std::string, std::string>& a) {
  const std::string out = get(a, "out", "cnot.payload.json");
  qcut::Circuit c = qcut::Circuit::make(2);
  const bool flip = a.count("flip") > 0;
  if (flip) c.add(qcut::standard_gate("x"), {0});
  c.add(qcut::standard_gate("cnot"), {0, 1});
  qcut::TensorNetwork tn = qcut::build_network(c);
  const int gate = flip ? 3 : 2, meas0 = flip ? 4 : 3;
  int victim = -1;
  for (const auto& e : tn.edges)
    if (e.u == gate && e.v == meas0) victim = e.id;
  if (victim < 0) throw std::runtime_error("victim edge not found");
  qcut::JobSpec job = qcut::make_job(tn, {victim}, 2, 1);
  qcut::Payload pl{job.tn, job.cut, job.plan, job.max_rank};
  write_file(out, qcut::encode_payload(pl));
  std::cout << "{\"serial\":" << cx_json(qcut::run_serial(job)) << ",\"victim\":" << victim << "}\n";
  return 0;
}

qcut::JobSpec load_job(const std::string& path) {
  qcut::Payload p = qcut::decode_payload(read_file(path));
  qcut::JobSpec job;
  job.tn = std::move(p.tn);
  job.cut = std::move(p.cut);
  job.plan = std::move(p.plan);
  job.max_rank = p.max_rank;
  return job;
}

int cmd_run(const std::map<std::string, std::string>& a) {
  qcut::JobSpec job = load_job(get(a, "payload", ""));
  std::uint64_t total = job.jobs();
  std::uint64_t lo = std::stoull(get(a, "lo", "0"));
  std::uint64_t hi = a.count("hi") ? std::stoull(a.at("hi")) : total;
  double t0 = now_s();
  cx v = qcut::sum_range(job, lo, hi);
  double dt = now_s() - t0;
  std::string s = "{\"jobs\":" + std::to_string(total) + ",\"lo\":" + std::to_string(lo) +
                  ",\"hi\":" + std::to_string(hi) + ",\"value\":" + cx_json(v) +
                  ",\"secs\":" + d17(dt) + ",\"plan\":" + plan_stats_json(job.plan);
  if (get(a, "slices", "0") == "1") {
    s += ",\"slices\":[";
    for (std::uint64_t i = lo; i < hi; ++i)
      s += (i > lo ? "," : "") + cx_json(qcut::sum_range(job, i, i + 1));
    s += "]";
  }
  if (get(a, "steps", "0") == "1") {
    s += ",\"steps\":[";
    for (std::size_t i = 0; i < job.plan.steps.size(); ++i) {
      const auto& st = job.plan.steps[i];
      s += (i ? "," : "") + std::string("[") + std::to_string(st.rank_a) + "," +
           std::to_string(st.rank_b) + "," + std::to_string(st.edges.size()) + "," +
           std::to_string(st.result_rank) + "]";
    }
    s += "]";
  }
  std::cout << s << "}\n";
  return 0;
}

// Per-slice reference values sum_range(job, s, s+1) for an explicit id list (--ids a,b,...),
// split over --workers threads (each slice is independent; the values do not depend on it).
int cmd_slices(const std::map<std::string, std::string>& a) {
  qcut::JobSpec job = load_job(get(a, "payload", ""));
  std::vector<std::uint64_t> ids;
  {
    std::string s = get(a, "ids", "");
    std::size_t at = 0;
    while (at < s.size()) {
      std::size_t e = s.find(',', at);
      if (e == std::string::npos) e = s.size();
      ids.push_back(std::stoull(s.substr(at, e - at)));
      at = e + 1;
    }
  }
  int workers = std::stoi(get(a, "workers", "1"));
  if (workers < 1) workers = static_cast<int>(std::thread::hardware_concurrency());
  std::vector<cx> vals(ids.size());
  std::atomic<std::size_t> next{0};
  double t0 = now_s();
  std::vector<std::thread> th;
  for (int w = 0; w < workers; ++w)
    th.emplace_back([&] {
      for (std::size_t i; (i = next++) < ids.size();) vals[i] = qcut::sum_range(job, ids[i], ids[i] + 1);
    });
  for (auto& t : th) t.join();
  double dt = now_s() - t0;
  std::string s = "{\"jobs\":" + std::to_string(job.jobs()) + ",\"secs\":" + d17(dt) + ",\"ids\":[";
  for (std::size_t i = 0; i < ids.size(); ++i) s += (i ? "," : "") + std::to_string(ids[i]);
  s += "],\"slices\":[";
  for (std::size_t i = 0; i < ids.size(); ++i) s += (i ? "," : "") + cx_json(vals[i]);
  std::cout << s << "]}\n";
  return 0;
}

int cmd_bench(const std::map<std::string, std::string>& a) {
  qcut::JobSpec job = load_job(get(a, "payload", ""));
  const std::uint64_t total = job.jobs();
  std::uint64_t slices = std::min<std::uint64_t>(total, std::stoull(get(a, "slices", "16")));
  int workers = std::stoi(get(a, "workers", "1"));
  if (workers < 1) workers = static_cast<int>(std::thread::hardware_concurrency());
  const int reps = std::stoi(get(a, "reps", "1"));
  std::vector<double> times;
  cx v{};
  for (int r = 0; r < reps; ++r) {
    // run_pool's default grid: ceil(jobs/workers) contiguous batches.
    std::uint64_t batch = (slices + workers - 1) / workers;
    std::vector<cx> parts(static_cast<std::size_t>(workers));
    double t0 = now_s();
    std::vector<std::thread> th;
    for (int w = 0; w < workers; ++w) {
      th.emplace_back([&, w] {
        std::uint64_t lo = std::min<std::uint64_t>(slices, w * batch);
        std::uint64_t hi = std::min<std::uint64_t>(slices, lo + batch);
        parts[static_cast<std::size_t>(w)] = lo < hi ? qcut::sum_range(job, lo, hi) : cx{};
      });
    }
    for (auto& t : th) t.join();
    times.push_back(now_s() - t0);
    v = {};
    for (const cx& p : parts) v += p;
  }
  std::string s = "{\"jobs\":" + std::to_string(total) + ",\"slices\":" +
                  std::to_string(slices) + ",\"workers\":" + std::to_string(workers) +
                  ",\"hw_threads\":" + std::to_string(std::thread::hardware_concurrency()) +
                  ",\"value\":" + cx_json(v) + ",\"secs\":[";
  for (std::size_t i = 0; i < times.size(); ++i) s += (i ? "," : "") + d17(times[i]);
  std::cout << s << "]}\n";
  return 0;
}

std::vector<int> parse_ints(const std::string& s) {
  std::vector<int> v;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) v.push_back(std::stoi(tok));
  return v;
}

// qcut::contract_pair on caller-provided tensors (--in: rank_a then rank_b row-major complex
// tensors as raw doubles); writes the result tensor's doubles to --out.
int cmd_pair(const std::map<std::string, std::string>& a) {
  const int ra = std::stoi(get(a, "rank-a", "2")), rb = std::stoi(get(a, "rank-b", "2"));
  const std::vector<int> la = parse_ints(get(a, "legs-a", "1")), lb = parse_ints(get(a, "legs-b", "0"));
  const int max_rank = std::stoi(get(a, "max-rank", "30"));
  const int reps = std::stoi(get(a, "reps", "0"));
  qcut::Tensor ta, tb;
  ta.rank = ra;
  tb.rank = rb;
  ta.data.resize(qcut::pow4(ra));
  tb.data.resize(qcut::pow4(rb));
  {
    std::ifstream f(get(a, "in", ""), std::ios::binary);
    if (!f) throw std::runtime_error("cannot open --in");
    f.read(reinterpret_cast<char*>(ta.data.data()), static_cast<std::streamsize>(ta.data.size() * sizeof(cx)));
    f.read(reinterpret_cast<char*>(tb.data.data()), static_cast<std::streamsize>(tb.data.size() * sizeof(cx)));
    if (!f) throw std::runtime_error("short --in file");
  }
  qcut::Tensor g = qcut::contract_pair(ta, la, tb, lb, max_rank);
  {
    std::ofstream f(get(a, "out", "pair.out.bin"), std::ios::binary);
    f.write(reinterpret_cast<const char*>(g.data.data()), static_cast<std::streamsize>(g.data.size() * sizeof(cx)));
  }
  std::string s = "{\"rank\":" + std::to_string(g.rank) + ",\"size\":" + std::to_string(g.data.size()) + ",\"secs\":[";
  for (int r = 0; r < reps; ++r) {
    const double t0 = now_s();
    qcut::Tensor h = qcut::contract_pair(ta, la, tb, lb, max_rank);
    const double dt = now_s() - t0;
    if (h.data.size() != g.data.size()) throw std::runtime_error("size changed");
    s += (r ? "," : "") + d17(dt);
  }
  std::cout << s << "]}\n";
  return 0;
}

}  // namespace

// The unmodified reference master (master.cpp:52-272) on a payload: prints the
// bound port, waits for --workers workers, prints the RunReport.
int cmd_master(const std::map<std::string, std::string>& a) {
  qcut::JobSpec job = load_job(get(a, "payload", ""));
  qcut::MasterConfig cfg;
  cfg.port = std::stoi(get(a, "port", "0"));
  cfg.workers = std::stoi(get(a, "workers", "1"));
  cfg.batch_size = std::stoull(get(a, "batch", "0"));
  cfg.timeout_secs = std::stod(get(a, "timeout", "120"));
  cfg.connect_timeout_secs = std::stod(get(a, "connect-timeout", "60"));
  cfg.on_listening = [](int port) {
    std::cout << "{\"event\":\"listening\",\"port\":" << port << "}" << std::endl;
  };
  qcut::RunReport r = qcut::run_distributed(cfg, job);
  std::cout << "{\"amplitude\":" << cx_json(r.amplitude) << ",\"jobs\":" << r.jobs
            << ",\"batches\":" << r.batches << ",\"recomputed_batches\":" << r.recomputed_batches
            << ",\"wall_secs\":" << d17(r.wall_secs) << "}" << std::endl;
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: qcut_refgen gen|random|run|bench [--key value ...]\n";
    return 2;
  }
  std::string cmd = argv[1];
  auto a = parse_args(argc, argv, 2);
  try {
    if (cmd == "gen") return cmd_gen(a);
    if (cmd == "random") return cmd_random(a);
    if (cmd == "run") return cmd_run(a);
    if (cmd == "bench") return cmd_bench(a);
    if (cmd == "slices") return cmd_slices(a);
    if (cmd == "mixed") return cmd_mixed(a);
    if (cmd == "cnot") return cmd_cnot(a);
    if (cmd == "pair") return cmd_pair(a);
    if (cmd == "master") return cmd_master(a);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  std::cerr << "unknown command " << cmd << "\n";
  return 2;
}
