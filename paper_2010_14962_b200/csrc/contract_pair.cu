// contract_pair on the device (include/qcut_gpu.h: qc_contract_pair, qc_contract_pair_bench).
//
// Mirrors qcut::contract_pair (proj/core/include/qcut/contraction.hpp:46-53,
// proj/core/src/contraction.cpp:71-116): the same argument checks in the same order with
// the same messages, the rank guard, result legs = free(a) in order ++ free(b) in order,
// row-major. The permutes of the reference (permute_legs, tensor.cpp:30-62) become the
// host-built offset tables of zgemm.cuh; dense shapes run on the FP64 tensor pipe.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/qcut_gpu.h"
#include "program.hpp"
#include "zgemm.cuh"

namespace qcg {
void set_last_error(const std::string& msg);  // engine.cu (thread-local, read by qc_last_error)
}

using namespace qcg;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

int ilog2(int64_t x) {
  int n = 0;
  while ((int64_t{1} << n) < x) ++n;
  return n;
}

// contraction.cpp:40-56
void check_leg_list(int rank, const std::vector<int>& legs, const char* side) {
  std::vector<char> seen(static_cast<size_t>(std::max(rank, 0)), 0);
  for (int l : legs) {
    if (l < 0 || l >= rank)
      throw std::invalid_argument("leg " + std::to_string(l) + " out of range for rank-" + std::to_string(rank) +
                                  " tensor (" + side + ")");
    if (seen[static_cast<size_t>(l)]) throw std::invalid_argument("leg " + std::to_string(l) + " repeated (" + side + ")");
    seen[static_cast<size_t>(l)] = 1;
  }
}

std::vector<int> free_legs(int rank, const std::vector<int>& shared) {
  std::vector<char> is(static_cast<size_t>(rank), 0);
  for (int l : shared) is[static_cast<size_t>(l)] = 1;
  std::vector<int> out;
  for (int l = 0; l < rank; ++l)
    if (!is[static_cast<size_t>(l)]) out.push_back(l);
  return out;
}

// offsets of the index x over `legs` (first leg most significant, as permute_legs orders
// them) inside a rank-`rank` row-major tensor of leg dimension 2^w
std::vector<int64_t> leg_table(int rank, int w, const std::vector<int>& legs) {
  const int nb = w * static_cast<int>(legs.size());
  std::vector<int64_t> t(size_t{1} << nb);
  const int64_t dmask = (int64_t{1} << w) - 1;
  for (int64_t x = 0; x < static_cast<int64_t>(t.size()); ++x) {
    int64_t off = 0;
    for (size_t i = 0; i < legs.size(); ++i) {
      const int64_t digit = (x >> (w * static_cast<int>(legs.size() - 1 - i))) & dmask;
      off |= digit << (w * (rank - 1 - legs[i]));
    }
    t[static_cast<size_t>(x)] = off;
  }
  return t;
}

struct PairJob {
  int w = 2;  // bits per leg (dim 4: 2, dim 2: 1)
  int ra = 0, rb = 0, k = 0, out_rank = 0;
  int64_t M = 1, N = 1, K = 1;
  std::vector<int64_t> tabs;  // kA kB mA nB mC nC
  int a_kfast = 0, b_kfast = 0, c_pair = 0;
  int path = QC_PAIR_AUTO;
};

PairJob plan_pair_job(int dim, int rank_a, const int32_t* legs_a, int rank_b, const int32_t* legs_b, int nshared,
                      int max_rank, int path) {
  if (dim != 2 && dim != 4) throw std::invalid_argument("leg dimension must be 2 or 4");
  if (rank_a < 0 || rank_b < 0) throw std::invalid_argument("negative tensor rank");
  if (nshared < 0) throw std::invalid_argument("negative shared-leg count");
  if (path < QC_PAIR_AUTO || path > QC_PAIR_SMALL) throw std::invalid_argument("unknown contract_pair path");
  // contract_pair's own checks, in its order (contraction.cpp:74-87)
  if (nshared == 0) throw std::invalid_argument("contract_pair needs at least one shared leg");
  const std::vector<int> la(legs_a, legs_a + nshared), lb(legs_b, legs_b + nshared);
  check_leg_list(rank_a, la, "left");
  check_leg_list(rank_b, lb, "right");
  PairJob j;
  j.w = dim == 4 ? 2 : 1;
  j.ra = rank_a;
  j.rb = rank_b;
  j.k = nshared;
  j.out_rank = rank_a + rank_b - 2 * nshared;
  if (max_rank >= 0 && j.out_rank > max_rank) throw RankGuard(j.out_rank, max_rank);
  const std::vector<int> fe = free_legs(rank_a, la), ff = free_legs(rank_b, lb);
  const int bits_total = j.w * std::max(std::max(rank_a, rank_b), j.out_rank);
  if (bits_total > 34) throw std::invalid_argument("tensor exceeds 2^34 elements");
  j.M = int64_t{1} << (j.w * static_cast<int>(fe.size()));
  j.K = int64_t{1} << (j.w * nshared);
  j.N = int64_t{1} << (j.w * static_cast<int>(ff.size()));
  const std::vector<int64_t> kA = leg_table(rank_a, j.w, la), kB = leg_table(rank_b, j.w, lb);
  const std::vector<int64_t> mA = leg_table(rank_a, j.w, fe), nB = leg_table(rank_b, j.w, ff);
  j.tabs.reserve(static_cast<size_t>(2 * j.K + 2 * j.M + 2 * j.N));
  j.tabs.insert(j.tabs.end(), kA.begin(), kA.end());
  j.tabs.insert(j.tabs.end(), kB.begin(), kB.end());
  j.tabs.insert(j.tabs.end(), mA.begin(), mA.end());
  j.tabs.insert(j.tabs.end(), nB.begin(), nB.end());
  for (int64_t m = 0; m < j.M; ++m) j.tabs.push_back(m * j.N);  // result: row-major M x N
  for (int64_t n = 0; n < j.N; ++n) j.tabs.push_back(n);
  // staging order: walk k across threads when the operand's fastest leg is a shared one
  j.a_kfast = std::find(la.begin(), la.end(), rank_a - 1) != la.end();
  j.b_kfast = std::find(lb.begin(), lb.end(), rank_b - 1) != lb.end();
  j.c_pair = j.N >= 2;
  const bool dense = j.K >= kGemmBK && j.M >= 8 && j.N >= 8;
  if (path == QC_PAIR_AUTO) path = dense ? QC_PAIR_DMMA : QC_PAIR_SMALL;
  if ((path == QC_PAIR_DMMA || path == QC_PAIR_DFMA) && j.K < kGemmBK)
    throw std::invalid_argument("the GEMM paths need at least " + std::to_string(kGemmBK) + " summed index values");
  j.path = path;
  return j;
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t bytes, const char* what) { ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), what); }
};

void launch_pair(const PairJob& j, const GemmDesc& d, const double2* A, const double2* B, double2* C, cudaStream_t s) {
  static bool attr_done[64] = {};
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 64 && !attr_done[dev]) {
    ck(cudaFuncSetAttribute(k_zgemm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmemBytes), "smem attr");
    ck(cudaFuncSetAttribute(k_zgemm_dfma, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmemBytes), "smem attr");
    attr_done[dev] = true;
  }
  if (j.path == QC_PAIR_SMALL) {
    const int64_t total = j.M * j.N;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    k_contract_small<<<dim3(grid, 1, 1), 256, 0, s>>>(d, A, B, C);
  } else {
    const int64_t tiles = ((j.M + kGemmBM - 1) / kGemmBM) * ((j.N + kGemmBN - 1) / kGemmBN);
    if (tiles > 0x7fffffff) throw std::invalid_argument("too many result tiles");
    const dim3 grid(static_cast<unsigned>(tiles), 1, 1);
    if (j.path == QC_PAIR_DMMA) k_zgemm_dmma<<<grid, kGemmThreads, kGemmSmemBytes, s>>>(d, A, B, C);
    else k_zgemm_dfma<<<grid, kGemmThreads, kGemmSmemBytes, s>>>(d, A, B, C);
  }
  ck(cudaGetLastError(), "contract_pair launch");
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return QC_OK;
  } catch (const RankGuard& e) {
    set_last_error(e.what());
    return QC_ERANK;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return QC_EINVAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return QC_EINTERNAL;
  } catch (...) {
    set_last_error("unknown error");
    return QC_EINTERNAL;
  }
}

// One resident problem: operands, tables and result on the device.
struct PairRun {
  PairJob job;
  GemmDesc desc{};
  DevBuf a, b, c, tabs, flush;
  cudaStream_t stream = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  size_t na = 0, nb = 0, nc = 0;
  ~PairRun() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (stream) cudaStreamDestroy(stream);
  }
  void setup(int device, int dim, int rank_a, const int32_t* legs_a, int rank_b, const int32_t* legs_b, int nshared,
             int max_rank, int path) {
    job = plan_pair_job(dim, rank_a, legs_a, rank_b, legs_b, nshared, max_rank, path);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
      throw std::runtime_error("CUDA device " + std::to_string(device) + " is not available (no CPU fallback)");
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    na = size_t{1} << (job.w * job.ra);
    nb = size_t{1} << (job.w * job.rb);
    nc = size_t{1} << (job.w * job.out_rank);
    a.alloc(na * 16, "cudaMalloc a");
    b.alloc(nb * 16, "cudaMalloc b");
    c.alloc(nc * 16, "cudaMalloc out");
    tabs.alloc(job.tabs.size() * 8, "cudaMalloc tables");
    ck(cudaMemcpyAsync(tabs.p, job.tabs.data(), job.tabs.size() * 8, cudaMemcpyHostToDevice, stream), "upload tables");
    desc.M = job.M;
    desc.N = job.N;
    desc.K = job.K;
    desc.batch = 1;
    desc.btabs = nullptr;
    desc.tabs = static_cast<const int64_t*>(tabs.p);
    desc.a_kfast = job.a_kfast;
    desc.b_kfast = job.b_kfast;
    desc.c_pair = job.c_pair;
  }
  void upload(const double* ha, const double* hb) {
    ck(cudaMemcpyAsync(a.p, ha, na * 16, cudaMemcpyHostToDevice, stream), "upload a");
    ck(cudaMemcpyAsync(b.p, hb, nb * 16, cudaMemcpyHostToDevice, stream), "upload b");
  }
  void run() {
    launch_pair(job, desc, static_cast<const double2*>(a.p), static_cast<const double2*>(b.p),
                static_cast<double2*>(c.p), stream);
  }
  void download(double* out) {
    ck(cudaMemcpyAsync(out, c.p, nc * 16, cudaMemcpyDeviceToHost, stream), "download");
    ck(cudaStreamSynchronize(stream), "sync");
  }
};

}  // namespace

extern "C" {

QC_API int qc_contract_pair(int device, int dim, int rank_a, const double* a, const int32_t* legs_a, int rank_b,
                            const double* b, const int32_t* legs_b, int nshared, int max_rank, int path,
                            double* out) {
  return guarded([&] {
    if (legs_a == nullptr || legs_b == nullptr) {
      if (nshared > 0) throw std::invalid_argument("null leg list");
    }
    PairRun r;
    r.setup(device, dim, rank_a, legs_a, rank_b, legs_b, nshared, max_rank, path);
    if (a == nullptr || b == nullptr || out == nullptr) throw std::invalid_argument("null tensor buffer");
    r.upload(a, b);
    r.run();
    r.download(out);
  });
}

QC_API int qc_contract_pair_bench(int device, int dim, int rank_a, const double* a, const int32_t* legs_a,
                                  int rank_b, const double* b, const int32_t* legs_b, int nshared, int path,
                                  int reps, int warmup, int flush_l2, double* out, double* kernel_ms,
                                  double* e2e_ms, int32_t* path_used) {
  return guarded([&] {
    if (reps < 1 || warmup < 0) throw std::invalid_argument("reps must be >= 1 and warmup >= 0");
    if (a == nullptr || b == nullptr || legs_a == nullptr || legs_b == nullptr)
      throw std::invalid_argument("null argument");
    PairRun r;
    r.setup(device, dim, rank_a, legs_a, rank_b, legs_b, nshared, -1, path);
    if (path_used) *path_used = r.job.path;
    r.upload(a, b);
    constexpr size_t kFlushBytes = size_t{512} << 20;
    if (flush_l2) r.flush.alloc(kFlushBytes, "cudaMalloc flush");
    for (int i = 0; i < warmup; ++i) r.run();
    ck(cudaStreamSynchronize(r.stream), "sync");
    // kernel time: CUDA events on the launch stream around each launch, inputs resident
    double total = 0;
    for (int i = 0; i < reps; ++i) {
      if (flush_l2) ck(cudaMemsetAsync(r.flush.p, i & 0xff, kFlushBytes, r.stream), "flush");
      ck(cudaEventRecord(r.e0, r.stream), "event");
      r.run();
      ck(cudaEventRecord(r.e1, r.stream), "event");
      ck(cudaEventSynchronize(r.e1), "sync");
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, r.e0, r.e1), "elapsed");
      total += ms;
    }
    if (kernel_ms) *kernel_ms = total / reps;
    // end to end: host operands in, host result out (pinned staging is the caller's choice)
    if (e2e_ms) {
      std::vector<double> tmp;
      double* dst = out;
      if (dst == nullptr) {
        tmp.resize(2 * r.nc);
        dst = tmp.data();
      }
      double tot2 = 0;
      for (int i = 0; i < reps; ++i) {
        ck(cudaEventRecord(r.e0, r.stream), "event");
        r.upload(a, b);
        r.run();
        ck(cudaMemcpyAsync(dst, r.c.p, r.nc * 16, cudaMemcpyDeviceToHost, r.stream), "download");
        ck(cudaEventRecord(r.e1, r.stream), "event");
        ck(cudaEventSynchronize(r.e1), "sync");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, r.e0, r.e1), "elapsed");
        tot2 += ms;
      }
      *e2e_ms = tot2 / reps;
    } else if (out) {
      r.download(out);
    }
  });
}

}  // extern "C"
