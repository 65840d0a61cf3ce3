// sm_100a kernels of the sliced-contraction engine.
//
// The hot path of the reference is sum_range -> apply_cut -> execute_plan ->
// contract_pair (proj/core/src/executor.cpp:45-68, cutting.cpp:67-129,
// contraction.cpp:288-319, contraction.cpp:71-116). On the device a pass runs
// one reference plan over a batch of 2^b slices at once:
//   k_advance  picks the pass's RunState (slice-id base, range, output slot)
//   k_prep     apply_cut as a gather: initial tensors whose cut legs are fixed by
//              the pass's high slice-id bits (slice bits decoded on the device)
//   k_tiles    one launch per dependency wave: every non-gate PlanStep of the
//              wave as shared-memory-staged batched tile contractions
//   k_gate<K>  gate-shaped PlanSteps: small operand in shared memory, big operand
//              streamed once (the dominant steps)
//   k_final    product of the rank-0 factors per slice (execute_plan's acc *=),
//              range mask, per-slice values, fixed-shape block tree reduction
// and k_reduce folds all pass partials in a fixed order (no float atomics), so
// results are bitwise reproducible run to run.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "desc.hpp"

namespace qcg {

constexpr int kStepThreads = 256;
constexpr int kFinalThreads = 256;
constexpr int kReduceThreads = 1024;

__device__ __forceinline__ uint64_t apply_runs(const Runs& r, uint64_t x) {
  uint64_t y = 0;
  for (int i = 0; i < r.n; ++i)
    y |= ((x >> r.src[i]) & ((uint64_t{1} << r.len[i]) - 1)) << r.dst[i];
  return y;
}

__device__ __forceinline__ void cmac(double2& acc, const double2 a, const double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

__device__ __forceinline__ double2 cmul(const double2 a, const double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void k_advance(const RunState* __restrict__ states, uint64_t* __restrict__ counter,
                          RunState* __restrict__ cur) {
  const uint64_t i = *counter;
  *cur = states[i];
  *counter = i + 1;
}

__global__ void k_prep(const PrepDesc* __restrict__ descs, double2* __restrict__ arena,
                       const RunState* __restrict__ st) {
  const PrepDesc& d = descs[blockIdx.y];
  const uint64_t base_id = st->pass_base;
  int64_t base = d.src;
  for (int f = 0; f < d.nfix; ++f)
    if ((base_id >> d.fix_pos[f]) & 1) base += d.fix_stride[f];
  const uint64_t n = uint64_t{1} << d.nbits;
  for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    arena[d.dst + e] = arena[base + apply_runs(d.map, e)];
}

// A wave of small/medium reference PlanSteps (all steps of one dependency level
// that are not gate-shaped) in one launch. Work item = (step, tile); prefix[i]
// is the first item of step i. Per tile: stage the A-tile and B-tile in shared
// memory (coalesced gathers), contract over the summed bits, write the C tile
// (contiguous in C). See StepDesc (desc.hpp).
__global__ void __launch_bounds__(kStepThreads) k_tiles(const StepDesc* __restrict__ descs,
                                                        const uint64_t* __restrict__ prefix, int nsteps,
                                                        uint64_t items, double2* __restrict__ arena) {
  __shared__ StepDesc d;
  __shared__ int cur;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int loaded = -1;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    if (threadIdx.x == 0) {
      int lo = 0, hi = nsteps - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= item) lo = mid;
        else hi = mid - 1;
      }
      cur = lo;
    }
    __syncthreads();
    const int step = cur;
    if (step != loaded) {
      const int4* src = reinterpret_cast<const int4*>(descs + step);
      int4* dst = reinterpret_cast<int4*>(&d);
      for (int i = threadIdx.x; i < static_cast<int>(sizeof(StepDesc) / 16); i += blockDim.x) dst[i] = src[i];
      __syncthreads();
      loaded = step;
    }
    const int nA = 1 << d.nTA, nB = 1 << d.nTB, nS = 1 << d.nS, nC = 1 << d.nTC;
    double2* As = reinterpret_cast<double2*>(smem_raw);
    double2* Bs = As + nA;
    int* sa = reinterpret_cast<int*>(Bs + nB);
    int* sb = sa + nS;
    for (int s = threadIdx.x; s < nS; s += blockDim.x) {
      sa[s] = static_cast<int>(apply_runs(d.sA, s));
      sb[s] = static_cast<int>(apply_runs(d.sB, s));
    }
    const uint64_t g = item - prefix[step];
    const double2* __restrict__ A = arena + d.offA + static_cast<int64_t>(apply_runs(d.gA, g));
    const double2* __restrict__ B = arena + d.offB + static_cast<int64_t>(apply_runs(d.gB, g));
    for (int e = threadIdx.x; e < nA; e += blockDim.x) As[e] = A[apply_runs(d.lA, e)];
    for (int e = threadIdx.x; e < nB; e += blockDim.x) Bs[e] = B[apply_runs(d.lB, e)];
    __syncthreads();
    double2* Cg = arena + d.offC + (g << d.nTC);
    for (int c = threadIdx.x; c < nC; c += blockDim.x) {
      const int ia = static_cast<int>(apply_runs(d.cA, c));
      const int ib = static_cast<int>(apply_runs(d.cB, c));
      double2 acc = make_double2(0.0, 0.0);
      for (int s = 0; s < nS; ++s) cmac(acc, As[ia + sa[s]], Bs[ib + sb[s]]);
      Cg[c] = acc;
    }
    __syncthreads();
  }
}

// Gate-shaped PlanStep (see GateDesc): small operand G whole in shared memory,
// big operand X streamed once; each thread owns columns j of X, holds its K
// summed values in registers and writes the 2^nF outputs of the column.
template <int K>
__global__ void __launch_bounds__(kStepThreads) k_gate(const __grid_constant__ GateDesc d,
                                                       double2* __restrict__ arena) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Gs = reinterpret_cast<double2*>(smem_raw);
  const int nGe = 1 << d.nG, nFe = 1 << d.nF;
  int* gft = reinterpret_cast<int*>(Gs + nGe);
  for (int e = threadIdx.x; e < nGe; e += blockDim.x) Gs[e] = arena[d.offG + e];
  for (int f = threadIdx.x; f < nFe; f += blockDim.x) gft[f] = static_cast<int>(apply_runs(d.gf, f));
  int64_t xs[K];
  int gs[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    xs[s] = static_cast<int64_t>(apply_runs(d.xs, s));
    gs[s] = static_cast<int>(apply_runs(d.gs, s));
  }
  __syncthreads();
  const double2* __restrict__ X = arena + d.offX;
  double2* __restrict__ C = arena + d.offC;
  const uint64_t ncol = uint64_t{1} << d.nCol;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < ncol; j += stride) {
    const int64_t xo = static_cast<int64_t>(apply_runs(d.xcol, j));
    const int go = static_cast<int>(apply_runs(d.gcol, j));
    double2 b[K];
#pragma unroll
    for (int s = 0; s < K; ++s) b[s] = __ldcs(X + xo + xs[s]);
    for (int f = 0; f < nFe; ++f) {
      const double2* gp = Gs + go + gft[f];
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < K; ++s) cmac(acc, gp[gs[s]], b[s]);
      C[(static_cast<uint64_t>(f) << d.nCol) + j] = acc;
    }
  }
}

__device__ __forceinline__ double2 block_reduce(double2 v, double2* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sh[threadIdx.x].x += sh[threadIdx.x + w].x;
      sh[threadIdx.x].y += sh[threadIdx.x + w].y;
    }
    __syncthreads();
  }
  return sh[0];
}

// Per-slice value = product of the rank-0 factors (step order, then leftover
// vertices ascending), masked to [lo, hi), summed with a fixed tree.
__global__ void __launch_bounds__(kFinalThreads) k_final(const FactorDesc* __restrict__ f, int nf, int b,
                                                         int per_thread, const double2* __restrict__ arena,
                                                         const RunState* __restrict__ st,
                                                         double2* __restrict__ partials) {
  __shared__ double2 sh[kFinalThreads];
  const RunState s = *st;
  const uint64_t nloc = uint64_t{1} << b;
  const uint64_t k0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * per_thread;
  double2 sum = make_double2(0.0, 0.0);
  double2* out = reinterpret_cast<double2*>(s.slice_out);
  for (int i = 0; i < per_thread; ++i) {
    const uint64_t k = k0 + i;
    if (k >= nloc) break;
    const uint64_t gid = s.pass_base + k;
    double2 v = make_double2(1.0, 0.0);
    for (int j = 0; j < nf; ++j) v = cmul(v, arena[f[j].off + apply_runs(f[j].map, k)]);
    if (gid >= s.lo && gid < s.hi) {
      sum.x += v.x;
      sum.y += v.y;
      if (out) out[gid - s.out_base] = v;
    }
  }
  const double2 tot = block_reduce(sum, sh);
  if (threadIdx.x == 0) partials[s.slot * gridDim.x + blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kReduceThreads) k_reduce(const double2* __restrict__ partials, uint64_t n,
                                                           double2* __restrict__ result) {
  __shared__ double2 sh[kReduceThreads];
  double2 sum = make_double2(0.0, 0.0);
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
    sum.x += partials[i].x;
    sum.y += partials[i].y;
  }
  const double2 tot = block_reduce(sum, sh);
  if (threadIdx.x == 0) *result = tot;
}

}  // namespace qcg
