// sm_100a kernels of the sliced-contraction engine.
//
// The hot path of the reference is sum_range -> apply_cut -> execute_plan ->
// contract_pair (proj/core/src/executor.cpp:45-68, cutting.cpp:67-129,
// contraction.cpp:288-319, contraction.cpp:71-116). On the device a pass runs
// one reference plan over a batch of 2^b slices at once:
//   k_advance  picks the pass's RunState (slice-id base, range, output slot)
//   k_prep     apply_cut as a gather: initial tensors whose cut legs are fixed by
//              the pass's high slice-id bits (slice bits decoded on the device)
//   k_flow     persistent dataflow executor: every small PlanStep between two big
//              ops, as shared-memory-staged batched tile contractions, with
//              per-step completion counters resolving dependencies on the device
//   k_gate<K>  gate-shaped PlanSteps: small operand in shared memory, big operand
//              streamed once (the dominant steps)
//   k_chain    consecutive gate steps fused: intermediates stay in shared memory
//   k_pair     two gate steps fused at register level (large intermediates)
//   k_final    product of the rank-0 factors per slice (execute_plan's acc *=),
//              range mask, per-slice values, fixed-shape block tree reduction; the
//              last CTA of a call's last pass folds all pass partials in a fixed
//              order (no float atomics), so results are bitwise reproducible
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "desc.hpp"

namespace qcg {

constexpr int kStepThreads = 256;
#ifndef QCG_FLOW_THREADS
#define QCG_FLOW_THREADS 256
#endif
constexpr int kFlowThreads = QCG_FLOW_THREADS;  // k_flow CTA size (tiles are <= 2^8 outputs)
#ifndef QCG_FLOW_SLEEP
#define QCG_FLOW_SLEEP 64  // ns between k_flow's dependency polls
#endif
constexpr int kFinalThreads = 256;
constexpr uint64_t kMaxCallPasses = 1 << 14;  // pass-state / partial buffers per call chunk

__device__ __forceinline__ uint64_t apply_runs(const Runs& r, uint64_t x) {
  uint64_t y = 0;
  for (int i = 0; i < r.n; ++i)
    y |= ((x >> r.src[i]) & ((uint64_t{1} << r.len[i]) - 1)) << r.dst[i];
  return y;
}

// Programmatic dependent launch (the engine launches every kernel with programmatic stream
// serialization): wait for the previous kernel's completion and memory before touching
// anything it produced (a no-op for a kernel launched without the attribute). No kernel
// triggers early: measured, dependents that launch at the primary's start hold SM slots
// while they wait and slow the primary down (config 2 0.295 -> 0.365 ms).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Experiment knob: kernels whose bit is set trigger their dependents at their own start
// (bit 0 forest, 1 gate, 2 chain, 3 pair, 4 flow, 5 advance/prep/final).
#ifndef QCG_PDL_EARLY
#define QCG_PDL_EARLY 0
#endif
template <int BIT>
__device__ __forceinline__ void pdl_early() {
  if constexpr ((QCG_PDL_EARLY >> BIT) & 1) pdl_trigger();
}

// Operand staging with asynchronous 16-byte copies: every element's copy is issued before
// any completes (one L2/HBM round trip for the whole tile instead of one per loop trip).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
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

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// QCG_KTRACE (build flag, measurement only): CTA (0,0) of every kernel prints its start,
// the end of its dependency wait and its end (globaltimer ns) -- the in-graph timeline of a pass.
#ifdef QCG_KTRACE
// (records go to a device array through one atomic slot counter -- ~1 us at the end of CTA 0;
// the engine prints and clears them after every call)
constexpr int kKtMax = 4096;
__device__ unsigned int g_kt_n;
__device__ unsigned long long g_kt[kKtMax * 8];
#define KT_BEGIN const unsigned long long kt0 = globaltimer();
#define KT_WAIT const unsigned long long kt1 = globaltimer();
// (every CTA also folds its end time into a small table keyed by kernel name and grid: the
// last CTA's end of same-shaped launches within one call)
__device__ unsigned long long g_kt_last[256];
#define KT_END_M(name, m)                                                                      \
  if (threadIdx.x == 0)                                                                          \
    atomicMax(&g_kt_last[(static_cast<unsigned>(name[0]) * 7u + gridDim.x * 131u + gridDim.y) & 255u], globaltimer()); \
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {                                  \
    const unsigned long long kt2 = globaltimer();                                                \
    const unsigned slot = atomicAdd(&g_kt_n, 1u);                                                \
    if (slot < kKtMax) {                                                                         \
      g_kt[8 * slot] = (static_cast<unsigned long long>(name[0]) << 56) |                        \
                       (static_cast<unsigned long long>(name[1]) << 48) |                        \
                       (static_cast<unsigned long long>(gridDim.x) << 16) | gridDim.y;           \
      g_kt[8 * slot + 1] = kt0;                                                                  \
      g_kt[8 * slot + 2] = kt1;                                                                  \
      g_kt[8 * slot + 3] = kt2;                                                                  \
      for (int q_ = 0; q_ < 4; ++q_) g_kt[8 * slot + 4 + q_] = (m)[q_];                          \
    }                                                                                            \
  }
#define KT_END(name)                                   \
  {                                                    \
    const unsigned long long kz_[4] = {0, 0, 0, 0};    \
    KT_END_M(name, kz_)                                \
  }
#define KT_MARKS unsigned long long km_[4] = {0, 0, 0, 0};
#define KT_MARKS_PTR km_
#else
#define KT_BEGIN
#define KT_WAIT
#define KT_END(name)
#define KT_END_M(name, m)
#define KT_MARKS
#define KT_MARKS_PTR nullptr
#endif

// First node of a pass: select the pass's RunState and zero the dataflow counters
// (per-step completion/claim counters and per-launch work counters).
__global__ void k_advance(const RunState* __restrict__ states, uint64_t* __restrict__ counter,
                          RunState* __restrict__ cur, int* __restrict__ done, int n_done,
                          unsigned long long* __restrict__ work, int n_work,
                          unsigned long long* __restrict__ stamps) {
  KT_BEGIN
  pdl_early<5>();
  pdl_wait();
  KT_WAIT
  if (stamps && threadIdx.x == 0) stamps[0] = globaltimer();  // QCG_PASS_STAMPS: pass start
  KT_END("advance")
  for (int i = threadIdx.x; i < n_done; i += blockDim.x) done[i] = 0;
  for (int i = threadIdx.x; i < n_work; i += blockDim.x) work[i] = 0;
  if (threadIdx.x == 0) {
    const uint64_t i = *counter;
    *cur = states[i];
    *counter = i + 1;
  }
}

__device__ __forceinline__ void prep_body(const PrepDesc& d, double2* __restrict__ arena,
                                          const RunState* __restrict__ st, unsigned bx, unsigned gx) {
  const uint64_t base_id = st->pass_base;
  int64_t base = d.src;
  for (int f = 0; f < d.nfix; ++f)
    if ((base_id >> d.fix_pos[f]) & 1) base += d.fix_stride[f];
  const uint64_t n = uint64_t{1} << d.nbits;
  for (uint64_t e = static_cast<uint64_t>(bx) * blockDim.x + threadIdx.x; e < n; e += static_cast<uint64_t>(gx) * blockDim.x)
    arena[d.dst + e] = __ldcg(arena + base + apply_runs(d.map, e));
}

__global__ void k_prep(const PrepDesc* __restrict__ descs, double2* __restrict__ arena,
                       const RunState* __restrict__ st) {
  pdl_early<5>();
  pdl_wait();
  prep_body(descs[blockIdx.y], arena, st, blockIdx.x, gridDim.x);
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}


__device__ __forceinline__ int atom_add_acqrel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Persistent dataflow executor for a group of small/medium tile-kind PlanSteps
// (everything between two big fused/gate ops). CTAs take work items (step, tile)
// in topological order from a device counter; before a tile runs, its step's
// producers inside the group must have finished all their tiles (per-step
// completion counters, release/acquire at GPU scope). Items are handed out in
// order and only wait on earlier items, so the schedule cannot deadlock. One
// launch replaces one launch per dependency level.
//
// Continuation (the latency path of the deep, narrow dependency chains): a
// single-tile step c whose in-group producers all feed only c is "continuation-only"
// (conly[c]): the queue skips it, and the CTA that completes the last of its
// producers runs it next -- detected by the value an acq_rel atomic returns, so a
// chain level costs the release of the producer, at most one more atomic and the
// operand loads, with no polling. Its descriptor is prefetched (cp.async) into a
// second shared-memory buffer while the producer runs.
__global__ void __launch_bounds__(kFlowThreads) k_flow(const StepDesc* __restrict__ descs,
                                                       const uint64_t* __restrict__ prefix,
                                                       const int* __restrict__ dep_off,
                                                       const int* __restrict__ deps, int* __restrict__ done,
                                                       const int* __restrict__ cont, const int* __restrict__ conly,
                                                       int* __restrict__ pend, unsigned long long* __restrict__ work,
                                                       int nsteps, uint64_t items, int npre,
                                                       double2* __restrict__ arena,
                                                       unsigned long long* __restrict__ trace) {
  __shared__ StepDesc dbuf[2];
  __shared__ int cur, s_cont;
  __shared__ unsigned long long s_dbg;
  __shared__ unsigned long long s_item;
  __shared__ int64_t s_ab[2];
  // schedule tables in shared memory (the step lookup is a binary search: keep its
  // probes off the L2 latency path)
  constexpr int kFlowSmemSteps = 1024;
  __shared__ uint64_t s_prefix[kFlowSmemSteps + 1];
  __shared__ int s_depoff[kFlowSmemSteps + 1];
  const bool in_smem = nsteps <= kFlowSmemSteps;
  if (in_smem) {
    for (int i = threadIdx.x; i <= nsteps; i += blockDim.x) {
      s_prefix[i] = prefix[i];
      s_depoff[i] = dep_off[i];
    }
  }
  const uint64_t* pf = in_smem ? s_prefix : prefix;
  const int* dof = in_smem ? s_depoff : dep_off;
  pdl_early<4>();
  pdl_wait();  // the schedule tables above are static; the operands are not
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int bstep0 = -1, bstep1 = -1;  // step whose descriptor each buffer holds (uniform across the CTA)
  int use = 0;
  // shared-memory hand-off: the last single-tile output of this CTA stays in Cs (the
  // first kFlowCs elements of the dynamic shared memory); a continuation reads that
  // operand from there. When the continuation has no other in-group producer the
  // output is not written to HBM and not released at all (nobody else reads it).
  int64_t cs_off = -1;  // arena offset of the tensor held in Cs, -1: none
  __shared__ int s_next;  // continuation step this CTA runs next, or -1
  // operand prefetch for a CTA-private continuation: its other operand comes from outside
  // the group (complete since pdl_wait), so it is staged into P[pbuf] while the producer
  // computes; pre_op = 0/1: A/B of the next item is already in P[pbuf], -1: none
  int pbuf = 0, pre_op = -1;
  if (threadIdx.x == 0) s_next = -1;
  constexpr int kDescChunks = static_cast<int>(sizeof(StepDesc) / 16);
  __syncthreads();
  for (;;) {
    unsigned long long t0 = 0, t1 = 0, t2 = 0;
    if (threadIdx.x < 32) {
      // warp 0: pick the next item (lane 0), then wait until the step's in-group
      // producers are complete -- one dependency per lane, converged, relaxed polls with
      // a short sleep, one acquire per dependency once reached -- all before the CTA
      // barrier below, so no other warp can touch the operands early. A continuation's
      // producers are complete by construction.
      const int lane = threadIdx.x;
      if (lane == 0) {
        if (s_next >= 0) {
          cur = s_next;
          s_item = pf[s_next];
          s_cont = 1;
        } else {
          s_cont = 0;
          for (;;) {
            const unsigned long long it = atomicAdd(work, 1ull);
            s_item = it;
            if (it >= items) break;
            int lo = 0, hi = nsteps - 1;
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (pf[mid] <= it) lo = mid;
              else hi = mid - 1;
            }
            cur = lo;
            if (conly[lo]) continue;  // run by the CTA that completes its last producer
            break;
          }
        }
        if (trace) t0 = globaltimer();
      }
      __syncwarp();
      if (s_item < items && cur != bstep0 && cur != bstep1) {
        // descriptor not staged: warp 0 fetches it (cp.async) while it waits below, into
        // the buffer every thread will select after the barrier (same rule, uniform state)
        const char* src = reinterpret_cast<const char*>(descs + cur);
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&dbuf[1 - use]));
        for (int i = lane; i < kDescChunks; i += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * i), "l"(src + 16 * i)
                       : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      }
      if (s_item < items && !s_cont) {
        const int st = cur;
        const int k0 = dof[st], nd = dof[st + 1] - k0;
        const int q = lane < nd ? deps[k0 + lane] : 0;
        const int need = lane < nd ? static_cast<int>(pf[q + 1] - pf[q]) : 0;
        for (;;) {
          const bool ok = lane >= nd || ld_relaxed(done + q) >= need;
          if (__all_sync(0xffffffffu, ok)) break;
#if QCG_FLOW_SLEEP > 0
          __nanosleep(QCG_FLOW_SLEEP);
#endif
        }
        if (lane < nd) (void)ld_acquire(done + q);
        __syncwarp();
      }
      if (trace && lane == 0) t1 = globaltimer();
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");  // a prefetched descriptor has landed
    __syncthreads();
    const uint64_t item = s_item;
    if (item >= items) break;
    const int step = cur;
    if (bstep0 == step) {
      use = 0;
    } else if (bstep1 == step) {
      use = 1;
    } else {
      use = 1 - use;  // staged by warp 0 before the barrier above
      (use ? bstep1 : bstep0) = step;
    }
    const StepDesc& d = dbuf[use];
    {
      // prefetch the continuation's descriptor into the other buffer
      const int c = cont[step];
      if (c >= 0 && bstep0 != c && bstep1 != c) {
        const int other = 1 - use;
        const char* src = reinterpret_cast<const char*>(descs + c);
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&dbuf[other]));
        for (int i = threadIdx.x; i < kDescChunks; i += blockDim.x)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * i), "l"(src + 16 * i)
                       : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        (other ? bstep1 : bstep0) = c;
      }
    }
    const int nA = 1 << d.nTA, nB = 1 << d.nTB, nS = 1 << d.nS, nC = 1 << d.nTC;
    double2* Cs = reinterpret_cast<double2*>(smem_raw);
    double2* P = Cs + kFlowCs;  // two prefetch buffers of npre elements
    double2* As = P + 2 * npre;
    double2* Bs = As + nA;
    int* sa = reinterpret_cast<int*>(Bs + nB);
    const int pre_in = s_cont ? pre_op : -1;  // operand staged by the previous item
    pre_op = -1;
    int* sb = sa + nS;
    // index tables first: they do not depend on the producers
    for (int s2 = threadIdx.x; s2 < nS; s2 += blockDim.x) {
      sa[s2] = static_cast<int>(apply_runs(d.sA, s2));
      sb[s2] = static_cast<int>(apply_runs(d.sB, s2));
    }
    const uint64_t g = item - pf[step];
    if (threadIdx.x == 0) s_ab[0] = static_cast<int64_t>(apply_runs(d.gA, g));
    if (threadIdx.x == 32) s_ab[1] = static_cast<int64_t>(apply_runs(d.gB, g));
    __syncthreads();
    const bool a_sm = s_cont && d.offA == cs_off, b_sm = s_cont && d.offB == cs_off;
    const double2* A = a_sm ? Cs + s_ab[0] : arena + d.offA + s_ab[0];
    const double2* B = b_sm ? Cs + s_ab[1] : arena + d.offB + s_ab[1];
    // L2-coherent loads: producers ran on other SMs within this launch
    if (pre_in == 0) As = P + pbuf * npre;
    else if (a_sm) for (int e = threadIdx.x; e < nA; e += blockDim.x) As[e] = A[apply_runs(d.lA, e)];
    else for (int e = threadIdx.x; e < nA; e += blockDim.x) cp_async16(As + e, A + apply_runs(d.lA, e));
    if (pre_in == 1) Bs = P + pbuf * npre;
    else if (b_sm) for (int e = threadIdx.x; e < nB; e += blockDim.x) Bs[e] = B[apply_runs(d.lB, e)];
    else for (int e = threadIdx.x; e < nB; e += blockDim.x) cp_async16(Bs + e, B + apply_runs(d.lB, e));
    cp_async_wait();
    unsigned long long tm = 0;
    if (trace && (threadIdx.x & 31) == 0) {
      // per-warp: when this warp's loads returned (first use of the loaded values)
      double2 v = threadIdx.x < nA ? As[threadIdx.x] : make_double2(0, 0);
      tm = globaltimer() + (v.x == 12345.678 ? 1 : 0);
    }
    __syncthreads();
    if (trace && threadIdx.x == 0) t2 = globaltimer();
    if (trace) {
      __shared__ unsigned long long s_tm[kFlowThreads / 32];
      if ((threadIdx.x & 31) == 0) s_tm[threadIdx.x >> 5] = tm;
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long mx = 0;
        int wmx = 0;
        for (int w = 0; w < kFlowThreads / 32; ++w)
          if (s_tm[w] > mx) mx = s_tm[w], wmx = w;
        t1 = (t1 & 0xffffffffffull) | (static_cast<unsigned long long>(wmx) << 56) |
             ((s_tm[0] - t1) & 0xffff) << 40;  // warp 0's own load latency (ns), slowest warp
      }
    }
    double2* Cg = arena + d.offC + (g << d.nTC);
    const int cnext = cont[step];
    const int ntiles = static_cast<int>(pf[step + 1] - pf[step]);
    // single-tile step with a continuation: keep the tile in Cs; with no other in-group
    // producer of the continuation (a CTA-private hand-off) skip HBM and the release
    const bool keep = ntiles == 1 && cnext >= 0 && nC <= kFlowCs;
    const bool priv = keep && dof[cnext + 1] - dof[cnext] <= 1;
#if QCG_FLOW_PREFETCH
    if (priv && npre > 0) {
      // c runs next on this CTA; its descriptor landed with the loads above (cp.async
      // group waited, then the barrier). One operand is this step's output (kept in Cs);
      // issue the other's loads now, they complete while this step computes
      const StepDesc* dn = bstep0 == cnext ? &dbuf[0] : (bstep1 == cnext ? &dbuf[1] : nullptr);
      if (dn != nullptr) {
        const int which = dn->offA == d.offC ? 1 : (dn->offB == d.offC ? 0 : -1);
        const int nX = which == 0 ? 1 << dn->nTA : 1 << dn->nTB;
        if (which >= 0 && nX <= npre) {
          const int64_t off = which == 0 ? dn->offA + static_cast<int64_t>(apply_runs(dn->gA, 0))
                                         : dn->offB + static_cast<int64_t>(apply_runs(dn->gB, 0));
          const double2* X = arena + off;
          double2* Pn = P + (pbuf ^ 1) * npre;
          if (which == 0) for (int e = threadIdx.x; e < nX; e += blockDim.x) cp_async16(Pn + e, X + apply_runs(dn->lA, e));
          else for (int e = threadIdx.x; e < nX; e += blockDim.x) cp_async16(Pn + e, X + apply_runs(dn->lB, e));
          asm volatile("cp.async.commit_group;\n" ::: "memory");
          pbuf ^= 1;
          pre_op = which;
        }
      }
    }
#endif
    for (int c = threadIdx.x; c < nC; c += blockDim.x) {
      const int ia = static_cast<int>(apply_runs(d.cA, c));
      const int ib = static_cast<int>(apply_runs(d.cB, c));
      double2 acc = make_double2(0.0, 0.0);
      for (int s2 = 0; s2 < nS; ++s2) cmac(acc, As[ia + sa[s2]], Bs[ib + sb[s2]]);
      if (keep) Cs[c] = acc;
      if (!priv) __stcg(Cg + c, acc);
    }
    cs_off = keep ? d.offC : -1;
    __syncthreads();
    if (threadIdx.x == 0) {
      int nxt = -1;
      if (priv) {
        nxt = cnext;  // c's only in-group producer: run it here, nothing to publish
      } else if (ntiles == 1 && cnext >= 0) {
        // c (continuation-only, never polled) is this step's only consumer: its pending
        // count alone publishes the tile (acq_rel), no completion counter needed
        const int nd = dof[cnext + 1] - dof[cnext];
        if (atom_add_acqrel(pend + cnext, 1) == nd - 1) nxt = cnext;
      } else {
        // release at GPU scope: the CTA's stores (ordered before by the barrier) are
        // visible to any thread that acquires this counter
        bool complete = true;
        if (ntiles == 1) asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(done + step) : "memory");
        else complete = atom_add_acqrel(done + step, 1) == ntiles - 1;  // acquires the other tiles
        if (complete && cnext >= 0) {
          const int nd = dof[cnext + 1] - dof[cnext];
          // the last of c's producers to complete runs c
          if (nd <= 1 || atom_add_acqrel(pend + cnext, 1) == nd - 1) nxt = cnext;
        }
      }
      s_next = nxt;
      if (trace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* tr = trace + 8 * item;
        tr[6] = static_cast<unsigned long long>(d.offA + s_ab[0]);

        tr[0] = (static_cast<unsigned long long>(step) << 32) | (static_cast<unsigned long long>(d.nTB) << 24) |
                (static_cast<unsigned long long>(d.nTA) << 16) | (static_cast<unsigned long long>(smid) << 8) |
                static_cast<unsigned long long>(s_cont);
        tr[1] = t0;
        tr[2] = t1;
        tr[3] = t2;
        tr[4] = globaltimer();
        tr[5] = s_dbg;
        tr[7] = 0;
        s_dbg = 0;
      }
    }
  }
}

// ---- TMA bulk copies (cp.async.bulk) completing on a CTA-local mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ uint32_t fmap_apply(const FMap& m, uint32_t x) {
  uint32_t y = 0;
  const int n = m.n;
  for (int i = 0; i < n; ++i) {
    const uint32_t r = m.r[i];
    y |= ((x >> (r & 31u)) & ((1u << ((r >> 5) & 31u)) - 1u)) << (r >> 10);
  }
  return y;
}

// A dataflow group of small steps (desc.hpp, k_forest): CTA = one unit (independent
// subtrees). Prologue: the unit's image (phases, work items, step descriptors) and every
// staged leaf operand arrive by bulk copy (TMA) on one mbarrier -- the image is static, so
// its copy is issued before the dependency wait and overlaps the previous kernel's tail.
// Then the unit's phases run back to back: warps take 32-output chunks of the phase's
// steps (a warp's lanes share one step, so descriptor reads are broadcasts), one barrier
// per phase. Intermediates stay in shared memory where they fit; roots and rank-0 factors
// go to the arena.
#ifndef QCG_FOREST_THREADS
#define QCG_FOREST_THREADS 512
#endif
constexpr int kForestThreads = QCG_FOREST_THREADS;
constexpr int kForestTracePhases = 29, kForestTraceWords = 3 + kForestTracePhases;
// One lane, one column of a forest step (FStep): the K values of X in registers, then the
// 2^nLoop outputs of the column with independent accumulators.
// (K = 16 runs as two halves of 8: the X values of one half in registers at a time.)
template <int K>
__device__ __forceinline__ void forest_column(const FStep& d, const double2* G, const double2* X, double2* C,
                                              uint32_t xo, uint32_t go, uint32_t co) {
  constexpr int KH = K > 8 ? 8 : K;
  const int nl = 1 << d.nLoop;
  double2 acc[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) acc[l] = make_double2(0.0, 0.0);
#pragma unroll
  for (int h = 0; h < K / KH; ++h) {
    double2 xv[KH];
#pragma unroll
    for (int s2 = 0; s2 < KH; ++s2) xv[s2] = X[xo + d.tx[h * KH + s2]];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      if (l < nl) {
        const uint32_t gl = go + d.loopG[l];
#pragma unroll
        for (int s2 = 0; s2 < KH; ++s2) cmac(acc[l], G[gl + d.tg[h * KH + s2]], xv[s2]);
      }
    }
  }
#pragma unroll
  for (int l = 0; l < 4; ++l)
    if (l < nl) C[co + d.loopC[l]] = acc[l];
}
// One unit on one CTA; `smem` = dynamic shared memory base (mbarrier, image, data region).
// `dep_wait`: wait for the previous grid (PDL) after issuing the static image copy.
__device__ __forceinline__ void forest_body(const ForestUnit& u, const int32_t* __restrict__ img_all, double2* arena,
                                            unsigned char* smem, bool dep_wait, unsigned long long* trace = nullptr) {
  unsigned long long t0 = 0, t1 = 0;
  if (trace && threadIdx.x == 0) t0 = globaltimer();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  const int32_t* gimg = img_all + u.img;
  int32_t* img = reinterpret_cast<int32_t*>(smem + 16);
  double2* data = reinterpret_cast<double2*>(smem + u.data_off);
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, static_cast<unsigned>(u.img_words) * 4u + static_cast<unsigned>(u.leaf_bytes));
    bulk_g2s(img, gimg, static_cast<unsigned>(u.img_words) * 4u, bar);
  }
  int4 lf = make_int4(0, 0, 0, 0);  // this thread's first leaf entry (static)
  if (static_cast<int>(threadIdx.x) < u.nleaves) lf = __ldg(reinterpret_cast<const int4*>(gimg + u.leaf_off) + threadIdx.x);
  if (dep_wait) pdl_early<0>();
  if (dep_wait) pdl_wait();  // leaf operands may come from the previous launch
  for (int t = threadIdx.x; t < u.nleaves; t += blockDim.x) {
    if (t != static_cast<int>(threadIdx.x)) lf = __ldg(reinterpret_cast<const int4*>(gimg + u.leaf_off) + t);
    int64_t off;
    memcpy(&off, &lf, 8);
    bulk_g2s(data + lf.z, arena + off, static_cast<unsigned>(lf.w), bar);
  }
  mbar_wait(bar, 0);
  if (trace && threadIdx.x == 0) t1 = globaltimer();
  const int nph = img[0];
  const int32_t* phase_off = img + 4;
  const uint32_t* items = reinterpret_cast<const uint32_t*>(img + 4 + ((nph + 1 + 3) & ~3));
  const FStep* steps = reinterpret_cast<const FStep*>(img + u.leaf_off + 4 * u.nleaves);
  const int warp = static_cast<int>(threadIdx.x >> 5), nw = static_cast<int>(blockDim.x >> 5);
  const uint32_t lane = threadIdx.x & 31u;
  for (int p = 0; p < nph; ++p) {
    const int end = phase_off[p + 1];
    for (int it = phase_off[p] + warp; it < end; it += nw) {
      const uint32_t item = items[it];
      const FStep& d = steps[item >> 16];
      const uint32_t chunk = (item & 0xffffu) << 5;
      if ((chunk | lane) < (1u << d.nCol)) {
        const double2* G = d.sG >= 0 ? data + d.sG : arena + d.gG;
        const double2* X = d.sX >= 0 ? data + d.sX : arena + d.gX;
        double2* C = d.sC >= 0 ? data + d.sC : arena + d.gC;
        // chunk part once per item (uniform), lane part from the tables
        const uint32_t m = (chunk >> 5) & 31u, hi = (chunk >> 10) & 15u;
        const uint32_t xo = d.highX[hi] + d.midX[m] + d.laneX[lane];
        const uint32_t go = d.highG[hi] + d.midG[m] + d.laneG[lane];
        const uint32_t co = d.highC[hi] + d.midC[m] + d.laneC[lane];
        switch (d.nS) {
          case 1: forest_column<2>(d, G, X, C, xo, go, co); break;
          case 2: forest_column<4>(d, G, X, C, xo, go, co); break;
          case 3: forest_column<8>(d, G, X, C, xo, go, co); break;
          default: forest_column<16>(d, G, X, C, xo, go, co); break;
        }
      }
    }
    __syncthreads();
    if (trace && threadIdx.x == 0 && p < kForestTracePhases) trace[3 + p] = globaltimer();
  }
  if (threadIdx.x == 0) {
    mbar_inval(bar);  // the memory is ordinary shared memory again
    if (trace) {  // QCG_FOREST_TRACE: per unit {start, operands landed, end} (ns)
      trace[0] = t0;
      trace[1] = t1;
      trace[2] = globaltimer();
    }
  }
}

__global__ void __launch_bounds__(kForestThreads, 1) k_forest(const ForestUnit* __restrict__ units,
                                                               const int32_t* __restrict__ img_all,
                                                               double2* arena, unsigned long long* trace) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  KT_BEGIN
  KT_WAIT
  forest_body(units[blockIdx.x], img_all, arena, smem_raw, true,
              trace ? trace + kForestTraceWords * blockIdx.x : nullptr);
  KT_END("forest")
}

// Gate-shaped PlanStep (see GateDesc): small operand G whole in shared memory,
// big operand X streamed once; each thread owns columns j of X, holds its K
// summed values in registers and writes the 2^nF outputs of the column.
// blockIdx.y = (H_hi, F_hi): a G tile per CTA row.
template <int K>
__device__ __forceinline__ void gate_body(const GateDesc& d, double2* __restrict__ arena, unsigned char* smem_raw,
                                          unsigned bx, unsigned by, unsigned gx) {
  double2* Gs = reinterpret_cast<double2*>(smem_raw);
  const int nGe = 1 << d.nG, nFe = 1 << d.nF;
  int* gft = reinterpret_cast<int*>(Gs + nGe);
  const uint64_t fhi = by & ((1u << d.nFhi) - 1), hhi = by >> d.nFhi;
  const int64_t gbase_hi =
      d.offG + static_cast<int64_t>(apply_runs(d.gfhi, fhi)) + static_cast<int64_t>(apply_runs(d.ghhi, hhi));
  for (int e = threadIdx.x; e < nGe; e += blockDim.x) cp_async16(Gs + e, arena + gbase_hi + apply_runs(d.gtile, e));
  for (int f = threadIdx.x; f < nFe; f += blockDim.x) gft[f] = static_cast<int>(apply_runs(d.gf, f));
  int64_t xs[K];
  int gs[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    xs[s] = d.xs_tab[s];
    gs[s] = d.gs_tab[s];
  }
  const double2* __restrict__ X = arena + d.offX + static_cast<int64_t>(apply_runs(d.xhhi, hhi));
  double2* __restrict__ C = arena + d.offC + ((static_cast<int64_t>(fhi) << d.nF) << d.nCol) +
                            static_cast<int64_t>(apply_runs(d.chhi, hhi));
  const uint64_t ncol = uint64_t{1} << (d.nCol - d.nHhi);
  const uint64_t stride = static_cast<uint64_t>(gx) * blockDim.x;
  uint64_t j = static_cast<uint64_t>(bx) * blockDim.x + threadIdx.x;
  // the first column's K values of X are requested before the staged G tile is waited for:
  // one memory round trip covers both operands
  double2 b[K];
  if (j < ncol) {
    const int64_t xo = static_cast<int64_t>(apply_runs(d.xcol, j));
#pragma unroll
    for (int s = 0; s < K; ++s) b[s] = __ldcs(X + xo + xs[s]);
  }
  cp_async_wait();
  __syncthreads();
  if constexpr (K <= 4) {
    // software-pipelined: the next column's K values are in flight while this column's
    // outputs are computed and stored (twice the loads in flight per thread)
    double2 bn[K];
    for (; j < ncol; j += stride) {
      const uint64_t jn = j + stride;
      if (jn < ncol) {
        const int64_t xn = static_cast<int64_t>(apply_runs(d.xcol, jn));
#pragma unroll
        for (int s = 0; s < K; ++s) bn[s] = __ldcs(X + xn + xs[s]);
      }
      const int go = static_cast<int>(apply_runs(d.gcol, j));
      const uint64_t cj = d.nHhi ? apply_runs(d.ccol, j) : j;
      for (int f = 0; f < nFe; ++f) {
        const double2* gp = Gs + go + gft[f];
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int s = 0; s < K; ++s) cmac(acc, gp[gs[s]], b[s]);
        C[(static_cast<uint64_t>(f) << d.nCol) + cj] = acc;
      }
#pragma unroll
      for (int s = 0; s < K; ++s) b[s] = bn[s];
    }
  } else {
    for (bool first = true; j < ncol; j += stride, first = false) {
      const int go = static_cast<int>(apply_runs(d.gcol, j));
      const uint64_t cj = d.nHhi ? apply_runs(d.ccol, j) : j;
      if (!first) {
        const int64_t xo = static_cast<int64_t>(apply_runs(d.xcol, j));
#pragma unroll
        for (int s = 0; s < K; ++s) b[s] = __ldcs(X + xo + xs[s]);
      }
      for (int f = 0; f < nFe; ++f) {
        const double2* gp = Gs + go + gft[f];
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int s = 0; s < K; ++s) cmac(acc, gp[gs[s]], b[s]);
        C[(static_cast<uint64_t>(f) << d.nCol) + cj] = acc;
      }
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kStepThreads) k_gate(const __grid_constant__ GateDesc d,
                                                       double2* __restrict__ arena) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KT_BEGIN
  pdl_early<1>();
  pdl_wait();
  KT_WAIT
#ifdef QCG_NULL_GATE  // timing experiment: the launch floor of a gate kernel without its body
  if (d.nCol >= 0) return;
#endif
  gate_body<K>(d, arena, smem_raw, blockIdx.x, blockIdx.y, gridDim.x);
  KT_END("gate")
}

// 256-bit global accesses (sm_100): two adjacent double2 (columns j, j+1)
__device__ __forceinline__ void ld256cs(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];\n"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p));
}
__device__ __forceinline__ void st256(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
               : "memory");
}

// k_gate with two adjacent columns per thread (GateDesc.pair2 = 1: column bit 0 is X's
// and C's lowest bit): 256-bit loads of X and 256-bit stores of C -- half the memory
// instructions of k_gate for the HBM-bound expanding steps.
template <int K>
__device__ __forceinline__ void gate2_body(const GateDesc& d, double2* __restrict__ arena, unsigned char* smem_raw,
                                           unsigned bx, unsigned by, unsigned gx) {
  double2* Gs = reinterpret_cast<double2*>(smem_raw);
  const int nGe = 1 << d.nG, nFe = 1 << d.nF;
  int* gft = reinterpret_cast<int*>(Gs + nGe);
  const uint64_t fhi = by & ((1u << d.nFhi) - 1), hhi = by >> d.nFhi;
  const int64_t gbase_hi =
      d.offG + static_cast<int64_t>(apply_runs(d.gfhi, fhi)) + static_cast<int64_t>(apply_runs(d.ghhi, hhi));
  for (int e = threadIdx.x; e < nGe; e += blockDim.x) cp_async16(Gs + e, arena + gbase_hi + apply_runs(d.gtile, e));
  for (int f = threadIdx.x; f < nFe; f += blockDim.x) gft[f] = static_cast<int>(apply_runs(d.gf, f));
  cp_async_wait();
  int64_t xs[K];
  int gs[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    xs[s] = d.xs_tab[s];
    gs[s] = d.gs_tab[s];
  }
  __syncthreads();
  const double2* __restrict__ X = arena + d.offX + static_cast<int64_t>(apply_runs(d.xhhi, hhi));
  double2* __restrict__ C = arena + d.offC + ((static_cast<int64_t>(fhi) << d.nF) << d.nCol) +
                            static_cast<int64_t>(apply_runs(d.chhi, hhi));
  const uint64_t npair = uint64_t{1} << (d.nCol - d.nHhi - 1);
  const uint64_t stride = static_cast<uint64_t>(gx) * blockDim.x;
  for (uint64_t jp = static_cast<uint64_t>(bx) * blockDim.x + threadIdx.x; jp < npair; jp += stride) {
    const uint64_t j = jp << 1;
    const int64_t xo = static_cast<int64_t>(apply_runs(d.xcol, j));
    const int go0 = static_cast<int>(apply_runs(d.gcol, j)), go1 = static_cast<int>(apply_runs(d.gcol, j + 1));
    const uint64_t cj = d.nHhi ? apply_runs(d.ccol, j) : j;
    double2 b0[K], b1[K];
#pragma unroll
    for (int s = 0; s < K; ++s) ld256cs(X + xo + xs[s], b0[s], b1[s]);
    for (int f = 0; f < nFe; ++f) {
      const double2* gp0 = Gs + go0 + gft[f];
      const double2* gp1 = Gs + go1 + gft[f];
      double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < K; ++s) {
        cmac(a0, gp0[gs[s]], b0[s]);
        cmac(a1, gp1[gs[s]], b1[s]);
      }
      st256(C + (static_cast<uint64_t>(f) << d.nCol) + cj, a0, a1);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kStepThreads) k_gate2(const __grid_constant__ GateDesc d,
                                                        double2* __restrict__ arena) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KT_BEGIN
  pdl_early<1>();
  pdl_wait();
  KT_WAIT
  gate2_body<K>(d, arena, smem_raw, blockIdx.x, blockIdx.y, gridDim.x);
  KT_END("gate2")
}

// ---- shared-memory access by 32-bit shared addresses (always LDS/STS) ----
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ double2 lds2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts2(unsigned a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1,%2};\n" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ int lds_i32(unsigned a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ long long lds_i64(unsigned a) {
  long long v;
  asm volatile("ld.shared.s64 %0, [%1];\n" : "=l"(v) : "r"(a));
  return v;
}

// Bit-scatter maps of a chain are tabulated once per CTA as two-level tables:
// map(x) = lo[x & 255] + hi[x >> 8] (bits are disjoint, so maps are additive).
constexpr int kTabLo = 256, kTabHi = 8;  // covers indices of up to 11 bits
// Per-stage tables (shared memory, byte addresses):
//   sin[K] gS[K] gF[nf] colLo[256] colHi[8] gHLo[256] gHHi[8]   (int32)
//   cF[nf] ccLo[256] ccHi[8]                                      (int64, 8-B aligned)
struct ChainTabs {
  unsigned sin, gS, gF, colLo, colHi, gHLo, gHHi, cF, ccLo, ccHi;
};

__device__ __forceinline__ ChainTabs chain_tabs(unsigned base, int K, int nf) {
  ChainTabs t;
  t.sin = base;
  t.gS = t.sin + 4 * K;
  t.gF = t.gS + 4 * K;
  t.colLo = t.gF + 4 * nf;
  t.colHi = t.colLo + 4 * kTabLo;
  t.gHLo = t.colHi + 4 * kTabHi;
  t.gHHi = t.gHLo + 4 * kTabLo;
  unsigned e = t.gHHi + 4 * kTabHi;
  e = (e + 7) & ~7u;
  t.cF = e;
  t.ccLo = t.cF + 8 * nf;
  t.ccHi = t.ccLo + 8 * kTabLo;
  return t;
}

// One stage of a fused chain, column form (see ChainStage). Element offsets into
// the dynamic shared memory; two outputs per iteration with four independent
// partial sums each (re*re, im*im, re*im, im*re) keep eight DFMA chains in flight.
template <int K>
__device__ __forceinline__ void chain_stage(const ChainStage& st, const ChainTabs& t, int in_e, int out_e, int g_e,
                                            int gbase, double2* __restrict__ dst, bool last, unsigned sbase) {
  const unsigned in_s = sbase + 16u * in_e, out_s = sbase + 16u * out_e, g_s = sbase + 16u * g_e;
  const unsigned tsin = sbase + t.sin, tgS = sbase + t.gS, tgF = sbase + t.gF, tcolLo = sbase + t.colLo,
                 tcolHi = sbase + t.colHi, tgHLo = sbase + t.gHLo, tgHHi = sbase + t.gHHi, tcF = sbase + t.cF,
                 tccLo = sbase + t.ccLo, tccHi = sbase + t.ccHi;
  const int cols = 1 << st.nKp, nf = 1 << st.nF;
  int lsplit = 0;
  while ((cols << lsplit) < static_cast<int>(blockDim.x) && (1 << lsplit) < nf) ++lsplit;
  const int fper = nf >> lsplit;
  unsigned si[K], gs[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    si[s] = 16u * lds_i32(tsin + 4 * s);
    gs[s] = 16u * lds_i32(tgS + 4 * s);
  }
  for (int w = threadIdx.x; w < (cols << lsplit); w += blockDim.x) {
    const int c = w & (cols - 1);
    const int f0 = (w >> st.nKp) * fper;
    const int ib = lds_i32(tcolLo + 4 * (c & 255)) + lds_i32(tcolHi + 4 * (c >> 8));
    const int gb = gbase + lds_i32(tgHLo + 4 * (c & 255)) + lds_i32(tgHHi + 4 * (c >> 8));
    double2 x[K];
    const unsigned xa = in_s + 16u * ib;
#pragma unroll
    for (int s = 0; s < K; ++s) x[s] = lds2(xa + si[s]);
    const unsigned ga0 = g_s + 16u * gb;
    double2* o = last ? dst + lds_i64(tccLo + 8 * (c & 255)) + lds_i64(tccHi + 8 * (c >> 8)) : nullptr;
    int f = f0;
    for (; f + 1 < f0 + fper; f += 2) {
      const unsigned gaA = ga0 + 16u * lds_i32(tgF + 4 * f);
      const unsigned gaB = ga0 + 16u * lds_i32(tgF + 4 * (f + 1));
      double rrA = 0, iiA = 0, riA = 0, irA = 0, rrB = 0, iiB = 0, riB = 0, irB = 0;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const double2 a = lds2(gaA + gs[s]);
        const double2 b = lds2(gaB + gs[s]);
        rrA = fma(a.x, x[s].x, rrA);
        iiA = fma(a.y, x[s].y, iiA);
        riA = fma(a.x, x[s].y, riA);
        irA = fma(a.y, x[s].x, irA);
        rrB = fma(b.x, x[s].x, rrB);
        iiB = fma(b.y, x[s].y, iiB);
        riB = fma(b.x, x[s].y, riB);
        irB = fma(b.y, x[s].x, irB);
      }
      const double2 vA = make_double2(rrA - iiA, riA + irA), vB = make_double2(rrB - iiB, riB + irB);
      if (last) {
        o[lds_i64(tcF + 8 * f)] = vA;
        o[lds_i64(tcF + 8 * (f + 1))] = vB;
      } else {
        sts2(out_s + 16u * (c + (f << st.nKp)), vA);
        sts2(out_s + 16u * (c + ((f + 1) << st.nKp)), vB);
      }
    }
    if (f < f0 + fper) {
      const unsigned ga = ga0 + 16u * lds_i32(tgF + 4 * f);
      double rr = 0, ii = 0, ri = 0, ir = 0;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const double2 a = lds2(ga + gs[s]);
        rr = fma(a.x, x[s].x, rr);
        ii = fma(a.y, x[s].y, ii);
        ri = fma(a.x, x[s].y, ri);
        ir = fma(a.y, x[s].x, ir);
      }
      const double2 v = make_double2(rr - ii, ri + ir);
      if (last) o[lds_i64(tcF + 8 * f)] = v;
      else sts2(out_s + 16u * (c + (f << st.nKp)), v);
    }
  }
}

__device__ __forceinline__ void cp_async16(unsigned saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int kChainIterMax = 128;  // tiles per CTA (power of two)

// Fused chain of gate steps (see ChainDesc). CTA b owns the 2^nIter consecutive
// grid indices g = (b << nIter) | i; grid maps are additive over these bit
// fields, so per-tile bases are a CTA constant plus a table lookup. Per tile:
// the input tile (prefetched with cp.async while the previous tile computes),
// every stage in shared memory, the last stage's tile written to HBM.
// KMAX = largest 2^|S| of the chain's stages (fewer registers for K <= 8).
#ifndef QCG_CHAIN_THREADS
#define QCG_CHAIN_THREADS 256
#endif
constexpr int kChainThreads = QCG_CHAIN_THREADS;
template <int KMAX>
__device__ __forceinline__ void chain_body(const ChainHead& h, const ChainDesc* __restrict__ gdesc,
                                           const int* __restrict__ img, double2* __restrict__ arena,
                                           unsigned char* smem_raw, unsigned bx, unsigned gx,
                                           unsigned long long* kt = nullptr) {
  __shared__ int64_t baseIn, baseOut;
  __shared__ int baseG[kMaxChain];
  // (baseIn/baseOut/baseG hold the maps of the current hi part, see set_hi)
  const int n0 = 1 << h.nT0, nW0 = 1 << h.nTmax, nW1 = 1 << h.nW1;
  const unsigned s0 = smem_addr(smem_raw);
  const unsigned inbuf0 = s0, inbuf1 = s0 + 16u * n0;
  // element offsets of the buffers for the stage code
  const int e_in0 = 0, e_in1 = n0, e_w0 = 2 * n0, e_w1 = 2 * n0 + nW0, e_g = 2 * n0 + nW0 + nW1;
  double2* Gs = reinterpret_cast<double2*>(smem_raw) + 2 * n0 + nW0 + nW1;
  int* tabs = reinterpret_cast<int*>(Gs + h.gElems);
  const unsigned tabs_s = smem_addr(tabs) - smem_addr(smem_raw);  // bytes from the dynamic base
  ChainDesc* sd = reinterpret_cast<ChainDesc*>(tabs + h.imgInts);  // the descriptor's shared copy
  // Prologue: everything it needs up front is in the kernel parameter `h`, so the table
  // image, the small operands, the full descriptor (bulk copies, TMA engine, one mbarrier, one
  // issuing thread) and the first input tile (16-byte async copies addressed through h's
  // own maps) are all in flight after one pass over the parameter block -- one memory round
  // trip in front of the first stage (measured before: descriptor -> table image -> first
  // tile, three dependent cold round trips, 3.3-5 us of the kernel's 6-11 us).
  __shared__ __align__(8) uint64_t cbar;
  if (threadIdx.x == 0) {
    mbar_init(&cbar, 1);
    unsigned total = static_cast<unsigned>(h.imgInts) * 4u + static_cast<unsigned>(sizeof(ChainDesc));
    for (int j = 0; j < h.nStages; ++j) total += 16u << h.nG[j];
    mbar_arrive_expect_tx(&cbar, total);
    bulk_g2s(sd, gdesc, static_cast<unsigned>(sizeof(ChainDesc)), &cbar);
    bulk_g2s(tabs, img + h.img, static_cast<unsigned>(h.imgInts) * 4u, &cbar);
    for (int j = 0; j < h.nStages; ++j) bulk_g2s(Gs + h.gsm[j], arena + h.offG[j], 16u << h.nG[j], &cbar);
  }
  const int nlo = 1 << h.nIter;
  const uint64_t n_tiles = uint64_t{1} << h.nGrid;
  const uint64_t t_begin = n_tiles * bx / gx;
  const uint64_t t_end = n_tiles * (bx + 1) / gx;
  if (t_begin < t_end) {
    const double2* src = arena + h.offIn + static_cast<int64_t>(apply_runs(h.grid2in, t_begin));
    for (int e = threadIdx.x; e < n0; e += blockDim.x) cp_async16(inbuf0 + 16u * e, src + apply_runs(h.load, e));
    cp_async_commit();
  }
  if (kt && threadIdx.x == 0) kt[0] = globaltimer();  // every prologue copy issued
  __syncthreads();       // cbar initialised for every thread
  mbar_wait(&cbar, 0);   // descriptor, table image and small operands landed (tile 0 may still be in flight)
  const ChainDesc& d = *sd;
  const int64_t* loadLo = reinterpret_cast<const int64_t*>(tabs + d.extraOff);
  const int64_t* loadHi = loadLo + kTabLo;
  const int64_t* itIn = loadHi + kTabHi;
  const int64_t* itOut = itIn + kChainIterMax;
  const int* itGb = reinterpret_cast<const int*>(itOut + kChainIterMax);
  __shared__ uint64_t hiIn;  // hi value baseIn/baseOut/baseG are valid for
  __shared__ int64_t baseInNext;
  auto set_hi = [&](uint64_t hi) {  // all threads call; one thread per map
    const uint64_t gh = hi << d.nIter;
    if (threadIdx.x == 0) baseIn = static_cast<int64_t>(apply_runs(d.grid2in, gh));
    if (threadIdx.x == 32) baseOut = static_cast<int64_t>(apply_runs(d.grid2out, gh));
    if (threadIdx.x >= 64 && threadIdx.x < 64 + d.nStages)
      baseG[threadIdx.x - 64] = static_cast<int>(apply_runs(d.st[threadIdx.x - 64].grid2g, gh));
    if (threadIdx.x == 96) hiIn = hi;
  };
  if (t_begin < t_end) set_hi(t_begin >> d.nIter);
  __syncthreads();
  auto in_base = [&](uint64_t g) -> int64_t {  // input base of tile g (hi part recomputed if needed)
    const uint64_t hi = g >> d.nIter;
    return (hi == hiIn ? baseIn : static_cast<int64_t>(apply_runs(d.grid2in, hi << d.nIter))) + itIn[g & (nlo - 1)];
  };
  auto prefetch = [&](int64_t base, unsigned buf) {
    const double2* src = arena + d.offIn + base;
    for (int e = threadIdx.x; e < n0; e += blockDim.x)
      cp_async16(buf + 16u * e, src + loadLo[e & 255] + loadHi[e >> 8]);
    cp_async_commit();
  };
  if (kt && threadIdx.x == 0) kt[1] = globaltimer();  // tables and small operands landed
  int par = 0;
  for (uint64_t g = t_begin; g < t_end; ++g, par ^= 1) {
    const int cur = par ? e_in1 : e_in0;
    if (g + 1 < t_end) {
      // next tile's input base: one thread computes it if the hi part changes
      if (threadIdx.x == 0) baseInNext = in_base(g + 1);
      __syncthreads();
      prefetch(baseInNext, par ? inbuf0 : inbuf1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    if ((g >> d.nIter) != hiIn) {  // uniform across the CTA
      __syncthreads();
      set_hi(g >> d.nIter);
    }
    __syncthreads();
    if (kt && threadIdx.x == 0 && g == t_begin) kt[2] = globaltimer();  // first tile landed
    const int i = static_cast<int>(g & (nlo - 1));
    int in = cur;
    int out = e_w0;
    double2* dst = arena + d.offOut + baseOut + itOut[i];
    for (int j = 0; j < d.nStages; ++j) {
      const ChainStage& st = d.st[j];
      const int gbase = baseG[j] + itGb[j * kChainIterMax + i];
      const bool last = j + 1 == d.nStages;
      const ChainTabs t = chain_tabs(tabs_s + 4u * st.tab, 1 << st.nS, 1 << st.nF);
      switch (st.nS) {
        case 1: chain_stage<2>(st, t, in, out, e_g, gbase, dst, last, s0); break;
        case 2: chain_stage<4>(st, t, in, out, e_g, gbase, dst, last, s0); break;
        case 3:
          if constexpr (KMAX >= 8) chain_stage<8>(st, t, in, out, e_g, gbase, dst, last, s0);
          break;
        default:
          if constexpr (KMAX >= 16) chain_stage<16>(st, t, in, out, e_g, gbase, dst, last, s0);
          break;
      }
      __syncthreads();
      in = out;
      out = (out == e_w0) ? e_w1 : e_w0;
    }
  }
}

template <int KMAX>
__global__ void __launch_bounds__(kChainThreads, kChainThreads > 256 ? 1 : (KMAX <= 8 ? 3 : 2)) k_chain(const __grid_constant__ ChainHead head,
                                                                          const ChainDesc* __restrict__ desc,
                                                                          const int* __restrict__ img,
                                                                          double2* __restrict__ arena) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KT_BEGIN
  pdl_early<2>();
  pdl_wait();
  KT_WAIT
  KT_MARKS
  chain_body<KMAX>(head, desc, img, arena, smem_raw, blockIdx.x, gridDim.x, KT_MARKS_PTR);
  KT_END_M("chain", km_)
}

// Two gate steps fused at register level (see PairDesc). blockIdx.y = r_hi (one
// G1 tile per CTA); each thread owns columns j' of X: NP x K1 values of X in
// registers, then for every r_mid NA accumulators (r_lo x f2). Shared operands use
// the expanded layouts of PairDesc, so the inner loop's shared addresses are one
// base per (q, accumulator) plus compile-time offsets in p and s1.
#ifndef QCG_PAIR_ZS
#define QCG_PAIR_ZS 1
#endif
constexpr int kPairMaskMax = 1024;  // (r_mid, q) zero masks kept in shared memory
#ifndef QCG_PAIR_MINB
#define QCG_PAIR_MINB 2
#endif
template <int NP, int K1, int NRL, int NF2>
__device__ __forceinline__ void pair_body(const PairDesc& d, double2* __restrict__ arena,
                                          unsigned long long* __restrict__ executed, unsigned char* smem_raw,
                                          unsigned bx, unsigned by, unsigned gx) {
  const int g1t = d.nG1x - d.nHhi;  // staged G1x sub-block (this CTA's H_hi value)
  const int n1 = 1 << g1t, n2 = 1 << d.nG2;
  const int nrt = 1 << (d.nRmid + d.nRlo), nq = 1 << d.nQ;
  double2* G1s = reinterpret_cast<double2*>(smem_raw);
  double2* G2s = G1s + n1 + (1 << (g1t - d.sh1));
  int* g2r_t = reinterpret_cast<int*>(G2s + n2 + (1 << (d.nG2 - d.sh2)));
  const uint64_t rhi = by & ((1u << d.nRhi) - 1), hhi = by >> d.nRhi;
  const int64_t rhi_off = static_cast<int64_t>(rhi) << (d.nRmid + d.nRlo);
  const int64_t g1base = d.offG1 + static_cast<int64_t>(apply_runs(d.g1hi, rhi));
  const uint64_t e_hi = hhi << g1t;  // first expanded G1 index of the sub-block
  // shared index of expanded index e (bank skew, e + (e >> sh1)) relative to the sub-block
  const int h_base = static_cast<int>(e_hi + (e_hi >> d.sh1));
  for (int e = threadIdx.x; e < n1; e += blockDim.x)
    cp_async16(G1s + e + (e >> d.sh1), arena + g1base + apply_runs(d.g1stage, e_hi + e));
  for (int e = threadIdx.x; e < n2; e += blockDim.x)
    cp_async16(G2s + e + (e >> d.sh2), arena + d.offG2 + apply_runs(d.g2stage, e));
  for (int i = threadIdx.x; i < nrt; i += blockDim.x)
    g2r_t[i] = static_cast<int>(apply_runs(d.g2r, static_cast<uint64_t>(rhi_off) | i));
  cp_async_wait();
  __syncthreads();
  // G2 independent of the column (no hc2 bits): its zero pattern is a CTA constant. One
  // bit per p of every (r_mid, q): set when some (r_lo, f2) entry is nonzero -- the
  // zero-skip (contraction.cpp:107-108) then costs a register test, not NRL x NF2 loads.
  const int nmask = (1 << d.nRmid) * nq;
  const bool masked = d.g2hc.n == 0 && nmask <= kPairMaskMax;
  unsigned* nzm = reinterpret_cast<unsigned*>(g2r_t + nrt);
  const int f2s = nq * NP;
  if (masked) {
    for (int e = threadIdx.x; e < nmask; e += blockDim.x) {
      const int rm = e / nq, q = e - rm * nq;
      unsigned m = 0;
      for (int p = 0; p < NP; ++p)
        for (int rl = 0; rl < NRL; ++rl)
          for (int f = 0; f < NF2; ++f) {
            const double2 v = G2s[g2r_t[rm * NRL + rl] + f * f2s + q * NP + p];
            if (v.x != 0.0 || v.y != 0.0) m |= 1u << p;
          }
      nzm[e] = m;
    }
    __syncthreads();
  }
  constexpr int KQ = NP * K1;                 // G1x elements per q
  const int r1stride = nq * KQ;               // G1x elements per r
  const int f2stride = nq * NP;               // G2x elements per f2
  const uint64_t ncol = uint64_t{1} << (d.nCol - d.nHhi);
  const uint64_t jhi = apply_runs(d.jhhi, hhi);
  const uint64_t stride = static_cast<uint64_t>(gx) * blockDim.x;
  const double2* __restrict__ X = arena + d.offX;
  double2* __restrict__ C = arena + d.offC;
  unsigned n_exec = 0;  // (column, r_mid, q, p) iterations not zero-skipped (profiling)
  for (uint64_t jl = static_cast<uint64_t>(bx) * blockDim.x + threadIdx.x; jl < ncol; jl += stride) {
    const uint64_t j = jhi | (d.nHhi ? apply_runs(d.jcol, jl) : jl);
    const int64_t xo = static_cast<int64_t>(apply_runs(d.xcol, j));
    const int h1 = static_cast<int>(apply_runs(d.g1hc, j) + apply_runs(d.g1hcx, j)) - h_base;
    const int h2 = static_cast<int>(apply_runs(d.g2hc, j) + apply_runs(d.g2hcx, j));
    double2 x[NP][K1];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int s = 0; s < K1; ++s) x[p][s] = __ldcs(X + xo + d.xoff_tab[p * K1 + s]);
    for (int rm = 0; rm < (1 << d.nRmid); ++rm) {
      double2 acc[NRL][NF2];
      int g1u[NRL], g2u[NRL];  // per-r_lo G1x / G2x bases of this r_mid
#pragma unroll
      for (int rl = 0; rl < NRL; ++rl) {
        const int ridx = rm * NRL + rl;
        g1u[rl] = h1 + ridx * r1stride;
        g2u[rl] = h2 + g2r_t[ridx];
#pragma unroll
        for (int f = 0; f < NF2; ++f) acc[rl][f] = make_double2(0.0, 0.0);
      }
      for (int q = 0; q < nq; ++q) {
        const unsigned m = masked ? nzm[rm * nq + q] : ~0u;
        if (m == 0) continue;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (!((m >> p) & 1u)) continue;
          double2 gb[NRL][NF2];
#pragma unroll
          for (int rl = 0; rl < NRL; ++rl)
#pragma unroll
            for (int f = 0; f < NF2; ++f) gb[rl][f] = G2s[g2u[rl] + f * f2stride + q * NP + p];
#if QCG_PAIR_ZS >= 1
          if (!masked) {
            // zero-skip on the second step's small operand, as the reference's
            // contract_pair skips zero left-operand entries (contraction.cpp:107-108):
            // a zero G2 entry makes the first-step products it weights unnecessary
            bool any = false;
#pragma unroll
            for (int rl = 0; rl < NRL; ++rl)
#pragma unroll
              for (int f = 0; f < NF2; ++f) any |= (gb[rl][f].x != 0.0) | (gb[rl][f].y != 0.0);
            if (!any) continue;
          }
#endif
          ++n_exec;
#pragma unroll
          for (int rl = 0; rl < NRL; ++rl) {
            // first step once per r (shared by every f2 of the second step)
            const double2* g1 = G1s + g1u[rl] + q * KQ + p * K1;
            double tr = 0.0, ti = 0.0, tr2 = 0.0, ti2 = 0.0;
#pragma unroll
            for (int s = 0; s < K1; ++s) {
              const double2 a = g1[s];
              tr = fma(a.x, x[p][s].x, tr);
              tr2 = fma(a.y, x[p][s].y, tr2);
              ti = fma(a.x, x[p][s].y, ti);
              ti2 = fma(a.y, x[p][s].x, ti2);
            }
            const double2 t = make_double2(tr - tr2, ti + ti2);
#pragma unroll
            for (int f = 0; f < NF2; ++f) cmac(acc[rl][f], gb[rl][f], t);
          }
        }
      }
#pragma unroll
      for (int rl = 0; rl < NRL; ++rl)
#pragma unroll
        for (int f = 0; f < NF2; ++f) {
          const int64_t r = rhi_off | (static_cast<int64_t>(rm) * NRL + rl);
          C[(((static_cast<int64_t>(f) << d.nR) | r) << d.nCol) + static_cast<int64_t>(j)] = acc[rl][f];
        }
    }
  }
  if (executed) {  // instrumented passes only: executed work for the roofline
    const unsigned w = __reduce_add_sync(0xffffffffu, n_exec);
    if ((threadIdx.x & 31) == 0) atomicAdd(executed, static_cast<unsigned long long>(w));
  }
}

// Register budget per instantiation: the large register tiles (X values x accumulators >=
// QCG_PAIR_BIG) run one CTA per SM scheduling slot pair less (255 registers, no spills); the
// small ones keep two CTAs per SM (128 registers).
#ifndef QCG_PAIR_BIG
#define QCG_PAIR_BIG 1000000  // off by default: measured, see DESIGN
#endif
template <int NP, int K1, int NRL, int NF2>
__global__ void __launch_bounds__(kStepThreads, (NP * K1 * NRL * NF2 >= QCG_PAIR_BIG) ? 1 : QCG_PAIR_MINB) k_pair(const __grid_constant__ PairDesc d,
                                                                      double2* __restrict__ arena,
                                                                      unsigned long long* __restrict__ executed) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KT_BEGIN
  pdl_early<3>();
  pdl_wait();
  KT_WAIT
  pair_body<NP, K1, NRL, NF2>(d, arena, executed, smem_raw, blockIdx.x, blockIdx.y, gridDim.x);
  KT_END("pair")
}

// Deterministic block sum: a fixed-order warp-shuffle tree per warp, then warp 0 folds the
// per-warp sums the same way (one shared-memory level, two barriers). `sh` holds >= 32
// entries; callers separate two uses of `sh` by a barrier.
__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}
__device__ __forceinline__ double2 block_reduce(double2 v, double2* sh) {
  v = warp_sum(v);
  const int w = static_cast<int>(threadIdx.x >> 5), nw = static_cast<int>(blockDim.x >> 5);
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = static_cast<int>(threadIdx.x) < nw ? sh[threadIdx.x] : make_double2(0.0, 0.0);
    v = warp_sum(v);
    if (threadIdx.x == 0) sh[32] = v;
  }
  __syncthreads();
  return sh[32];
}

// k_gate whose result is the pass's lead rank-0 factor (GateDesc.reduce): the epilogue of
// execute_plan (contraction.cpp:304-317, acc *= every rank-0 value) and the slice sum run
// here. Each output element is one slice's lead factor: its slice index comes from the lead
// factor's inverse-map table, the other factors from their tables (Program::final_tab, the
// same image k_final uses), the product is range-masked and summed per CTA in a fixed tree
// into gpart[CTA]; k_final then only folds those partials. The result tensor is written (and
// k_final walks it as usual) only when per-slice values are requested (RunState.slice_out).
struct GateReduceArgs {
  const RunState* st;
  const FactorDesc* f;
  const uint32_t* ftab;
  double2* gpart;
  int32_t nf, lead, b, pad;
};
template <int K>
__global__ void __launch_bounds__(kStepThreads) k_gate_reduce(const __grid_constant__ GateDesc d,
                                                              double2* __restrict__ arena,
                                                              const __grid_constant__ GateReduceArgs r) {
  static_assert(K <= 4, "the fused epilogue covers the pipelined gate form");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double2 sh[33];
  __shared__ __align__(8) uint64_t tbar;
  KT_BEGIN
  double2* Gs = reinterpret_cast<double2*>(smem_raw);
  const int nGe = 1 << d.nG, nFe = 1 << d.nF;
  int* gft = reinterpret_cast<int*>(Gs + nGe);
  const uint32_t(*tab)[2][1024] = reinterpret_cast<const uint32_t(*)[2][1024]>(
      smem_raw + ((static_cast<size_t>(nGe) * 16 + static_cast<size_t>(nFe) * 4 + 15) & ~size_t{15}));
  if (threadIdx.x == 0) {  // static lookup tables: one bulk copy, in flight across the dependency wait
    const unsigned bytes = static_cast<unsigned>(r.nf + 1) * 2048u * 4u;
    mbar_init(&tbar, 1);
    mbar_arrive_expect_tx(&tbar, bytes);
    bulk_g2s(const_cast<uint32_t*>(&tab[0][0][0]), r.ftab, bytes, &tbar);
  }
  pdl_early<1>();
  pdl_wait();
  KT_WAIT
  const RunState s = *r.st;
  const bool write_c = s.slice_out != nullptr;
  const unsigned by = blockIdx.y;
  const uint64_t fhi = by & ((1u << d.nFhi) - 1), hhi = by >> d.nFhi;
  const int64_t gbase_hi =
      d.offG + static_cast<int64_t>(apply_runs(d.gfhi, fhi)) + static_cast<int64_t>(apply_runs(d.ghhi, hhi));
  for (int e = threadIdx.x; e < nGe; e += blockDim.x) cp_async16(Gs + e, arena + gbase_hi + apply_runs(d.gtile, e));
  for (int f = threadIdx.x; f < nFe; f += blockDim.x) gft[f] = static_cast<int>(apply_runs(d.gf, f));
  int64_t xs[K];
  int gs[K];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    xs[q] = d.xs_tab[q];
    gs[q] = d.gs_tab[q];
  }
  const double2* __restrict__ X = arena + d.offX + static_cast<int64_t>(apply_runs(d.xhhi, hhi));
  // element offset of this CTA row's outputs inside the result tensor
  const uint64_t cbase = ((fhi << d.nF) << d.nCol) + apply_runs(d.chhi, hhi);
  double2* __restrict__ C = arena + d.offC + cbase;
  const uint64_t ncol = uint64_t{1} << (d.nCol - d.nHhi);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double2 b[K], bn[K];
  if (j < ncol) {
    const int64_t xo = static_cast<int64_t>(apply_runs(d.xcol, j));
#pragma unroll
    for (int q = 0; q < K; ++q) b[q] = __ldcs(X + xo + xs[q]);
  }
  int64_t foff[kFinalTabFactors];  // the other factors' bases
#pragma unroll
  for (int q = 0; q < kFinalTabFactors; ++q) foff[q] = q < r.nf ? r.f[q].off : 0;
  cp_async_wait();
  __syncthreads();
  mbar_wait(&tbar, 0);
  const uint64_t nloc = uint64_t{1} << r.b;
  double2 sum = make_double2(0.0, 0.0);
  for (; j < ncol; j += stride) {
    const uint64_t jn = j + stride;
    if (jn < ncol) {
      const int64_t xn = static_cast<int64_t>(apply_runs(d.xcol, jn));
#pragma unroll
      for (int q = 0; q < K; ++q) bn[q] = __ldcs(X + xn + xs[q]);
    }
    const int go = static_cast<int>(apply_runs(d.gcol, j));
    const uint64_t cj = d.nHhi ? apply_runs(d.ccol, j) : j;
    for (int f = 0; f < nFe; ++f) {
      const double2* gp = Gs + go + gft[f];
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < K; ++q) cmac(acc, gp[gs[q]], b[q]);
      const uint64_t co = (static_cast<uint64_t>(f) << d.nCol) + cj;
      if (write_c) {
        C[co] = acc;
      } else {
        const uint64_t e = cbase + co;  // storage offset in the lead factor = one slice
        const uint64_t k = tab[r.nf][0][e & 1023] | tab[r.nf][1][e >> 10];
        const int lo = static_cast<int>(k & 1023), hi = static_cast<int>(k >> 10);
        double2 v = acc;
        bool first = true;
#pragma unroll
        for (int q = 0; q < kFinalTabFactors; ++q) {
          if (q >= r.nf) continue;
          // (the other factors were completed by earlier launches: read-only here, L1-cacheable)
          const double2 t = q == r.lead ? acc : __ldg(arena + foff[q] + tab[q][0][lo] + tab[q][1][hi]);
          v = first ? t : cmul(v, t);  // the reference's order: factors in plan order
          first = false;
        }
        const uint64_t gid = s.pass_base + k;
        if (k < nloc && gid >= s.lo && gid < s.hi) {
          sum.x += v.x;
          sum.y += v.y;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < K; ++q) b[q] = bn[q];
  }
  if (!write_c) {
    const double2 tot = block_reduce(sum, sh);
    if (threadIdx.x == 0) r.gpart[blockIdx.y * gridDim.x + blockIdx.x] = tot;
  }
  KT_END("gr")
}

// Per-slice value = product of the rank-0 factors (step order, then leftover vertices
// ascending), masked to [lo, hi), summed with a fixed tree. On the last pass of a call the
// last CTA to finish also reduces every partial of the call in a fixed order (the call's
// result; no separate reduction launch).
// Slices per k_final thread: a CTA owns kFinalThreads * per_thread consecutive pass-local
// slices, and pass j of a thread's loop covers the CTA's j-th block of kFinalThreads slices
// (a warp's 32 slices are consecutive: coalesced factor reads where a factor's low bits are
// slice bits). Four slices' factor values are loaded before any is multiplied, so a thread
// keeps 4 x nf independent loads in flight (the reduction is latency-, not bandwidth-bound).
#ifndef QCG_FINAL_GROUP
#define QCG_FINAL_GROUP 4
#endif
constexpr int kFinalGroup = QCG_FINAL_GROUP;
constexpr int kFinalSmemBytes = (kFinalTabFactors + 1) * 2 * 1024 * 4 + kFinalSmemFactors * static_cast<int>(sizeof(FactorDesc));
__device__ __forceinline__ void final_body(const FactorDesc* f, int nf, int b, int per_thread,
                                           const double2* __restrict__ arena, const RunState* __restrict__ st,
                                           double2* __restrict__ partials, unsigned* __restrict__ fin_ctr,
                                           double2* __restrict__ result, const uint32_t* __restrict__ ftab,
                                           unsigned char* smem, unsigned bx, unsigned gx, unsigned amp,
                                           unsigned namp, bool dep_wait, unsigned long long* stamps = nullptr,
                                           uint64_t* pass_counter = nullptr, int lead = -1,
                                           const double2* __restrict__ gpart = nullptr, int n_gpart = 0) {
  __shared__ double2 sh[33];
  __shared__ bool last_cta;
  // few factors over <= 20 slice bits: each map (a bit scatter, so additive over disjoint
  // bit fields) tabulated per 10-bit half of the slice index -- two shared-memory lookups
  // per factor and slice instead of walking every run
  constexpr int kTabFactors = kFinalTabFactors;
  uint32_t(*tab)[2][1024] = reinterpret_cast<uint32_t(*)[2][1024]>(smem);
  // factor maps staged in shared memory with one cooperative copy (apply_runs then
  // walks shared memory instead of issuing dependent global loads per run)
  FactorDesc* sf = reinterpret_cast<FactorDesc*>(smem + (kTabFactors + 1) * 2 * 1024 * 4);
  const bool use_tab = ftab != nullptr;
  __shared__ __align__(8) uint64_t tbar;
  const FactorDesc* fg = f;
  auto stage_static = [&]() {  // factor descriptors and lookup tables (static data) into shared memory
    if (nf <= kFinalSmemFactors) {
      const int4* src = reinterpret_cast<const int4*>(fg);
      int4* dst = reinterpret_cast<int4*>(sf);
      for (int i = threadIdx.x; i < nf * static_cast<int>(sizeof(FactorDesc) / 16); i += blockDim.x) dst[i] = src[i];
    }
    if (use_tab && threadIdx.x == 0) {  // host-built tables (Program::final_tab): one bulk copy (TMA engine)
      const unsigned bytes = static_cast<unsigned>(nf + (lead >= 0 ? 1 : 0)) * 2048u * 4u;
      mbar_init(&tbar, 1);
      mbar_arrive_expect_tx(&tbar, bytes);
      bulk_g2s(&tab[0][0][0], ftab, bytes, &tbar);
    }
  };
  if (nf <= kFinalSmemFactors) f = sf;
  // A program whose lead factor's gate does the product and the sum (k_gate_reduce, gpart !=
  // null) needs the walk below only when per-slice values are requested: the static staging
  // waits until that is known. Otherwise it runs ahead of the dependency wait.
  const bool maybe_fused = gpart != nullptr;
  if (!maybe_fused) stage_static();
  if (dep_wait) pdl_early<5>();
  if (dep_wait) pdl_wait();  // factor maps above are static; the factors and the run state are not
  const RunState s = *st;
  if (maybe_fused && s.slice_out == nullptr) {
    // fold the gate's per-CTA partials: CTA (0, 0) alone (one amplitude per pass in this mode)
    if (bx != 0 || amp != 0) return;
    double2 gs = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < n_gpart; i += blockDim.x) {
      const double2 pv = __ldcg(gpart + i);
      gs.x += pv.x;
      gs.y += pv.y;
    }
    const double2 tot = block_reduce(gs, sh);
    // this pass's slot of the call's partials: the sum in entry 0, zeros behind it
    for (unsigned c = threadIdx.x; c < gx; c += blockDim.x)
      partials[s.slot * namp * gx + c] = c == 0 ? tot : make_double2(0.0, 0.0);
    if (stamps && threadIdx.x == 0) atomicMax(stamps + 1, globaltimer());  // QCG_PASS_STAMPS: pass end
    if (s.nparts == 0) return;
    __threadfence();
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);  // the call's passes in order, in the same fixed tree
    const uint64_t n = s.nparts * gx;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double2 pv = __ldcg(partials + i);
      acc.x += pv.x;
      acc.y += pv.y;
    }
    const double2 r = block_reduce(acc, sh);
    if (threadIdx.x == 0) {
      result[0] = r;
      if (pass_counter) *pass_counter = 0;  // the next call's first pass reads states[0]
    }
    return;
  }
  if (maybe_fused) stage_static();
  __syncthreads();
  if (use_tab) mbar_wait(&tbar, 0);
  const uint64_t nloc = uint64_t{1} << b;
  const uint64_t cta0 = static_cast<uint64_t>(bx) * blockDim.x * per_thread;
  // pass-local factor index: the amplitude (blockIdx.y) above the b batched slice bits
  const uint64_t kamp = static_cast<uint64_t>(amp) << b;
  double2 sum = make_double2(0.0, 0.0);
  double2* out = reinterpret_cast<double2*>(s.slice_out);
  if (out) out += amp * s.out_stride;
  auto take = [&](uint64_t k, double2 v, bool valid = true) {
    const uint64_t gid = s.pass_base + k;
    if (valid && k < nloc && gid >= s.lo && gid < s.hi) {
      sum.x += v.x;
      sum.y += v.y;
      if (out) out[gid - s.out_base] = v;
    }
  };
  if (use_tab) {
    for (int i0 = 0; i0 < per_thread; i0 += kFinalGroup) {
      const uint64_t k0 = cta0 + static_cast<uint64_t>(i0) * blockDim.x + threadIdx.x;
      double2 t[kFinalGroup][kTabFactors];
      uint64_t ks[kFinalGroup];
#pragma unroll
      for (int u = 0; u < kFinalGroup; ++u) {
        const uint64_t kr = k0 + static_cast<uint64_t>(u) * blockDim.x;
        uint64_t k = (kr < nloc ? kr : 0) | kamp;
        const uint64_t e = k;  // lead mode: the walk index is the lead factor's storage offset
        if (lead >= 0) k = tab[nf][0][e & 1023] | tab[nf][1][e >> 10];
        ks[u] = k;
        const int lo = static_cast<int>(k & 1023), hi = static_cast<int>(k >> 10);
#pragma unroll
        for (int j = 0; j < kTabFactors; ++j)
          t[u][j] = j == lead ? __ldcg(arena + f[j].off + e)
                              : (j < nf ? __ldcg(arena + f[j].off + tab[j][0][lo] + tab[j][1][hi])
                                        : make_double2(1.0, 0.0));
      }
#pragma unroll
      for (int u = 0; u < kFinalGroup; ++u) {
        double2 v = t[u][0];
#pragma unroll
        for (int j = 1; j < kTabFactors; ++j) v = cmul(v, t[u][j]);
        const uint64_t kr = k0 + static_cast<uint64_t>(u) * blockDim.x;
        take(lead >= 0 ? ks[u] : kr, v, kr < nloc);
      }
    }
  } else {
    for (int i = 0; i < per_thread; ++i) {
      const uint64_t k = cta0 + static_cast<uint64_t>(i) * blockDim.x + threadIdx.x;
      if (k >= nloc) break;
      double2 v = make_double2(1.0, 0.0);
      for (int j0 = 0; j0 < nf; j0 += 8) {
        double2 t[8];
#pragma unroll
        for (int w = 0; w < 8; ++w)
          t[w] = j0 + w < nf ? __ldcg(arena + f[j0 + w].off + apply_runs(f[j0 + w].map, k | kamp))
                             : make_double2(1.0, 0.0);
#pragma unroll
        for (int w = 0; w < 8; ++w) v = cmul(v, t[w]);
      }
      take(k, v);
    }
  }
  const double2 tot = block_reduce(sum, sh);
  // partials of a call: [pass slot][amplitude][CTA]
  if (threadIdx.x == 0) partials[(s.slot * namp + amp) * gx + bx] = tot;
  if (stamps && threadIdx.x == 0) atomicMax(stamps + 1, globaltimer());  // QCG_PASS_STAMPS: pass end
  if (s.nparts == 0) return;
  if (threadIdx.x == 0) {
    __threadfence();
    last_cta = atomicAdd(fin_ctr, 1u) == gx * namp - 1;
  }
  __syncthreads();
  if (!last_cta) return;
  __threadfence();
  // every amplitude's partials, passes in order, in a fixed tree
  for (unsigned a2 = 0; a2 < namp; ++a2) {
    double2 acc = make_double2(0.0, 0.0);
    const uint64_t n = s.nparts * gx;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t slot = i / gx, c = i - slot * gx;
      const double2 pv = __ldcg(partials + (slot * namp + a2) * gx + c);
      acc.x += pv.x;
      acc.y += pv.y;
    }
    const double2 r = block_reduce(acc, sh);
    if (threadIdx.x == 0) result[a2] = r;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *fin_ctr = 0;
    if (pass_counter) *pass_counter = 0;  // the next call's first pass reads states[0]
  }
}

__global__ void __launch_bounds__(kFinalThreads) k_final(const FactorDesc* f, int nf, int b, int per_thread,
                                                         const double2* __restrict__ arena,
                                                         const RunState* __restrict__ st,
                                                         double2* __restrict__ partials,
                                                         unsigned* __restrict__ fin_ctr,
                                                         double2* __restrict__ result,
                                                         const uint32_t* __restrict__ ftab,
                                                         unsigned long long* __restrict__ stamps,
                                                         uint64_t* __restrict__ pass_counter, int lead,
                                                         const double2* __restrict__ gpart, int n_gpart) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KT_BEGIN
  KT_WAIT
  final_body(f, nf, b, per_thread, arena, st, partials, fin_ctr, result, ftab, smem_raw, blockIdx.x, gridDim.x,
             blockIdx.y, gridDim.y, true, stamps, pass_counter, lead, gpart, n_gpart);
  KT_END("final")
}



}  // namespace qcg
