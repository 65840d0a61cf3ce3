/*
 * qcut_gpu.h — C-ABI of the B200 sliced-contraction engine.
 *
 * Drop-in for the reference's per-slice hot path (arXiv 2010.14962 `qcut`):
 *
 *   cx qcut::sum_range(const JobSpec& job, uint64_t lo, uint64_t hi)
 *        proj/core/include/qcut/executor.hpp:46, proj/core/src/executor.cpp:45-68
 *
 * An engine is built from the reference's lossless payload
 * (`qcut::encode_payload`, proj/core/src/serialize.cpp:147-154 — the network,
 * the sorted cut set, the shared ContractionPlan and max_rank; the same bytes the
 * reference master ships to its workers, proj/core/src/master.cpp:52-272) and
 * answers sum_range queries on one CUDA device. Plain pointers and sizes only.
 *
 * Views:
 *   QC_MODE_DENSITY  the reference's own view: every leg has dimension 4, slice
 *                    ids s in [0, 4^M) with base-4 digits, MSB = smallest cut
 *                    edge id (proj/core/src/cutting.cpp:41-52). sum_range returns
 *                    exactly the reference quantity (p = tr(E U rho U^+)).
 *   QC_MODE_KET      the binary-variable view of the same plan:
 *                    legs of dimension 2, ket slice ids k in [0, 2^M), bit i
 *                    (MSB first) = ket bit of cut edge i. Requires every tensor to
 *                    factorise as K (x) conj(K) (pure inputs, unitary gates,
 *                    projector measurements — all QAOA instances). Density-id
 *                    queries are answered exactly from the ket slice values:
 *                    V(s) = A(k(s)) * conj(A(b(s))) with digit d_i = 2 k_i + b_i.
 *                    A(k) carries one global phase fixed by the factorisation
 *                    convention; |sum_k A(k)|^2 and every V(s) are phase-free.
 *
 * Errors: every entry point returns a status code that maps 1:1 onto the
 * reference's exception classes (proj/core/src/executor.cpp:48-64):
 *   QC_EINVAL     std::invalid_argument  (bad range, bad payload / plan)
 *   QC_ERANK      qcut::RankGuardError    (a plan step exceeds max_rank;
 *                                          proj/core/src/contraction.cpp:280-286)
 *   QC_EINTERNAL  std::runtime_error      (CUDA failure, out of memory, ...)
 * qc_last_error() returns the message of the calling thread's last failure.
 *
 * Threading: calls on one engine are serialised by the engine; engines on
 * different devices may run concurrently (one host thread or process per GPU).
 */
#ifndef QCUT_GPU_H_
#define QCUT_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef QC_API
#define QC_API __attribute__((visibility("default")))
#endif

#define QC_OK 0
#define QC_EINVAL 1
#define QC_ERANK 2
#define QC_EINTERNAL 3

#define QC_MODE_DENSITY 0
#define QC_MODE_KET 1

typedef struct qc_engine qc_engine;

typedef struct qc_plan_stats {
  int32_t mode;            /* QC_MODE_* */
  int32_t n_cut;           /* M */
  int32_t n_steps;         /* plan steps (identical to the reference plan) */
  int32_t peak_rank;       /* reference peak_rank (legs of the cut network) */
  int32_t max_rank;        /* payload max_rank (the rank guard) */
  int32_t batch_bits;      /* cut bits batched inside one device pass */
  uint64_t jobs;           /* reference job count 4^M */
  uint64_t ket_jobs;       /* 2^M (ket view) */
  uint64_t chunks;         /* device passes for the full range */
  uint64_t arena_bytes;    /* device workspace */
  int32_t n_kernels;       /* kernel launches per device pass */
  int32_t n_invariant_steps; /* steps whose operands carry no cut variable */
  double essential_bytes;  /* SURVEY §8(d) unshared count: per-slice bytes x slices, full range */
  double moved_bytes;      /* algorithmic bytes: every tensor the engine materialises in HBM,
                              read once + written once (fused intermediates excluded), full range */
  double flops;            /* 8 * sum 2^work per slice-dependent step, full range */
  int32_t dominant_kernel; /* index (in plan-step order) of the step kernel moving the most bytes */
  int32_t pad0;
  double dominant_bytes;   /* bytes that kernel reads + writes per pass */
  double algo_flops;       /* engine plan flops at the batched shapes (8 per complex MAC of every
                              step, fused or not), full range */
  int32_t n_amplitudes;    /* payloads batched in this engine (qc_engine_create_batch; 1 otherwise) */
  int32_t amp_bits;        /* ceil(log2 n_amplitudes): extra batch bits of every pass */
} qc_plan_stats;

/* Per-step shapes for the shape-parity check: arrays of n_steps entries
 * (rank_a, rank_b, shared legs, result_rank), same order as the reference plan. */
QC_API int qc_engine_step_shapes(const qc_engine* e, int32_t* rank_a, int32_t* rank_b,
                          int32_t* shared, int32_t* result_rank, size_t n);

/* Build an engine from encode_payload() JSON. device < 0 builds the host-side
 * program only (no CUDA calls; stats and shape checks work, compute calls
 * return QC_EINTERNAL). mem_budget_bytes = 0 picks 70% of free device memory. */
QC_API int qc_engine_create(const char* payload_json, size_t len, int device, int mode,
                     uint64_t mem_budget_bytes, qc_engine** out);
/* As qc_engine_create, with the batched slice bits (slices per device pass = 2^b) capped
 * at max_batch_bits (-1: no cap). A caller that owns 2^k slices of a sharded range passes
 * k so a pass does not compute slices outside its shard. */
QC_API int qc_engine_create_ex(const char* payload_json, size_t len, int device, int mode,
                               uint64_t mem_budget_bytes, int max_batch_bits, qc_engine** out);
/* Amplitude batch (no reference counterpart; plans depend only on structure):
 * n payloads of ONE network, cut and plan whose tensor values differ -- output bitstrings
 * (the measurement vectors, tensor_network.cpp:82-87) or angle sets -- run as one program whose
 * passes carry ceil(log2 n) extra batch bits (tensors independent of the differing vertices
 * are computed once for all amplitudes). Structural mismatch -> QC_EINVAL. The single-amplitude
 * compute calls return QC_EINVAL on a batch engine (n > 1); use the *_batch calls. */
QC_API int qc_engine_create_batch(const char* const* payloads, const size_t* lens, int n, int device, int mode,
                                  uint64_t mem_budget_bytes, int max_batch_bits, qc_engine** out);
QC_API int qc_engine_destroy(qc_engine* e);
QC_API int qc_engine_plan_stats(const qc_engine* e, qc_plan_stats* out);

/* Reference sum_range over density slice ids [lo, hi) (either mode). */
QC_API int qc_engine_sum_range(qc_engine* e, uint64_t lo, uint64_t hi, double out[2]);
/* Per-slice reference values sum_range(s, s+1) for s in [lo, hi): 2*(hi-lo) doubles. */
QC_API int qc_engine_slice_values(qc_engine* e, uint64_t lo, uint64_t hi, double* out);
/* Ket view only: sum of A(k) over ket ids [klo, khi). */
QC_API int qc_engine_ket_sum(qc_engine* e, uint64_t klo, uint64_t khi, double out[2]);
/* Ket view only: A(k) for k in [klo, khi): 2*(khi-klo) doubles. */
QC_API int qc_engine_ket_values(qc_engine* e, uint64_t klo, uint64_t khi, double* out);

/* Ket view, batch engine: out[2a], out[2a+1] = sum of A_a(k) over [klo, khi) for every
 * amplitude a < n (2n doubles); ket_values_batch: A_a(k) at out[2(a (khi-klo) + k - klo)]. */
QC_API int qc_engine_ket_sum_batch(qc_engine* e, uint64_t klo, uint64_t khi, double* out);
QC_API int qc_engine_ket_values_batch(qc_engine* e, uint64_t klo, uint64_t khi, double* out);

/* Device time (CUDA events on the engine stream) and kernel launches of the
 * last compute call; upload/readback included in the time. */
QC_API int qc_engine_last_run(const qc_engine* e, double* device_ms, uint64_t* launches,
                       uint64_t* h2d_bytes, uint64_t* d2h_bytes);

/* Benchmark hook: run the full range `reps` times on device-resident inputs
 * (no host copies) and report per-rep device time of the whole pass and of
 * the dominant (largest-traffic) step kernel. out[2] = last ket/density sum. */
QC_API int qc_engine_bench(qc_engine* e, int reps, uint64_t lo, uint64_t hi, double* pass_ms,
                    double* dominant_ms, double* dominant_bytes, double out[2]);

/* qc_engine_bench's timed calls with a cold L2: a device write of flush_bytes (>= the L2 size;
 * 0 = none) is enqueued on the engine stream before every timed call, outside its CUDA-event
 * bracket (the call is already enqueued when the write finishes, so the bracket does not
 * include the host's submission latency of an idle stream). pass_ms: reps entries. */
QC_API int qc_engine_bench_cold(qc_engine* e, int reps, uint64_t lo, uint64_t hi, uint64_t flush_bytes,
                                double* pass_ms, double out[2]);

/* One instrumented (non-graph) pass over [lo, hi): per launch, its device time
 * (CUDA events on the engine stream), algorithmic bytes, dense plan flops (8 per complex
 * MAC of every step it runs), executed flops (the dense count minus the work the zero-skip
 * removed -- measured by the fused pair kernel, equal to the dense count elsewhere) and
 * kind (0 tile wave, 1 gate, 2 fused chain, 3 fused pair). Arrays hold max_launches
 * entries (any may be NULL); *n_launches receives the program's launch count. */
QC_API int qc_engine_profile_pass(qc_engine* e, uint64_t lo, uint64_t hi, int max_launches, double* ms,
                                  double* bytes, double* flops, double* exec_flops, int32_t* kind,
                                  int32_t* n_launches);

/* Human-readable device program (launch kinds, geometry, bytes), NUL-terminated. */
QC_API int qc_engine_describe(const qc_engine* e, char* buf, size_t len);

/* ---- contract_pair on the device ----------------------------------------------------
 * Drop-in for qcut::contract_pair (proj/core/include/qcut/contraction.hpp:46-53,
 * proj/core/src/contraction.cpp:71-116): contracts legs legs_a[i] of `a` against legs_b[i]
 * of `b` (i < nshared); result legs = a's remaining legs in order, then b's; all tensors
 * row-major complex128 (interleaved re, im) with leg dimension `dim` (4 = the reference's
 * view, 2 = the binary view). Host buffers in, host buffer out (2 * dim^(ra+rb-2k) doubles).
 * The reference's permute_legs + i-s-j loop becomes a gather-staged complex GEMM: dense
 * shapes (K = dim^nshared >= 8 and both free sides >= 8 wide) run on the FP64 tensor pipe
 * (DMMA, mma.sync m8n8k4), thin shapes as one thread per output element.
 * Errors as the reference: no shared leg / leg out of range / leg repeated -> QC_EINVAL
 * with the reference's message; result rank > max_rank -> QC_ERANK (max_rank < 0: no
 * guard; the reference default is 13). A missing device is QC_EINTERNAL (no CPU path). */
#define QC_PAIR_AUTO 0   /* DMMA when dense, else the thin-shape kernel */
#define QC_PAIR_DMMA 1   /* FP64 tensor-pipe GEMM (needs K >= 8) */
#define QC_PAIR_DFMA 2   /* the same tiling on the FP64 FMA pipe (A/B partner) */
#define QC_PAIR_SMALL 3  /* one thread per output element */
QC_API int qc_contract_pair(int device, int dim, int rank_a, const double* a, const int32_t* legs_a, int rank_b,
                            const double* b, const int32_t* legs_b, int nshared, int max_rank, int path,
                            double* out);
/* The reference's BM_ContractPair (proj/benchmarks/bench_main.cpp:42-65) on the device:
 * operands uploaded once, `warmup` untimed and `reps` timed launches, each bracketed by CUDA
 * events on the launch stream (flush_l2 != 0: a 512 MB write between launches). kernel_ms =
 * mean per launch with resident operands; e2e_ms (may be NULL) = mean of upload + launch +
 * download per call; out (may be NULL) receives the result; path_used the kernel taken. */
QC_API int qc_contract_pair_bench(int device, int dim, int rank_a, const double* a, const int32_t* legs_a,
                                  int rank_b, const double* b, const int32_t* legs_b, int nshared, int path,
                                  int reps, int warmup, int flush_l2, double* out, double* kernel_ms,
                                  double* e2e_ms, int32_t* path_used);

QC_API const char* qc_last_error(void);
QC_API const char* qc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QCUT_GPU_H_ */
