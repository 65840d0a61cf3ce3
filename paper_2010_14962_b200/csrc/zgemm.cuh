// Dense pairwise contraction as a batched complex128 GEMM on the FP64 tensor pipe (DMMA).
//
// The reference's contract_pair (proj/core/src/contraction.cpp:71-116) permutes both
// operands (permute_legs, tensor.cpp:30-62) to [free, shared] / [shared, free] and runs an
// i-s-j triple loop: an M x K times K x N complex matrix product with M = d^|free(a)|,
// K = d^|shared|, N = d^|free(b)| (d = 4 in the reference's view, 2 in the binary view).
// Here the permutes are never materialised: every leg is a bit field of the operand's
// row-major index, so the permuted element (m, s) of A sits at mA[m] + kA[s] -- two
// additive host-built tables -- and the tile staging gathers through them with 16-byte
// asynchronous copies into a multi-stage shared-memory pipeline.
//
//   k_zgemm_dmma   CTA tile 64 x 64 complex, 8 warps as 4 (M) x 2 (N), warp tile 16 x 32 =
//                  2 x 4 DMMA tiles (mma.sync m8n8k4 f64). Complex arithmetic is the real
//                  embedding with split accumulators: Cre += Are*Bre; Cre += (-Aim)*Bim;
//                  Cim += Are*Bim; Cim += Aim*Bre -- four real DMMAs per 8 x 8 x 4 complex
//                  block, i.e. exactly 4 real FMAs per complex MAC (no padding waste).
//                  Operands stay interleaved (re, im) in shared memory: one LDS.128 per
//                  fragment element yields both planes. Row stride 192 B (8 k-elements +
//                  64 B skew) makes every quarter-warp's fragment load conflict-free.
//   k_zgemm_dfma   the same staging with a classical 4 x 4 register micro-tile of DFMAs per
//                  thread: the A/B partner of the DMMA kernel (tools/pair_bench.py).
//   k_contract_small  one thread per output element: the shapes that are not dense
//                  contractions (K < 8 or a free side < 8 wide), where a GEMM tile would
//                  be mostly padding.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace qcg {

struct GemmDesc {
  int64_t M, N, K;       // powers of two (d^legs)
  int64_t batch;         // independent products; operand/result offsets from `btabs`
  // batch tables gA[batch] gB[batch] gC[batch] (element offsets), or null for batch = 1
  const int64_t* btabs;
  // table image (int64 element offsets): kA[K] kB[K] mA[M] nB[N] mC[M] nC[N]
  const int64_t* tabs;
  int32_t a_kfast, b_kfast;  // staging order: 1 = consecutive threads walk k, 0 = walk rows
  int32_t c_pair;            // 1: nC[n + 1] == nC[n] + 1 for even n (256-bit result stores)
};

constexpr int kGemmThreads = 256;
constexpr int kGemmBM = 64, kGemmBN = 64, kGemmBK = 8;
constexpr int kGemmStages = 4;
constexpr int kGemmRowBytes = kGemmBK * 16 + 64;  // 192: skewed row of a staged tile
constexpr int kGemmStageBytes = (kGemmBM + kGemmBN) * kGemmRowBytes;
constexpr int kGemmSmemBytes = kGemmStages * kGemmStageBytes + (kGemmBM + kGemmBN) * 8;

__device__ __forceinline__ void zg_cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void zg_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void zg_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ double2 zg_lds(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
// D(8x8) += A(8x4, row) * B(4x8, col) on the FP64 tensor pipe
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Stage k-step `kt` of both operand tiles into pipeline stage `st` (rows skewed, see above).
// LAYOUT 0: [row][k] (DMMA fragments); LAYOUT 1: [k][row] rows contiguous (DFMA micro-tiles).
template <int LAYOUT>
__device__ __forceinline__ void zg_stage(const GemmDesc& d, const double2* __restrict__ A,
                                         const double2* __restrict__ B, unsigned sbase, int st, int64_t kt,
                                         const int64_t* sRowA, const int64_t* sRowB) {
  const int64_t* kA = d.tabs;
  const int64_t* kB = d.tabs + d.K;
  const unsigned sa = sbase + st * kGemmStageBytes;
  const unsigned sb = sa + kGemmBM * kGemmRowBytes;
  const int tid = threadIdx.x;
  auto dst = [&](unsigned base, int row, int k, int rows) -> unsigned {
    if constexpr (LAYOUT == 0) return base + row * kGemmRowBytes + k * 16;
    else return base + (k * rows + row) * 16;
  };
  const int64_t k0 = kt * kGemmBK;
  if (d.a_kfast) {
    const int k = tid & (kGemmBK - 1);
    const int64_t ko = __ldg(kA + k0 + k);
#pragma unroll
    for (int i = 0; i < kGemmBM * kGemmBK / kGemmThreads; ++i) {
      const int row = (tid / kGemmBK) + i * (kGemmThreads / kGemmBK);
      zg_cp16(dst(sa, row, k, kGemmBM), A + sRowA[row] + ko);
    }
  } else {
    const int row = tid & (kGemmBM - 1);
    const int64_t ro = sRowA[row];
#pragma unroll
    for (int i = 0; i < kGemmBM * kGemmBK / kGemmThreads; ++i) {
      const int k = (tid / kGemmBM) + i * (kGemmThreads / kGemmBM);
      zg_cp16(dst(sa, row, k, kGemmBM), A + ro + __ldg(kA + k0 + k));
    }
  }
  if (d.b_kfast) {
    const int k = tid & (kGemmBK - 1);
    const int64_t ko = __ldg(kB + k0 + k);
#pragma unroll
    for (int i = 0; i < kGemmBN * kGemmBK / kGemmThreads; ++i) {
      const int row = (tid / kGemmBK) + i * (kGemmThreads / kGemmBK);
      zg_cp16(dst(sb, row, k, kGemmBN), B + sRowB[row] + ko);
    }
  } else {
    const int row = tid & (kGemmBN - 1);
    const int64_t ro = sRowB[row];
#pragma unroll
    for (int i = 0; i < kGemmBN * kGemmBK / kGemmThreads; ++i) {
      const int k = (tid / kGemmBN) + i * (kGemmThreads / kGemmBN);
      zg_cp16(dst(sb, row, k, kGemmBN), B + ro + __ldg(kB + k0 + k));
    }
  }
}

// Common prologue: row tables of this CTA's tile (rows past M / N repeat row 0 and are
// never stored), then the first kGemmStages - 1 k-steps in flight.
struct ZgTile {
  int64_t m0, n0;
  const double2 *A, *B;
  double2* C;
  int64_t* sRowA;
  int64_t* sRowB;
  unsigned sbase;
};

template <int LAYOUT>
__device__ __forceinline__ ZgTile zg_prologue(const GemmDesc& d, const double2* __restrict__ A0,
                                              const double2* __restrict__ B0, double2* __restrict__ C0,
                                              unsigned char* smem) {
  ZgTile t;
  const int64_t tiles_n = (d.N + kGemmBN - 1) / kGemmBN, tiles_m = (d.M + kGemmBM - 1) / kGemmBM;
  const int64_t z = blockIdx.x / (tiles_m * tiles_n), tile = blockIdx.x % (tiles_m * tiles_n);
  t.m0 = (tile / tiles_n) * kGemmBM;
  t.n0 = (tile % tiles_n) * kGemmBN;
  t.A = A0 + (d.btabs ? d.btabs[z] : 0);
  t.B = B0 + (d.btabs ? d.btabs[d.batch + z] : 0);
  t.C = C0 + (d.btabs ? d.btabs[2 * d.batch + z] : 0);
  t.sRowA = reinterpret_cast<int64_t*>(smem + kGemmStages * kGemmStageBytes);
  t.sRowB = t.sRowA + kGemmBM;
  t.sbase = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int64_t* mA = d.tabs + 2 * d.K;
  const int64_t* nB = mA + d.M;
  for (int i = threadIdx.x; i < kGemmBM + kGemmBN; i += blockDim.x) {
    if (i < kGemmBM) t.sRowA[i] = mA[t.m0 + i < d.M ? t.m0 + i : 0];
    else t.sRowB[i - kGemmBM] = nB[t.n0 + (i - kGemmBM) < d.N ? t.n0 + (i - kGemmBM) : 0];
  }
  // inside the engine the kernel is launched with programmatic stream serialization: the
  // tables above are static, the operands are the previous launches' outputs
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();
  const int64_t KT = d.K / kGemmBK;
#pragma unroll
  for (int s = 0; s < kGemmStages - 1; ++s) {
    if (s < KT) zg_stage<LAYOUT>(d, t.A, t.B, t.sbase, s, s, t.sRowA, t.sRowB);
    zg_commit();
  }
  return t;
}

static __global__ void __launch_bounds__(kGemmThreads, 2) k_zgemm_dmma(const __grid_constant__ GemmDesc d,
                                                                 const double2* __restrict__ A0,
                                                                 const double2* __restrict__ B0,
                                                                 double2* __restrict__ C0) {
  extern __shared__ __align__(128) unsigned char zg_smem[];
  const ZgTile t = zg_prologue<0>(d, A0, B0, C0, zg_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
  double cre[2][4][2], cim[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) cre[i][j][c] = cim[i][j][c] = 0.0;
  const int64_t KT = d.K / kGemmBK;
  // fragment element of this lane inside a staged tile: row g (+ sub-tile), k-element q
  const unsigned fa = (wm + g) * kGemmRowBytes + q * 16;
  const unsigned fb = kGemmBM * kGemmRowBytes + (wn + g) * kGemmRowBytes + q * 16;
  for (int64_t kt = 0; kt < KT; ++kt) {
    zg_wait<kGemmStages - 2>();
    __syncthreads();  // stage kt landed for every thread; stage kt - 1 is free again
    {
      const int64_t nx = kt + kGemmStages - 1;
      if (nx < KT) zg_stage<0>(d, t.A, t.B, t.sbase, static_cast<int>(nx % kGemmStages), nx, t.sRowA, t.sRowB);
      zg_commit();
    }
    const unsigned sb = t.sbase + static_cast<unsigned>(kt % kGemmStages) * kGemmStageBytes;
#pragma unroll
    for (int k4 = 0; k4 < kGemmBK / 4; ++k4) {
      double2 a[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = zg_lds(sb + fa + i * 8 * kGemmRowBytes + k4 * 64);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = zg_lds(sb + fb + j * 8 * kGemmRowBytes + k4 * 64);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double nai = -a[i].y;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(cre[i][j][0], cre[i][j][1], a[i].x, b[j].x);
          dmma(cim[i][j][0], cim[i][j][1], a[i].x, b[j].y);
          dmma(cre[i][j][0], cre[i][j][1], nai, b[j].y);
          dmma(cim[i][j][0], cim[i][j][1], a[i].y, b[j].x);
        }
      }
    }
  }
  // result: lane holds (row g, columns 2q and 2q + 1) of every 8 x 8 tile
  const int64_t* mC = d.tabs + 2 * d.K + d.M + d.N;
  const int64_t* nC = mC + d.M;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t m = t.m0 + wm + 8 * i + g;
    if (m >= d.M) continue;
    const int64_t ro = __ldg(mC + m);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = t.n0 + wn + 8 * j + 2 * q;
      if (n >= d.N) continue;
      if (d.c_pair) {
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(t.C + ro + __ldg(nC + n)), "d"(cre[i][j][0]),
                     "d"(cim[i][j][0]), "d"(cre[i][j][1]), "d"(cim[i][j][1])
                     : "memory");
      } else {
        t.C[ro + __ldg(nC + n)] = make_double2(cre[i][j][0], cim[i][j][0]);
        if (n + 1 < d.N) t.C[ro + __ldg(nC + n + 1)] = make_double2(cre[i][j][1], cim[i][j][1]);
      }
    }
  }
}

// The DFMA partner: thread (ty, tx) owns the 4 x 4 complex micro-tile rows 4 ty .. 4 ty + 3,
// columns 4 tx .. 4 tx + 3 of the 64 x 64 CTA tile; operands staged [k][row].
static __global__ void __launch_bounds__(kGemmThreads, 2) k_zgemm_dfma(const __grid_constant__ GemmDesc d,
                                                                 const double2* __restrict__ A0,
                                                                 const double2* __restrict__ B0,
                                                                 double2* __restrict__ C0) {
  extern __shared__ __align__(128) unsigned char zg_smem[];
  const ZgTile t = zg_prologue<1>(d, A0, B0, C0, zg_smem);
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
  const int64_t KT = d.K / kGemmBK;
  for (int64_t kt = 0; kt < KT; ++kt) {
    zg_wait<kGemmStages - 2>();
    __syncthreads();
    {
      const int64_t nx = kt + kGemmStages - 1;
      if (nx < KT) zg_stage<1>(d, t.A, t.B, t.sbase, static_cast<int>(nx % kGemmStages), nx, t.sRowA, t.sRowB);
      zg_commit();
    }
    const unsigned sa = t.sbase + static_cast<unsigned>(kt % kGemmStages) * kGemmStageBytes;
    const unsigned sb = sa + kGemmBM * kGemmRowBytes;
#pragma unroll
    for (int k = 0; k < kGemmBK; ++k) {
      double2 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = zg_lds(sa + (k * kGemmBM + 4 * ty + i) * 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = zg_lds(sb + (k * kGemmBN + 4 * tx + j) * 16);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fma(a[i].x, b[j].x, acc[i][j].x);
          acc[i][j].x = fma(-a[i].y, b[j].y, acc[i][j].x);
          acc[i][j].y = fma(a[i].x, b[j].y, acc[i][j].y);
          acc[i][j].y = fma(a[i].y, b[j].x, acc[i][j].y);
        }
    }
  }
  const int64_t* mC = d.tabs + 2 * d.K + d.M + d.N;
  const int64_t* nC = mC + d.M;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = t.m0 + 4 * ty + i;
    if (m >= d.M) continue;
    const int64_t ro = __ldg(mC + m);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = t.n0 + 4 * tx + j;
      if (n < d.N) t.C[ro + __ldg(nC + n)] = acc[i][j];
    }
  }
}

// Thin shapes: one thread per output element, the K products accumulated in s order
// (the reference's own summation order, contraction.cpp:104-113).
static __global__ void __launch_bounds__(256) k_contract_small(const __grid_constant__ GemmDesc d,
                                                        const double2* __restrict__ A0,
                                                        const double2* __restrict__ B0,
                                                        double2* __restrict__ C0) {
  const int64_t* kA = d.tabs;
  const int64_t* kB = kA + d.K;
  const int64_t* mA = kB + d.K;
  const int64_t* nB = mA + d.M;
  const int64_t* mC = nB + d.N;
  const int64_t* nC = mC + d.M;
  const double2* A = A0;
  const double2* B = B0;
  double2* C = C0;
  const int64_t total = d.M * d.N;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = e / d.N, n = e - m * d.N;
    const int64_t ao = mA[m], bo = nB[n];
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t s = 0; s < d.K; ++s) {
      const double2 a = A[ao + kA[s]], b = B[bo + kB[s]];
      acc.x = fma(a.x, b.x, acc.x);
      acc.x = fma(-a.y, b.y, acc.x);
      acc.y = fma(a.x, b.y, acc.y);
      acc.y = fma(a.y, b.x, acc.y);
    }
    C[mC[m] + nC[n]] = acc;
  }
}

}  // namespace qcg
