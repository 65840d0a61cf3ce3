// Descriptors shared by the host program builder (program.cpp) and the
// sm_100a kernels (kernels.cu). Plain structs, no CUDA types, so the host side
// compiles with g++ alone.
//
// Everything in the engine is a binary index variable ("bit"). A tensor is a
// list of bits in storage order (MSB first) over a dense complex128 array of
// 2^nbits elements. A reference leg of dimension 4 (density view) is the bit
// pair (ket, bra) with the ket bit more significant, which makes the byte layout
// identical to the reference's row-major 4^rank layout (tensor.hpp:27-40).
#pragma once

#include <cstdint>

namespace qcg {

constexpr int kMaxRuns = 48;
constexpr int kFlowCs = 256;  // k_flow: elements of its shared-memory hand-off tile (Cs)
constexpr int kFinalTabFactors = 4;  // k_final: factors served by lookup tables
constexpr int kFlowSmemMax = 200 * 1024;  // k_flow's dynamic shared-memory attribute
constexpr int kForestSmemMax = 227 * 1024;  // k_forest's dynamic shared-memory attribute (the per-CTA maximum)
#ifndef QCG_FLOW_PREFETCH
#define QCG_FLOW_PREFETCH 1  // k_flow: stage a private continuation's outside operand early
#endif

// A bit-scatter map x -> y: for each run i, bits [src, src+len) of x land at
// bits [dst, dst+len) of y. Bits are disjoint, so y = sum of the runs. This is
// how every index translation (grid index -> operand offset, tile index ->
// operand offset, slice id -> factor element) is expressed; merging runs of
// consecutive bits keeps the device loop short.
struct Runs {
  int32_t n;
  uint8_t src[kMaxRuns];
  uint8_t len[kMaxRuns];
  uint8_t dst[kMaxRuns];
};

// One pairwise contraction (one reference PlanStep) over a batch of slices:
//   C[h, fa, fb] = sum_s A[h, fa, s] * B[h, s, fb]
// h = cut variables shared by A and B (batch), s = the step's shared legs.
// The output is tiled: a CTA owns the 2^nTC lowest C bits (the tile, contiguous
// in C) for one value of the 2^nG high C bits (the grid index g). The A-tile
// (2^nTA elements: A's bits that are summed or in the C tile) and the B-tile are
// staged in shared memory with coalesced loads, contracted, and the C tile is
// written with coalesced stores.
struct alignas(16) StepDesc {
  int64_t offA, offB, offC;  // element offsets into the arena
  int32_t nS, nTA, nTB, nTC, nG;
  int32_t pad;
  Runs gA, gB;  // grid index g -> element offset in A / B
  Runs lA, lB;  // A-tile index -> element offset in A (relative to the g base)
  Runs cA, cB;  // C-tile index -> A-tile / B-tile index
  Runs sA, sB;  // summed index s -> A-tile / B-tile index
};
static_assert(sizeof(StepDesc) % 16 == 0, "StepDesc is copied to shared memory as int4");

// A step whose small operand G (<= 2^12 elements) is staged whole in shared
// memory while the big operand X streams through once: every thread owns one
// "column" j of X (X's non-summed bits, in X's storage order), loads its K = 2^nS
// summed values into registers and emits all 2^nF outputs of that column:
//   C[f, j] = sum_s G[h(j), f, s] * X[j, s],   C offset = (f << nCol) + j.
// This is the state-vector pattern (apply a small gate to a large state): X is
// read exactly once, C is written once, both coalesced along j.
// When G is too large for shared memory its highest free bits F_hi become a grid
// dimension (blockIdx.y): each CTA stages the G tile of one F_hi value and X is
// re-read per F_hi value (only allowed when X is L2-resident).
struct alignas(16) GateDesc {
  int64_t offG, offX, offC;
  int32_t nG;    // bits of the staged G tile (G's bits minus F_hi and H_hi)
  int32_t nS;    // summed bits (template K = 2^nS)
  int32_t nF;    // G's free bits in the tile (outputs per column per CTA = 2^nF)
  int32_t nCol;  // X's non-summed bits
  int32_t nFhi;  // G's free bits on the grid (blockIdx.y low bits; X re-read per value)
  int32_t nHhi;  // G's batch bits shared with X columns on the grid (blockIdx.y high bits;
                 // each value owns a disjoint column subset, no re-read)
  int32_t pair2;  // 1: column bit 0 is X's and C's lowest bit (k_gate2, 256-bit access)
  int32_t reduce; // 1: C is the pass's lead rank-0 factor (every batched slice bit): k_gate_reduce
                  // multiplies each output by the other factors and sums -- C and k_final's walk
                  // over it disappear unless per-slice values are requested
  Runs xcol;     // thread column index -> X offset
  Runs xs;       // summed index -> X offset
  Runs gcol;     // thread column index -> G-tile index (batch bits shared with G)
  Runs gs;       // summed index -> G-tile index
  Runs gf;       // free (tile) index -> G-tile index
  Runs gtile;    // G-tile index -> G offset
  Runs gfhi;     // F_hi index -> G offset
  Runs ghhi, xhhi, chhi;  // H_hi index -> G offset / X offset / C column index
  Runs ccol;     // thread column index -> C column index (identity when nHhi = 0)
  int64_t xs_tab[16];  // xs(s) for s < 2^nS (host-evaluated: no per-thread map setup)
  int32_t gs_tab[16];  // gs(s)
};

// Two consecutive gate steps fused at register level (no intermediate in memory):
//   step 1: C1 = sum_{s1} G1[r, q, s1, h1] X[j', p, s1]       (C1 = [F1] ++ [X cols])
//   step 2: C2 = sum_{q, p} G2[f2, q, p, h2] C1[r, q, j', p]   (C2 = [F2] ++ [R] ++ [cols'])
// with P = step-2 summed bits among X's columns, Q = those among G1's free bits,
// R = G1's free bits that survive, cols' = X's columns minus P. A thread owns one
// column j': it loads its 2^nP x K1 values of X into registers once, then for each
// r emits C2[f2, r, j'] for all f2. R splits into r_lo (register accumulators),
// r_mid (a loop) and r_hi (blockIdx.y: one G1 tile per CTA in shared memory).
// Both small operands are staged in shared memory in an "expanded" layout whose
// innermost bits are the ones the inner loops walk, so every shared load in the
// loop nest is one per-(q, accumulator) base plus a compile-time offset:
//   G1x[hc1][r_mid, r_lo][q][p][s1]   (p expanded over P bits G1 does not carry)
//   G2x[hc2][r in G2][f2][q][p]
struct alignas(16) PairDesc {
  int64_t offG1, offG2, offX, offC;
  int32_t nS1, nS2, nP, nQ;
  int32_t nRlo, nRmid, nRhi, nF2;
  int32_t nCol;  // bits of cols'
  int32_t nG1x;  // bits of the expanded G1 tile (shared memory)
  int32_t nG2;   // bits of G2 (staged whole, permuted)
  int32_t nR;    // nRlo + nRmid + nRhi
  int32_t nHhi;  // G1-carried cols' bits on the grid (blockIdx.y high bits, the top bits of the
                 // expanded G1 tile): each value owns a disjoint column subset and stages
                 // only its G1x sub-block (no re-read)
  int32_t nG1h;  // |hc1|: cols' bits G1 carries
  Runs jcol;     // thread column index -> cols' index (the H_hi bits zero)
  Runs jhhi;     // H_hi index -> cols' index bits
  Runs xcol;            // cols' -> X offset
  Runs g1stage, g1hi;   // expanded G1 index -> G1 offset; r_hi -> G1 offset
  Runs g1hc;            // cols' -> expanded G1 index (hc1 block)
  Runs g2stage;         // expanded G2 index -> G2 offset
  Runs g2hc, g2r;       // cols' -> expanded G2 index; r (lo, mid, hi) -> expanded G2 index
  // bank skew: the hc blocks (top bits, selected by the lane's column) are padded by one
  // element each, so lanes reading different blocks hit different shared-memory banks:
  // shared index = expanded index + (expanded index >> sh)
  int32_t sh1, sh2;     // nG1x - |hc1|, nG2 - |hc2|
  Runs g1hcx, g2hcx;    // cols' -> hc1 / hc2 block number
  int64_t xoff_tab[16];  // X offset of (p, s1) at p * 2^nS1 + s1
};

// A fused chain of gate-shaped PlanSteps (state-vector gate fusion): step j
// contracts the running state with a small tensor G_j. A CTA owns one value of
// the "outer" state bits (never summed in the chain): it loads the input tile
// (the chain's summed input bits + coalescing bits, 2^nT0 elements) from HBM,
// runs every stage in shared memory (tile T_j = T_{j-1} minus S_j plus G_j's free
// bits), and writes only the last stage's tile. Intermediates never touch HBM.
constexpr int kMaxChain = 8;
// Stage j of a chain, in "column" form: the input tile's bits that survive the
// stage (kept bits Kp) index columns c; a thread loads the K = 2^nS summed values
// of a column into registers once and emits all 2^nF outputs of that column:
//   out[c + (f << nKp)] = sum_s G[gH(c) + gF[f] + gS[s] + grid2g(g)] * in[col(c) + sin[s]]
// (last stage: written to HBM at grid2out(g) + ccol(c) + cF[f]).
struct ChainStage {
  int64_t offG;   // G_j in the arena
  int32_t gsm;    // G_j's element offset in shared memory
  int32_t nG;     // bits of G_j
  int32_t nS, nKp, nF;
  int32_t tab;    // offset of this stage's int tables in shared memory
  Runs col;       // column index -> input tile index (summed bits zero)
  Runs gH;        // column index -> G index (G's batch bits inside the tile)
  Runs grid2g;    // CTA grid index -> G index (G's batch bits among the outer bits)
  Runs ccol;      // last stage: column index -> output offset
  Runs sin, gS;   // summed index -> input tile index / G index     (tabulated)
  Runs gF, cF;    // free index -> G index / output offset (last)   (tabulated)
};
struct alignas(16) ChainDesc {
  int64_t offIn, offOut;
  int32_t nStages, nT0, nGrid, nTmax, gElems, tabInts;
  int32_t nIter;        // CTA b runs grid indices (b << nIter) | i, i < 2^nIter
  int32_t nW1;          // bits of the second stage buffer (stages 2, 4, ...); nTmax covers 1, 3, ...
  int32_t imgInts;      // shared-memory table image (ints), host-built, copied verbatim per CTA
  int64_t img;          // its offset (ints) in the engine's chain-image buffer
  int32_t extraOff;     // ints from the image start to loadLo|loadHi|itIn|itOut|itG (8-B aligned)
  int32_t pad3;
  Runs load;      // input tile index -> input offset
  Runs grid2in;   // grid index -> input offset
  Runs grid2out;  // grid index -> output offset
  ChainStage st[kMaxChain];
};
static_assert(sizeof(ChainDesc) % 16 == 0, "ChainDesc is copied to shared memory as int4");
// What k_chain's prologue needs before any memory arrives (a kernel parameter, ~0.5 KB): the
// sizes, where the table image / small operands / descriptor live, and the two maps that
// address the first input tile. The full ChainDesc follows by bulk copy into shared memory.
struct ChainHead {
  int64_t offIn, img;
  int32_t nT0, nTmax, nW1, gElems, nStages, imgInts, nIter, nGrid;
  int64_t offG[kMaxChain];
  int32_t gsm[kMaxChain], nG[kMaxChain];
  Runs load, grid2in;
};

// ---- k_forest: a dataflow group of small steps as independent subtrees, one per CTA ----
// A group's tile steps form a forest (each tensor has one consumer). Every subtree (or a
// pack of small ones) is a "unit" run by one CTA: its steps in phases (ALAP depth), all
// steps of a phase at once, one barrier between phases, operands and intermediates in
// shared memory where they fit (the rest in the arena, read back through L2). No
// cross-CTA dependency exists inside a group, so a phase costs a barrier, not an L2
// round trip.
constexpr int kFMapRuns = 15;
// A bit-scatter map over indices of <= 16 bits, each run packed src | len << 5 | dst << 10.
struct FMap {
  uint16_t n;
  uint16_t r[kFMapRuns];
};
// One plan step in "column" form: C's bits split into column bits (every C bit of the
// streamed operand X -- including batch bits X shares with G -- and G-only bits beyond the
// first two) and up to two loop bits (C bits only the small operand G carries). A lane owns
// one column: it loads its K = 2^nS values of X into registers once, then for every loop
// value l (unrolled, independent accumulators) emits
//   C[colC(col) + loopC[l]] = sum_s G[colG(col) + loopG[l] + tg[s]] * X[colX(col) + tx[s]].
// A work item is 32 consecutive columns (one warp). The column maps are bit scatters, so they
// are additive over disjoint bit fields: host-built tables serve column bits 0-4, 5-9 and
// 10-13 -- three lookups per operand, no map walk on the device.
struct alignas(16) FStep {
  int64_t gG, gX, gC;   // arena element offsets (operands in global memory)
  int32_t sG, sX, sC;   // data-region element offsets in shared memory, -1: global
  int32_t nCol, nLoop, nS;  // column bits (<= 14), loop bits (<= 2), summed bits (<= 4)
  uint16_t tg[16], tx[16];  // G / X offsets of the summed index (operands have <= 2^16 elements)
  uint16_t loopG[4], loopC[4];
  uint16_t laneC[32], laneG[32], laneX[32];  // column maps of column bits 0-4 (the lane)
  uint16_t midC[32], midG[32], midX[32];     // column bits 5-9
  uint16_t highC[16], highG[16], highX[16];  // column bits 10-13
};
static_assert(sizeof(FStep) % 16 == 0, "FStep is copied to shared memory in 16-byte units");
// Per unit: its image (int32 words, 16-byte aligned) in Program::forest_image:
//   [nphases, nsteps, nitems, nleaves] phase_off[nphases + 1] (pad to 4) items[nitems] (pad to 4)
//   leaves[nleaves] {int64 arena offset, int32 data-region offset, int32 bytes} FStep[nsteps]
// item = step << 16 | 32-column chunk; the image and every leaf arrive by bulk copy (TMA).
struct ForestUnit {
  int64_t img;         // word offset of the image
  int32_t img_words;   // image size (multiple of 4)
  int32_t leaf_off;    // word offset of leaves[] in the image
  int32_t nleaves;
  int32_t leaf_bytes;  // sum of leaf bytes (bulk-copy transaction count)
  int32_t data_off;    // byte offset of the data region in dynamic shared memory
  int32_t smem;        // dynamic shared memory the unit needs (bytes)
};

// Per-pass slicing of an initial tensor whose cut legs are fixed by the pass's
// high slice-id bits (apply_cut, cutting.cpp:67-129, done as a gather).
struct alignas(16) PrepDesc {
  int64_t src;      // full (uncut) tensor in the static region
  int64_t dst;      // sliced copy in the arena
  int32_t nbits;    // bits of the sliced copy
  int32_t nfix;     // fixed cut bits
  uint8_t fix_pos[16];     // slice-id bit position of each fixed bit
  int64_t fix_stride[16];  // element stride of that bit in the full tensor
  Runs map;         // sliced index -> full-tensor element offset
};

// k_final's dynamic shared memory: factor-map lookup tables, then the staged factor descriptors
constexpr int kFinalSmemFactors = 32;

static_assert(sizeof(GateDesc) % 16 == 0 && sizeof(PairDesc) % 16 == 0 && sizeof(PrepDesc) % 16 == 0,
              "descriptor arrays are copied to shared memory in 16-byte units");

// A rank-0 (in the reference's sense) result: the reference multiplies it into
// the slice's accumulator (contraction.cpp:304-306, 311-317). Here it is a
// tensor over the batched cut bits it depends on.
struct FactorDesc {
  int64_t off;
  Runs map;  // pass-local slice index -> element offset
};
static_assert(sizeof(FactorDesc) % 16 == 0, "k_final copies FactorDesc arrays as int4");

// Device-resident per-pass state, written by the host before each pass.
struct RunState {
  uint64_t pass_base;   // global slice id of the pass's first slice
  uint64_t lo, hi;      // requested slice-id range (in the engine's id space)
  uint64_t slot;        // partial-sum slot of this pass within the call
  uint64_t out_base;    // global id of slice_out[0]
  uint64_t nparts;      // last pass of the call: the call's passes, whose partials it reduces (else 0)
  void* slice_out;      // per-slice values (double2, [amplitude][id - out_base]), or nullptr
  uint64_t out_stride;  // slice_out entries per amplitude
};

}  // namespace qcg
