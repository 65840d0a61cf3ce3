// Host side of the engine: payload decoding (mirrors decode_payload,
// proj/core/src/serialize.cpp:156-167), validation with the reference's error
// classes, the ket factorisation of density-basis tensors, and the translation
// of the reference ContractionPlan into a device program over binary variables
// (layouts, tiles, memory plan). No CUDA here.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "desc.hpp"

namespace qcg {

struct cxd {
  double re, im;
};

struct Vertex {
  int id = 0;
  int rank = 0;
  std::vector<cxd> data;  // 4^rank, row-major, leg 0 most significant
};

struct NetEdge {
  int id, u, leg_u, v, leg_v;
};

struct PlanStep {
  int a = -1, b = -1, out = -1;
  std::vector<int> edges, legs_a, legs_b;
  int rank_a = 0, rank_b = 0, result_rank = 0, work_rank = 0;
};

// The reference Payload {network, cut, plan, max_rank} (serialize.hpp:32-37).
struct Payload {
  std::vector<Vertex> vertices;  // ascending id (TensorNetwork::vertices is a std::map)
  std::vector<NetEdge> edges;
  std::vector<int> cut;
  std::vector<PlanStep> steps;
  std::vector<int> scalars;
  int peak_rank = 0;
  double cost_estimate = 0;
  int max_rank = 13;
};

// qcut::RankGuardError (contraction.hpp:34-44, message contraction.cpp:29-36).
class RankGuard : public std::runtime_error {
 public:
  RankGuard(int rank, int max_rank);
  int rank, max_rank;
};

Payload decode_payload(const char* text, size_t len);
void check_closed(const Payload& p);  // tensor_network.cpp:128-153
void check_cut(const Payload& p);     // cutting.cpp:67-92 argument checks
void check_rank_guard(const Payload& p);  // contraction.cpp:280-286
// Batched amplitudes: same network, cut and plan (std::invalid_argument otherwise).
void check_same_structure(const Payload& a, const Payload& b);

// K with T[(k1 b1)...(kr br)] = K[k1..kr] conj(K[b1..br]); the largest |K| entry
// is made real positive. Throws std::invalid_argument if T is not of that form.
std::vector<cxd> ket_factor(const std::vector<cxd>& t, int rank);

enum Mode { kDensity = 0, kKet = 1 };
enum StepKind { kTile = 0, kGate = 1, kChain = 2, kPair = 3, kForest = 4, kGemm = 5 };

struct Program {
  Mode mode = kKet;
  int M = 0;           // cut edges
  int bpc = 1;         // bits per cut variable (1 ket, 2 density)
  int id_bits = 0;     // slice-id bits: M * bpc
  int b = 0;           // batched (pass-local) slice-id bits
  int n_amps = 1;      // amplitudes batched in every pass (payloads differing only in values)
  int amp_bits = 0;    // ceil(log2 n_amps): pass-local index = amplitude << b | slice
  uint64_t passes = 1; // 2^(id_bits - b)

  int64_t static_elems = 0;  // arena[0, static_elems) holds uploaded tensors
  int64_t arena_elems = 0;   // total elements (static + workspace)
  std::vector<cxd> static_data;

  std::vector<PrepDesc> prep;
  // Per plan step (plan order): which kernel family runs it and its traffic.
  std::vector<int> step_kind;        // kTile or kGate
  std::vector<int> step_level;       // dependency level (launch wave) of the op running the step
  std::vector<int> step_fused;       // 1 if the step runs inside a fused chain
  std::vector<double> kernel_bytes;  // bytes moved per step per pass
  std::vector<double> kernel_flops;  // real flops per step per pass
  std::vector<int> kernel_dep;       // 1 if the step's operands carry cut variables
  // Device work, in launch order.
  std::vector<StepDesc> tiles;       // tile-kernel steps, grouped by launch
  std::vector<uint64_t> tile_prefix; // per launch: prefix tile counts (count+1 entries each)
  // Dataflow dependencies of tile steps inside their launch (CSR, launch-local step
  // indices): steps of launch L are flow_dep_off[L.dep_off + k] .. [+k+1].
  std::vector<int> flow_dep_off, flow_deps;
  std::vector<int> flow_cont;   // per tile step: launch-local continuation step or -1
  std::vector<int> flow_conly;  // per tile step: 1 = run only as a continuation (never queued)
  std::vector<GateDesc> gates;
  std::vector<ChainDesc> chains;
  std::vector<PairDesc> pairs;
  std::vector<int32_t> chain_image;  // concatenated k_chain shared-memory table images
  std::vector<ForestUnit> forest_units;  // k_forest units, grouped by launch
  std::vector<int32_t> forest_image;     // concatenated unit images
  // A dense PlanStep (both operands large, >= 8 summed index values, both free sides >= 8
  // wide) as a batched complex GEMM on the FP64 tensor pipe (zgemm.cuh, k_zgemm_dmma):
  // C[g; m, n] = sum_k A[g; m, k] B[g; k, n] with every index map a host-built table.
  struct GemmOp {
    int64_t offA, offB, offC;  // arena element offsets
    int32_t nM, nN, nK, nG;    // log2 extents (g = batch: bits both operands carry, not summed)
    int64_t tab;               // gemm_image offset (int64 entries): kA[K] kB[K] mA[M] nB[N] mC[M] nC[N]
                               // gA[G] gB[G] gC[G]
    int32_t a_kfast, b_kfast, c_pair;
  };
  std::vector<GemmOp> gemms;
  std::vector<int64_t> gemm_image;
  struct Launch {
    int kind;            // kTile (a wave of tile steps), kForest (a forest of small steps), kGate (one
                         // step), kChain / kPair (fused steps)
    int first, count;    // tiles[first, first+count), forest_units[first, first+count), gates[first],
                         // chains[first] or pairs[first]
    int prefix_off;      // kTile: offset into tile_prefix
    int dep_off;         // kTile: offset into flow_dep_off (count + 1 entries)
    uint64_t items;      // kTile: total tiles; kGate: columns
    int smem;            // dynamic shared memory bytes
    int npre;            // kTile: elements of each of k_flow's two continuation-operand prefetch buffers
    int plan_step;       // kGate: plan step index; kTile: -1
    double bytes;        // bytes its steps read + write per pass
    double flops;        // real flops of its steps per pass (8 per complex MAC)
    int per_pass;        // 1: reads a tensor that depends on the pass's fixed slice bits
  };
  std::vector<Launch> launches;
  std::vector<std::vector<int>> launch_deps;  // per launch: the launches producing its inputs
  std::vector<FactorDesc> factors;
  // k_final lookup tables (<= kFinalTabFactors factors over <= 20 batch bits): per factor,
  // its map evaluated on the low and the high 10 bits of the pass-local slice index
  // (2 x 1024 entries); empty when k_final walks the maps instead
  std::vector<uint32_t> final_tab;
  int final_fused = -1;  // launch (a kGate) whose epilogue does the final product and sum, or -1
  int final_lead = -1;  // factor whose storage order k_final walks (its inverse map is the last table pair)

  // shape parity (one entry per reference plan step)
  std::vector<int> ra, rb, rk, rr;
  int n_invariant = 0;
  double essential_bytes = 0;  // SURVEY §8(d), full range
  double moved_bytes = 0;      // engine kernels, full range
  double flops = 0;            // SURVEY §8(d), full range
  double algo_flops = 0;       // engine plan flops at the batched shapes, full range

  uint64_t jobs_density() const;  // 4^M
  uint64_t jobs_ket() const;      // 2^M
};

// Thrown by build_program when an intermediate needs more than 2^56 elements (the arena offsets would
// overflow); plan_program turns it into the memory-budget error.
struct WorkspaceTooLarge : std::runtime_error {
  explicit WorkspaceTooLarge(int bits);
  int bits;
};

Program build_program(const Payload& p, Mode mode, int batch_bits);
// Several payloads of one network, cut and plan whose tensor values differ (output bitstrings,
// angle sets): one program, their amplitudes as extra batch bits (Program::amp_bits).
Program build_program(const std::vector<const Payload*>& amps, Mode mode, int batch_bits);
// Human-readable launch list (kinds, geometry, bytes) for profiling and tests.
std::string describe_program(const Program& prog);
// Largest batch (<= max_batch_bits when >= 0) such that the arena fits `budget_bytes`.
Program plan_program(const Payload& p, Mode mode, uint64_t budget_bytes, int max_batch_bits = -1);
Program plan_program(const std::vector<const Payload*>& amps, Mode mode, uint64_t budget_bytes,
                     int max_batch_bits = -1);

}  // namespace qcg
