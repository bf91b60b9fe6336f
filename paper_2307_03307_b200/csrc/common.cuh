// common.cuh — shared types, constants and block/grid reduction helpers for the MWU hot path.
//
// All reductions are deterministic: every kernel that reduces writes one partial per block
// (fixed block -> work assignment), and the LAST block to finish (threadfence + atomic ticket,
// the classic "last block" pattern) combines the partials in a fixed order and runs the
// control logic of that phase (finalize).  So one MWU phase = one kernel launch, with no
// host round trip, which is what lets a whole probe run as one CUDA-graph launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define MWU_NT 256            // threads per block for every kernel
#define MWU_MAXC 8            // step-search candidates evaluated per HBM pass
#define MWU_SLOTS 32          // reduction slots per block partial (4 * MAXC)
#define MWU_TILE 2048         // items per seg tile (a tile loads <= 2*TILE items into smem)
#define MWU_LCH 8192          // items per chunk of a long row (deg > TILE)

namespace mwu {

enum Status : int { ST_RUNNING = 0, ST_FEASIBLE = 1, ST_INFEASIBLE = 2, ST_ITER_LIMIT = 3 };
enum Reason : int { R_NONE = 0, R_MAXD_ZERO = 1, R_ALPHA_LT_1 = 2, R_EMPTY_COVER = 3, R_ITER_LIMIT = 4, R_MIN_Z = 5 };
enum RedOp : int { OP_SUM = 0, OP_MAX = 1, OP_MIN = 2 };
// candidate evaluation modes of one side in a search pass (DESIGN.md §3 Q16)
enum CandMode : int { CM_EXPM1 = 0, CM_LSE = 1, CM_EXT = 2 };
// search phases (Alg. 3)
enum SPhase : int { SP_DOUBLE = 0, SP_BISECT = 1, SP_DONE = 2, SP_FIXED = 3 };

// Finalize actions (what the last block does after a kernel's reduction).
enum Action : int {
  A_NONE = 0,
  A_COL = 1,        // column phase done: max d, sum(invB*d) -> infeasibility test, singleton deltas
  A_STEP_MAXDY = 2, // forward product of P done: store max d^(y)
  A_STEP_DONE = 3,  // all forward products done: set up the step search
  A_SEARCH = 4,     // a search pass done: Alg. 3 replay / next pass / accept alpha
  A_UPDATE = 5,     // y, z, weights updated: sums S_P, S_C, termination test
  A_INIT_SING = 6,  // init: singleton-row value sum(invB * x)
  A_INIT_EXT = 7,   // init: shifts s_P = max y, s_C = min z
  A_INIT_W = 8,     // init: S_P, S_C, termination test at t = 0
  A_SUM = 9,        // generic: store the reduced slots in ctl->scratch
};

// Device-resident control block of one probe (one per context).
struct Ctl {
  // ---- probe constants
  double eta, sigma, eps, B, invB;     // eta, sigma = 1/(2eta) or 1/eta
  int64_t max_iter;
  int32_t pSing, cSing;                // side is the embedded singleton row
  int32_t mode;                        // 0 mixed, 1 pure packing, 2 pure covering
  int32_t tol_prose, max_evals, bisect_depth, use_graph;
  // ---- iteration state
  int64_t t;                           // completed MWU iterations
  int64_t iter_stop;                   // graph loop stops when t reaches this (benchmarks)
  int32_t status, reason;
  int32_t apply_prev, record;          // lazy x += alpha_prev d_prev pending
  double alpha_prev, alpha;            // accepted step sizes
  double sP, SP, sC, SC;               // shifts (max y / min z) and weight sums (Q4)
  double yS, dyS, zS, dzS;             // singleton-side values
  double maxd, maxdy;                  // column / step reductions
  double newsP, newsC;                 // shifts of the accepted alpha (from its search pass)
  // ---- step search (Alg. 3)
  int32_t sphase, sactive;             // phase, another pass needed
  int32_t ncand, evals;                // candidates in this pass; f evaluations this iteration
  double sa, lb, ub;                   // doubling alpha, bisection bracket
  double lb_mx, lb_mn, ok_mx, ok_mn;   // ext values of lb / the last accepted doubling alpha
  double fixed_alpha;
  double cand[MWU_MAXC], cea[MWU_MAXC], shP[MWU_MAXC], shC[MWU_MAXC];
  int32_t cmP[MWU_MAXC], cmC[MWU_MAXC];
  // ---- statistics (accumulated over the probe)
  int64_t evals_total, passes_total;
  double alpha_last;
  double scratch[MWU_SLOTS];
  // ---- CUDA graph conditional handles (0 when host-driven)
  unsigned long long h_iter, h_search;
  int32_t nan_flag, pad_;
};

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double red_identity(int op) {
  return op == OP_SUM ? 0.0 : (op == OP_MAX ? -INFINITY : INFINITY);
}
__device__ __forceinline__ double red_combine(int op, double a, double b) {
  return op == OP_SUM ? __dadd_rn(a, b) : (op == OP_MAX ? fmax(a, b) : fmin(a, b));
}

// Reduce NS per-thread values across the block and write this block's partial row.
// ops: compile-time-unknown but warp-uniform op per slot.
template <int NS>
__device__ __forceinline__ void block_partials(double (&v)[NS], const int* ops, double* part) {
  __shared__ double sh[MWU_NT / 32][MWU_SLOTS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    double a = v[s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = red_combine(ops[s], a, __shfl_down_sync(0xffffffffu, a, o));
    if (lane == 0) sh[warp][s] = a;
  }
  __syncthreads();
  if (threadIdx.x < NS) {
    const int s = threadIdx.x;
    double a = sh[0][s];
    for (int w = 1; w < MWU_NT / 32; ++w) a = red_combine(ops[s], a, sh[w][s]);
    part[(size_t)blockIdx.x * MWU_SLOTS + s] = a;
  }
}

// Returns true in the last block to finish; in that block out[0..NS) holds the grid result
// (combined over blocks 0..gridDim.x-1 in a fixed order).  Must be called by all threads.
template <int NS>
__device__ __forceinline__ bool last_block_reduce(const int* ops, const double* part,
                                                  unsigned int* counter, double (&out)[NS]) {
  __shared__ int am_last;
  __shared__ double sh2[MWU_NT][1];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  const int L = MWU_NT / NS;              // lanes per slot
  const int s = threadIdx.x % NS, k = threadIdx.x / NS;
  double a = red_identity(ops[s]);
  if (k < L)
    for (unsigned int b = k; b < gridDim.x; b += L)
      a = red_combine(ops[s], a, __ldcg(part + (size_t)b * MWU_SLOTS + s));
  sh2[threadIdx.x][0] = a;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    double r = red_identity(ops[q]);
    for (int kk = 0; kk < L; ++kk) r = red_combine(ops[q], r, sh2[kk * NS + q][0]);
    out[q] = r;
  }
  if (threadIdx.x == 0) *counter = 0u;    // ready for the next kernel on this stream
  __syncthreads();
  return true;
}

// Direction d_i = sigma * max{0, 1 - g_i/h_i} * x_i (P:279 / P:666); h_i = 0 -> 0 (Q5).
// Evaluated in the oracle's operation order; the library is built with --fmad=false so no
// multiply-add is contracted.
__device__ __forceinline__ double mwu_direction(double g, double h, double x, double sigma) {
  if (!(h > 0.0)) return 0.0;
  const double r = 1.0 - g / h;
  return (sigma * fmax(0.0, r)) * x;
}

}  // namespace mwu
