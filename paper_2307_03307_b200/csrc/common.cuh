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
#define MWU_SLOTS 50          // reduction slots per block partial (6 * MAXC + 2 Newton derivative sums)
#ifndef MWU_CT
#define MWU_CT 1024           // edges per column tile (compacted covering-row records)
#endif
#define MWU_TILE 2048         // items per seg tile (a tile loads <= 2*TILE items into smem)
#define MWU_LCH 8192          // items per chunk of a long row (deg > TILE)

namespace mwu {

constexpr int kColEdges = MWU_CT / MWU_NT;         // edges per thread per column tile
constexpr int kWarpSeg = MWU_CT / (MWU_NT / 32);   // edges (and record slots) per warp per tile

enum Status : int { ST_RUNNING = 0, ST_FEASIBLE = 1, ST_INFEASIBLE = 2, ST_ITER_LIMIT = 3 };
enum Reason : int { R_NONE = 0, R_MAXD_ZERO = 1, R_ALPHA_LT_1 = 2, R_EMPTY_COVER = 3, R_ITER_LIMIT = 4, R_MIN_Z = 5 };
enum RedOp : int { OP_SUM = 0, OP_MAX = 1, OP_MIN = 2, OP_FIRST = 3 };
// candidate evaluation modes of one side in a search pass (DESIGN.md §3 Q16)
enum CandMode : int { CM_EXPM1 = 0, CM_LSE = 1, CM_EXT = 2 };
// search phases (Alg. 3)
enum SPhase : int { SP_DOUBLE = 0, SP_BISECT = 1, SP_DONE = 2, SP_FIXED = 3, SP_TCFIX = 4,
                    SP_NEWTON = 5, SP_NBACK = 6 };   // Newton steps, its (1 - eps)^p back-off
// step rules (mwu_options.step_rule): Alg. 3, Newton, alpha = 1 (Alg. 1)
enum StepRule : int { STEP_BINARY = 0, STEP_NEWTON = 1, STEP_STANDARD = 2 };
#define MWU_NEWTON_MAX_STEPS 20     // Q35 (oracle NEWTON_MAX_STEPS)
#define MWU_NEWTON_MAX_BACKOFF 64   // Q36 (oracle NEWTON_MAX_BACKOFF)
// candidate layout of a search pass: explicit list, doubling a0*2^j, bisection grid a0 + k*delta
// PT_G16 (8 candidates): a bisection pass over the 1/16 grid lb + j (ub - lb)/16 of the bracket
// evaluating j = 1, 2, 4, 6, 8, 10, 12, 14 — the first three levels plus the most likely node of
// the fourth — from TWO transcendentals (at lb + delta and delta) and a 13-step recurrence
enum PType : int { PT_LIST = 0, PT_DOUBLE = 1, PT_GRID = 2, PT_G16 = 3 };

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
  A_COL_FAST = 10,  // fast densest column: max d, inactive covering aggregate (mzi, Vi)
  A_VI_EXACT = 11,  // exact inactive aggregate at shift mzi (rare path)
  A_STEP_DONE_C = 12,  // vcover forward product with compacted covering records: inactive
                       // aggregate (mzi, Vi), then as A_STEP_DONE
};

// Device-resident control block of one probe (one per context).
struct Ctl {
  // ---- probe constants
  double eta, sigma, eps, B, invB;     // eta, sigma = 1/(2eta) or 1/eta
  int64_t max_iter;
  int32_t pSing, cSing;                // side is the embedded singleton row
  int32_t mode;                        // 0 mixed, 1 pure packing, 2 pure covering
  int32_t tol_prose, max_evals, bisect_depth, use_graph;
  int32_t lazyC, compC;                 // covering rows of the fast densest path: z updated lazily in
                                       // the column kernel, weights v recomputed from z, S_C carried
                                       // from the accepted alpha's search pass
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
  double lb_tc, lb_sh, ok_tc, ok_sh, hi_tc, hi_sh;   // covering-side shifted sums (and their shifts)
  double acc_tc, acc_sh;               // of the accepted alpha (lazyC: S_C of the next iterate)
  int32_t vi_exact, pad4_;             // lazyC: the inactive aggregate needs the exact pass
  double mzi, Vi;                      // lazyC: inactive covering rows (d^(z) = 0): min z and
                                       // sum exp(-eta (z - mzi)) (candidate independent)
  double fixed_alpha;
  int32_t step_rule, nk;               // step rule; Newton evaluations of this iteration
  int32_t nfb, nb;                     // Newton fell back to Alg. 3; back-off factors applied
  int32_t ptype, pad2_;                // pass layout: PT_LIST, PT_DOUBLE (a0 2^j), PT_GRID (a0 + k delta)
  double pa0, pdelta;
  // doubling phase bookkeeping over exponents k (candidates 2^k, Alg. 3):
  // dk_lo = largest k known to pass (f >= 1 and no early exit), dk_hi = smallest k known to stop
  int32_t dk_lo, dk_hi, hi_exit, pad3_;
  double hi_mx, hi_mn;
  int32_t cexp[MWU_MAXC], csq[MWU_MAXC];
  double cand[MWU_MAXC], cea[MWU_MAXC], shP[MWU_MAXC], shC[MWU_MAXC];
  int32_t cmP[MWU_MAXC], cmC[MWU_MAXC];
  // ---- first-window guesses: accepted step sizes of the previous probe at the same iteration
  // index (only a choice of which candidates the first search pass evaluates)
  double aguess[32], ahist[32];
  // ---- statistics (accumulated over the probe)
  int64_t evals_total, passes_total;
  double alpha_last;
  double scratch[MWU_SLOTS];
  // ---- multi-GPU: partial phase reductions are deferred to the host-driven exchange
  int32_t world, dpending;             // ranks; a deferred reduction awaits finalize_multi
  int32_t repvars, partupd;            // variables replicated (vcover / domset); update reduction partial
  int32_t ownrows, pad_own;            // owner-partitioned packing rows (sharded bipartite matching)
  int32_t dn, daction;                 // its slot count and action
  double dslots[MWU_SLOTS];            // this rank's reduced slots
  int32_t dops[MWU_SLOTS];             // their combine ops
  // ---- CUDA graph conditional handles (0 when host-driven)
  unsigned long long h_iter, h_search;
  int32_t nan_flag, pad_;
  // ---- diagnostics: decisions within 1e-12 of their threshold (Q22) and device time by phase
  // (column, step, search, update), from %globaltimer at the end of each phase (ns)
  int64_t near_ties;
  unsigned long long tmark;
  double tph[4];
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// close the phase that ends now: the time since the previous phase end goes to phase p
__device__ __forceinline__ void phase_mark(Ctl* c, int p) {
  const unsigned long long t = globaltimer_ns();
  if (p >= 0 && c->tmark) c->tph[p] += (double)(t - c->tmark);
  c->tmark = t;
}
__device__ __forceinline__ bool near_tie(double a, double b) {
  return fabs(a - b) <= 1e-12 * fmax(fabs(a), fabs(b));
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double red_identity(int op) {
  return op == OP_SUM ? 0.0 : (op == OP_MAX ? -INFINITY : INFINITY);
}
__device__ __forceinline__ double red_combine(int op, double a, double b) {
  return op == OP_SUM ? __dadd_rn(a, b) : (op == OP_MAX ? fmax(a, b) : fmin(a, b));
}

// Reduce NS per-thread values across the block and write this block's partials into slots
// [slot0, slot0 + NS) of its partial row.  ops: warp-uniform op per slot.
template <int NS>
__device__ __forceinline__ void block_partials(const double (&v)[NS], const int* ops, double* part, int slot0 = 0) {
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
    part[(size_t)blockIdx.x * MWU_SLOTS + slot0 + s] = a;
  }
  __syncthreads();   // sh may be reused by the next call
}

// block_partials with one compile-time op for all NS slots (the search pass reduces 50 slots per
// block: with run-time ops the op switch around every shuffle round was ~40% of a small pass's
// stall samples).  Same per-slot shuffle tree and warp order as block_partials; the NS trees are
// interleaved.  slot1 >= 0: the partials are also written there.
template <int OP>
__device__ __forceinline__ double red_combine_c(double a, double b) {
  return OP == OP_SUM ? __dadd_rn(a, b) : (OP == OP_MAX ? fmax(a, b) : fmin(a, b));
}
template <int NS, int OP>
__device__ __forceinline__ void block_partials_op(const double (&v)[NS], double* part, int slot0, int slot1 = -1) {
  __shared__ double sh[MWU_NT / 32][NS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) a[s] = v[s];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int s = 0; s < NS; ++s) a[s] = red_combine_c<OP>(a[s], __shfl_down_sync(0xffffffffu, a[s], o));
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) sh[warp][s] = a[s];
  }
  __syncthreads();
  if (threadIdx.x < NS) {
    const int s = threadIdx.x;
    double r = sh[0][s];
#pragma unroll
    for (int w = 1; w < MWU_NT / 32; ++w) r = red_combine_c<OP>(r, sh[w][s]);
    part[(size_t)blockIdx.x * MWU_SLOTS + slot0 + s] = r;
    if (slot1 >= 0) part[(size_t)blockIdx.x * MWU_SLOTS + slot1 + s] = r;
  }
  __syncthreads();   // sh may be reused by the next call
}

// Returns true in the last block to finish; there res[0..nslots) (shared memory) holds the grid
// result of every slot, combined over blocks 0..gridDim.x-1 in a fixed order.  Must be called
// by all threads; ops[s] is the op of slot s.
__device__ __forceinline__ bool last_block_combine(const int* ops, int nslots, const double* part,
                                                   unsigned int* counter, double* res) {
  __shared__ int am_last;
  __shared__ double sh2[MWU_NT];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  const int L = MWU_NT / nslots;          // lanes per slot
  const int s = threadIdx.x % nslots, k = threadIdx.x / nslots;
  double a = red_identity(ops[s]);
  if (k < L) {
    // same combination order as a plain loop over b = k, k + L, ...; the loads of 8 partials are
    // issued together (a serial chain of L2 round trips was most of a small kernel's tail)
    constexpr int UB = 8;
    for (unsigned int b = k; b < gridDim.x; b += UB * L) {
      double t[UB];
#pragma unroll
      for (int i = 0; i < UB; ++i) {
        const unsigned int bb = b + i * L;
        t[i] = bb < gridDim.x ? __ldcg(part + (size_t)bb * MWU_SLOTS + s) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < UB; ++i)
        if (b + i * L < gridDim.x) a = red_combine(ops[s], a, t[i]);
    }
  }
  sh2[threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.x < nslots) {
    double r = red_identity(ops[threadIdx.x]);
    for (int kk = 0; kk < L; ++kk) r = red_combine(ops[threadIdx.x], r, sh2[kk * nslots + threadIdx.x]);
    res[threadIdx.x] = r;
  }
  if (threadIdx.x == 0) *counter = 0u;    // ready for the next kernel on this stream
  __syncthreads();
  return true;
}

// ---------------------------------------------------------------- TMA (1-D bulk copy) pipeline
// cp.async.bulk global -> shared with an mbarrier completion (the Hopper/Blackwell bulk-copy
// engine): streams contiguous row vectors into shared memory, so HBM parallelism does not
// depend on how many registers the consuming kernel needs.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// bulk copy with an L2 eviction-priority hint (streams: evict_first, so the gathered /
// scattered vertex vectors keep their L2 lines)
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 8-byte asynchronous gather global -> shared (LDGSTS): the loaded value never occupies a
// register, so a gather issued one tile ahead cannot stall the issuing warp
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

#ifndef MWU_SCH
#define MWU_SCH 1024   // rows per streamed chunk (search: 1024 x 3 stages measured 7% faster than 512 x 4)
#endif
#ifndef MWU_SST
#define MWU_SST 3      // pipeline stages
#endif

// Stream rows [0, n) of three fp64 arrays through shared memory in chunks of MWU_SCH, chunk k
// of the grid-stride sequence going to stage (it % MWU_SST).
// `it` continues across calls so mbarrier parities stay consistent.  Vectors must be allocated
// with >= 1 padding element (bulk copies move multiples of 16 bytes).  Rows go to the functor
// two at a time (f.pair), so their dependent FP64 chains interleave (c5 search 3.24 -> 3.12 ms).
template <class F>
__device__ __forceinline__ void stream_rows3(const double* A, const double* B, const double* C, int64_t n,
                                             double* buf, uint64_t* bars, uint32_t& it, F&& f) {
  const int64_t nchunks = (n + MWU_SCH - 1) / MWU_SCH;
  const int64_t first = blockIdx.x;
  const int64_t mine = (nchunks > first) ? (nchunks - first + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](int64_t k, uint32_t slot) {
    const int64_t ch = first + k * (int64_t)gridDim.x;
    const int64_t r0 = ch * MWU_SCH;
    const int64_t rows = (n - r0 < MWU_SCH) ? (n - r0) : MWU_SCH;
    const uint32_t bytes = (uint32_t)(((rows * 8) + 15) & ~15ll);
    double* s = buf + (size_t)slot * 3 * MWU_SCH;
    mbar_expect_tx(&bars[slot], 3 * bytes);
    tma_load_1d(s, A + r0, bytes, &bars[slot]);
    tma_load_1d(s + MWU_SCH, B + r0, bytes, &bars[slot]);
    tma_load_1d(s + 2 * MWU_SCH, C + r0, bytes, &bars[slot]);
  };
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < mine && k < MWU_SST; ++k) issue(k, (it + (uint32_t)k) % MWU_SST);
  for (int64_t k = 0; k < mine; ++k) {
    const uint32_t slot = it % MWU_SST, parity = (it / MWU_SST) & 1u;
    mbar_wait(&bars[slot], parity);
    const int64_t r0 = (first + k * (int64_t)gridDim.x) * MWU_SCH;
    const int rows = (int)((n - r0 < MWU_SCH) ? (n - r0) : MWU_SCH);
    const double* s = buf + (size_t)slot * 3 * MWU_SCH;
    // two rows per call (their dependent chains interleave); an absent second row is the
    // neutral (+-inf, 0, 0) of the functor's side (F::kAbsent)
    for (int r = threadIdx.x; r < rows; r += 2 * blockDim.x) {
      const int r1 = r + blockDim.x;
      if (r1 < rows) f.pair(s[r], s[MWU_SCH + r], s[2 * MWU_SCH + r], s[r1], s[MWU_SCH + r1], s[2 * MWU_SCH + r1]);
      else f.pair(s[r], s[MWU_SCH + r], s[2 * MWU_SCH + r], std::remove_reference_t<F>::kAbsent, 0.0, 0.0);
    }
    __syncthreads();                                   // everyone is done with this slot
    if (threadIdx.x == 0 && k + MWU_SST < mine) issue(k + MWU_SST, slot);
    ++it;
  }
}

// ---------------------------------------------------------------- L2 eviction-priority hints
// Streams (read or written once per sweep) are marked evict_first, so the small vertex vectors
// that are gathered / scattered at random (u, d^(y): tens of MB) keep their L2 lines (evict_last).
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldh(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldh_nc(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int ldh_nc(const int* a, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ldh_nc(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ldh2(const double2* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void sth(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void sth2(double2* a, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void redh_add(double* a, double v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
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
