// kernels.cuh — sm_100a kernels of the MWU hot path (Alg. 2 + Alg. 3 of arXiv 2307.03307).
//
// Phase kernels of one MWU iteration, each ending with a last-block finalize:
//   column  : x += alpha_prev d_prev (lazy P:677), g = P^T w_p, h = C^T w_c,
//             d = sigma max{0, 1 - g/h} x, reductions max d and sum(d)/M
//   step    : d^(y) = P d, d^(z) = C d, max d^(y)
//   search  : per candidate alpha: sum w expm1(.) or shifted exp sums, max(y+a dy), min(z+a dz)
//             (Q16) for up to MWU_MAXC candidates per HBM pass; the last block
//             replays Alg. 3 and either accepts alpha or stages the next pass
//   update  : y += alpha d^(y), z += alpha d^(z) fused with the new shifted weights
//             u = exp(eta(y - s_P)), v = exp(-eta(z - s_C)) and their sums (Q4)
// Sparse structure is never materialised as an incidence matrix: M, O, W are applied from
// the edge list and a vertex -> incident-slot CSR.  Segmented sums run on a
// tile plan (TILE items per tile staged in shared memory, long rows split into chunks) so
// power-law degree distributions load-balance and results stay deterministic.
#pragma once
#include "common.cuh"

namespace mwu {

// =====================================================================================
// CUDA graph conditional helper (device side)
// =====================================================================================
__device__ __forceinline__ void set_cond(unsigned long long h, unsigned int v) {
  if (h) cudaGraphSetConditional((cudaGraphConditionalHandle)h, v);
}

// =====================================================================================
// Search controller: Alg. 3 replayed over the candidates evaluated in one HBM pass
// =====================================================================================
// Result slots of a search pass, per candidate j (R_*(j) index into the reduced vector):
//   EP  sum_i u_i expm1(eta a dy_i)            (P side, expm1 form)
//   LP  sum_i exp(eta (y_i + a dy_i - shP_j))  (P side, shifted log-sum-exp form)
//   MX  max_i (y_i + a dy_i)
//   EC  sum_i v_i expm1(-eta a dz_i)           (C side, expm1 form)
//   TC  sum_i exp(-eta (z_i + a dz_i - shC_j)) (C side, shifted form; shC = s_C in DOUBLE/GRID
//                                               passes, where it equals sum_i v_i e^{-eta a dz_i})
//   MN  min_i (z_i + a dz_i)
#define R_EP(j) (j)
#define R_LP(j) (MWU_MAXC + (j))
#define R_MX(j) (2 * MWU_MAXC + (j))
#define R_EC(j) (3 * MWU_MAXC + (j))
#define R_TC(j) (4 * MWU_MAXC + (j))
#define R_MN(j) (5 * MWU_MAXC + (j))

__device__ void stage_modes(Ctl* c, int j) {
  c->cea[j] = c->eta * c->cand[j];
  if (c->pSing) c->cmP[j] = CM_EXT;
  else if (c->cea[j] * c->maxdy <= 700.0) c->cmP[j] = CM_EXPM1;                 // Q16 branch
  else { c->cmP[j] = CM_LSE; c->shP[j] = c->sP + c->cand[j] * c->maxdy; }        // >= max(y + a dy)
  c->cmC[j] = c->cSing ? CM_EXT : CM_EXPM1;
  c->shC[j] = c->sC;
}

// Doubling candidates alpha = 2^k for ascending exponents k[0..n) (alpha <- 2 alpha from 1).
// Rows derive 2^k[j] from 2^k[j-1] by csq[j] = k[j]-k[j-1] exact squarings of expm1 / exp.
__device__ void stage_double_exps(Ctl* c, const int* ks, int n) {
  for (int j = 0; j < n; ++j) {
    c->cexp[j] = ks[j];
    c->csq[j] = j ? ks[j] - ks[j - 1] : 0;
    c->cand[j] = ldexp(1.0, ks[j]);
    stage_modes(c, j);
  }
  c->ncand = n;
  c->ptype = PT_DOUBLE;
  c->pa0 = c->cand[0];
}

// Next exponents to evaluate given what is known (dk_lo passes, dk_hi stops).  By Prop. 4.2
// (f decreasing in alpha) and the monotonicity of min(z + alpha d^(z)), every k below a
// passing exponent passes and every k above a stopping exponent is never reached, so Alg. 3's
// sequential outcome is decided by the first stopping exponent; the candidates are chosen to find
// it in few passes (galloping up, then splitting the unknown gap).
__device__ void stage_double_next(Ctl* c) {
  int ks[MWU_MAXC], n = 0;
  if (c->dk_hi >= (1 << 20)) {                       // no stop seen yet: gallop upward
    const int offs[4] = {1, 2, 4, 8};
    for (int i = 0; i < MWU_MAXC && i < 4; ++i) ks[n++] = c->dk_lo + offs[i];
  } else {                                           // unknown exponents dk_lo+1 .. dk_hi-1
    const int lo = c->dk_lo + 1, hi = c->dk_hi - 1, cnt = hi - lo + 1;
    if (cnt <= MWU_MAXC) {
      for (int k = lo; k <= hi; ++k) ks[n++] = k;
    } else {
      for (int i = 0; i < MWU_MAXC; ++i) {
        const int k = lo + ((i + 1) * cnt) / (MWU_MAXC + 1);
        if (n == 0 || k > ks[n - 1]) ks[n++] = k;
      }
    }
  }
  stage_double_exps(c, ks, n);
}

// First pass of an iteration: a window of exponents around the previous accepted step size
// (the Table 3 caption's observation that consecutive step sizes are close, used
// here only to choose which candidates to evaluate, not to change Alg. 3's result).
__device__ void stage_double_first(Ctl* c) {
  c->dk_lo = -1;
  c->dk_hi = 1 << 20;
  int kg = 1;
  if (c->t > 0 && c->alpha_prev >= 1.0) kg = ilogb(c->alpha_prev);
  int k0 = kg - 1 < 0 ? 0 : kg - 1;
  int ks[MWU_MAXC];
  for (int j = 0; j < MWU_MAXC; ++j) ks[j] = k0 + j;
  stage_double_exps(c, ks, MWU_MAXC);
}

__device__ void stage_bisect(Ctl* c) {          // the 2^L - 1 midpoints of L bisection levels
  const int Lmax = (MWU_MAXC >= 7) ? 3 : ((MWU_MAXC >= 3) ? 2 : 1);
  const int L = c->bisect_depth < 1 ? 1 : (c->bisect_depth > Lmax ? Lmax : c->bisect_depth);
  const int n = (1 << L) - 1;
  // midpoints computed exactly as the sequential loop computes them, stored in ascending order
  double lo[8], hi[8], nlo[8], nhi[8], vals[8];
  int ni = 1, nv = 0;
  lo[0] = c->lb; hi[0] = c->ub;
  for (int lev = 0; lev < L; ++lev) {
    int nn = 0;
    for (int k = 0; k < ni; ++k) {
      const double m = (lo[k] + hi[k]) / 2.0;
      vals[nv++] = m;
      nlo[nn] = lo[k]; nhi[nn] = m; ++nn;
      nlo[nn] = m; nhi[nn] = hi[k]; ++nn;
    }
    for (int k = 0; k < nn; ++k) { lo[k] = nlo[k]; hi[k] = nhi[k]; }
    ni = nn;
  }
  for (int i = 1; i < nv; ++i)            // insertion sort (<= 7 values)
    for (int k = i; k > 0 && vals[k - 1] > vals[k]; --k) { const double t = vals[k]; vals[k] = vals[k - 1]; vals[k - 1] = t; }
  for (int k = 0; k < n; ++k) { c->cand[k] = vals[k]; stage_modes(c, k); }
  c->ncand = n;
  c->ptype = PT_GRID;
  c->pa0 = c->lb;
  c->pdelta = (c->ub - c->lb) / (double)(1 << L);
}

// eta*Psi and eta*Phi of candidate j (P:719-720, P:322 singletons, Q12, Q16).  The shifted
// forms use the pass's shift sh: eta*Psi = eta(sh - s_P) + log(sum exp(eta(t - sh))) - log S_P,
// eta*Phi = eta(sh - s_C) - log(sum exp(-eta(t - sh))) + log S_C, identical in value to the
// oracle's max/min-shifted forms; a sum that underflowed asks for an exact-shift re-pass.
__device__ void eval_cand(const Ctl* c, int j, const double* res, double& psi, double& phi,
                          int& needP, int& needC) {
  const double ea = c->cea[j];
  needP = needC = 0;
  psi = phi = 0.0;
  if (c->pSing) psi = ea * c->dyS;
  else if (c->cmP[j] == CM_EXPM1) psi = log1p(res[R_EP(j)] / c->SP);
  else if (c->cmP[j] == CM_LSE && res[R_LP(j)] > 1e-280)
    psi = c->eta * (c->shP[j] - c->sP) + log(res[R_LP(j)]) - log(c->SP);
  else needP = 1;
  if (c->cSing) phi = ea * c->dzS;
  else {
    const double e = (c->cmC[j] == CM_EXPM1) ? res[R_EC(j)] / c->SC : -1.0;
    if (c->cmC[j] == CM_EXPM1 && e >= -0.5) phi = -log1p(e);
    else if (c->cmC[j] != CM_EXT && res[R_TC(j)] > 1e-280)
      phi = c->eta * (c->shC[j] - c->sC) - log(res[R_TC(j)]) + log(c->SC);
    else needC = 1;
  }
}

__device__ __forceinline__ double cand_mx(const Ctl* c, int j, const double* res) {
  return c->pSing ? (c->yS + c->cand[j] * c->dyS) : res[R_MX(j)];
}
__device__ __forceinline__ double cand_mn(const Ctl* c, int j, const double* res) {
  return c->cSing ? (c->zS + c->cand[j] * c->dzS) : res[R_MN(j)];
}

__device__ void accept_alpha(Ctl* c, double a, double mx, double mn) {
  c->alpha = a;
  c->newsP = mx;
  c->newsC = mn;
  c->sphase = SP_DONE;
  c->sactive = 0;
  if (a < 1.0) { c->status = ST_INFEASIBLE; c->reason = R_ALPHA_LT_1; }
}

// res layout: see R_* above
__device__ void search_controller(Ctl* c, const double* res) {
  c->passes_total++;
  if (c->sphase == SP_FIXED) { accept_alpha(c, c->cand[0], cand_mx(c, 0, res), cand_mn(c, 0, res)); return; }
  if (c->sphase == SP_DOUBLE) {
    // classify the evaluated exponents (ascending): pass = f >= 1 and min(z + a dz) < 1
    int lse_j = -1;
    for (int j = 0; j < c->ncand; ++j) {
      const int k = c->cexp[j];
      if (k <= c->dk_lo || k >= c->dk_hi) continue;             // outcome already implied
      double psi, phi; int nP, nC;
      eval_cand(c, j, res, psi, phi, nP, nC);
      if (nP || nC) { if (lse_j < 0) lse_j = j; continue; }
      const double mxj = cand_mx(c, j, res), mnj = cand_mn(c, j, res);
      const bool ok = phi >= psi;                                  // eq:b4b_conv
      if (ok && mnj < 1.0) { c->dk_lo = k; c->ok_mx = mxj; c->ok_mn = mnj; }
      else { c->dk_hi = k; c->hi_exit = ok ? 1 : 0; c->hi_mx = mxj; c->hi_mn = mnj; }
    }
    if (lse_j >= 0 && c->cexp[lse_j] > c->dk_lo && c->cexp[lse_j] < c->dk_hi) {
      // Q16: re-evaluate this exponent with the exact max / min shift
      double psi, phi; int nP, nC;
      eval_cand(c, lse_j, res, psi, phi, nP, nC);
      const double mxj = cand_mx(c, lse_j, res), mnj = cand_mn(c, lse_j, res);
      const int k = c->cexp[lse_j];
      const int keepP = c->cmP[lse_j];
      const double kshP = c->shP[lse_j];
      c->cand[0] = ldexp(1.0, k); c->cea[0] = c->eta * c->cand[0]; c->cexp[0] = k; c->csq[0] = 0;
      c->cmP[0] = c->pSing ? CM_EXT : (nP ? CM_LSE : keepP); c->shP[0] = nP ? mxj : kshP;
      c->cmC[0] = c->cSing ? CM_EXT : (nC ? CM_LSE : CM_EXPM1); c->shC[0] = nC ? mnj : c->sC;
      c->ncand = 1; c->ptype = PT_LIST; c->sactive = 1;
      return;
    }
    // the literal loop stops at the first stopping exponent k* = dk_hi (alpha = 2^k*) after k*+1
    // evaluations; the cap max_evals stops it earlier at alpha = 2^(max_evals-1)
    const int cap_k = c->max_evals - 1;
    if (c->dk_lo >= cap_k || (c->dk_hi == c->dk_lo + 1 && c->dk_hi > cap_k)) {
      c->evals = c->max_evals; c->evals_total += c->max_evals;
      if (c->dk_lo == cap_k) { accept_alpha(c, ldexp(1.0, cap_k), c->ok_mx, c->ok_mn); return; }
      c->sphase = SP_FIXED; c->ncand = 1; c->cand[0] = ldexp(1.0, cap_k); c->ptype = PT_LIST;   // shifts only
      c->cea[0] = c->eta * c->cand[0]; c->cmP[0] = CM_EXT; c->cmC[0] = CM_EXT; c->sactive = 1;
      return;
    }
    if (c->dk_hi == c->dk_lo + 1) {
      const int ks = c->dk_hi;
      c->evals = ks + 1; c->evals_total += ks + 1;
      if (c->hi_exit) { accept_alpha(c, ldexp(1.0, ks), c->hi_mx, c->hi_mn); return; }
      c->sphase = SP_BISECT; c->lb = ldexp(1.0, ks - 1); c->ub = ldexp(1.0, ks);
      c->lb_mx = c->ok_mx; c->lb_mn = c->ok_mn;
    } else {
      stage_double_next(c);
      c->sactive = 1;
      return;
    }
  }
  for (int guard = 0; guard < 4096; ++guard) {
    double need;
    {
      const double thr = c->tol_prose ? c->eps : (1.0 - c->eps);         // Q9
      if (!((c->ub - c->lb) > thr * c->lb && c->evals < c->max_evals)) {
        accept_alpha(c, c->lb, c->lb_mx, c->lb_mn);                         // return lb
        return;
      }
      need = (c->lb + c->ub) / 2.0;
    }
    int j = -1;
    for (int k = 0; k < c->ncand; ++k) if (c->cand[k] == need) { j = k; break; }
    if (j < 0) {                                                            // not evaluated yet
      stage_bisect(c);
      c->sactive = 1;
      return;
    }
    double psi, phi; int nP, nC;
    eval_cand(c, j, res, psi, phi, nP, nC);
    const double mxj = cand_mx(c, j, res), mnj = cand_mn(c, j, res);
    if (nP || nC) {                          // Q16 shifted form with the exact max / min shift
      const int keepP = c->cmP[j], keepC = c->cmC[j];
      const double kshP = c->shP[j];
      c->cand[0] = need; c->cea[0] = c->eta * need;
      c->cmP[0] = c->pSing ? CM_EXT : (nP ? CM_LSE : keepP); c->shP[0] = nP ? mxj : kshP;
      c->cmC[0] = c->cSing ? CM_EXT : (nC ? CM_LSE : CM_EXPM1); c->shC[0] = nC ? mnj : c->sC;
      c->ncand = 1;
      c->ptype = PT_LIST;
      c->sactive = 1;
      return;
    }
    const bool ok = phi >= psi;                                             // eq:b4b_conv
    c->evals++;
    c->evals_total++;
    if (ok) { c->lb = need; c->lb_mx = mxj; c->lb_mn = mnj; } else { c->ub = need; }
  }
  c->status = ST_INFEASIBLE; c->reason = R_ALPHA_LT_1; c->sactive = 0;   // unreachable guard
}

// =====================================================================================
// Finalize: control logic run by thread 0 of the last block of a phase kernel
// =====================================================================================
__device__ void finalize(Ctl* c, int action, const double* r) {
  switch (action) {
    case A_COL: {
      c->apply_prev = 0;
      c->maxd = r[0];
      if (c->pSing) c->dyS = r[1];                 // d^(y) = (1/M) 1^T d   (pure covering)
      if (c->cSing) c->dzS = r[1];                 // d^(z) = (1/M) 1^T d   (pure packing)
      if (!(r[0] > 0.0)) { c->status = ST_INFEASIBLE; c->reason = R_MAXD_ZERO; }
      break;
    }
    case A_STEP_MAXDY:
      c->maxdy = r[0];
      break;
    case A_STEP_DONE:
    case A_STEP_DONE + 100: {
      if (action == A_STEP_DONE + 100) c->maxdy = r[0];
      c->evals = 0;
      if (c->fixed_alpha > 0.0) {
        c->sphase = SP_FIXED; c->ncand = 1; c->cand[0] = c->fixed_alpha; c->ptype = PT_LIST;
        c->cea[0] = c->eta * c->fixed_alpha; c->cmP[0] = CM_EXT; c->cmC[0] = CM_EXT;
      } else {
        c->sphase = SP_DOUBLE; c->sa = 1.0;                                 // alpha <- 1
        stage_double_first(c);
      }
      c->sactive = 1;
      set_cond(c->h_search, 1u);
      break;
    }
    case A_SEARCH:
      search_controller(c, r);
      set_cond(c->h_search, c->sactive ? 1u : 0u);
      break;
    case A_UPDATE: {
      c->t++;
      c->alpha_last = c->alpha; c->alpha_prev = c->alpha; c->apply_prev = 1;
      if (c->pSing) { c->yS = c->yS + c->alpha * c->dyS; c->sP = c->yS; c->SP = 1.0; }
      else { c->sP = c->newsP; c->SP = r[0]; }
      if (c->cSing) { c->zS = c->zS + c->alpha * c->dzS; c->sC = c->zS; c->SC = 1.0; }
      else { c->sC = c->newsC; c->SC = r[1]; }
      if (!(isfinite(c->SP) && isfinite(c->SC) && c->SP > 0.0 && c->SC > 0.0)) {
        c->nan_flag = 1; c->status = ST_INFEASIBLE;
      } else if (c->sC >= 1.0) { c->status = ST_FEASIBLE; c->reason = R_MIN_Z; }   // Q6
      else if (c->t >= c->max_iter) { c->status = ST_ITER_LIMIT; c->reason = R_ITER_LIMIT; }
      set_cond(c->h_iter, (c->status == ST_RUNNING && c->t < c->iter_stop) ? 1u : 0u);
      break;
    }
    case A_INIT_SING:
      if (c->pSing) c->yS = r[0];
      if (c->cSing) c->zS = r[0];
      break;
    case A_INIT_EXT:
      c->sP = c->pSing ? c->yS : r[0];
      c->sC = c->cSing ? c->zS : r[1];
      break;
    case A_INIT_W: {
      c->SP = c->pSing ? 1.0 : r[0];
      c->SC = c->cSing ? 1.0 : r[1];
      if (!(isfinite(c->SP) && isfinite(c->SC) && c->SP > 0.0 && c->SC > 0.0)) {
        c->nan_flag = 1; c->status = ST_INFEASIBLE;
      }
      if (c->status == ST_RUNNING) {
        if (c->sC >= 1.0) { c->status = ST_FEASIBLE; c->reason = R_MIN_Z; }
        else if (c->t >= c->max_iter) { c->status = ST_ITER_LIMIT; c->reason = R_ITER_LIMIT; }
      }
      break;
    }
    case A_SUM:
      for (int s = 0; s < MWU_SLOTS; ++s) c->scratch[s] = r[s];
      break;
    default:
      break;
  }
}

// Standard epilogue of a reducing kernel: block partials -> last block -> finalize.
template <int NS>
__device__ __forceinline__ void reduce_and_finalize(double (&acc)[NS], const int* ops, double* part,
                                                    unsigned int* counter, Ctl* c, int action) {
  block_partials<NS>(acc, ops, part);
  double out[NS];
  if (last_block_reduce<NS>(ops, part, counter, out)) {
    if (threadIdx.x == 0) {
      double r[MWU_SLOTS];
      for (int s = 0; s < MWU_SLOTS; ++s) r[s] = (s < NS) ? out[s] : 0.0;
      finalize(c, action, r);
    }
  }
}

// =====================================================================================
// Segmented row sums over a CSR-like structure (rows -> items)
// =====================================================================================
struct SegView {
  const int64_t* rowptr;    // [nrows+1]
  int64_t nrows;
  const uint32_t* idx;      // [nnz] item -> index into the gathered vector (>> shift)
  const double* val;        // [nnz] or nullptr (all ones)
  const int64_t* tile_row;  // [ntiles+1] first row starting in [k*TILE, (k+1)*TILE)
  int64_t ntiles;
  const int64_t* long_rows; // [nlong] rows with more than TILE items
  const int64_t* long_cptr; // [nlong+1] chunk prefix
  int64_t nlong, nchunks;
  double* chunk_sum;        // [nchunks]
};

// Item value: val[k] * vec[idx[k] >> shift]  (or scale * vec[..] / vec[..]), the oracle's
// per-term product order (scipy: data[k] * x[col]).
struct ItemGather {
  const uint32_t* idx;
  const double* val;
  const double* vec;
  int shift;
  const double* scale_ptr;  // per-probe scale (1/D of O/D) read from the control block
  __device__ __forceinline__ double load_scale() const { return scale_ptr ? *scale_ptr : 1.0; }
  __device__ __forceinline__ double operator()(int64_t k, double scale) const {
    double v = __ldg(vec + (__ldg(idx + k) >> shift));
    if (val) v = __ldg(val + k) * v;
    else if (scale_ptr) v = scale * v;
    return v;
  }
};

// Long rows, phase 1: chunk sums (one block per chunk, grid-stride).
template <class Item>
__global__ void __launch_bounds__(MWU_NT) seg_long_chunks(SegView sv, Item item, const Ctl* c) {
  if (c->status != ST_RUNNING) return;
  __shared__ double sh[MWU_NT / 32];
  const double scale = item.load_scale();
  for (int64_t ch = blockIdx.x; ch < sv.nchunks; ch += gridDim.x) {
    // find the long row owning chunk ch (binary search in long_cptr)
    int64_t lo = 0, hi = sv.nlong - 1;
    while (lo < hi) { int64_t mid = (lo + hi + 1) >> 1; if (sv.long_cptr[mid] <= ch) lo = mid; else hi = mid - 1; }
    const int64_t row = sv.long_rows[lo];
    const int64_t k0 = sv.rowptr[row] + (ch - sv.long_cptr[lo]) * (int64_t)MWU_LCH;
    const int64_t k1 = min(k0 + (int64_t)MWU_LCH, sv.rowptr[row + 1]);
    double a = 0.0;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += MWU_NT) a += item(k, scale);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < MWU_NT / 32; ++w) s += sh[w];
      sv.chunk_sum[ch] = s;
    }
    __syncthreads();
  }
}

// Main segmented kernel: short rows by tiles staged in shared memory, then long rows from
// their chunk sums; each complete row goes through the epilogue Ep, whose per-thread
// reductions are combined deterministically and finalized by the last block.
template <class Item, class Ep>
__global__ void __launch_bounds__(MWU_NT) seg_main(SegView sv, Item item, Ep ep, Ctl* c, double* part,
                                                   unsigned int* counter, int action) {
  if (c->status != ST_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && ep.kind_step) set_cond(c->h_search, 0u);
    return;
  }
  __shared__ double vals[2 * MWU_TILE];
  int ops[Ep::NS];
  double acc[Ep::NS];
#pragma unroll
  for (int s = 0; s < Ep::NS; ++s) { ops[s] = Ep::op(s); acc[s] = red_identity(ops[s]); }
  const double scale = item.load_scale();
  const int lane = threadIdx.x & 31;
  for (int64_t tile = blockIdx.x; tile < sv.ntiles; tile += gridDim.x) {
    const int64_t r0 = sv.tile_row[tile];
    int64_t r1 = sv.tile_row[tile + 1];
    if (r1 > r0 && sv.rowptr[r1] - sv.rowptr[r1 - 1] > MWU_TILE) --r1;   // trailing long row
    const int64_t R = r1 - r0;
    if (R <= 0) continue;
    const int64_t i0 = sv.rowptr[r0];
    const int64_t nit = sv.rowptr[r1] - i0;                              // <= 2*TILE
    // stage item values (coalesced index loads, independent gathers)
#pragma unroll 8
    for (int64_t j = threadIdx.x; j < nit; j += MWU_NT) vals[j] = item(i0 + j, scale);
    __syncthreads();
    // group size: power of two ~ average row length, 1..32
    const int64_t avg = (nit + R - 1) / R;
    int G = 1;
    while (G < 32 && G < avg) G <<= 1;
    const int groups = MWU_NT / G;
    const int gid = threadIdx.x / G, gl = threadIdx.x % G;
    for (int64_t base = 0; base < R; base += groups) {
      const int64_t rr = base + gid;
      double s = 0.0;
      int64_t row = r0 + rr;
      if (rr < R) {
        const int64_t a = sv.rowptr[row] - i0, b = sv.rowptr[row + 1] - i0;
        for (int64_t k = a + gl; k < b; k += G) s += vals[k];
      }
      for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, G);
      if (rr < R && gl == 0) ep(row, s, acc);
    }
    __syncthreads();
  }
  // long rows: one warp per row sums its chunk sums in order
  const int warp_global = (blockIdx.x * MWU_NT + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * MWU_NT) >> 5;
  for (int64_t l = warp_global; l < sv.nlong; l += nwarps) {
    const int64_t c0 = sv.long_cptr[l], c1 = sv.long_cptr[l + 1];
    double s = 0.0;
    for (int64_t q = c0 + lane; q < c1; q += 32) s += __ldcg(sv.chunk_sum + q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) ep(sv.long_rows[l], s, acc);
  }
  reduce_and_finalize<Ep::NS>(acc, ops, part, counter, c, action);
}

// ---------------------------------------------------------------- seg epilogues
// Forward product row: out[row] = sum; reduce max (max d^(y) for Q16's expm1 validity).
struct EpOut {
  static constexpr int NS = 1;
  static __device__ __forceinline__ int op(int) { return OP_MAX; }
  double* out;
  int kind_step;
  __device__ __forceinline__ void operator()(int64_t row, double s, double (&acc)[1]) const {
    out[row] = s;
    acc[0] = fmax(acc[0], s);
  }
};

// Store g_i = (P^T u)_i / S_P (first column pass of a mixed CSR instance).
struct EpStoreG {
  static constexpr int NS = 1;
  static __device__ __forceinline__ int op(int) { return OP_SUM; }
  double* g;
  const Ctl* c;
  int kind_step;
  __device__ __forceinline__ void operator()(int64_t row, double s, double (&acc)[1]) const {
    g[row] = s / c->SP;
  }
};

// Column epilogue: row = variable i.  s_is_h: the row sum is (C^T v)_i (h = s / S_C) and g
// comes from gtmp (mixed) or the singleton (1/M); else s is (P^T u)_i (g = s / S_P) and h is
// the singleton's 1/M.  Applies the lazy x update, writes d, reduces max d and sum(d/M).
struct EpColumn {
  static constexpr int NS = 2;
  static __device__ __forceinline__ int op(int s) { return s == 0 ? OP_MAX : OP_SUM; }
  double* x;
  double* d;
  const double* gtmp;
  double* gdbg;
  double* hdbg;
  const Ctl* c;
  int s_is_h;
  int kind_step;
  __device__ __forceinline__ void operator()(int64_t i, double s, double (&acc)[2]) const {
    double xi = x[i];
    if (c->apply_prev) { xi = xi + c->alpha_prev * d[i]; x[i] = xi; }   // P:677 (lazy)
    double g, h;
    if (s_is_h) { h = s / c->SC; g = gtmp ? gtmp[i] : c->invB; }
    else { g = s / c->SP; h = c->invB; }
    const double di = mwu_direction(g, h, xi, c->sigma);
    d[i] = di;
    if (gdbg) { gdbg[i] = g; hdbg[i] = h; }
    acc[0] = fmax(acc[0], di);
    acc[1] += c->invB * di;
  }
};

// =====================================================================================
// Edge-parallel kernels of the implicit graph operators
// =====================================================================================
// MATCH / BMATCH column (P = M, C = (1/M)1^T): g_e = w_p[r(src)] + w_p[r(dst)] (M^T),
// h_e = 1/M, d_e; lazy x update; reduce max d, sum(d/M).
__global__ void __launch_bounds__(MWU_NT, 2) col_match(int64_t E, const int32_t* __restrict__ srow,
                                                    const int32_t* __restrict__ drow, const double* __restrict__ u,
                                                    double* __restrict__ x, double* __restrict__ d,
                                                    double* gdbg, double* hdbg, Ctl* c, double* part,
                                                    unsigned int* counter) {
  if (c->status != ST_RUNNING) return;
  const double rSP = 1.0 / c->SP, invB = c->invB, sigma = c->sigma, ap = c->alpha_prev;
  const int apply = c->apply_prev;
  double acc[2] = {-INFINITY, 0.0};
  constexpr int U = 2;   // edges per thread per trip: all independent loads issued before use
  const int64_t stride = (int64_t)gridDim.x * MWU_NT;
  for (int64_t e0 = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e0 < E; e0 += U * stride) {
    double xe[U], dp[U], us[U], ud[U];
    int32_t sr[U], dr[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = e0 + k * stride;
      if (e < E) {
        xe[k] = x[e];
        dp[k] = apply ? d[e] : 0.0;
        sr[k] = __ldg(srow + e);
        dr[k] = __ldg(drow + e);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (e0 + k * stride < E) { us[k] = __ldg(u + sr[k]); ud[k] = __ldg(u + dr[k]); }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = e0 + k * stride;
      if (e >= E) break;
      if (apply) { xe[k] = xe[k] + ap * dp[k]; x[e] = xe[k]; }   // lazy x += alpha d
      const double g = us[k] * rSP + ud[k] * rSP;                 // M^T w_p
      const double de = mwu_direction(g, invB, xe[k], sigma);
      d[e] = de;
      if (gdbg) { gdbg[e] = g; hdbg[e] = invB; }
      acc[0] = fmax(acc[0], de);
      acc[1] += invB * de;
    }
  }
  const int ops[2] = {OP_MAX, OP_SUM};
  reduce_and_finalize<2>(acc, ops, part, counter, c, A_COL);
}

// DENSEST column (P = O/D, C = W): for edge e, slots s = 2e+b: g_s = (1/D) w_p[r_b] (O^T),
// h_s = w_c[e] (W^T), d_s (sigma = 1/(2 eta)), and d^(z)_e = d_2e + d_2e+1 (W d) fused.
__global__ void __launch_bounds__(MWU_NT, 2) col_densest(int64_t E, const int32_t* __restrict__ srow,
                                                      const int32_t* __restrict__ drow, const double* __restrict__ u,
                                                      const double* __restrict__ v, double* __restrict__ x,
                                                      double* __restrict__ d, double* __restrict__ dz,
                                                      double* gdbg, double* hdbg, Ctl* c, double* part,
                                                      unsigned int* counter) {
  if (c->status != ST_RUNNING) return;
  const double rSP = 1.0 / c->SP, rSC = 1.0 / c->SC, invD = c->invB, sigma = c->sigma, ap = c->alpha_prev;
  const int apply = c->apply_prev;
  double acc[2] = {-INFINITY, 0.0};
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* d2 = reinterpret_cast<double2*>(d);
  constexpr int U = 2;   // edges per thread per trip: all independent loads issued before use
  const int64_t stride = (int64_t)gridDim.x * MWU_NT;
  for (int64_t e0 = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e0 < E; e0 += U * stride) {
    double2 xe[U], dp[U];
    double vv[U], us[U], ud[U];
    int32_t sr[U], dr[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = e0 + k * stride;
      if (e < E) {
        xe[k] = x2[e];
        dp[k] = apply ? d2[e] : make_double2(0.0, 0.0);
        vv[k] = __ldg(v + e);
        sr[k] = __ldg(srow + e);
        dr[k] = __ldg(drow + e);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (e0 + k * stride < E) { us[k] = __ldg(u + sr[k]); ud[k] = __ldg(u + dr[k]); }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = e0 + k * stride;
      if (e >= E) break;
      if (apply) {                                               // lazy x += alpha d
        xe[k].x = xe[k].x + ap * dp[k].x;
        xe[k].y = xe[k].y + ap * dp[k].y;
        x2[e] = xe[k];
      }
      const double h = vv[k] * rSC;
      const double g0 = invD * (us[k] * rSP);
      const double g1 = invD * (ud[k] * rSP);
      double2 de;
      de.x = mwu_direction(g0, h, xe[k].x, sigma);
      de.y = mwu_direction(g1, h, xe[k].y, sigma);
      d2[e] = de;
      dz[e] = de.x + de.y;
      if (gdbg) { gdbg[2 * e] = g0; gdbg[2 * e + 1] = g1; hdbg[2 * e] = h; hdbg[2 * e + 1] = h; }
      acc[0] = fmax(acc[0], fmax(de.x, de.y));
    }
  }
  const int ops[2] = {OP_MAX, OP_SUM};
  reduce_and_finalize<2>(acc, ops, part, counter, c, A_COL);
}

// VCOVER forward product (C = M^T): out_e = in[src_e] + in[dst_e] (d^(z) or z at init).
__global__ void __launch_bounds__(MWU_NT) edge_sum(int64_t E, const int32_t* __restrict__ src,
                                                   const int32_t* __restrict__ dst, const double* __restrict__ in,
                                                   double* __restrict__ out, Ctl* c, double* part,
                                                   unsigned int* counter, int action) {
  if (c->status != ST_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && action == A_STEP_DONE) set_cond(c->h_search, 0u);
    return;
  }
  double acc[1] = {-INFINITY};
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT) {
    const double s = __ldg(in + __ldg(src + e)) + __ldg(in + __ldg(dst + e));
    out[e] = s;
    acc[0] = fmax(acc[0], s);
  }
  const int ops[1] = {OP_MAX};
  reduce_and_finalize<1>(acc, ops, part, counter, c, action);
}

// DENSEST init: z_e = x_2e + x_2e+1 (W x).
__global__ void __launch_bounds__(MWU_NT) pair_sum(int64_t E, const double* __restrict__ in, double* __restrict__ out,
                                                   const Ctl* c) {
  if (c->status != ST_RUNNING) return;
  const double2* in2 = reinterpret_cast<const double2*>(in);
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT) {
    const double2 a = in2[e];
    out[e] = a.x + a.y;
  }
}

// =====================================================================================
// Row kernels: search pass and update (P rows then C rows as one index space)
// =====================================================================================
constexpr size_t kSearchSmem = (size_t)MWU_SST * 3 * MWU_SCH * sizeof(double);

// One HBM pass evaluating the staged candidates (P:716-727 on cached vectors).
__global__ void __launch_bounds__(MWU_NT) search_pass(int64_t mP, const double* __restrict__ y,
                                                      const double* __restrict__ dy, const double* __restrict__ u,
                                                      int64_t mC, const double* __restrict__ z,
                                                      const double* __restrict__ dz, const double* __restrict__ v,
                                                      Ctl* c, double* part, unsigned int* counter) {
  if (c->status != ST_RUNNING || !c->sactive) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(c->h_search, 0u);
    return;
  }
  __shared__ double s_a[MWU_MAXC], s_ea[MWU_MAXC], s_shP[MWU_MAXC], s_shC[MWU_MAXC];
  __shared__ int s_mP[MWU_MAXC], s_mC[MWU_MAXC], s_sq[MWU_MAXC];
  if (threadIdx.x < MWU_MAXC) {
    const int j = threadIdx.x;
    s_a[j] = c->cand[j]; s_ea[j] = c->cea[j]; s_shP[j] = c->shP[j]; s_shC[j] = c->shC[j];
    s_mP[j] = c->cmP[j]; s_mC[j] = c->cmC[j]; s_sq[j] = c->csq[j];
  }
  __syncthreads();
  const int nc = c->ncand, pt = c->ptype;
  const double eta = c->eta, neta = -c->eta;
  // one transcendental per row and pass (per side): candidates follow by exact identities
  //   doubling  a -> 2a : expm1(2x) = e (e + 2),           exp(2x) = q^2
  //   grid  a -> a + delta: expm1(x + w) = e + e_w + e e_w, exp(x + w) = q q_w
  const double ea0 = eta * c->pa0, ead = eta * c->pdelta;
  double acc[6 * MWU_MAXC];
#pragma unroll
  for (int j = 0; j < MWU_MAXC; ++j) {
    acc[R_EP(j)] = 0.0; acc[R_LP(j)] = 0.0; acc[R_MX(j)] = -INFINITY;
    acc[R_EC(j)] = 0.0; acc[R_TC(j)] = 0.0; acc[R_MN(j)] = INFINITY;
  }
  extern __shared__ __align__(128) double sbuf[];
  __shared__ __align__(8) uint64_t bars[MWU_SST];
  if (threadIdx.x == 0) {
    for (int s = 0; s < MWU_SST; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t it = 0;
  stream_rows3(y, dy, u, mP, sbuf, bars, it, [&](double yi, double di, double ui, int64_t) {
    double em = 0.0, emd = 0.0;
    if (pt != PT_LIST) em = expm1(ea0 * di);
    if (pt == PT_GRID) emd = expm1(ead * di);
#pragma unroll
    for (int j = 0; j < MWU_MAXC; ++j) {
      if (j < nc) {
        if (pt == PT_DOUBLE) { for (int s = 0; s < s_sq[j]; ++s) em = em * (em + 2.0); }
        else if (pt == PT_GRID) em = em + emd + em * emd;
        else if (s_mP[j] == CM_EXPM1) em = expm1(s_ea[j] * di);
        const double t = yi + s_a[j] * di;
        acc[R_MX(j)] = fmax(acc[R_MX(j)], t);
        if (s_mP[j] == CM_EXPM1) acc[R_EP(j)] = __fma_rn(ui, em, acc[R_EP(j)]);   // sums: any order
        else if (s_mP[j] == CM_LSE) acc[R_LP(j)] += exp(eta * (t - s_shP[j]));
      }
    }
  });
  stream_rows3(z, dz, v, mC, sbuf, bars, it, [&](double zi, double di, double vi, int64_t) {
    double em = 0.0, q = 1.0, emd = 0.0, qd = 1.0;
    if (pt != PT_LIST) {
      const double xa = -(ea0 * di);
      if (xa >= -0.6931471805599453) { em = expm1(xa); q = 1.0 + em; } else { q = exp(xa); em = q - 1.0; }
      if (pt == PT_GRID) {
        const double xd = -(ead * di);
        if (xd >= -0.6931471805599453) { emd = expm1(xd); qd = 1.0 + emd; } else { qd = exp(xd); emd = qd - 1.0; }
      }
    }
#pragma unroll
    for (int j = 0; j < MWU_MAXC; ++j) {
      if (j < nc) {
        if (pt == PT_DOUBLE) { for (int s = 0; s < s_sq[j]; ++s) { em = em * (em + 2.0); q = q * q; } }
        else if (pt == PT_GRID) { em = em + emd + em * emd; q = q * qd; }
        else if (s_mC[j] == CM_EXPM1) {
          const double xa = -(s_ea[j] * di);
          if (xa >= -0.6931471805599453) { em = expm1(xa); q = 1.0 + em; } else { q = exp(xa); em = q - 1.0; }
        }
        const double t = zi + s_a[j] * di;
        acc[R_MN(j)] = fmin(acc[R_MN(j)], t);
        if (s_mC[j] == CM_EXPM1) { acc[R_EC(j)] = __fma_rn(vi, em, acc[R_EC(j)]); acc[R_TC(j)] = __fma_rn(vi, q, acc[R_TC(j)]); }
        else if (s_mC[j] == CM_LSE) acc[R_TC(j)] += exp(neta * (t - s_shC[j]));
      }
    }
  });
  int ops[6 * MWU_MAXC];
#pragma unroll
  for (int j = 0; j < MWU_MAXC; ++j) {
    ops[R_EP(j)] = OP_SUM; ops[R_LP(j)] = OP_SUM; ops[R_MX(j)] = OP_MAX;
    ops[R_EC(j)] = OP_SUM; ops[R_TC(j)] = OP_SUM; ops[R_MN(j)] = OP_MIN;
  }
  reduce_and_finalize<6 * MWU_MAXC>(acc, ops, part, counter, c, A_SEARCH);
}

// y += alpha d^(y), z += alpha d^(z) fused with u = exp(eta (y - s_P)),
// v = exp(-eta (z - s_C)) at the accepted alpha's shifts, and S_P, S_C.
// has_delta = 0: initial weights only (init) with shifts from A_INIT_EXT.
__global__ void __launch_bounds__(MWU_NT) update_rows(int64_t mP, double* __restrict__ y, const double* __restrict__ dy,
                                                      double* __restrict__ u, int64_t mC, double* __restrict__ z,
                                                      const double* __restrict__ dz, double* __restrict__ v, Ctl* c,
                                                      double* part, unsigned int* counter, int has_delta) {
  if (c->status != ST_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(c->h_iter, 0u);
    return;
  }
  const double a = c->alpha, eta = c->eta, neta = -c->eta;
  const double sP = has_delta ? c->newsP : c->sP, sC = has_delta ? c->newsC : c->sC;
  double acc[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * MWU_NT;
  const int64_t tid = (int64_t)blockIdx.x * MWU_NT + threadIdx.x;
  for (int64_t i = tid; i < mP; i += stride) {
    double yi = y[i];
    if (has_delta) { yi = yi + a * dy[i]; y[i] = yi; }
    const double w = exp(eta * (yi - sP));
    u[i] = w;
    acc[0] += w;
  }
  for (int64_t i = tid; i < mC; i += stride) {
    double zi = z[i];
    if (has_delta) { zi = zi + a * dz[i]; z[i] = zi; }
    const double w = exp(neta * (zi - sC));
    v[i] = w;
    acc[1] += w;
  }
  const int ops[2] = {OP_SUM, OP_SUM};
  reduce_and_finalize<2>(acc, ops, part, counter, c, has_delta ? A_UPDATE : A_INIT_W);
}

// Init: shifts s_P = max y, s_C = min z (Q4).
__global__ void __launch_bounds__(MWU_NT) init_ext(int64_t mP, const double* __restrict__ y, int64_t mC,
                                                   const double* __restrict__ z, Ctl* c, double* part,
                                                   unsigned int* counter) {
  if (c->status != ST_RUNNING) return;
  double acc[2] = {-INFINITY, INFINITY};
  const int64_t stride = (int64_t)gridDim.x * MWU_NT;
  const int64_t tid = (int64_t)blockIdx.x * MWU_NT + threadIdx.x;
  for (int64_t i = tid; i < mP; i += stride) acc[0] = fmax(acc[0], y[i]);
  for (int64_t i = tid; i < mC; i += stride) acc[1] = fmin(acc[1], z[i]);
  const int ops[2] = {OP_MAX, OP_MIN};
  reduce_and_finalize<2>(acc, ops, part, counter, c, A_INIT_EXT);
}

// Init: x_i = eps / (n ||P_{:,i}||_inf); colmax == nullptr: all columns have max cm
// (graph operators: 1, O/D: 1/D, embedded row: 1/M).  Reduces sum(x/M) for a singleton side.
__global__ void __launch_bounds__(MWU_NT) init_x(int64_t n, double* __restrict__ x, const double* __restrict__ colmax,
                                                 double cm, Ctl* c, double* part, unsigned int* counter) {
  const double eps = c->eps, nd = (double)n, invB = c->invB;
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * MWU_NT) {
    const double ci = colmax ? colmax[i] : cm;
    const double xi = eps / (nd * ci);
    x[i] = xi;
    acc[0] += invB * xi;
  }
  const int ops[1] = {OP_SUM};
  reduce_and_finalize<1>(acc, ops, part, counter, c, A_INIT_SING);
}

// x += alpha_prev d (flush of the lazy update at the end of a probe).
__global__ void flush_x(int64_t n, double* __restrict__ x, const double* __restrict__ d, Ctl* c) {
  if (!c->apply_prev) return;
  const double a = c->alpha_prev;
  for (int64_t i = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * MWU_NT)
    x[i] = x[i] + a * d[i];
}

// out = in / s  with s = *sp (x_out = x / min(Cx), Q15), or out = in / S (w = u / S).
__global__ void scale_div(int64_t n, const double* __restrict__ in, double* __restrict__ out, const double* sp) {
  const double s = *sp;
  for (int64_t i = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * MWU_NT)
    out[i] = in[i] / s;
}

// Generic sum / max reduction into ctl->scratch (bracket computations).
__global__ void __launch_bounds__(MWU_NT) reduce_vec(int64_t n, const double* __restrict__ a, Ctl* c, double* part,
                                                     unsigned int* counter) {
  double acc[2] = {0.0, -INFINITY};
  for (int64_t i = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * MWU_NT) {
    acc[0] += a[i];
    acc[1] = fmax(acc[1], a[i]);
  }
  const int ops[2] = {OP_SUM, OP_MAX};
  reduce_and_finalize<2>(acc, ops, part, counter, c, A_SUM);
}

}  // namespace mwu
