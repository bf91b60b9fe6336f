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
#include "fastmath.cuh"

#ifndef MWU_SEARCH_PTAB
#define MWU_SEARCH_PTAB 0     // packing side of the search: degree-14 Taylor expm1 (1: table-driven,
#endif                        // as fast but moved the densest-bu310 solve to 2.3% from the oracle's count
#ifndef MWU_CSR_GRID
#define MWU_CSR_GRID 4        // csr_scatter CTAs per SM (grid-stride, ids of the next chunk prefetched; 8 measured 4% slower)
#endif
#ifndef MWU_VC_GRID
#define MWU_VC_GRID 4         // vc_scatter CTAs per SM
#endif
#ifndef MWU_SEARCH_TAB
#define MWU_SEARCH_TAB 1      // covering side of the search: table-driven (expm1, exp) pair
#endif

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
//   NP  sum_i u_i e^{eta a0 dy_i} dy_i (candidate 0, P side; same shift as EP / LP) — Newton's Psi'
//   NC  sum_i v_i e^{-eta a0 dz_i} dz_i (candidate 0, C side; same shift as TC)    — Newton's Phi'
#define R_NP (6 * MWU_MAXC)
#define R_NC (6 * MWU_MAXC + 1)

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
  if (c->dk_hi >= (1 << 20)) {                       // no stop seen yet: the next MAXC exponents
    for (int i = 0; i < MWU_MAXC; ++i) ks[n++] = c->dk_lo + 1 + i;
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
  if (c->t < 32 && c->aguess[c->t] >= 1.0) kg = ilogb(c->aguess[c->t]);   // previous probe, same t
  else if (c->t > 0 && c->alpha_prev >= 1.0) kg = ilogb(c->alpha_prev);
  int k0 = kg - (MWU_MAXC / 2 - 1);
  if (k0 < 0) k0 = 0;
  int ks[MWU_MAXC];
  for (int j = 0; j < MWU_MAXC; ++j) ks[j] = k0 + j;
  stage_double_exps(c, ks, MWU_MAXC);
}

// The 2^L - 1 midpoints of L bisection levels of [lb, ub], computed exactly as the sequential
// loop computes them, ascending.
__device__ int bisect_tree(double lb, double ub, int L, double* vals) {
  double lo[8], hi[8], nlo[8], nhi[8];
  int ni = 1, nv = 0;
  lo[0] = lb; hi[0] = ub;
  for (int lev = 0; lev < L; ++lev) {
    int nn = 0;
    for (int k = 0; k < ni; ++k) {
      const double m = (lo[k] + hi[k]) / 2.0;
      vals[nv++] = m;
      if (lev + 1 < L) { nlo[nn] = lo[k]; nhi[nn] = m; ++nn; nlo[nn] = m; nhi[nn] = hi[k]; ++nn; }
    }
    for (int k = 0; k < nn; ++k) { lo[k] = nlo[k]; hi[k] = nhi[k]; }
    ni = nn;
  }
  for (int i = 1; i < nv; ++i)            // insertion sort (<= 15 values)
    for (int k = i; k > 0 && vals[k - 1] > vals[k]; --k) { const double t = vals[k]; vals[k] = vals[k - 1]; vals[k - 1] = t; }
  return nv;
}

// A bisection that may need four levels (the stop rule of Q9 with eps < 1/8 on a whole octave):
// one pass evaluates the first three levels and the fourth-level node of the lowest bracket
// (the most likely of the fourth level for a log-uniform step size), so only a step size in
// [lb + 2 delta, lb + 4 delta) needs a further, one-candidate pass.  search_controller replays
// the sequential bisection exactly over whatever was evaluated.
__device__ void stage_g16(Ctl* c) {
  double v[15];
  bisect_tree(c->lb, c->ub, 4, v);                     // v[j - 1] = lb + j (ub - lb)/16
  const int pick[MWU_MAXC] = {1, 2, 4, 6, 8, 10, 12, 14};
  for (int k = 0; k < MWU_MAXC; ++k) { c->cand[k] = v[pick[k] - 1]; stage_modes(c, k); }
  c->ncand = MWU_MAXC;
  c->ptype = PT_G16;
  c->pdelta = (c->ub - c->lb) / 16.0;
  c->pa0 = c->cand[0];
}

__device__ void stage_bisect(Ctl* c) {          // the 2^L - 1 midpoints of L bisection levels
  const int Lmax = (MWU_MAXC >= 7) ? 3 : ((MWU_MAXC >= 3) ? 2 : 1);
  int L = c->bisect_depth < 1 ? 1 : (c->bisect_depth > Lmax ? Lmax : c->bisect_depth);
  {   // no more levels than the stop rule can still ask for: lb only grows, so after l levels the
      // bracket is (ub - lb)/2^l <= thr * lb_final once (ub - lb)/2^l <= thr * lb (Q9)
    const double thr = c->tol_prose ? c->eps : (1.0 - c->eps);
    int need = 1;
    while (need < 4 && (c->ub - c->lb) / (double)(1 << need) > thr * c->lb) ++need;
    if (need >= 4 && L == 3 && MWU_MAXC == 8) { stage_g16(c); return; }
    L = need < L ? need : L;
  }
  double vals[8];
  const int n = bisect_tree(c->lb, c->ub, L, vals);
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

__device__ __forceinline__ double cand_tc(const Ctl* c, int j, const double* res) { return res[R_TC(j)]; }
__device__ __forceinline__ double cand_sh(const Ctl* c, int j) { return c->shC[j]; }

__device__ void accept_alpha(Ctl* c, double a, double mx, double mn, double tc, double tsh) {
  c->alpha = a;
  c->newsP = mx;
  c->newsC = mn;
  c->acc_tc = tc;
  c->acc_sh = tsh;
  c->sphase = SP_DONE;
  c->sactive = 0;
  if (a < 1.0) { c->status = ST_INFEASIBLE; c->reason = R_ALPHA_LT_1; return; }
  if (c->lazyC && !(tc > 1e-280 && isfinite(tc))) {
    // lazyC carries S_C of the next iterate from this sum; it underflowed at the old shift, so
    // re-evaluate the accepted alpha with the exact min shift (one extra pass, Q16)
    c->sphase = SP_TCFIX; c->ncand = 1; c->cand[0] = a; c->cea[0] = c->eta * a; c->cexp[0] = 0; c->csq[0] = 0;
    c->cmP[0] = CM_EXT; c->cmC[0] = CM_LSE; c->shC[0] = mn; c->ptype = PT_LIST; c->sactive = 1;
  }
}

// Newton: a pass evaluating one point a, with the derivative sums of candidate 0
__device__ void stage_newton(Ctl* c, double a) {
  c->cand[0] = a; c->cexp[0] = -1; c->csq[0] = 0;
  stage_modes(c, 0);
  c->ncand = 1; c->ptype = PT_LIST; c->sphase = SP_NEWTON; c->sactive = 1;
}
// the (1 - eps)^p back-off ladder after a, the multiplications done in sequence
__device__ void stage_backoff(Ctl* c, double a) {
  int n = MWU_MAXC;
  if (MWU_NEWTON_MAX_BACKOFF - c->nb < n) n = MWU_NEWTON_MAX_BACKOFF - c->nb;
  for (int j = 0; j < n; ++j) {
    a = a * (1.0 - c->eps);
    c->cand[j] = a; c->cexp[j] = -1; c->csq[j] = 0;
    stage_modes(c, j);
  }
  c->ncand = n; c->ptype = PT_LIST; c->sphase = SP_NBACK; c->sactive = 1;
}
// Newton gives up (Q35): Alg. 3 from alpha = 1 with its own evaluation count
__device__ void newton_fallback(Ctl* c) {
  c->nfb = 1; c->evals = 0;
  c->sphase = SP_DOUBLE;
  stage_double_first(c);
  c->sactive = 1;
}
// a candidate whose expm1 form is invalid (Q16): re-evaluate alone with the exact max / min shift
__device__ void stage_exact_shift(Ctl* c, int j, int nP, int nC, double mxj, double mnj, int keep_phase) {
  const double a = c->cand[j];
  const int keepP = c->cmP[j];
  const double kshP = c->shP[j];
  c->cand[0] = a; c->cea[0] = c->eta * a; c->cexp[0] = -1; c->csq[0] = 0;
  c->cmP[0] = c->pSing ? CM_EXT : (nP ? CM_LSE : keepP); c->shP[0] = nP ? mxj : kshP;
  c->cmC[0] = c->cSing ? CM_EXT : (nC ? CM_LSE : CM_EXPM1); c->shC[0] = nC ? mnj : c->sC;
  c->ncand = 1; c->ptype = PT_LIST; c->sphase = keep_phase; c->sactive = 1;
}

__device__ void newton_controller(Ctl* c, const double* res) {
  if (c->sphase == SP_NEWTON) {
    double psi, phi; int nP, nC;
    eval_cand(c, 0, res, psi, phi, nP, nC);
    const double mx0 = cand_mx(c, 0, res), mn0 = cand_mn(c, 0, res);
    if (nP || nC) { stage_exact_shift(c, 0, nP, nC, mx0, mn0, SP_NEWTON); return; }
    const double a = c->cand[0];
    const double dphi = c->cSing ? c->eta * c->dzS : c->eta * (res[R_NC] / res[R_TC(0)]);
    const double dpsi = c->pSing ? c->eta * c->dyS
                                 : c->eta * (res[R_NP] / (c->cmP[0] == CM_EXPM1 ? c->SP + res[R_EP(0)] : res[R_LP(0)]));
    c->evals++; c->evals_total++; c->nk++;
    const double P = phi, Q = psi;
    const double den = dphi * Q - P * dpsi;
    bool bad = !(isfinite(P) && isfinite(Q) && isfinite(den)) || !(den < 0.0) || !(Q > 0.0);
    double an = 0.0;
    if (!bad) { an = a - (P - Q) * Q / den; bad = !(isfinite(an) && an > 0.0); }
    if (bad) { newton_fallback(c); return; }
    if (fabs(an - a) <= c->eps * a) {                       // converged (Q35): keep the evaluated a
      if (P >= Q) { accept_alpha(c, a, mx0, mn0, cand_tc(c, 0, res), cand_sh(c, 0)); return; }
      c->nb = 0;
      stage_backoff(c, a);
      return;
    }
    if (c->nk >= MWU_NEWTON_MAX_STEPS) { newton_fallback(c); return; }
    stage_newton(c, an);
    return;
  }
  // SP_NBACK: the ladder a (1 - eps)^p in order; the first with f >= 1, or the 64th, is the answer
  for (int j = 0; j < c->ncand; ++j) {
    double psi, phi; int nP, nC;
    eval_cand(c, j, res, psi, phi, nP, nC);
    const double mxj = cand_mx(c, j, res), mnj = cand_mn(c, j, res);
    if (nP || nC) { stage_exact_shift(c, j, nP, nC, mxj, mnj, SP_NBACK); return; }
    c->nb++; c->evals++; c->evals_total++;
    if (near_tie(phi, psi)) c->near_ties++;
    if (phi >= psi || c->nb >= MWU_NEWTON_MAX_BACKOFF) {
      accept_alpha(c, c->cand[j], mxj, mnj, cand_tc(c, j, res), cand_sh(c, j));
      return;
    }
  }
  stage_backoff(c, c->cand[c->ncand - 1]);
}

// res layout: see R_* above
__device__ void search_controller(Ctl* c, const double* res) {
  c->passes_total++;
  if (c->sphase == SP_NEWTON || c->sphase == SP_NBACK) { newton_controller(c, res); return; }
  if (c->sphase == SP_FIXED) {
    accept_alpha(c, c->cand[0], cand_mx(c, 0, res), cand_mn(c, 0, res), cand_tc(c, 0, res), cand_sh(c, 0));
    return;
  }
  if (c->sphase == SP_TCFIX) {
    const double tc = cand_tc(c, 0, res);
    if (!(tc > 1e-280 && isfinite(tc))) { c->nan_flag = 1; c->status = ST_INFEASIBLE; c->sactive = 0; return; }
    accept_alpha(c, c->cand[0], c->newsP, c->newsC, tc, cand_sh(c, 0));
    return;
  }
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
      if (near_tie(phi, psi) || near_tie(mnj, 1.0)) c->near_ties++;
      if (ok && mnj < 1.0) { c->dk_lo = k; c->ok_mx = mxj; c->ok_mn = mnj; c->ok_tc = cand_tc(c, j, res); c->ok_sh = cand_sh(c, j); }
      else {
        c->dk_hi = k; c->hi_exit = ok ? 1 : 0; c->hi_mx = mxj; c->hi_mn = mnj;
        c->hi_tc = cand_tc(c, j, res); c->hi_sh = cand_sh(c, j);
      }
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
      if (c->dk_lo == cap_k) { accept_alpha(c, ldexp(1.0, cap_k), c->ok_mx, c->ok_mn, c->ok_tc, c->ok_sh); return; }
      c->sphase = SP_FIXED; c->ncand = 1; c->cand[0] = ldexp(1.0, cap_k); c->ptype = PT_LIST;   // shifts only
      c->cea[0] = c->eta * c->cand[0]; c->cmP[0] = CM_EXT; c->cmC[0] = c->lazyC ? CM_EXPM1 : CM_EXT;
      c->shC[0] = c->sC; c->sactive = 1;
      return;
    }
    if (c->dk_hi == c->dk_lo + 1) {
      const int ks = c->dk_hi;
      c->evals = ks + 1; c->evals_total += ks + 1;
      if (c->hi_exit) { accept_alpha(c, ldexp(1.0, ks), c->hi_mx, c->hi_mn, c->hi_tc, c->hi_sh); return; }
      if (c->step_rule == STEP_NEWTON && !c->nfb && ks >= 1) {   // Newton from the largest passing 2^p (Q34)
        c->nk = 0;
        stage_newton(c, ldexp(1.0, ks - 1));
        return;
      }
      c->sphase = SP_BISECT; c->lb = ldexp(1.0, ks - 1); c->ub = ldexp(1.0, ks);
      c->lb_mx = c->ok_mx; c->lb_mn = c->ok_mn; c->lb_tc = c->ok_tc; c->lb_sh = c->ok_sh;
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
        accept_alpha(c, c->lb, c->lb_mx, c->lb_mn, c->lb_tc, c->lb_sh);     // return lb
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
    if (near_tie(phi, psi)) c->near_ties++;
    c->evals++;
    c->evals_total++;
    if (ok) { c->lb = need; c->lb_mx = mxj; c->lb_mn = mnj; c->lb_tc = cand_tc(c, j, res); c->lb_sh = cand_sh(c, j); }
    else { c->ub = need; }
  }
  c->status = ST_INFEASIBLE; c->reason = R_ALPHA_LT_1; c->sactive = 0;   // unreachable guard
}

// =====================================================================================
// Finalize: control logic run by thread 0 of the last block of a phase kernel
// =====================================================================================
__device__ void finalize(Ctl* c, int action, double* r) {
  switch (action) {                        // phase timing: which phase ends with this action
    case A_COL: case A_COL_FAST: phase_mark(c, 0); break;
    case A_STEP_MAXDY: case A_STEP_DONE: case A_STEP_DONE + 100: case A_STEP_DONE_C: phase_mark(c, 1); break;
    case A_SEARCH: phase_mark(c, 2); break;
    case A_UPDATE: phase_mark(c, 3); break;
    case A_INIT_W: phase_mark(c, -1); break;
    default: break;
  }
  switch (action) {
    case A_COL_FAST: {                             // fast densest column: max d, inactive aggregate
      c->apply_prev = 0;
      c->maxd = r[0];
      c->mzi = r[1];
      // r[2] = sum of v = exp(-eta(z - s_C)) over inactive rows; rescaled to shift mzi.  Exact
      // unless eta(mzi - s_C) > 600, where terms may have underflowed: inactive_exact redoes it.
      c->vi_exact = 0;
      if (!(r[2] > 0.0)) c->Vi = 0.0;
      else if (c->eta * (c->mzi - c->sC) <= 600.0) c->Vi = r[2] * exp(c->eta * (c->mzi - c->sC));
      else c->vi_exact = 1;
      if (!(r[0] > 0.0)) { c->status = ST_INFEASIBLE; c->reason = R_MAXD_ZERO; }
      break;
    }
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
    case A_STEP_DONE_C:
      // r = (max d^(z), min z, sum v) over the rows with d^(z) = 0; v is stored at shift s_C,
      // the aggregate is carried at shift mzi (exact pass when terms may have underflowed)
      c->mzi = r[1];
      c->vi_exact = 0;
      if (!(r[2] > 0.0)) c->Vi = 0.0;
      else if (c->eta * (c->mzi - c->sC) <= 600.0) c->Vi = r[2] * exp(c->eta * (c->mzi - c->sC));
      else c->vi_exact = 1;
      // fall through
    case A_STEP_DONE:
    case A_STEP_DONE + 100: {
      if (action == A_STEP_DONE + 100) c->maxdy = r[0];
      c->evals = 0;
      c->nk = 0; c->nfb = 0; c->nb = 0;
      if (c->fixed_alpha > 0.0 || c->step_rule == STEP_STANDARD) {   // fixed steps; Alg. 1's alpha = 1
        const double fa = c->fixed_alpha > 0.0 ? c->fixed_alpha : 1.0;
        c->sphase = SP_FIXED; c->ncand = 1; c->cand[0] = fa; c->ptype = PT_LIST;
        c->cea[0] = c->eta * fa; c->cmP[0] = CM_EXT; c->cmC[0] = c->lazyC ? CM_EXPM1 : CM_EXT;
        c->shC[0] = c->sC;
      } else if (c->step_rule == STEP_NEWTON && c->t > 0 && c->alpha_prev >= 1.0) {
        stage_newton(c, c->alpha_prev);                   // warm start (Q34)
      } else {
        c->sphase = SP_DOUBLE; c->sa = 1.0;                                 // alpha <- 1
        stage_double_first(c);
      }
      c->sactive = 1;
      set_cond(c->h_search, 1u);
      break;
    }
    case A_SEARCH:
      if (c->lazyC || c->compC) {
        // covering rows with d^(z) = 0 were not streamed: they add exp(-eta(z - shC)) to the
        // shifted sums and z to the minima, for every candidate alike
        for (int j = 0; j < c->ncand; ++j) {
          r[R_MN(j)] = fmin(r[R_MN(j)], c->mzi);
          if (c->Vi > 0.0 && c->cmC[j] != CM_EXT) r[R_TC(j)] += c->Vi * exp(-c->eta * (c->mzi - c->shC[j]));
        }
      }
      search_controller(c, r);
      set_cond(c->h_search, c->sactive ? 1u : 0u);
      break;
    case A_UPDATE: {
      if (c->t < 32) c->ahist[c->t] = c->alpha;
      c->t++;
      c->alpha_last = c->alpha; c->alpha_prev = c->alpha; c->apply_prev = 1;
      if (near_tie(c->cSing ? c->zS + c->alpha * c->dzS : c->newsC, 1.0)) c->near_ties++;   // min z >= 1
      if (c->pSing) { c->yS = c->yS + c->alpha * c->dyS; c->sP = c->yS; c->SP = 1.0; }
      else { c->sP = c->newsP; c->SP = r[0] + r[2]; }          // r[2]: owned rows (0 unless sharded by owner)
      if (c->cSing) { c->zS = c->zS + c->alpha * c->dzS; c->sC = c->zS; c->SC = 1.0; }
      else if (c->lazyC) { c->sC = c->newsC; c->SC = c->acc_tc * exp(c->eta * (c->newsC - c->acc_sh)); }
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
      c->SP = c->pSing ? 1.0 : r[0] + r[2];
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
    case A_VI_EXACT:
      c->Vi = r[0];
      c->vi_exact = 0;
      break;
    default:
      break;
  }
}

// Phase reductions over rank-local rows are partial on a sharded run: the last block parks its
// reduced slots in the control block and the host exchanges them (allgather) before
// finalize_multi combines them in rank order and runs the same control logic on every rank.
__device__ __forceinline__ bool partial_action(const Ctl* c, int a) {
  if (a == A_COL || a == A_INIT_SING || a == A_SUM) return !c->repvars;   // over the (local) variables
  if (a == A_UPDATE) return c->partupd;                                  // local covering / owned rows
  if (a == A_STEP_DONE + 100) return c->ownrows;                         // max d^(y) over owned rows
  return a == A_COL_FAST || a == A_SEARCH || a == A_INIT_EXT || a == A_INIT_W || a == A_VI_EXACT;
}
__device__ void finish(Ctl* c, int action, double* res, const int* ops, int n) {
  if (c->world > 1 && partial_action(c, action)) {
    for (int s = 0; s < n; ++s) { c->dslots[s] = res[s]; c->dops[s] = ops[s]; }
    c->dn = n;
    c->daction = action;
    c->dpending = 1;
    return;
  }
  finalize(c, action, res);
}

__global__ void finalize_multi(Ctl* c, const double* __restrict__ g, int world) {
  if (threadIdx.x != 0 || !c->dpending) return;
  c->dpending = 0;
  double res[MWU_SLOTS];
  const int n = c->dn, act = c->daction;
  for (int s = 0; s < MWU_SLOTS; ++s) res[s] = 0.0;
  for (int s = 0; s < n; ++s) {
    int op = c->dops[s];
    if ((act == A_INIT_W || act == A_UPDATE) && s == 0) op = OP_FIRST;   // S_P of the replicated packing rows
    double a = g[s];
    for (int r = 1; r < world; ++r) {
      const double b = g[(size_t)r * MWU_SLOTS + s];
      a = (op == OP_FIRST) ? a : red_combine(op, a, b);
    }
    res[s] = a;
  }
  finalize(c, act, res);
}

// Standard epilogue of a reducing kernel: block partials -> last block -> finalize.
template <int NS>
__device__ __forceinline__ void reduce_and_finalize(double (&acc)[NS], const int* ops, double* part,
                                                    unsigned int* counter, Ctl* c, int action) {
  __shared__ double res[MWU_SLOTS];
  block_partials<NS>(acc, ops, part);
  if (last_block_combine(ops, NS, part, counter, res)) {
    if (threadIdx.x == 0) finish(c, action, res, ops, NS);
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

// VCOVER forward product d^(z) = M^T d (edge rows) fused with the compaction of the
// covering rows with d^(z) > 0 into per-warp records (z, d^(z), v) — the layout of the fast
// densest column kernel — and the candidate-independent aggregate (min z, sum v) of the others,
// so the search passes stream only the active rows.  src == nullptr: d^(z) is
// already in `in` (domset: scattered by csr_scatter); only the compaction runs.
__global__ void __launch_bounds__(MWU_NT) edge_sum_compact(int64_t E64, const int32_t* __restrict__ src,
                                                           const int32_t* __restrict__ dst,
                                                           const double* __restrict__ in, double* __restrict__ out,
                                                           const double* __restrict__ z, const double* __restrict__ v,
                                                           double* __restrict__ rz, double* __restrict__ rdz,
                                                           double* __restrict__ rv, int32_t* __restrict__ tcnt,
                                                           int64_t rcap, Ctl* c, double* part, unsigned int* counter) {
  if (c->status != ST_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(c->h_search, 0u);
    return;
  }
  const int E = (int)E64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ntiles = (E + MWU_CT - 1) / MWU_CT;
  double acc[3] = {-INFINITY, INFINITY, 0.0};
  const int64_t w0 = ((int64_t)blockIdx.x * (MWU_NT / 32) + warp) * rcap;   // this warp's record stream
  int64_t wp = w0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    double s[kColEdges], zz[kColEdges], vv[kColEdges];
#pragma unroll
    for (int k = 0; k < kColEdges; ++k) {
      const int e = tile * MWU_CT + k * MWU_NT + threadIdx.x;
      if (e < E) {
        s[k] = src ? __ldg(in + __ldcs(src + e)) + __ldg(in + __ldcs(dst + e)) : __ldcs(in + e);
        zz[k] = __ldcs(z + e); vv[k] = __ldcs(v + e);
      } else {
        s[k] = 0.0; zz[k] = INFINITY; vv[k] = 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kColEdges; ++k) {
      const int e = tile * MWU_CT + k * MWU_NT + threadIdx.x;
      const bool nz = s[k] > 0.0;
      const uint32_t bw = __ballot_sync(0xffffffffu, nz);
      if (e < E) {
        if (src) out[e] = s[k];
        acc[0] = fmax(acc[0], s[k]);
        if (nz) {
          const int64_t p = wp + __popc(bw & ((1u << lane) - 1u));
          rz[p] = zz[k]; rdz[p] = s[k]; rv[p] = vv[k];
        } else {
          acc[1] = fmin(acc[1], zz[k]);
          acc[2] += vv[k];
        }
      }
      wp += __popc(bw);
    }
  }
  if (lane == 0) tcnt[blockIdx.x * (MWU_NT / 32) + warp] = (int32_t)(wp - w0);
  const int ops[3] = {OP_MAX, OP_MIN, OP_SUM};
  reduce_and_finalize<3>(acc, ops, part, counter, c, A_STEP_DONE_C);
}

// Rare path of the vcover inactive aggregate (rows with d^(z) = 0), exactly at shift mzi.
__global__ void __launch_bounds__(MWU_NT) inactive_exact_dz(int64_t E, const double* __restrict__ dz,
                                                            const double* __restrict__ z, Ctl* c, double* part,
                                                            unsigned int* counter) {
  if (c->status != ST_RUNNING || !c->vi_exact) return;
  const double neta = -c->eta, m = c->mzi;
  double acc[1] = {0.0};
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT)
    if (!(dz[e] > 0.0)) acc[0] += exp(neta * (z[e] - m));
  const int ops[1] = {OP_SUM};
  reduce_and_finalize<1>(acc, ops, part, counter, c, A_VI_EXACT);
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

__device__ __forceinline__ int search_slot_op(int s) {
  const int g = s / MWU_MAXC;            // 0 EP, 1 LP, 2 MX, 3 EC, 4 TC, 5 MN, 6 NP / NC
  return g == 2 ? OP_MAX : (g == 5 ? OP_MIN : OP_SUM);
}

// (expm1(x), exp(x)) for x <= 0 with both accurate relative to themselves: expm1 while
// x >= -ln 2 (then exp = 1 + expm1 >= 1/2), exp below (then expm1 = exp - 1 <= -1/2).
__device__ __forceinline__ void expm1_exp(double x, double& em, double& q) {
  if (x >= -0.6931471805599453) { em = expm1(x); q = 1.0 + em; }
  else { q = exp(x); em = q - 1.0; }
}

// Candidate parameters of a pass, in registers (uniform over the grid).
struct Cands {
  double a[MWU_MAXC], ea[MWU_MAXC], shP[MWU_MAXC], shC[MWU_MAXC];
  int mP[MWU_MAXC], mC[MWU_MAXC], sq[MWU_MAXC];
  int nc, pt;
  double ea0, ead;
};

// PT_G16: the candidates are lb + j delta, j = 1, 2, 4, ..., 14; expm1 and exp advance from the
// first one by the exact identities e(t + delta) = e + ed + e ed, q(t + delta) = q qd: one step
// to candidate 1, two steps to each later one
template <int PT>
__device__ __forceinline__ int grid_steps(int j) { return PT == PT_G16 ? (j == 0 ? 0 : (j == 1 ? 1 : 2)) : 1; }

// Fast per-row bodies: every candidate of the pass uses the expm1 form (Q16) on the streamed
// side; the candidates follow from ONE transcendental per row by exact identities
//   doubling  a -> 2a   : expm1(2x) = e (e + 2),            exp(2x) = q^2
//   grid  a -> a + delta: expm1(x + w) = e + e_w + e e_w,  exp(x + w) = q q_w
template <int PT, int NC, bool SQ1>
struct PRowFast {
  static constexpr double kAbsent = -INFINITY;     // y of an absent row (stream_rows3 pairs)
  double a[NC], ea0, ead, eta;
  int sq[NC];
  double ep[NC], mx[NC];
  double shP[NC];
  bool lse[NC];        // Q16: candidates with eta alpha max d^(y) > 700 use the shifted exp sum
  const double *T, *Mh, *Ml;   // exp tables (shared memory)
  __device__ PRowFast(const Cands& k, double e, const double* tab) : ea0(k.ea0), ead(k.ead), eta(e),
                                                                      T(tab), Mh(tab + 256), Ml(tab + 512) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      a[j] = k.a[j]; sq[j] = k.sq[j]; ep[j] = 0.0; mx[j] = -INFINITY; shP[j] = k.shP[j]; lse[j] = (k.mP[j] == CM_LSE);
    }
  }
  __device__ __forceinline__ double xm1(double x) const {
#if MWU_SEARCH_PTAB
    double em, q;
    mwu_expm1_exp_tab(x, T, Mh, Ml, em, q);
    return em;
#else
    return mwu_expm1(x);
#endif
  }
  // two rows with their dependent chains interleaved; row 1 is masked by u1 = 0, y1 = -inf
  __device__ __forceinline__ void pair(double y0, double d0, double u0, double y1, double d1, double u1) {
    double e0 = xm1(ea0 * d0), e1 = xm1(ea0 * d1), ed0 = 0.0, ed1 = 0.0;
    if (PT == PT_GRID || PT == PT_G16) { ed0 = xm1(ead * d0); ed1 = xm1(ead * d1); }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (PT == PT_DOUBLE) {
        if (SQ1) { if (j > 0) { e0 = e0 * (e0 + 2.0); e1 = e1 * (e1 + 2.0); } }
        else { for (int s = 0; s < sq[j]; ++s) { e0 = e0 * (e0 + 2.0); e1 = e1 * (e1 + 2.0); } }
      } else if (PT == PT_GRID) { e0 = e0 + ed0 + e0 * ed0; e1 = e1 + ed1 + e1 * ed1; }
      else {
#pragma unroll
        for (int s = 0; s < grid_steps<PT>(j); ++s) { e0 = e0 + ed0 + e0 * ed0; e1 = e1 + ed1 + e1 * ed1; }
      }
      if (lse[j]) {
        ep[j] += mwu_exp(eta * ((y0 + a[j] * d0) - shP[j]));
        if (u1 != 0.0) ep[j] += mwu_exp(eta * ((y1 + a[j] * d1) - shP[j]));
      } else ep[j] = __fma_rn(u1, e1, __fma_rn(u0, e0, ep[j]));
    }
    const bool up0 = (y0 + a[NC - 1] * d0) > mx[0], up1 = (y1 + a[NC - 1] * d1) > mx[0];
    if (__any_sync(__activemask(), up0 || up1)) {
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const double t0 = y0 + a[j] * d0, t1 = y1 + a[j] * d1;
        if (up0 && t0 > mx[j]) mx[j] = t0;
        if (up1 && t1 > mx[j]) mx[j] = t1;
      }
    }
  }
  __device__ __forceinline__ void operator()(double y, double d, double u, int64_t = 0) {
    double em = xm1(ea0 * d), emd = 0.0;
    if (PT == PT_GRID || PT == PT_G16) emd = xm1(ead * d);
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (PT == PT_DOUBLE) {
        if (SQ1) { if (j > 0) em = em * (em + 2.0); }          // consecutive exponents
        else { for (int s = 0; s < sq[j]; ++s) em = em * (em + 2.0); }
      } else if (PT == PT_GRID) em = em + emd + em * emd;
      else {
#pragma unroll
        for (int s = 0; s < grid_steps<PT>(j); ++s) em = em + emd + em * emd;
      }
      if (lse[j]) ep[j] += mwu_exp(eta * ((y + a[j] * d) - shP[j]));   // packing side is short
      else ep[j] = __fma_rn(u, em, ep[j]);
    }
    // candidates ascend, so y + a_j d <= y + a_last d: a row can raise a maximum only if that
    // exceeds the smallest running max (warp-uniform branch)
    const bool upd = (y + a[NC - 1] * d) > mx[0];
    if (__any_sync(__activemask(), upd)) {
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const double t = y + a[j] * d;
        if (upd && t > mx[j]) mx[j] = t;
      }
    }
  }
};

template <int PT, int NC, bool SQ1>
struct CRowFast {
  static constexpr double kAbsent = INFINITY;      // z of an absent row
  double a[NC], ea0, ead;
  int sq[NC];
  double ec[NC], tc[NC], mn[NC];
  const double *T, *Mh, *Ml;   // exp tables (shared memory)
  __device__ CRowFast(const Cands& k, const double* tab) : ea0(k.ea0), ead(k.ead), T(tab), Mh(tab + 256), Ml(tab + 512) {
#pragma unroll
    for (int j = 0; j < NC; ++j) { a[j] = k.a[j]; sq[j] = k.sq[j]; ec[j] = 0.0; tc[j] = 0.0; mn[j] = INFINITY; }
  }
  __device__ __forceinline__ void ex(double x, double& em, double& q) const {
#if MWU_SEARCH_TAB
    mwu_expm1_exp_tab(x, T, Mh, Ml, em, q);
#else
    mwu_expm1_exp(x, em, q);
#endif
  }
  __device__ __forceinline__ void operator()(double z, double d, double v, int64_t = 0) {
    double em, q, emd = 0.0, qd = 1.0;
    ex(-(ea0 * d), em, q);
    if (PT == PT_GRID || PT == PT_G16) ex(-(ead * d), emd, qd);
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (PT == PT_DOUBLE) {
        if (SQ1) { if (j > 0) { em = em * (em + 2.0); q = q * q; } }
        else { for (int s = 0; s < sq[j]; ++s) { em = em * (em + 2.0); q = q * q; } }
      } else if (PT == PT_GRID) { em = em + emd + em * emd; q = q * qd; }
      else {
#pragma unroll
        for (int s = 0; s < grid_steps<PT>(j); ++s) { em = em + emd + em * emd; q = q * qd; }
      }
      ec[j] = __fma_rn(v, em, ec[j]);
      tc[j] = __fma_rn(v, q, tc[j]);
    }
    // z + a_j d >= z and the running minima ascend in j: a row can lower a minimum only if
    // z < mn[NC-1] (rare once the minima settle; warp-uniform branch)
    const bool upd = z < mn[NC - 1];
    if (__any_sync(__activemask(), upd)) {
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const double t = z + a[j] * d;
        if (upd && t < mn[j]) mn[j] = t;
      }
    }
  }
  // two rows with their dependent chains interleaved (FP64 latency is the limiter); row 1 is
  // masked by w1 = 0 (weight 0, z = +inf) when absent
  __device__ __forceinline__ void pair(double z0, double d0, double v0, double z1, double d1, double v1) {
    double e0, q0, e1, q1, ed0 = 0.0, qd0 = 1.0, ed1 = 0.0, qd1 = 1.0;
    ex(-(ea0 * d0), e0, q0);
    ex(-(ea0 * d1), e1, q1);
    if (PT == PT_GRID || PT == PT_G16) { ex(-(ead * d0), ed0, qd0); ex(-(ead * d1), ed1, qd1); }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (PT == PT_DOUBLE) {
        if (SQ1) {
          if (j > 0) { e0 = e0 * (e0 + 2.0); q0 = q0 * q0; e1 = e1 * (e1 + 2.0); q1 = q1 * q1; }
        } else {
          for (int s = 0; s < sq[j]; ++s) { e0 = e0 * (e0 + 2.0); q0 = q0 * q0; e1 = e1 * (e1 + 2.0); q1 = q1 * q1; }
        }
      } else {
#pragma unroll
        for (int s = 0; s < grid_steps<PT>(j); ++s) {
          e0 = e0 + ed0 + e0 * ed0; q0 = q0 * qd0;
          e1 = e1 + ed1 + e1 * ed1; q1 = q1 * qd1;
        }
      }
      ec[j] = __fma_rn(v1, e1, __fma_rn(v0, e0, ec[j]));
      tc[j] = __fma_rn(v1, q1, __fma_rn(v0, q0, tc[j]));
    }
    const bool u0 = z0 < mn[NC - 1], u1 = z1 < mn[NC - 1];
    if (__any_sync(__activemask(), u0 || u1)) {
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const double t0 = z0 + a[j] * d0, t1 = z1 + a[j] * d1;
        if (u0 && t0 < mn[j]) mn[j] = t0;
        if (u1 && t1 < mn[j]) mn[j] = t1;
      }
    }
  }
};

// Generic per-row bodies (any candidate list and modes: fixed steps, exact-shift re-passes).
struct PRowGen {
  static constexpr double kAbsent = -INFINITY;
  __device__ __forceinline__ void pair(double y0, double d0, double u0, double y1, double d1, double u1) {
    (*this)(y0, d0, u0);
    if (u1 != 0.0 || y1 != -INFINITY) (*this)(y1, d1, u1);
  }
  const Cands& k;
  double eta;
  double ep[MWU_MAXC], lp[MWU_MAXC], mx[MWU_MAXC];
  double nd;                           // Newton: sum of the candidate-0 terms times d^(y)
  __device__ PRowGen(const Cands& kk, double e) : k(kk), eta(e), nd(0.0) {
#pragma unroll
    for (int j = 0; j < MWU_MAXC; ++j) { ep[j] = 0.0; lp[j] = 0.0; mx[j] = -INFINITY; }
  }
  __device__ __forceinline__ void operator()(double y, double d, double u, int64_t = 0) {
#pragma unroll
    for (int j = 0; j < MWU_MAXC; ++j) {
      if (j < k.nc) {
        const double t = y + k.a[j] * d;
        mx[j] = fmax(mx[j], t);
        if (k.mP[j] == CM_EXPM1) {
          const double em = expm1(k.ea[j] * d);
          ep[j] = __fma_rn(u, em, ep[j]);
          if (j == 0) nd = __fma_rn(u + u * em, d, nd);                     // u e^{eta a dy} dy
        } else if (k.mP[j] == CM_LSE) {
          const double e = exp(eta * (t - k.shP[j]));
          lp[j] += e;
          if (j == 0) nd = __fma_rn(e, d, nd);
        }
      }
    }
  }
};

struct CRowGen {
  static constexpr double kAbsent = INFINITY;
  __device__ __forceinline__ void pair(double z0, double d0, double v0, double z1, double d1, double v1) {
    (*this)(z0, d0, v0);
    if (v1 != 0.0 || z1 != INFINITY) (*this)(z1, d1, v1);
  }
  const Cands& k;
  double neta;
  double ec[MWU_MAXC], tc[MWU_MAXC], mn[MWU_MAXC];
  double nd;                           // Newton: sum of the candidate-0 terms times d^(z)
  __device__ CRowGen(const Cands& kk, double ne) : k(kk), neta(ne), nd(0.0) {
#pragma unroll
    for (int j = 0; j < MWU_MAXC; ++j) { ec[j] = 0.0; tc[j] = 0.0; mn[j] = INFINITY; }
  }
  __device__ __forceinline__ void operator()(double z, double d, double v, int64_t = 0) {
#pragma unroll
    for (int j = 0; j < MWU_MAXC; ++j) {
      if (j < k.nc) {
        const double t = z + k.a[j] * d;
        mn[j] = fmin(mn[j], t);
        if (k.mC[j] == CM_EXPM1) {
          double em, q;
          expm1_exp(-(k.ea[j] * d), em, q);
          ec[j] = __fma_rn(v, em, ec[j]);
          tc[j] = __fma_rn(v, q, tc[j]);
          if (j == 0) nd = __fma_rn(v * q, d, nd);                          // v e^{-eta a dz} dz
        } else if (k.mC[j] == CM_LSE) {
          const double e = exp(neta * (t - k.shC[j]));
          tc[j] += e;
          if (j == 0) nd = __fma_rn(e, d, nd);
        }
      }
    }
  }
};

// Compacted covering rows: `ns` dense record streams (one per warp of the compacting kernel),
// stream w holding cnt[w] records (z, d^(z), v) from w * cap.  A search block takes the streams
// w = blockIdx.x, + gridDim.x, ... and streams them through shared memory in MWU_SCH-row chunks
// with the bulk-copy engine (the same stage ring as stream_rows3), two rows per thread at a time.
template <class F>
__device__ __forceinline__ void stream_recs3(const double* rz, const double* rdz, const double* rv,
                                             const int32_t* __restrict__ cnt, int64_t ns, int64_t cap,
                                             double* buf, uint64_t* bars, uint32_t& it, F& f) {
  int64_t iw = blockIdx.x, ioff = 0;               // producer cursor (thread 0)
  int64_t cw = blockIdx.x, coff = 0;               // consumer cursor (all threads)
  auto len = [&](int64_t w) -> int64_t { return (int64_t)__ldg(cnt + w); };
  auto skip_empty = [&](int64_t& w, int64_t& off) {
    while (w < ns && off >= len(w)) { w += gridDim.x; off = 0; }
  };
  auto issue = [&](uint32_t slot) {                // the chunk at the producer cursor
    skip_empty(iw, ioff);
    if (iw >= ns) return;
    const int64_t r0 = iw * cap + ioff;
    const int64_t rows = min((int64_t)MWU_SCH, len(iw) - ioff);
    const uint32_t bytes = (uint32_t)(((rows * 8) + 15) & ~15ll);
    double* s = buf + (size_t)slot * 3 * MWU_SCH;
    mbar_expect_tx(&bars[slot], 3 * bytes);
    const uint64_t pf = pol_first();
    tma_load_1d_hint(s, rz + r0, bytes, &bars[slot], pf);
    tma_load_1d_hint(s + MWU_SCH, rdz + r0, bytes, &bars[slot], pf);
    tma_load_1d_hint(s + 2 * MWU_SCH, rv + r0, bytes, &bars[slot], pf);
    ioff += rows;
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < MWU_SST; ++k) issue((it + (uint32_t)k) % MWU_SST);
  for (;;) {
    skip_empty(cw, coff);
    if (cw >= ns) break;
    const uint32_t slot = it % MWU_SST, parity = (it / MWU_SST) & 1u;
    mbar_wait(&bars[slot], parity);
    const int rows = (int)min((int64_t)MWU_SCH, len(cw) - coff);
    const double* s = buf + (size_t)slot * 3 * MWU_SCH;
    for (int r = threadIdx.x; r < rows; r += 2 * MWU_NT) {
      const int r1 = r + MWU_NT;
      if (r1 < rows) f.pair(s[r], s[MWU_SCH + r], s[2 * MWU_SCH + r], s[r1], s[MWU_SCH + r1], s[2 * MWU_SCH + r1]);
      else f.pair(s[r], s[MWU_SCH + r], s[2 * MWU_SCH + r], INFINITY, 0.0, 0.0);
    }
    coff += rows;
    __syncthreads();                                 // everyone is done with this slot
    if (threadIdx.x == 0) issue(slot);
    ++it;
  }
}

constexpr size_t kSearchSmem = (size_t)MWU_SST * 3 * MWU_SCH * sizeof(double);

struct SearchArgs {
  int64_t mP; const double *y, *dy, *u;                  // this rank's slice of the packing rows
  int64_t mP2; const double *y2, *dy2, *u2;              // + its own rows (owner-partitioned sharding)
  int64_t mC; const double *z, *dz, *v;                  // dense covering rows (v: weights)
  const double *rz, *rdz, *rv; const int32_t* tcnt; int64_t nstreams, rcap;   // compacted (rz != nullptr)
  const double* emtab;                                   // 768: T, T-1 hi, T-1 lo (fastmath.cuh)
};

template <int PT, int NC, bool SQ1>
__device__ __forceinline__ void search_body_fast(const SearchArgs& A, const Cands& K, const Ctl* c, double* sbuf,
                                                 uint64_t* bars, double* part,
                                                 const double* tab) {
  uint32_t it = 0;
  {
    PRowFast<PT, NC, SQ1> f(K, c->eta, tab);
    if (!c->pSing) stream_rows3(A.y, A.dy, A.u, A.mP, sbuf, bars, it, f);
    if (!c->pSing && A.mP2 > 0) stream_rows3(A.y2, A.dy2, A.u2, A.mP2, sbuf, bars, it, f);
    block_partials_op<NC, OP_SUM>(f.ep, part, R_EP(0), R_LP(0));   // LSE-mode candidates read R_LP
    block_partials_op<NC, OP_MAX>(f.mx, part, R_MX(0));
  }
  {
    CRowFast<PT, NC, SQ1> f(K, tab);
    if (!c->cSing) {
      if (A.rz) stream_recs3(A.rz, A.rdz, A.rv, A.tcnt, A.nstreams, A.rcap, sbuf, bars, it, f);
      else stream_rows3(A.z, A.dz, A.v, A.mC, sbuf, bars, it, f);
    }
    block_partials_op<NC, OP_SUM>(f.ec, part, R_EC(0));
    block_partials_op<NC, OP_SUM>(f.tc, part, R_TC(0));
    block_partials_op<NC, OP_MIN>(f.mn, part, R_MN(0));
  }
  if (threadIdx.x < 2) part[(size_t)blockIdx.x * MWU_SLOTS + R_NP + threadIdx.x] = 0.0;   // no Newton sums
}

__device__ __forceinline__ void search_body_gen(const SearchArgs& A, const Cands& K, const Ctl* c, double* sbuf,
                                                uint64_t* bars, double* part) {
  uint32_t it = 0;
  double nd[2] = {0.0, 0.0};           // Newton derivative sums (P side, C side)
  {
    PRowGen f(K, c->eta);
    if (!c->pSing) stream_rows3(A.y, A.dy, A.u, A.mP, sbuf, bars, it, f);
    if (!c->pSing && A.mP2 > 0) stream_rows3(A.y2, A.dy2, A.u2, A.mP2, sbuf, bars, it, f);
    nd[0] = f.nd;
    block_partials_op<MWU_MAXC, OP_SUM>(f.ep, part, R_EP(0));
    block_partials_op<MWU_MAXC, OP_SUM>(f.lp, part, R_LP(0));
    block_partials_op<MWU_MAXC, OP_MAX>(f.mx, part, R_MX(0));
  }
  {
    CRowGen f(K, -c->eta);
    if (!c->cSing) {
      if (A.rz) stream_recs3(A.rz, A.rdz, A.rv, A.tcnt, A.nstreams, A.rcap, sbuf, bars, it, f);
      else stream_rows3(A.z, A.dz, A.v, A.mC, sbuf, bars, it, f);
    }
    block_partials_op<MWU_MAXC, OP_SUM>(f.ec, part, R_EC(0));
    block_partials_op<MWU_MAXC, OP_SUM>(f.tc, part, R_TC(0));
    block_partials_op<MWU_MAXC, OP_MIN>(f.mn, part, R_MN(0));
    nd[1] = f.nd;
  }
  block_partials_op<2, OP_SUM>(nd, part, R_NP);
}

// One HBM pass evaluating the staged candidates (P:716-727 on cached vectors); the
// last block replays Alg. 3 (search_controller).
#ifndef MWU_SEARCH_MINB
#define MWU_SEARCH_MINB 2     // resident search CTAs per SM (grid = MWU_SEARCH_MINB x SMs)
#endif
__global__ void __launch_bounds__(MWU_NT, MWU_SEARCH_MINB) search_pass(SearchArgs A, Ctl* c, double* part, unsigned int* counter) {
  if (c->status != ST_RUNNING || !c->sactive) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(c->h_search, 0u);
    return;
  }
  Cands K;
  K.nc = c->ncand; K.pt = c->ptype;
  K.ea0 = c->eta * c->pa0; K.ead = c->eta * c->pdelta;
  bool fast = (K.pt == PT_DOUBLE || K.pt == PT_GRID || (K.pt == PT_G16 && K.nc == MWU_MAXC));
  bool sq1 = true;
#pragma unroll
  for (int j = 0; j < MWU_MAXC; ++j) {
    K.a[j] = c->cand[j]; K.ea[j] = c->cea[j]; K.shP[j] = c->shP[j]; K.shC[j] = c->shC[j];
    K.mP[j] = c->cmP[j]; K.mC[j] = c->cmC[j]; K.sq[j] = c->csq[j];
    if (j < K.nc) {
      if (K.pt == PT_DOUBLE && j > 0 && K.sq[j] != 1) sq1 = false;
      if (!(c->pSing || K.mP[j] == CM_EXPM1 || K.mP[j] == CM_LSE)) fast = false;
      if (!(c->cSing || K.mC[j] == CM_EXPM1)) fast = false;
    }
  }
  extern __shared__ __align__(128) double sbuf[];
  __shared__ __align__(8) uint64_t bars[MWU_SST];
  __shared__ double s_tab[768];
  for (int i = threadIdx.x; i < 768; i += MWU_NT) s_tab[i] = A.emtab[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < MWU_SST; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (fast) {
#define MWU_FAST_CASE(PTV, N, S) \
    if (K.pt == PTV && K.nc == N && sq1 == S) search_body_fast<PTV, N, S>(A, K, c, sbuf, bars, part, s_tab); else
    MWU_FAST_CASE(PT_DOUBLE, 8, true) MWU_FAST_CASE(PT_DOUBLE, 7, true) MWU_FAST_CASE(PT_DOUBLE, 6, true)
    MWU_FAST_CASE(PT_DOUBLE, 5, true) MWU_FAST_CASE(PT_DOUBLE, 4, true) MWU_FAST_CASE(PT_DOUBLE, 3, true)
    MWU_FAST_CASE(PT_DOUBLE, 2, true) MWU_FAST_CASE(PT_DOUBLE, 1, true)
    MWU_FAST_CASE(PT_DOUBLE, 8, false) MWU_FAST_CASE(PT_DOUBLE, 7, false) MWU_FAST_CASE(PT_DOUBLE, 6, false)
    MWU_FAST_CASE(PT_DOUBLE, 5, false) MWU_FAST_CASE(PT_DOUBLE, 4, false) MWU_FAST_CASE(PT_DOUBLE, 3, false)
    MWU_FAST_CASE(PT_DOUBLE, 2, false)
    MWU_FAST_CASE(PT_GRID, 7, true) MWU_FAST_CASE(PT_GRID, 3, true) MWU_FAST_CASE(PT_GRID, 1, true)
    MWU_FAST_CASE(PT_G16, MWU_MAXC, true)
    search_body_gen(A, K, c, sbuf, bars, part);
#undef MWU_FAST_CASE
  } else {
    search_body_gen(A, K, c, sbuf, bars, part);
  }
  __shared__ double res[MWU_SLOTS];
  int ops[MWU_SLOTS];
#pragma unroll
  for (int s = 0; s < MWU_SLOTS; ++s) ops[s] = search_slot_op(s);
  if (last_block_combine(ops, MWU_SLOTS, part, counter, res)) {
    if (threadIdx.x == 0) finish(c, A_SEARCH, res, ops, MWU_SLOTS);
  }
}

// y += alpha d^(y), z += alpha d^(z) fused with u = exp(eta (y - s_P)),
// v = exp(-eta (z - s_C)) at the accepted alpha's shifts, and S_P, S_C.
// has_delta = 0: initial weights only (init) with shifts from A_INIT_EXT.
// Packing rows [0, mP) — or, on an owner-partitioned sharded matching, the
// replicated rows [0, mP) plus this rank's own rows [R0, R1), whose weight sum goes to slot 2.
__global__ void __launch_bounds__(MWU_NT) update_rows(int64_t mP, double* __restrict__ y, const double* __restrict__ dy,
                                                      double* __restrict__ u, int64_t mC, double* __restrict__ z,
                                                      const double* __restrict__ dz, double* __restrict__ v, Ctl* c,
                                                      double* part, unsigned int* counter, int has_delta,
                                                      int64_t R0, int64_t R1) {
  if (c->status != ST_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(c->h_iter, 0u);
    return;
  }
  const double a = c->alpha, eta = c->eta, neta = -c->eta;
  const double sP = has_delta ? c->newsP : c->sP, sC = has_delta ? c->newsC : c->sC;
  double acc[3] = {0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * MWU_NT;
  const int64_t tid = (int64_t)blockIdx.x * MWU_NT + threadIdx.x;
  for (int64_t i = tid; i < mP; i += stride) {
    double yi = y[i];
    if (has_delta) { yi = yi + a * dy[i]; y[i] = yi; }
    const double w = exp(eta * (yi - sP));
    if (u) u[i] = w;
    acc[0] += w;
  }
  for (int64_t i = R0 + tid; i < R1; i += stride) {
    double yi = y[i];
    if (has_delta) { yi = yi + a * dy[i]; y[i] = yi; }
    const double w = exp(eta * (yi - sP));
    if (u) u[i] = w;
    acc[2] += w;
  }
  for (int64_t i = tid; i < mC; i += stride) {
    double zi = z[i];
    if (has_delta) { zi = zi + a * dz[i]; z[i] = zi; }
    const double w = exp(neta * (zi - sC));
    if (v) v[i] = w;
    acc[1] += w;
  }
  const int ops[3] = {OP_SUM, OP_SUM, OP_SUM};
  reduce_and_finalize<3>(acc, ops, part, counter, c, has_delta ? A_UPDATE : A_INIT_W);
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
                                                 double cm, Ctl* c, double* part, unsigned int* counter,
                                                 int64_t n_all) {
  const double eps = c->eps, nd = (double)n_all, invB = c->invB;   // n = #variables of the LP (Q3)
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
// owner-partitioned rows: keep the replicated prefix [0, nL) on rank 0 only and the own rows
// [R0, R1); zeros elsewhere (a sum over ranks then assembles the whole vector exactly)
__global__ void own_mask(int64_t m, const double* __restrict__ in, double* __restrict__ out, int64_t nL, int64_t R0,
                         int64_t R1, int keep_prefix) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ((i < nL && keep_prefix) || (i >= R0 && i < R1)) ? in[i] : 0.0;
}
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


// =====================================================================================
// Fast densest path: column kernel fused with the lazy z update, the weights
// v = exp(-eta (z - s_C)) recomputed from z, the forward product d^(y) = (1/D) O d scattered
// with fp64 reductions into the (L2-resident) vertex vector, and per-tile compaction of the
// covering rows with d^(z) > 0 for the search passes.
// =====================================================================================
// Warp-segmented sum over runs of equal keys held by consecutive lanes (edges sorted by src row,
// or any order: a key that reappears after a different key starts a new run).  The last lane
// of each run returns the run's sum in `out` (others return false).  The scan adds lane - o only
// when it lies inside the lane's own run (run start from a ballot of the heads), so keys
// A, B, A in one warp are three runs, never one.
__device__ __forceinline__ bool warp_run_sum(int key, double val, double& out) {
  const int lane = threadIdx.x & 31;
  const int pk = __shfl_up_sync(0xffffffffu, key, 1);
  const uint32_t heads = __ballot_sync(0xffffffffu, lane == 0 || pk != key);
  const int start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));   // first lane of my run
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double ov = __shfl_up_sync(0xffffffffu, val, o);
    if (lane - o >= start) val += ov;
  }
  const int nk = __shfl_down_sync(0xffffffffu, key, 1);
  out = val;
  return lane == 31 || nk != key;
}

__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}


// act: bit e = (d_2e, d_2e+1) != 0 in the last computed direction (word e >> 5, bit e & 31).
// Edges with a clear bit have d = 0 (their d slots in memory are stale and never read), so the
// kernel reads x and d, and writes x, z and d, only for edges active in this or the last step.
__device__ __forceinline__ bool act_bit(const uint32_t* act, int e) { return (__ldg(act + (e >> 5)) >> (e & 31)) & 1u; }

// The per-edge stream of each 1024-edge tile (z, src/dst rows, activity words) is staged into
// shared memory by the bulk-copy engine (cp.async.bulk + mbarrier) kColStages tiles ahead; the
// u gathers of tile i+1 are issued (registers) before tile i is computed.  Stages are released per warp (an 8-arrival "empty" mbarrier), so
// only the producer thread waits for the slowest warp; no block-wide barrier in the loop.
#ifndef MWU_COL_MINB
#define MWU_COL_MINB 2        // resident column CTAs per SM (grid = MWU_COL_MINB x SMs)
#endif
#ifndef MWU_COL_STAGES
#define MWU_COL_STAGES 4
#endif
constexpr int kColStages = MWU_COL_STAGES;
constexpr int kColOffS = MWU_CT * 8, kColOffD = kColOffS + MWU_CT * 4, kColOffA = kColOffD + MWU_CT * 4;
constexpr int kColStageBytes = ((kColOffA + (MWU_CT / 32) * 4) + 127) / 128 * 128;
constexpr size_t kColSmem = (size_t)kColStages * kColStageBytes;

__device__ __forceinline__ uint32_t r16(uint32_t b) { return (b + 15u) & ~15u; }

__device__ __forceinline__ void col_issue(char* stage, uint64_t* bar, int tile, int E, const double* z,
                                          const int32_t* srow, const int32_t* drow, const uint32_t* act) {
  const int e0 = tile * MWU_CT;
  const int rows = min(MWU_CT, E - e0);
  const uint32_t bz = r16(rows * 8u), bi = r16(rows * 4u), ba = r16(((rows + 31) / 32) * 4u);
  mbar_expect_tx(bar, bz + 2 * bi + ba);
  const uint64_t pf = pol_first();
  tma_load_1d_hint(stage, z + e0, bz, bar, pf);
  tma_load_1d_hint(stage + kColOffS, srow + e0, bi, bar, pf);
  tma_load_1d_hint(stage + kColOffD, drow + e0, bi, bar, pf);
  tma_load_1d(stage + kColOffA, act + (e0 >> 5), ba, bar);
}

// this thread's u gathers of a staged tile (registers; issued one tile ahead of their use)
__device__ __forceinline__ void col_gather(const char* stage, int rows, const double* __restrict__ u, double* us,
                                           double* ud) {
  const int32_t* ssr = reinterpret_cast<const int32_t*>(stage + kColOffS);
  const int32_t* sdr = reinterpret_cast<const int32_t*>(stage + kColOffD);
#pragma unroll
  for (int k = 0; k < kColEdges; ++k) {
    const int j = k * MWU_NT + threadIdx.x;
    if (j < rows) { us[k] = __ldg(u + ssr[j]); ud[k] = __ldg(u + sdr[j]); }
  }
}

__global__ void __launch_bounds__(MWU_NT, MWU_COL_MINB) col_densest_fast(
    int64_t E64, const int32_t* __restrict__ srow, const int32_t* __restrict__ drow, const double* __restrict__ u,
    double* __restrict__ x, double* __restrict__ d, double* __restrict__ z, double* __restrict__ dy,
    uint32_t* __restrict__ act, double* __restrict__ rz, double* __restrict__ rdz, double* __restrict__ rv,
    int32_t* __restrict__ tcnt, int64_t rcap, double* gdbg, double* hdbg, Ctl* c, double* part,
    unsigned int* counter, const double* __restrict__ exptab) {
  if (c->status != ST_RUNNING) return;
  __shared__ double s_tab[256];                                   // 2^(j/256), host-rounded
  s_tab[threadIdx.x] = exptab[threadIdx.x];                       // MWU_NT == 256
  const double rSP = 1.0 / c->SP, rSC = 1.0 / c->SC, invD = c->invB, sigma = c->sigma, ap = c->alpha_prev;
  const double neta = -c->eta, sC = c->sC;
  const int apply = c->apply_prev;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int E = (int)E64;                  // the fast path requires E < 2^31 - MWU_CT (host check)
  double maxd = 0.0;                       // every d >= 0 and E > 0: max d >= 0 (inactive rows add 0)
  double im = INFINITY, is = 0.0;          // inactive rows: min z and sum of v (shift s_C)
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* d2 = reinterpret_cast<double2*>(d);
  extern __shared__ __align__(128) char csm[];
  __shared__ __align__(8) uint64_t full[kColStages], empty[kColStages];
  const int ntiles = (E + MWU_CT - 1) / MWU_CT;
  const int mine = (ntiles > (int)blockIdx.x) ? (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kColStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MWU_NT / 32); }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < mine && k < kColStages; ++k)
      col_issue(csm + k * kColStageBytes, &full[k], blockIdx.x + k * gridDim.x, E, z, srow, drow, act);
  // compaction of the active covering rows: each warp appends its records to its own dense
  // stream [w0, w0 + rcap) in (tile, k, lane) order; the count goes to tcnt at the end
  const int64_t w0 = ((int64_t)blockIdx.x * (MWU_NT / 32) + warp) * rcap;
  int64_t wp = w0;
  double us[kColEdges], ud[kColEdges], nus[kColEdges], nud[kColEdges];
  if (mine > 0) {
    mbar_wait(&full[0], 0u);
    col_gather(csm, min(MWU_CT, E - (int)blockIdx.x * MWU_CT), u, us, ud);
  }
  // double-buffered gather registers (no register moves that would wait on the loads)
  auto body = [&](int kt, double (&us)[kColEdges], double (&ud)[kColEdges], double (&nus)[kColEdges],
                  double (&nud)[kColEdges]) {
    const int tile = blockIdx.x + kt * gridDim.x;
    const int slot = kt % kColStages;
    char* stg = csm + slot * kColStageBytes;
    const int e0 = tile * MWU_CT;
    const int rows = min(MWU_CT, E - e0);
    // the next tile's gathers are in flight while this one is computed
    if (kt + 1 < mine) {
      const int ns = (kt + 1) % kColStages;
      mbar_wait(&full[ns], (uint32_t)(((kt + 1) / kColStages) & 1));
      col_gather(csm + ns * kColStageBytes, min(MWU_CT, E - (tile + (int)gridDim.x) * MWU_CT), u, nus, nud);
    }
    const double* sz = reinterpret_cast<const double*>(stg);
    const int32_t* ssr = reinterpret_cast<const int32_t*>(stg + kColOffS);
    const int32_t* sdr = reinterpret_cast<const int32_t*>(stg + kColOffD);
    const uint32_t* sac = reinterpret_cast<const uint32_t*>(stg + kColOffA);
    double2 xe[kColEdges], dp[kColEdges];
    bool had[kColEdges];
    uint32_t pw[kColEdges];
#pragma unroll
    for (int k = 0; k < kColEdges; ++k) {                        // x, d of the previously active
      const int j = k * MWU_NT + threadIdx.x;
      pw[k] = j < rows ? sac[j >> 5] : 0u;
      had[k] = (pw[k] >> lane) & 1u;
      // x of EVERY edge, issued at the tile start: an edge that turns active needs it for its
      // direction, and a load issued only then stalls the warp (measured: column 4.03 -> 3.73 ms
      // on c4 despite the extra reads of edges that stay inactive)
      if (j < rows) xe[k] = x2[e0 + j];
      if (had[k]) dp[k] = d2[e0 + j];
    }
#pragma unroll
    for (int k = 0; k < kColEdges; ++k) {
      const int j = k * MWU_NT + threadIdx.x;
      const int e = e0 + j;
      const bool valid = j < rows;
      double zz = valid ? sz[j] : INFINITY;
      const int sr = valid ? ssr[j] : -1, dr = valid ? sdr[j] : -1;
      double d0 = 0.0, d1 = 0.0, v = 0.0;
      if (valid) {
        if (apply && had[k]) {                                    // lazy x, z += alpha d
          xe[k].x = xe[k].x + ap * dp[k].x;
          xe[k].y = xe[k].y + ap * dp[k].y;
          x2[e] = xe[k];
          const double dzp = dp[k].x + dp[k].y;                   // d^(z)_e = (W d)_e of the last step
          zz = zz + ap * dzp;
          z[e] = zz;
        }
        v = mwu_exp_tab(neta * (zz - sC), s_tab);                 // covering weight (Q4)
        const double h = v * rSC;                                 // W^T w_c
        const double g0 = invD * (us[k] * rSP);                   // (1/D) O^T w_p
        const double g1 = invD * (ud[k] * rSP);
        if (gdbg) { gdbg[2 * e] = g0; gdbg[2 * e + 1] = g1; hdbg[2 * e] = h; hdbg[2 * e + 1] = h; }
        // g >= h gives fl(g/h) >= 1, i.e. d = 0 exactly
        const bool a0 = g0 < h, a1 = g1 < h;
        if (a0) d0 = mwu_direction(g0, h, xe[k].x, sigma);
        if (a1) d1 = mwu_direction(g1, h, xe[k].y, sigma);
      }
      const double dz = d0 + d1;
      const bool nz = dz > 0.0;
      const uint32_t bw = __ballot_sync(0xffffffffu, nz);
      if (nz) {
        d2[e] = make_double2(d0, d1);
        const double m01 = d0 > d1 ? d0 : d1;
        maxd = m01 > maxd ? m01 : maxd;
        const int64_t p = wp + __popc(bw & ((1u << lane) - 1u));
        rz[p] = zz; rdz[p] = dz; rv[p] = v;
      } else if (valid) { im = zz < im ? zz : im; is += v; }       // candidate-independent row
      wp += __popc(bw);
      if (lane == 0 && valid && bw != pw[k]) act[e >> 5] = bw;
      if (d1 > 0.0) red_add_f64(dy + dr, invD * d1);              // dst side: random rows
      // src side: edges are sorted by src within an L2 block, so lanes hold runs of equal rows
      const double val = d0 > 0.0 ? invD * d0 : 0.0;
      if (__any_sync(0xffffffffu, val > 0.0)) {
        double run;
        if (warp_run_sum(sr, val, run) && run > 0.0) red_add_f64(dy + sr, run);
      }
    }
    // this warp is done with the stage: release it
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (threadIdx.x == 0 && kt + kColStages < mine) {           // producer: refill once all warps left
      mbar_wait(&empty[slot], (uint32_t)((kt / kColStages) & 1));
      col_issue(stg, &full[slot], blockIdx.x + (kt + kColStages) * gridDim.x, E, z, srow, drow, act);
    }
  };
  for (int kt = 0; kt < mine; ++kt) {
    body(kt, us, ud, nus, nud);
#pragma unroll
    for (int q = 0; q < kColEdges; ++q) { us[q] = nus[q]; ud[q] = nud[q]; }
  }
  if (lane == 0) tcnt[blockIdx.x * (MWU_NT / 32) + warp] = (int32_t)(wp - w0);
  double acc[3] = {maxd, im, is};
  const int ops[3] = {OP_MAX, OP_MIN, OP_SUM};
  reduce_and_finalize<3>(acc, ops, part, counter, c, A_COL_FAST);
}

// Fast MATCH / BMATCH column (P = M, C = (1/M) 1^T): lazy x += alpha d,
// g_e = w_p[r(src)] + w_p[r(dst)] (M^T), d_e, and the forward product
// d^(y) = M d scattered into the vertex vector (src side: warp-segmented runs of the sorted edge
// list; dst side: one fp64 reduction per nonzero d_e).  Reduces max d and sum(d)/M.
// Fed like the c4 kernel: each 1024-edge tile's stream (src / dst rows, activity words) is
// staged in shared memory by the bulk-copy engine kColStages tiles ahead, and the u gathers of
// tile i+1 are in flight while tile i is computed, so every thread keeps 2 kColEdges random
// gathers outstanding (the kernel is bound by the latency of the random destination-side
// gathers; c5 column 24.3 -> 20.4 ms against a grid-stride loop).
constexpr int kMOffD = MWU_CT * 4, kMOffA = kMOffD + MWU_CT * 4;
constexpr int kMStageBytes = ((kMOffA + (MWU_CT / 32) * 4) + 127) / 128 * 128;
constexpr size_t kMSmem = (size_t)kColStages * kMStageBytes;
#ifndef MWU_MT_MINB
#define MWU_MT_MINB 2
#endif

__device__ __forceinline__ void mt_issue(char* stage, uint64_t* bar, int tile, int64_t E, const int32_t* srow,
                                         const int32_t* drow, const uint32_t* act) {
  const int64_t e0 = (int64_t)tile * MWU_CT;
  const int rows = (int)min((int64_t)MWU_CT, E - e0);
  const uint32_t bi = r16(rows * 4u), ba = r16(((rows + 31) / 32) * 4u);
  mbar_expect_tx(bar, 2 * bi + ba);
  const uint64_t pf = pol_first();
  tma_load_1d_hint(stage, srow + e0, bi, bar, pf);
  tma_load_1d_hint(stage + kMOffD, drow + e0, bi, bar, pf);
  tma_load_1d_hint(stage + kMOffA, act + (e0 >> 5), ba, bar, pf);
}

__device__ __forceinline__ void mt_gather(const char* stage, int rows, const double* __restrict__ u, double* us,
                                          double* ud) {
  const int32_t* ssr = reinterpret_cast<const int32_t*>(stage);
  const int32_t* sdr = reinterpret_cast<const int32_t*>(stage + kMOffD);
#pragma unroll
  for (int k = 0; k < kColEdges; ++k) {
    const int j = k * MWU_NT + threadIdx.x;
    if (j < rows) { us[k] = __ldg(u + ssr[j]); ud[k] = __ldg(u + sdr[j]); }
  }
}

__global__ void __launch_bounds__(MWU_NT, MWU_MT_MINB) col_match_fast(
    int64_t E64, const int32_t* __restrict__ srow, const int32_t* __restrict__ drow, const double* __restrict__ u,
    double* __restrict__ x, double* __restrict__ d, double* __restrict__ dy, double* gdbg, double* hdbg, Ctl* c,
    double* part, unsigned int* counter, uint32_t* __restrict__ act) {
  if (c->status != ST_RUNNING) return;
  const double rSP = 1.0 / c->SP, invB = c->invB, sigma = c->sigma, ap = c->alpha_prev;
  const int apply = c->apply_prev;
  const int lane = threadIdx.x & 31;
  const int64_t E = E64;
  double acc[2] = {-INFINITY, 0.0};
  extern __shared__ __align__(128) char csm[];
  __shared__ __align__(8) uint64_t full[kColStages], empty[kColStages];
  const int ntiles = (int)((E + MWU_CT - 1) / MWU_CT);
  const int mine = (ntiles > (int)blockIdx.x) ? (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kColStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MWU_NT / 32); }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < mine && k < kColStages; ++k)
      mt_issue(csm + k * kMStageBytes, &full[k], blockIdx.x + k * gridDim.x, E, srow, drow, act);
  double us[kColEdges], ud[kColEdges], nus[kColEdges], nud[kColEdges];
  if (mine > 0) {
    mbar_wait(&full[0], 0u);
    mt_gather(csm, (int)min((int64_t)MWU_CT, E - (int64_t)blockIdx.x * MWU_CT), u, us, ud);
  }
  auto body = [&](int kt, double (&us)[kColEdges], double (&ud)[kColEdges], double (&nus)[kColEdges],
                  double (&nud)[kColEdges]) {
    const int tile = blockIdx.x + kt * gridDim.x;
    const int slot = kt % kColStages;
    char* stg = csm + slot * kMStageBytes;
    const int64_t e0 = (int64_t)tile * MWU_CT;
    const int rows = (int)min((int64_t)MWU_CT, E - e0);
    if (kt + 1 < mine) {
      const int ns = (kt + 1) % kColStages;
      mbar_wait(&full[ns], (uint32_t)(((kt + 1) / kColStages) & 1));
      const int nrows = (int)min((int64_t)MWU_CT, E - (int64_t)(tile + (int)gridDim.x) * MWU_CT);
      mt_gather(csm + ns * kMStageBytes, nrows, u, nus, nud);
    }
    const int32_t* ssr = reinterpret_cast<const int32_t*>(stg);
    const int32_t* sdr = reinterpret_cast<const int32_t*>(stg + kMOffD);
    const uint32_t* sac = reinterpret_cast<const uint32_t*>(stg + kMOffA);
    double xe[kColEdges], dp[kColEdges];
    uint32_t pw[kColEdges];
#pragma unroll
    for (int k = 0; k < kColEdges; ++k) {                        // x, d of the previously active
      const int j = k * MWU_NT + threadIdx.x;
      pw[k] = j < rows ? sac[j >> 5] : 0u;
      dp[k] = 0.0;
      const bool had = (pw[k] >> lane) & 1u;
      // x of EVERY edge, issued at the tile start (an edge that turns active needs it for its
      // direction; a load issued only then stalls the warp: c5 column 22.7 -> 20.4 ms)
      if (j < rows) xe[k] = x[e0 + j];
      if (had) dp[k] = d[e0 + j];
    }
#pragma unroll
    for (int k = 0; k < kColEdges; ++k) {
      const int j = k * MWU_NT + threadIdx.x;
      const int64_t e = e0 + j;
      const bool valid = j < rows;
      const int sr = valid ? ssr[j] : -1, dr = valid ? sdr[j] : -1;
      const bool had = (pw[k] >> lane) & 1u;
      double de = 0.0;
      if (valid) {
        if (apply && had) { xe[k] = xe[k] + ap * dp[k]; x[e] = xe[k]; }             // P:677 (lazy)
        const double g = us[k] * rSP + ud[k] * rSP;                                 // M^T w_p
        if (g < invB) {                                                             // g >= h: d = 0
          de = mwu_direction(g, invB, xe[k], sigma);
        }
        if (de > 0.0 && de != dp[k]) d[e] = de;                                     // zeros live in `act`
        if (gdbg) { gdbg[e] = g; hdbg[e] = invB; }
        acc[0] = fmax(acc[0], de);
        acc[1] += invB * de;
      }
      const bool want = de > 0.0;
      const uint32_t bw = __ballot_sync(0xffffffffu, want);
      if (lane == 0 && valid && bw != pw[k]) act[e >> 5] = bw;
      if (want) red_add_f64(dy + dr, de);                         // dst side
      if (__any_sync(0xffffffffu, want)) {                        // src side: sorted runs
        double run;
        if (warp_run_sum(sr, de, run) && run > 0.0) red_add_f64(dy + sr, run);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (threadIdx.x == 0 && kt + kColStages < mine) {
      mbar_wait(&empty[slot], (uint32_t)((kt / kColStages) & 1));
      mt_issue(stg, &full[slot], blockIdx.x + (kt + kColStages) * gridDim.x, E, srow, drow, act);
    }
  };
  for (int kt = 0; kt < mine; ++kt) {
    body(kt, us, ud, nus, nud);
#pragma unroll
    for (int q = 0; q < kColEdges; ++q) { us[q] = nus[q]; ud[q] = nud[q]; }
  }
  const int ops[2] = {OP_MAX, OP_SUM};
  reduce_and_finalize<2>(acc, ops, part, counter, c, A_COL);
}

// Init forward product y = P x of the edge-variable kinds by scatter (fast path):
// MATCH: y_r += x_e for both endpoints (P = M); DENSEST: y_r += (1/D) x_{2e+b} (P = O/D).
__global__ void scatter_init(int64_t E, const int32_t* __restrict__ srow, const int32_t* __restrict__ drow,
                             const double* __restrict__ x, double* __restrict__ y, const Ctl* c, int pairs) {
  const double s = c->invB;
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT) {
    if (pairs) {
      red_add_f64(y + srow[e], s * x[2 * e]);
      red_add_f64(y + drow[e], s * x[2 * e + 1]);
    } else {
      red_add_f64(y + srow[e], x[e]);
      red_add_f64(y + drow[e], x[e]);
    }
  }
}

// =====================================================================================
// Fast transposed / forward products of the pure covering kinds (vcover c2, domset c3)
// =====================================================================================
// VCOVER (C = M^T): hs_v += v_e for both endpoints of every edge (h = M w_c), the src
// side as warp-segmented runs of the sorted edge list, the dst side one fp64 reduction per edge
// into the (L2-resident) vertex vector.
__global__ void __launch_bounds__(MWU_NT) vc_scatter(int64_t E, const int32_t* __restrict__ src,
                                                     const int32_t* __restrict__ dst, const double* __restrict__ v,
                                                     double* __restrict__ hs, const Ctl* c) {
  if (c->status != ST_RUNNING) return;
  constexpr int U = 4;
  const int64_t chunk = (int64_t)U * MWU_NT;
  for (int64_t base = (int64_t)blockIdx.x * chunk; base < E; base += (int64_t)gridDim.x * chunk) {
    double val[U];
    int sr[U], dr[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = base + k * MWU_NT + threadIdx.x;
      if (e < E) { val[k] = __ldcs(v + e); sr[k] = __ldcs(src + e); dr[k] = __ldcs(dst + e); }
      else { val[k] = 0.0; sr[k] = -1; dr[k] = -1; }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (dr[k] >= 0) red_add_f64(hs + dr[k], val[k]);
      double run;
      if (warp_run_sum(sr[k], val[k], run) && sr[k] >= 0) red_add_f64(hs + sr[k], run);
    }
  }
}

// CSR rows sorted (row id per nonzero): out_r += w[col_k] (all values 1.0: C = I + A)
__global__ void __launch_bounds__(MWU_NT) csr_scatter(int64_t nnz, const int32_t* __restrict__ rowid,
                                                      const uint32_t* __restrict__ col, const double* __restrict__ w,
                                                      double* __restrict__ out, const Ctl* c, int64_t row_base) {
  if (c->status != ST_RUNNING) return;
  // each thread sums 4 consecutive nonzeros (rows are sorted, so they hold at most a head
  // segment, interior segments and a tail segment); interior segments are emitted directly,
  // heads / tails are joined across lanes by one segmented scan: ~14 shuffles per 4 nonzeros
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)U * MWU_NT;
  const bool al16 = (((uintptr_t)rowid | (uintptr_t)col) & 15) == 0;      // q0 is a multiple of 4
  // row / column ids of the 4 nonzeros at q0 (16-byte loads where aligned and in range)
  auto load_ids = [&](int64_t q0, int (&rr)[U], uint32_t (&cc)[U]) {
    if (q0 + U <= nnz && al16) {
      const int4 a = __ldcs(reinterpret_cast<const int4*>(rowid + q0));
      const uint4 b = __ldcs(reinterpret_cast<const uint4*>(col + q0));
      rr[0] = a.x; rr[1] = a.y; rr[2] = a.z; rr[3] = a.w;
      cc[0] = b.x; cc[1] = b.y; cc[2] = b.z; cc[3] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const bool in = q0 + k < nnz;
        rr[k] = in ? __ldcs(rowid + q0 + k) : -1;
        cc[k] = in ? __ldcs(col + q0 + k) : 0u;
      }
    }
  };
  int rn[U];
  uint32_t cn[U];
  const int64_t stride = (int64_t)gridDim.x * chunk;
  int64_t base = (int64_t)blockIdx.x * chunk;
  if (base < nnz) load_ids(base + (int64_t)threadIdx.x * U, rn, cn);
  for (; base < nnz; base += stride) {
    int r[U];
    uint32_t ci[U];
    double val[U];
#pragma unroll
    for (int k = 0; k < U; ++k) { r[k] = rn[k]; ci[k] = cn[k]; }
    // ids of the next chunk are requested before this chunk's gathers (two chunks in flight)
    if (base + stride < nnz) load_ids(base + stride + (int64_t)threadIdx.x * U, rn, cn);
#pragma unroll
    for (int k = 0; k < U; ++k) val[k] = (r[k] >= 0) ? __ldg(w + ci[k]) : 0.0;
    // out-of-range entries (r = -1) only occur at the end, after every valid one
    const int kh = r[0], kt = r[U - 1];
    double head = 0.0, tail = 0.0;
    const bool single = (kh == kt);
    if (single) {
#pragma unroll
      for (int k = 0; k < U; ++k) tail += val[k];
    } else {
      int cur = kh;
      double acc = 0.0;
      bool first = true;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (r[k] != cur) {
          if (first) { head = acc; first = false; }
          else if (cur >= 0) red_add_f64(out + (cur - row_base), acc);     // interior segment
          cur = r[k]; acc = 0.0;
        }
        acc += val[k];
      }
      tail = acc;                                                          // cur == kt
    }
    const int kt_prev = __shfl_up_sync(0xffffffffu, kt, 1);
    const int kh_next = __shfl_down_sync(0xffffffffu, kh, 1);
    const bool cont = lane > 0 && single && kt_prev == kh;                 // continues lane - 1's run
    const uint32_t heads = __ballot_sync(0xffffffffu, !cont);
    const int start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));   // first lane of my run
    double P = tail;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, P, o);
      if (lane - o >= start) P += t;
    }
    const double P_prev = __shfl_up_sync(0xffffffffu, P, 1);
    if (!single && lane > 0 && kt_prev == kh) head += P_prev;              // run entering my head
    if (!single && kh >= 0) red_add_f64(out + (kh - row_base), head);
    if (kt >= 0 && (lane == 31 || kh_next != kt)) red_add_f64(out + (kt - row_base), P);
  }
}

// Sharded domset: the local rows' contribution to C^T v (C symmetric): out[col_k] += w[row_k - base]
__global__ void __launch_bounds__(MWU_NT) csr_scatter_T(int64_t nnz, const int32_t* __restrict__ rowid,
                                                        const uint32_t* __restrict__ col, const double* __restrict__ w,
                                                        int64_t row_base, double* __restrict__ out, const Ctl* c) {
  if (c->status != ST_RUNNING) return;
  for (int64_t q = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * MWU_NT)
    red_add_f64(out + __ldcs(col + q), __ldg(w + (__ldcs(rowid + q) - row_base)));
}

// Column epilogue over the variables (pure covering, P = (1/M) 1^T): lazy x += alpha d,
// h = (C^T v)_i / S_C, g = 1/M, d; reduces max d and sum(d)/M.
__global__ void __launch_bounds__(MWU_NT) col_vertex(int64_t n, const double* __restrict__ hs, double* __restrict__ x,
                                                     double* __restrict__ d, double* gdbg, double* hdbg, Ctl* c,
                                                     double* part, unsigned int* counter) {
  if (c->status != ST_RUNNING) return;
  const double SC = c->SC, g = c->invB, sigma = c->sigma, ap = c->alpha_prev, invB = c->invB;
  const int apply = c->apply_prev;
  double acc[2] = {-INFINITY, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * MWU_NT) {
    double xi = x[i];
    const double dp = d[i];
    if (apply && dp != 0.0) { xi = xi + ap * dp; x[i] = xi; }
    const double h = hs[i] / SC;
    const double di = (g < h) ? mwu_direction(g, h, xi, sigma) : 0.0;
    if (di != dp) d[i] = di;
    if (gdbg) { gdbg[i] = g; hdbg[i] = h; }
    acc[0] = fmax(acc[0], di);
    acc[1] += invB * di;
  }
  const int ops[2] = {OP_MAX, OP_SUM};
  reduce_and_finalize<2>(acc, ops, part, counter, c, A_COL);
}

// Forward product done (scattered): set up the step search.
__global__ void step_done(Ctl* c) {
  if (threadIdx.x != 0) return;
  if (c->status != ST_RUNNING) { set_cond(c->h_search, 0u); return; }
  double r[MWU_SLOTS];
  for (int s = 0; s < MWU_SLOTS; ++s) r[s] = 0.0;
  finalize(c, A_STEP_DONE, r);
}

// Rare path of the inactive-row aggregate: when min_inactive z - s_C exceeds 600/eta the sum of
// v at shift s_C may have lost terms to underflow; recompute it at shift mzi exactly.
__global__ void __launch_bounds__(MWU_NT) inactive_exact(int64_t E, const uint32_t* __restrict__ act,
                                                         const double* __restrict__ z, Ctl* c, double* part,
                                                         unsigned int* counter) {
  if (c->status != ST_RUNNING || !c->vi_exact) return;
  const double neta = -c->eta, m = c->mzi;
  double acc[1] = {0.0};
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT)
    if (!act_bit(act, (int)e)) acc[0] += exp(neta * (z[e] - m));
  const int ops[1] = {OP_SUM};
  reduce_and_finalize<1>(acc, ops, part, counter, c, A_VI_EXACT);
}

// max d^(y) over the packing rows once the scattered forward product is complete; sets up the
// step search (A_STEP_DONE).
__global__ void __launch_bounds__(MWU_NT) dy_finalize(int64_t mP, const double* __restrict__ dy, Ctl* c, double* part,
                                                      unsigned int* counter) {
  if (c->status != ST_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(c->h_search, 0u);
    return;
  }
  double acc[1] = {-INFINITY};
  for (int64_t i = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; i < mP; i += (int64_t)gridDim.x * MWU_NT)
    acc[0] = fmax(acc[0], dy[i]);
  const int ops[1] = {OP_MAX};
  reduce_and_finalize<1>(acc, ops, part, counter, c, A_STEP_DONE + 100);
}

// Apply the pending lazy update x += alpha d, z += alpha (W d) (end of probe / vector hooks).
__global__ void flush_pairs(int64_t E, double* __restrict__ x, const double* __restrict__ d, double* __restrict__ z,
                            const uint32_t* __restrict__ act, const Ctl* c) {
  if (!c->apply_prev) return;
  const double a = c->alpha_prev;
  double2* x2 = reinterpret_cast<double2*>(x);
  const double2* d2 = reinterpret_cast<const double2*>(d);
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT) {
    if (act_bit(act, (int)e)) {
      const double2 dp = d2[e];
      double2 xe = x2[e];
      xe.x = xe.x + a * dp.x;
      xe.y = xe.y + a * dp.y;
      x2[e] = xe;
      const double dzp = dp.x + dp.y;
      z[e] = z[e] + a * dzp;
    }
  }
}

// Vector hooks of the fast densest path: d (zeros where the activity bit is clear) and
// d^(z)_e = d_2e + d_2e+1 (W d), regardless of the probe status.
__global__ void d_from_act1(int64_t E, const double* __restrict__ d, const uint32_t* __restrict__ act,
                            double* __restrict__ dout) {     // one variable per edge (matching)
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT)
    dout[e] = act_bit(act, (int)e) ? d[e] : 0.0;
}

// x += alpha_prev d where the activity bit is set (end of probe / hooks), one variable per edge
__global__ void flush_act1(int64_t E, double* __restrict__ x, const double* __restrict__ d,
                           const uint32_t* __restrict__ act, const Ctl* c) {
  if (!c->apply_prev) return;
  const double a = c->alpha_prev;
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT)
    if (act_bit(act, (int)e)) x[e] = x[e] + a * d[e];
}

__global__ void d_from_act(int64_t E, const double* __restrict__ d, const uint32_t* __restrict__ act,
                           double* __restrict__ dout, double* __restrict__ dzout) {
  const double2* d2 = reinterpret_cast<const double2*>(d);
  for (int64_t e = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; e < E; e += (int64_t)gridDim.x * MWU_NT) {
    const double2 a = act_bit(act, (int)e) ? d2[e] : make_double2(0.0, 0.0);
    if (dout) { dout[2 * e] = a.x; dout[2 * e + 1] = a.y; }
    if (dzout) dzout[e] = a.x + a.y;
  }
}

// w_c = exp(-eta (z - s_C)) / S_C from z (vector hook of the lazy covering side).
__global__ void wc_from_z(int64_t m, const double* __restrict__ z, double* __restrict__ out, const Ctl* c) {
  const double neta = -c->eta, sC = c->sC, SC = c->SC;
  for (int64_t i = (int64_t)blockIdx.x * MWU_NT + threadIdx.x; i < m; i += (int64_t)gridDim.x * MWU_NT)
    out[i] = exp(neta * (z[i] - sC)) / SC;
}

}  // namespace mwu
