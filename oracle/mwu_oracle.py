"""Plain, slow, single-threaded fp64 CPU oracle of the MWU positive-LP solver of
Ju, Yesil, Sun, Chekuri, Solomonik, "Efficient Parallel Implementation of the
Multiplicative Weight Update Method for Graph-based Linear Programs" (arXiv 2307.03307).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg, never by the product path, and sharing no code
with it (the seeded inputs come from graphgen/, which holds no MWU arithmetic).

Citation key: "P:n" = /root/reference/PAPER.md line n.  Readings of silent, ambiguous
or garbled passages are tagged (Q#) and listed in DESIGN.md §3 (numbering follows
SURVEY.md §8(c)).  Everything is the algorithm step by step in the paper's order and
notation: Alg. 1 initialisation, Alg. 2 loop with cached
y = Px, z = Cx, d^(y) = Pd, d^(z) = Cd, Alg. 3 step search, and the outer
bisections over the objective bound M or density D.  scipy.sparse
products and numpy reductions are the only library steps.

Pins (tests/test_oracle_*.py) tie each part to something other than itself; the
per-iteration vectors of a long run have no printed values in the paper and are pinned
only through their parts ("parity unpinned" beyond the primitive pins).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import scipy.sparse as sp

MIXED, PACKING, COVERING = "mixed", "packing", "covering"
RUNNING, FEASIBLE, INFEASIBLE, ITER_LIMIT = "running", "feasible", "infeasible", "iter_limit"
EXPM1_MAX_ARG = 700.0     # Q16: expm1 form of Psi only while eta*alpha*max d^(y) <= 700
EXPM1_MIN_SUM = -0.5      # Q16: expm1 form of Phi only while sum w_c expm1(.) >= -1/2


# --------------------------------------------------------------------------------------
# Constraint matrices from the paper's definitions (§3)
# --------------------------------------------------------------------------------------
def incidence_M(src, dst, n_vertices: int) -> sp.csr_matrix:
    """Vertex-edge incidence M in {0,1}^{n x m}: M[u,e] = 1 iff u in e (eq:incidence)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    E = src.size
    rows = np.concatenate([src, dst])
    cols = np.concatenate([np.arange(E), np.arange(E)])
    M = sp.csr_matrix((np.ones(2 * E), (rows, cols)), shape=(n_vertices, E))
    M.sort_indices()
    return M


def adjacency_A(src, dst, n_vertices: int) -> sp.csr_matrix:
    """Symmetric 0/1 adjacency matrix with a nonzero for each edge."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    rows = np.concatenate([src, dst])
    cols = np.concatenate([dst, src])
    A = sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(n_vertices, n_vertices))
    A.sort_indices()
    return A


def closed_neighborhood(src, dst, n_vertices: int) -> sp.csr_matrix:
    """Dominating-set covering matrix I + A."""
    C = (sp.identity(n_vertices, format="csr") + adjacency_A(src, dst, n_vertices)).tocsr()
    C.sort_indices()
    return C


def pair_matrix_O(src, dst, n_vertices: int) -> sp.csr_matrix:
    """Vertex-edge pair matrix O in {0,1}^{n x 2m} (eq:oddshifted_incidence):
    O[u, 2e+b] = 1 for b = 0 if e = (u, v) and for b = 1 if e = (v, u); here b = 0 is
    src[e] and b = 1 is dst[e] (Q29)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    E = src.size
    rows = np.concatenate([src, dst])
    cols = np.concatenate([2 * np.arange(E), 2 * np.arange(E) + 1])
    O = sp.csr_matrix((np.ones(2 * E), (rows, cols)), shape=(n_vertices, 2 * E))
    O.sort_indices()
    return O


def interweaved_W(n_edges: int) -> sp.csr_matrix:
    """Interweaved identity W: W[e,2e] = W[e,2e+1] = 1 (eq:interweaved), read as
    m x 2m (Q18: the printed n x 2m has row index e ranging over edges)."""
    E = int(n_edges)
    rows = np.repeat(np.arange(E), 2)
    cols = np.arange(2 * E)
    return sp.csr_matrix((np.ones(2 * E), (rows, cols)), shape=(E, 2 * E))


def singleton_row(n: int, bound: float) -> sp.csr_matrix:
    """Embedded objective row (1/M) 1^T."""
    return sp.csr_matrix(np.full((1, n), 1.0 / bound))


def drop_empty_rows(A: sp.csr_matrix):
    """Q17: empty packing rows (isolated vertices) are vacuous and dropped.
    Returns (A restricted to non-empty rows, kept original row ids)."""
    A = A.tocsr()
    keep = np.flatnonzero(np.diff(A.indptr) > 0)
    return A[keep], keep


def matvec(A: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    """A x with per-row sums in CSR index order (scipy).  A matrix of ONE row — the embedded
    objective row (1/M) 1^T of the pure modes — is a global sum over all n variables: it
    is summed exactly rounded (math.fsum of the products), the compensated global sum of reading
    Q22, since a sequential sum of n = 10^7 terms is off by up to n/2 ulps."""
    if A.shape[0] == 1:
        row = A.data * x[A.indices]
        return np.array([math.fsum(row.tolist())])
    return A @ x


# --------------------------------------------------------------------------------------
# LP instances (normalised form  Px <= 1, Cx >= 1, x >= 0 of eq:NormFeasibleLP)
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class LP:
    P: sp.csr_matrix
    C: sp.csr_matrix
    mode: str                       # MIXED / PACKING (C = singleton) / COVERING (P = singleton)
    p_rows: np.ndarray | None = None  # original ids of kept packing rows (Q17)

    @property
    def n(self) -> int:
        return self.P.shape[1]

    @property
    def m(self) -> int:               # m := m_P + m_C, embedded row counted (Q2)
        return self.P.shape[0] + self.C.shape[0]


def packing_lp(P: sp.csr_matrix, bound: float) -> LP:
    """Pure packing max <1,x> s.t. Px <= 1 as feasibility with (1/M)1^T x >= 1."""
    P2, keep = drop_empty_rows(P)
    return LP(P2, singleton_row(P.shape[1], bound), PACKING, keep)


def covering_lp(C: sp.csr_matrix, bound: float) -> LP:
    """Pure covering min <1,x> s.t. Cx >= 1 as feasibility with (1/M)1^T x <= 1."""
    return LP(singleton_row(C.shape[1], bound), C.tocsr(), COVERING, None)


def mixed_lp(P: sp.csr_matrix, C: sp.csr_matrix) -> LP:
    P2, keep = drop_empty_rows(P)
    return LP(P2, C.tocsr(), MIXED, keep)


def gmatch_matrices(src, dst, n_vertices: int, lb, ub):
    """Generalized matching l <= M x <= u in the normalised form of eq:NormFeasibleLP:
    P = diag(1/u) M over the vertices with finite u, C = diag(1/l) M over the vertices with l > 0
    (rows in vertex order, M = eq:incidence)."""
    lb = np.asarray(lb, dtype=np.float64)
    ub = np.asarray(ub, dtype=np.float64)
    M = incidence_M(src, dst, n_vertices)
    pr = np.flatnonzero(np.isfinite(ub))
    cr = np.flatnonzero(lb > 0)
    P = (sp.diags(1.0 / ub[pr]) @ M[pr]).tocsr()
    C = (sp.diags(1.0 / lb[cr]) @ M[cr]).tocsr()
    P.sort_indices()
    C.sort_indices()
    return P, C


def gmatch_lp(src, dst, n_vertices: int, lb, ub) -> LP:
    """Generalized matching as a mixed LP (empty packing rows dropped, Q17)."""
    return mixed_lp(*gmatch_matrices(src, dst, n_vertices, lb, ub))


def densest_lp(src, dst, n_vertices: int, D: float) -> LP:
    """Feasibility form of the densest-subgraph dual (eq:densest_linalg):
    W z >= 1, O z <= D 1, i.e. P = (1/D) O, C = W (mixed)."""
    O = pair_matrix_O(src, dst, n_vertices)
    P = O.multiply(1.0 / D).tocsr()
    return mixed_lp(P, interweaved_W(len(src)))


def graph_lp(kind: str, src, dst, n_vertices: int, bound: float) -> LP:
    """The §3 LPs at objective bound M (or density D for 'densest')."""
    if kind in ("bmatch", "match"):               # max <1,x> s.t. Mx <= 1
        return packing_lp(incidence_M(src, dst, n_vertices), bound)
    if kind == "vcover":                          # min <1,x> s.t. M^T x >= 1
        return covering_lp(incidence_M(src, dst, n_vertices).T.tocsr(), bound)
    if kind == "domset":                          # min <1,x> s.t. (I+A) x >= 1
        return covering_lp(closed_neighborhood(src, dst, n_vertices), bound)
    if kind == "densest":
        return densest_lp(src, dst, n_vertices, bound)
    raise KeyError(kind)


# --------------------------------------------------------------------------------------
# Smoothed max / min and their gradients
# --------------------------------------------------------------------------------------
def smax(v, eta: float) -> float:
    """smax_eta(v) = (1/eta) log sum exp(eta v_i), evaluated with the max shift (Q4)."""
    v = np.asarray(v, dtype=np.float64)
    s = v.max()
    return s + math.log(np.sum(np.exp(eta * (v - s)))) / eta


def smin(v, eta: float) -> float:
    """smin_eta(v) = -(1/eta) log sum exp(-eta v_i), evaluated with the min shift (Q4)."""
    v = np.asarray(v, dtype=np.float64)
    s = v.min()
    return s - math.log(np.sum(np.exp(-eta * (v - s)))) / eta


def grad_smax(v, eta: float) -> np.ndarray:
    """grad smax_eta(v) = exp(eta v) / <1, exp(eta v)>."""
    v = np.asarray(v, dtype=np.float64)
    u = np.exp(eta * (v - v.max()))
    return u / np.sum(u)


def grad_smin(v, eta: float) -> np.ndarray:
    """grad smin_eta(v) = exp(-eta v) / <1, exp(-eta v)>."""
    v = np.asarray(v, dtype=np.float64)
    u = np.exp(-eta * (v - v.min()))
    return u / np.sum(u)


# --------------------------------------------------------------------------------------
# Alg. 1 / Alg. 2 building blocks
# --------------------------------------------------------------------------------------
def eta_parameter(m: int, eps: float, factor: float = 10.0) -> float:
    """eta <- 10 log(m) / eps, m := m_P + m_C; natural log (Q1)."""
    return factor * math.log(m) / eps


def column_inf_norms(P: sp.csr_matrix) -> np.ndarray:
    """||P_{:,i}||_inf for each column."""
    return np.asarray(abs(P).max(axis=0).todense()).ravel()


def init_x(P: sp.csr_matrix, eps: float) -> np.ndarray:
    """x_i <- eps / (n ||P_{:,i}||_inf) (Alg. 1 line init_vec); n = #variables (Q3, Q32)."""
    n = P.shape[1]
    cn = column_inf_norms(P)
    if np.any(cn <= 0):
        raise ValueError("all-zero packing column: initialisation undefined (SPEC S:212)")
    return eps / (n * cn)


def step_sigma(mode: str, eta: float) -> float:
    """1/(2 eta); pure modes scale by a factor of 2 -> 1/eta (Q13)."""
    return 1.0 / eta if mode in (PACKING, COVERING) else 1.0 / (2.0 * eta)


def direction(g, h, x, sigma: float) -> np.ndarray:
    """d_i <- sigma max{0, 1 - g_i/h_i} x_i (P:279 / P:666); h_i = 0 -> d_i = 0 (Q5)."""
    g = np.asarray(g, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    d = np.zeros_like(x)
    pos = h > 0
    with np.errstate(over="ignore"):     # g/h = inf where h underflowed: clipped to 0 below
        d[pos] = sigma * np.maximum(0.0, 1.0 - g[pos] / h[pos]) * x[pos]
    return d


def shifted_weights_packing(y, eta: float):
    """Unnormalised weights of grad smax_eta(y) with shift s_P = max y (Q4):
    u = exp(eta (y - s_P)), S_P = sum u; w_p = u / S_P."""
    s = y.max()
    u = np.exp(eta * (y - s))
    return s, u, np.sum(u)


def shifted_weights_covering(z, eta: float):
    """Unnormalised weights of grad smin_eta(z) with shift s_C = min z (Q4):
    v = exp(-eta (z - s_C)), S_C = sum v; w_c = v / S_C."""
    s = z.min()
    v = np.exp(-eta * (z - s))
    return s, v, np.sum(v)


# --------------------------------------------------------------------------------------
# Bang-for-buck f(alpha) = Phi(alpha) / Psi(alpha) on the cached vectors
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class SearchInputs:
    y: np.ndarray
    dy: np.ndarray
    z: np.ndarray
    dz: np.ndarray
    eta: float
    sP: float
    SP: float
    sC: float
    SC: float
    wp: np.ndarray
    wc: np.ndarray

    @property
    def maxdy(self) -> float:
        return float(self.dy.max())


def eta_psi(si: SearchInputs, alpha: float) -> float:
    """eta*Psi(alpha) = eta(smax(y + alpha d^(y)) - smax(y)), no SpMV.
    Single packing row: smax is exact, eta*Psi = eta*alpha*d^(y) (Q12).
    Q16 numerics: log1p(sum w_p expm1(eta alpha d^(y))) while eta*alpha*max d^(y) <= 700,
    otherwise the max-shifted log-sum-exp difference."""
    ea = si.eta * alpha
    if si.y.size == 1:
        return ea * si.dy[0]
    if ea * si.maxdy <= EXPM1_MAX_ARG:
        return math.log1p(np.sum(si.wp * np.expm1(ea * si.dy)))
    t = si.y + alpha * si.dy
    s2 = t.max()
    return si.eta * (s2 - si.sP) + math.log(np.sum(np.exp(si.eta * (t - s2)))) - math.log(si.SP)


def eta_phi(si: SearchInputs, alpha: float) -> float:
    """eta*Phi(alpha) = eta(smin(z + alpha d^(z)) - smin(z)).
    Single covering row: exact, eta*Phi = eta*alpha*d^(z) (Q12).
    Q16 numerics: -log1p(sum w_c expm1(-eta alpha d^(z))) while that sum >= -1/2,
    otherwise the min-shifted log-sum-exp difference."""
    ea = si.eta * alpha
    if si.z.size == 1:
        return ea * si.dz[0]
    e = np.sum(si.wc * np.expm1(-(ea * si.dz)))
    if e >= EXPM1_MIN_SUM:
        return -math.log1p(e)
    t = si.z + alpha * si.dz
    s2 = t.min()
    return si.eta * (s2 - si.sC) - math.log(np.sum(np.exp(-si.eta * (t - s2)))) + math.log(si.SC)


def f_at_least_one(si: SearchInputs, alpha: float) -> bool:
    """Invariant eq:b4b_conv f(alpha) = Phi/Psi >= 1, tested as eta*Phi >= eta*Psi;
    Psi = 0 reads as f = +inf, which the comparison also gives."""
    return eta_phi(si, alpha) >= eta_psi(si, alpha)


def covering_min_after(si: SearchInputs, alpha: float) -> float:
    """min(z + alpha d^(z)) for the early exit of Alg. 3 (Q11)."""
    return float(np.min(si.z + alpha * si.dz))


@dataclasses.dataclass
class SearchResult:
    alpha: float
    evals: int
    early: bool


def binsearch(si: SearchInputs, eps: float, tol_mode: str = "prose", max_evals: int = 200) -> SearchResult:
    """Alg. 3 BinSearch: exponential search from alpha = 1 (Q10), early
    return when min(z + alpha d^(z)) >= 1, then bisection on [alpha/2, alpha]
     returning lb.  Stop rule (Q9): 'prose' ub - lb <= eps*lb;
    'listing' ub - lb <= (1-eps)*lb.  max_evals caps the evaluations."""
    alpha = 1.0
    evals = 0
    while True:
        ok = f_at_least_one(si, alpha)
        evals += 1
        if not ok:
            break
        if covering_min_after(si, alpha) >= 1.0:
            return SearchResult(alpha, evals, True)
        if evals >= max_evals:
            return SearchResult(alpha, evals, False)
        alpha = 2.0 * alpha
    lb, ub = alpha / 2.0, alpha
    thr = eps if tol_mode == "prose" else (1.0 - eps)
    while ub - lb > thr * lb and evals < max_evals:
        beta = (lb + ub) / 2.0
        if f_at_least_one(si, beta):
            lb = beta
        else:
            ub = beta
        evals += 1
    return SearchResult(lb, evals, False)


# --------------------------------------------------------------------------------------
# Newton step search (readings Q34-Q37 in DESIGN.md §3)
# --------------------------------------------------------------------------------------
NEWTON_MAX_STEPS = 20      # Q35: Newton steps before falling back to Alg. 3
NEWTON_MAX_BACKOFF = 64    # Q36: at most this many (1 - eps) back-off factors


def eta_psi_prime(si: SearchInputs, alpha: float) -> float:
    """d/dalpha of eta*Psi(alpha) = eta <grad smax(y + alpha d^(y)), d^(y)> (P:720 differentiated):
    eta sum_i w_i dy_i e^{eta alpha dy_i} / sum_i w_i e^{eta alpha dy_i}, evaluated with the
    exponents shifted by their maximum.  Single packing row: eta d^(y)."""
    if si.y.size == 1:
        return si.eta * si.dy[0]
    a = si.eta * alpha * si.dy
    e = si.wp * np.exp(a - a.max())
    return si.eta * float(np.sum(e * si.dy) / np.sum(e))


def eta_phi_prime(si: SearchInputs, alpha: float) -> float:
    """d/dalpha of eta*Phi(alpha) = eta <grad smin(z + alpha d^(z)), d^(z)> (P:719 differentiated):
    eta sum_i w_i dz_i e^{-eta alpha dz_i} / sum_i w_i e^{-eta alpha dz_i}, shifted by the
    largest exponent.  Single covering row: eta d^(z)."""
    if si.z.size == 1:
        return si.eta * si.dz[0]
    a = -(si.eta * alpha) * si.dz
    e = si.wc * np.exp(a - a.max())
    return si.eta * float(np.sum(e * si.dz) / np.sum(e))


def newton_search(si: SearchInputs, eps: float, alpha0: float | None, tol_mode: str = "prose",
                  max_evals: int = 200) -> SearchResult:
    """Newton's method on g(alpha) = f(alpha) - 1: alpha <- alpha - g/g', with
    f = Phi/Psi and g' = (Phi' Psi - Phi Psi')/Psi^2, i.e. with P = eta Phi, Q = eta Psi,
    alpha <- alpha - (P - Q) Q / (P' Q - P Q').
      Q34 start: the previous accepted step size; without one, Alg. 3's exponential
          search gives the largest passing power of two (its early exit and alpha < 1 outcomes
          are returned as Alg. 3 returns them).
      Q35 convergence: stop at the evaluated iterate alpha once the next Newton update would move
          it by <= eps * alpha; a non-finite or non-negative g' (f must decrease, Prop. P:746-758),
          a non-positive update or NEWTON_MAX_STEPS steps fall back to Alg. 3 from scratch.
      Q36 back-off: alpha <- alpha (1 - eps) until f(alpha) >= 1 (at most
          NEWTON_MAX_BACKOFF times); the first factor tested is (1 - eps)^0.
    Every f evaluation counts one evaluation (the derivative comes from the same pass)."""
    evals = 0
    if alpha0 is None or not (alpha0 >= 1.0):
        alpha = 1.0
        while True:                                     # Alg. 3 exponential search
            ok = f_at_least_one(si, alpha)
            evals += 1
            if not ok:
                break
            if covering_min_after(si, alpha) >= 1.0:
                return SearchResult(alpha, evals, True)
            if evals >= max_evals:
                return SearchResult(alpha, evals, False)
            alpha = 2.0 * alpha
        if alpha == 1.0:                                # f(1) < 1: Alg. 3's own answer (< 1)
            r = binsearch(si, eps, tol_mode, max_evals)
            return SearchResult(r.alpha, evals + r.evals, r.early)
        alpha0 = alpha / 2.0
    a = float(alpha0)
    P = Q = 0.0
    converged = False
    for _ in range(NEWTON_MAX_STEPS):
        P, Q = eta_phi(si, a), eta_psi(si, a)
        Pd, Qd = eta_phi_prime(si, a), eta_psi_prime(si, a)
        evals += 1
        den = Pd * Q - P * Qd
        if not (math.isfinite(P) and math.isfinite(Q) and math.isfinite(den)) or not (den < 0.0) or not (Q > 0.0):
            break
        a_new = a - (P - Q) * Q / den
        if not (math.isfinite(a_new) and a_new > 0.0):
            break
        if abs(a_new - a) <= eps * a:
            converged = True
            break
        a = a_new
    if not converged:                                   # Q35 fallback
        r = binsearch(si, eps, tol_mode, max_evals)
        return SearchResult(r.alpha, evals + r.evals, r.early)
    ok = P >= Q                                         # f(a) >= 1, from the converged pass
    p = 0
    while not ok and p < NEWTON_MAX_BACKOFF:            # Q36 back-off by (1 - eps)^p
        a = a * (1.0 - eps)
        p += 1
        ok = f_at_least_one(si, a)
        evals += 1
    return SearchResult(a, evals, False)


# --------------------------------------------------------------------------------------
# Alg. 2 probe: one feasibility solve of  Px <= 1, Cx >= 1
# --------------------------------------------------------------------------------------
STEP_RULES = ("binary", "newton", "standard")   # Alg. 3 / Newton / alpha = 1 (Alg. 1)


class Probe:
    """Alg. 2 with a step rule — Alg. 3 (default), Newton or the standard step
    alpha = 1 of Alg. 1 ("Std" of Table 3) — or a caller-supplied fixed step
    sequence, one iteration per step() so tests can run it in lockstep with the GPU."""

    def __init__(self, lp: LP, eps: float, max_iter: int = 5000, eta_factor: float = 10.0,
                 tol_mode: str = "prose", max_evals: int = 200, x0_scale: float = 1.0,
                 step_rule: str = "binary"):
        if step_rule not in STEP_RULES:
            raise ValueError(step_rule)
        self.lp, self.eps, self.max_iter = lp, eps, max_iter
        self.tol_mode, self.max_evals, self.step_rule = tol_mode, max_evals, step_rule
        self.P, self.C = lp.P, lp.C
        self.PT, self.CT = lp.P.T.tocsr(), lp.C.T.tocsr()
        self.eta = eta_parameter(lp.m, eps, eta_factor)                 # P:271 (line init2 P:656)
        self.sigma = step_sigma(lp.mode, self.eta)
        self.t = 0
        self.evals = 0
        self.alphas: list[float] = []
        self.status, self.reason = RUNNING, ""
        if lp.C.shape[0] > 0 and np.any(np.diff(lp.C.indptr) == 0):
            self.status, self.reason = INFEASIBLE, "EMPTY_COVER_ROW"    # Q17: 0 >= 1 fails
        self.x = init_x(lp.P, eps)
        if x0_scale != 1.0:   # test knob: one-ulp perturbation to measure fp sensitivity
            self.x = self.x * x0_scale
        self.y = matvec(self.P, self.x)
        self.z = matvec(self.C, self.x)
        self._weights()
        self.last: dict = {}
        self.perturb = None   # test knob: callable (g, h) -> (g, h), rounding-noise models

    def _weights(self):
        self.sP, self.u, self.SP = shifted_weights_packing(self.y, self.eta)
        self.sC, self.v, self.SC = shifted_weights_covering(self.z, self.eta)
        if not (np.isfinite(self.SP) and np.isfinite(self.SC) and self.SP > 0 and self.SC > 0):
            raise FloatingPointError("non-finite weight sums")

    def search_inputs(self, dy, dz) -> SearchInputs:
        return SearchInputs(self.y, dy, self.z, dz, self.eta, self.sP, self.SP, self.sC, self.SC,
                            self.u / self.SP, self.v / self.SC)

    def step(self, alpha: float | None = None) -> str:
        """One pass of the while-loop body of Alg. 2."""
        if self.status != RUNNING:
            return self.status
        # loop guard (Q6): terminate once every covering row is satisfied
        if self.z.min() >= 1.0:
            self.status = FEASIBLE
            return self.status
        if self.t >= self.max_iter:
            self.status, self.reason = ITER_LIMIT, "ITER_LIMIT"
            return self.status
        wp = self.u / self.SP                                             # grad smax(y)
        wc = self.v / self.SC                                             # grad smin(z)
        g = self.PT @ wp
        h = self.CT @ wc
        if self.perturb is not None:
            g, h = self.perturb(g, h)
        d = direction(g, h, self.x, self.sigma)
        if d.size == 0 or d.max() == 0.0:
            self.status, self.reason = INFEASIBLE, "MAXD_ZERO"
            self.last = dict(wp=wp, wc=wc, g=g, h=h, d=d)
            return self.status
        dy = matvec(self.P, d)
        dz = matvec(self.C, d)
        if alpha is None and self.step_rule == "standard":
            alpha = 1.0                                                   # Alg. 1
        elif alpha is None:
            si = self.search_inputs(dy, dz)
            if self.step_rule == "newton":                                # warm start (Q34)
                sr = newton_search(si, self.eps, self.alphas[-1] if self.alphas else None, self.tol_mode,
                                   self.max_evals)
            else:
                sr = binsearch(si, self.eps, self.tol_mode, self.max_evals)
            alpha = sr.alpha
            self.evals += sr.evals
        self.last = dict(wp=wp, wc=wc, g=g, h=h, d=d, dy=dy, dz=dz, alpha=alpha)
        if alpha < 1.0:
            self.status, self.reason = INFEASIBLE, "ALPHA_LT_1"
            return self.status
        self.x = self.x + alpha * d
        self.y = self.y + alpha * dy
        self.z = self.z + alpha * dz
        self._weights()
        self.alphas.append(alpha)
        self.t += 1
        return RUNNING

    def run(self) -> str:
        while self.step() == RUNNING:
            pass
        return self.status

    # ---- outputs -------------------------------------------------------------------
    def x_out(self) -> np.ndarray:
        """Q15: on FEASIBLE return x / min(Cx) so min(C x_out) = 1 exactly."""
        return self.x / self.z.min()

    def certificate(self) -> float:
        """rho = max(y) / min(z): packing level of x_out (Q6)."""
        return float(self.y.max() / self.z.min())


def run_probe(lp: LP, eps: float, **kw) -> Probe:
    p = Probe(lp, eps, **kw)
    p.run()
    return p


# --------------------------------------------------------------------------------------
# Outer searches over the objective bound M / density D
# --------------------------------------------------------------------------------------
def packing_bracket(P: sp.csr_matrix, eps: float):
    """Q14: L = sum x0 / max(P x0) (x0 of P:272 rescaled to a feasible witness);
    H = sum_i max_{j: p_ji > 0} 1/p_ji."""
    P2, _ = drop_empty_rows(P)
    x0 = init_x(P2, eps)
    w = x0 / np.max(P2 @ x0)
    Pc = P2.tocsc()
    H = 0.0
    for i in range(P2.shape[1]):
        vals = Pc.data[Pc.indptr[i]:Pc.indptr[i + 1]]
        H += np.max(1.0 / vals[vals > 0])
    return float(np.sum(w)), float(H), w


def covering_bracket(C: sp.csr_matrix):
    """Q14: L = m_C / max_i ||C_{:,i}||_1 (weak duality); H = sum_i max_{j: c_ji>0} 1/c_ji with
    witness x_i = max_j 1/c_ji (0 for empty columns)."""
    Cc = C.tocsc()
    colsum = np.asarray(Cc.sum(axis=0)).ravel()
    L = C.shape[0] / colsum.max()
    w = np.zeros(C.shape[1])
    for i in range(C.shape[1]):
        vals = Cc.data[Cc.indptr[i]:Cc.indptr[i + 1]]
        vals = vals[vals > 0]
        if vals.size:
            w[i] = np.max(1.0 / vals)
    return float(L), float(np.sum(w)), w


def densest_bracket(src, dst, n_vertices: int):
    """Q14: L = m / n' (density of G over its n' non-isolated vertices, <= max density);
    H = Delta/2 (z = 1/2 everywhere satisfies eq:dualDS at D = Delta/2)."""
    deg = np.bincount(np.concatenate([np.asarray(src), np.asarray(dst)]).astype(np.int64),
                      minlength=n_vertices)
    nprime = int(np.count_nonzero(deg))
    return len(src) / nprime, deg.max() / 2.0, np.full(2 * len(src), 0.5)


@dataclasses.dataclass
class SolveResult:
    outcome: str
    objective: float
    bound: float
    x: np.ndarray
    probes: list
    iters_total: int
    evals_total: int
    certificate: float


def solve(kind: str, src=None, dst=None, n_vertices: int = 0, eps: float = 0.1,
          max_iter: int = 5000, P: sp.csr_matrix | None = None, C: sp.csr_matrix | None = None,
          tol_mode: str = "prose", max_evals: int = 200, eta_factor: float = 10.0,
          outer_rel_tol: float | None = None, x0_scale: float = 1.0, step_rule: str = "binary") -> SolveResult:
    """Full solve: outer geometric bisection (Q14) over M (pure modes) or D (densest) with a
    fresh Alg. 2 probe per bound; IterLimit counts as infeasible.  kind in {bmatch, match,
    vcover, domset, densest, packing, covering, mixed}; the last three take explicit P / C."""
    rt = eps / 4.0 if outer_rel_tol is None else outer_rel_tol
    kw = dict(max_iter=max_iter, eta_factor=eta_factor, tol_mode=tol_mode, max_evals=max_evals, step_rule=step_rule,
              x0_scale=x0_scale)
    if kind == "mixed":
        p = run_probe(mixed_lp(P, C), eps, **kw)
        ok = p.status == FEASIBLE
        return SolveResult(p.status, float("nan"), float("nan"), p.x_out() if ok else p.x,
                           [(None, p.status, p.t, p.evals)], p.t, p.evals,
                           p.certificate() if ok else float("nan"))
    if kind in ("bmatch", "match"):
        P = incidence_M(src, dst, n_vertices)
        kind = "packing"
    elif kind == "vcover":
        C = incidence_M(src, dst, n_vertices).T.tocsr()
        kind = "covering"
    elif kind == "domset":
        C = closed_neighborhood(src, dst, n_vertices)
        kind = "covering"

    if kind == "packing":
        L, H, best = packing_bracket(P, eps)
        make = lambda B: packing_lp(P, B)  # noqa: E731
        sense = +1
    elif kind == "covering":
        L, H, best = covering_bracket(C)
        make = lambda B: covering_lp(C, B)  # noqa: E731
        sense = -1
    elif kind == "densest":
        L, H, best = densest_bracket(src, dst, n_vertices)
        make = lambda B: densest_lp(src, dst, n_vertices, B)  # noqa: E731
        sense = -1
    else:
        raise KeyError(kind)

    probes = []
    iters = evals = 0
    cert = float("nan")
    any_feasible = False
    while H > (1.0 + rt) * L:
        B = math.sqrt(L * H)
        p = run_probe(make(B), eps, **kw)
        iters += p.t
        evals += p.evals
        ok = p.status == FEASIBLE
        probes.append((B, p.status, p.t, p.evals))
        if ok:
            best, cert, any_feasible = p.x_out(), p.certificate(), True
        if (ok and sense > 0) or (not ok and sense < 0):
            L = B
        else:
            H = B
    bound = L if sense > 0 else H
    objective = bound if kind == "densest" else float(np.sum(best))
    # a witness always exists for the pure modes (bracket end points), so the outcome is
    # FEASIBLE; `certificate` is NaN when no probe succeeded and the witness is returned
    return SolveResult(FEASIBLE, objective, bound, best, probes, iters, evals,
                       cert if any_feasible else float("nan"))
