"""Shared helpers for the GPU parity tests: build the same instance for the oracle and the CUDA
path (through the C ABI), run them in lockstep and compare element by element.

Two kinds of per-iteration parity:
 (A) phase parity — the oracle recomputes every phase of iteration t from the GPU's own inputs
     to that phase (weights from the GPU's y, z; g, h from its w; d from its g, h, x; d^(y),
     d^(z) from its d; alpha from Alg. 3 on its cached vectors; the update from its state).
     Elementwise 1e-10, d and the updates bit-exact, alpha exact.
 (B) trajectory parity — an independent oracle run with the same fixed steps (or its own
     search); state vectors x, y = Px, z = Cx within 1e-10 relative (BASELINE north_star);
     derived vectors (w, g, h, d, d^(y), d^(z)) within 1e-10 plus the first-order propagation of
     the measured state difference through exp (condition number eta*|y|) and 1 - g/h.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

import graphgen as gg
import oracle as O

RTOL = 1e-10   # BASELINE north_star: per-iteration vectors within 1e-10 relative


def solver_for(kind, G, **opts):
    from paper_2307_03307_b200 import Solver
    return Solver.graph(kind, G.src.cuda(), G.dst.cuda(), G.n_vertices,
                        G.n_left if kind == "bmatch" else 0, **opts)


def csr_tuple(A: sp.csr_matrix):
    A = A.tocsr()
    A.sort_indices()
    return (torch.from_numpy(A.indptr.astype(np.int64)), torch.from_numpy(A.indices.astype(np.int32)),
            torch.from_numpy(A.data.astype(np.float64)))


def lp_mats(lp: gg.CsrLP):
    P = sp.csr_matrix((lp.p_val.numpy(), lp.p_col.numpy(), lp.p_rowptr.numpy()),
                      shape=(lp.p_rowptr.numel() - 1, lp.n)) if lp.p_rowptr is not None else None
    C = sp.csr_matrix((lp.c_val.numpy(), lp.c_col.numpy(), lp.c_rowptr.numpy()),
                      shape=(lp.c_rowptr.numel() - 1, lp.n)) if lp.c_rowptr is not None else None
    return P, C


def np_(t):
    return t.detach().cpu().numpy() if torch.is_tensor(t) else np.asarray(t, dtype=np.float64)


def rel_err(a, b, floor=1e-300):
    a, b = np_(a), np_(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.size == 0:
        return 0.0
    den = np.maximum(np.abs(b), floor)
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.abs(a - b) / den
    return float(np.nanmax(r))


def excess(a, b, bound):
    """max(|a-b| - bound) (<= 0 means within bound)."""
    a, b = np_(a), np_(b)
    return float(np.max(np.abs(a - b) - bound)) if a.size else -1.0


def assert_vec(name, gpu, ref, rtol=RTOL, floor=1e-300):
    e = rel_err(gpu, ref, floor)
    assert e <= rtol, f"{name}: max rel err {e:.3e} > {rtol:.1e}"
    return e


class Gpu:
    """Snapshot of the GPU probe state through the C ABI."""

    def __init__(self, S):
        self.S = S

    def state(self):
        S = self.S
        sc = S.scalars()
        return dict(x=np_(S.vec("x")), y=np_(S.vec("y")), z=np_(S.vec("z")), wp=np_(S.vec("wp")),
                    wc=np_(S.vec("wc")), sc=sc)

    def phase(self):
        S = self.S
        return dict(g=np_(S.vec("g")), h=np_(S.vec("h")), d=np_(S.vec("d")), dy=np_(S.vec("dy")),
                    dz=np_(S.vec("dz")), alpha=S.scalars()["alpha_last"])


def phase_parity(lp: O.LP, eta, sigma, eps, before, ph, after, alpha_fixed, tol_mode="prose"):
    """(A): oracle phases recomputed from the GPU's own inputs; returns a dict of errors and
    asserts.  before/after: Gpu.state() around one mwu_step; ph: Gpu.phase() after it."""
    e = {}
    x0, y0, z0 = before["x"], before["y"], before["z"]
    # weights of the current state (Q4)
    sP, u, SP = O.shifted_weights_packing(y0, eta)
    sC, v, SC = O.shifted_weights_covering(z0, eta)
    e["wp"] = assert_vec("A:wp", before["wp"], u / SP)
    e["wc"] = assert_vec("A:wc", before["wc"], v / SC)
    # transposed products from the GPU's weights
    g = lp.P.T @ before["wp"]
    h = lp.C.T @ before["wc"]
    e["g"] = assert_vec("A:g", ph["g"], g)
    e["h"] = assert_vec("A:h", ph["h"], h)
    # direction from the GPU's g, h, x: same operation order -> bit-exact
    d = O.direction(ph["g"], ph["h"], x0, sigma)
    assert np.array_equal(ph["d"], d), f"A:d not bit-exact (max diff {np.max(np.abs(ph['d'] - d)):.3e})"
    # forward products from the GPU's d
    e["dy"] = assert_vec("A:dy", ph["dy"], lp.P @ ph["d"])
    e["dz"] = assert_vec("A:dz", ph["dz"], lp.C @ ph["d"])
    # step size: Alg. 3 on the GPU's cached vectors (exact decisions barring near-ties)
    a = ph["alpha"]
    if alpha_fixed is None:
        sc = before["sc"]
        si = O.SearchInputs(y0, ph["dy"], z0, ph["dz"], eta, sc["sP"], sc["SP"], sc["sC"], sc["SC"],
                            before["wp"], before["wc"])
        ref = O.binsearch(si, eps, tol_mode).alpha
        assert a == ref, f"A:alpha gpu {a} vs oracle-on-gpu-state {ref}"
    else:
        assert a == alpha_fixed
    # update: elementwise, same operation order -> bit-exact
    if after is not None:
        assert np.array_equal(after["x"], x0 + a * ph["d"]), "A:x update not bit-exact"
        assert np.array_equal(after["y"], y0 + a * ph["dy"]), "A:y update not bit-exact"
        assert np.array_equal(after["z"], z0 + a * ph["dz"]), "A:z update not bit-exact"
    return e


def trajectory_errors(probe: O.Probe, st, ph, eta):
    """(B): GPU state/phase vs the independent oracle run; returns max relative errors and the
    excess over the propagated allowance for derived vectors."""
    L = probe.last
    r = {}
    for k, ref in (("x", probe.x), ("y", probe.y), ("z", probe.z)):
        r[k] = rel_err(st[k], ref)
    dy_state = np.abs(st["y"] - probe.y)
    dz_state = np.abs(st["z"] - probe.z)
    wp_ref, wc_ref = probe.u / probe.SP, probe.v / probe.SC
    # first-order propagation: w_i = exp(eta (y_i - s)) / S  =>  |dw_i| <= w_i eta (|dy_i| + max|dy|) * 2
    r["wp"] = rel_err(st["wp"], wp_ref)
    r["wc"] = rel_err(st["wc"], wc_ref)
    r["wp_excess"] = excess(st["wp"], wp_ref, RTOL * wp_ref + wp_ref * eta * 2 * (dy_state + dy_state.max()) + 1e-300)
    r["wc_excess"] = excess(st["wc"], wc_ref, RTOL * wc_ref + wc_ref * eta * 2 * (dz_state + dz_state.max()) + 1e-300)
    if ph is not None and "g" in L:
        for k in ("g", "h", "dy", "dz", "d"):
            r[k] = rel_err(ph[k], L[k])
    return r


DRIFT_KEYS = ("x", "y", "z", "wp", "wc", "g", "h", "d", "dy", "dz")
DRIFT_FACTOR = 10.0   # GPU vs oracle allowed: max(1e-10, DRIFT_FACTOR x the oracle's own drift(t))


def _probe_vecs(p: O.Probe):
    v = dict(x=p.x, y=p.y, z=p.z, wp=p.u / p.SP, wc=p.v / p.SC)
    for k in ("g", "h", "d", "dy", "dz"):
        if k in p.last:
            v[k] = p.last[k]
    return v


SEPARATED = 1e-3      # state drift beyond which two fp64 trajectories are no longer comparable
NOISE = 2.0 ** -49    # rounding noise per iteration and per summed term: 8 ulps (a 2-ulp exp, a
                      # product, the shift and its reordered sums; times sqrt(#terms))


def noise_amplitudes(lp: O.LP, noise: float = None):
    """Relative rounding-noise amplitude per element of the vectors the drift model perturbs: a sum
    of n terms evaluated in another order (the GPU's atomics / trees against the oracle's CSR-order
    sums) differs by ~sqrt(n) ulps, so y, z (rows of P, C), g, h (columns of P, C) get
    NOISE * sqrt(max(1, n)) with n their number of terms, x gets NOISE."""
    noise = NOISE if noise is None else noise
    def rows(A):
        return noise * np.sqrt(np.maximum(1.0, np.diff(A.tocsr().indptr)))
    def cols(A):
        return noise * np.sqrt(np.maximum(1.0, np.diff(A.tocsc().indptr)))
    return {"x": noise, "y": rows(lp.P), "z": rows(lp.C), "g": cols(lp.P), "h": cols(lp.C)}


def self_drift(lp: O.LP, eps, alphas, iters, tol_mode="prose"):
    """The ORACLE's own fp64 conditioning along the compared trajectory.  Two reruns inject
    rounding noise of the size another correct fp64 evaluation makes (other summation order, a
    2-ulp exp): x0 scaled by 1 + s 2^-52; every iteration every element of g = P^T w_p and
    h = C^T w_c (before the direction, so the noise passes through the 1 - g/h cancellation as the
    GPU's does) and, after the update, of x, y, z scaled by 1 + s r a_i (s = +1 / -1 per rerun,
    r = +-1 at random per element, a_i = noise_amplitudes: 8 ulps times sqrt of the element's
    number of summed terms).  drift[t][k] is the largest elementwise relative difference (floor
    1e-300) of vector k between the reruns and the reference run after iteration t (t = 0: the
    initial state).  drift[t]["split"] is True once a rerun accepted a different step size or
    terminated differently (a decision within the rounding noise of Alg. 3, or of
    min z >= 1, Q6) or its state drifted beyond SEPARATED: from there the trajectories separate
    by the method itself."""
    runs = [O.Probe(lp, eps, tol_mode=tol_mode)] + [O.Probe(lp, eps, tol_mode=tol_mode, x0_scale=sc)
                                                    for sc in (1 + 2.0 ** -52, 1 - 2.0 ** -52)]

    def rec(split):
        ref = _probe_vecs(runs[0])
        r = {"split": split}
        for k in DRIFT_KEYS:
            if k in ref:
                r[k] = max(rel_err(_probe_vecs(q)[k], ref[k]) for q in runs[1:])
        return r
    rng = np.random.default_rng(12345)
    amp = noise_amplitudes(lp)
    for q, sg in zip(runs[1:], (1.0, -1.0)):      # noise on every element of g and h, random signs
        q.perturb = (lambda g, h, sg=sg: (g * (1.0 + sg * amp["g"] * rng.choice((-1.0, 1.0), size=g.shape)),
                                          h * (1.0 + sg * amp["h"] * rng.choice((-1.0, 1.0), size=h.shape))))
    out = [rec(False)]
    gone = {"split": True, **{k: float("inf") for k in DRIFT_KEYS}}
    for t in range(iters):
        al = None if alphas is None else alphas[t]
        sts = [q.step(al) for q in runs]
        if any(q.status != runs[0].status for q in runs[1:]) or \
                any(q.last.get("alpha") != runs[0].last.get("alpha") for q in runs[1:]):
            out.append(gone)                   # a decision inside the rounding noise
            break
        if sts[0] != O.RUNNING:                # all terminated alike: nothing more to compare
            break
        for q, sg in zip(runs[1:], (1.0, -1.0)):        # elementwise noise, random signs
            q.x, q.y, q.z = (v * (1.0 + sg * amp[k] * rng.choice((-1.0, 1.0), size=v.shape))
                             for k, v in (("x", q.x), ("y", q.y), ("z", q.z)))
            q._weights()
        r = rec(False)
        if max(r["x"], r["y"], r["z"]) > SEPARATED:
            out.append(gone)
            break
        out.append(r)
    return out


def drift_tol(drift, t, k, factor=DRIFT_FACTOR):
    """Allowed GPU-vs-oracle relative error of vector k after iteration t."""
    if t >= len(drift):
        return float("inf")
    return max(RTOL, factor * drift[t].get(k, 0.0))


def self_sensitivity_window(lp: O.LP, eps, alphas, iters, level=1e-12):
    """Number of leading iterations over which the ORACLE, rerun from x0 perturbed by one ulp,
    stays within `level` relative of itself (x, y, z) — reported as a diagnostic."""
    dr = self_drift(lp, eps, alphas, iters)
    for t, r in enumerate(dr):
        if r["split"] or max(r["x"], r["y"], r["z"]) > level:
            return max(0, t - 1)
    return len(dr) - 1


def lockstep(solver, probe: O.Probe, bound, eps, iters, alphas=None, phase_check=True, drift=None,
             strict_derived=False, factor=DRIFT_FACTOR):
    """Run `iters` MWU iterations on both sides (fixed steps `alphas`, or the Alg. 3 search on
    both when None).  Asserts (A) every iteration; asserts (B) — every compared vector within
    max(1e-10, factor x the oracle's own one-ulp drift(t)) relative, identical step sizes — for
    ALL iterations, with drift = self_drift(...) (None: the plain 1e-10 bound everywhere).
    After the oracle's own reruns split (a decision inside the rounding noise) the trajectories
    legitimately separate: (B) stops there, (A) continues from the GPU's own states.  Returns
    the per-iteration (B) error records (with the bound used)."""
    solver.set_record(True)
    solver.probe_begin(bound, eps)
    sc = solver.scalars()
    assert sc["eta"] == probe.eta and sc["sigma"] == probe.sigma
    gpu = Gpu(solver)
    st = gpu.state()
    recs = [trajectory_errors(probe, st, None, probe.eta)]
    for k in ("x", "y", "z"):
        assert recs[0][k] <= RTOL, (k, recs[0])
    coupled = True                               # oracle trajectory still comparable under (B)
    for t in range(iters):
        a = None if alphas is None else alphas[t]
        split = drift is not None and t + 1 < len(drift) and drift[t + 1]["split"]
        st_o = probe.step(alpha=a) if coupled else O.RUNNING
        st_g = solver.step(0.0 if a is None else a)
        if coupled and st_o == O.RUNNING and st_g in (O.FEASIBLE, O.ITER_LIMIT):
            # the GPU tests termination right after the update; the oracle at the top of its next
            # step — one more oracle call must terminate without iterating
            t0 = probe.t
            st_o = probe.step(alpha=None if a is None else a)
            assert probe.t == t0 or split, "oracle iterated where the GPU terminated"
        if coupled and st_o != st_g and not split:
            raise AssertionError(f"iteration {t}: oracle {st_o}/{probe.reason} vs gpu {st_g}")
        ph = gpu.phase() if st_g == O.RUNNING or st_g in (O.FEASIBLE, O.ITER_LIMIT) else None
        new = gpu.state()
        if phase_check and ph is not None and st_g != O.INFEASIBLE:
            phase_parity(probe.lp, probe.eta, probe.sigma, eps, st, ph, new, a)
        if st_g != O.RUNNING or (coupled and st_o != O.RUNNING and not split):
            break
        if coupled and split:
            coupled = False
        if not coupled:
            st = new
            continue
        rec = trajectory_errors(probe, new, ph, probe.eta)
        rec["alpha_gpu"], rec["alpha_oracle"] = ph["alpha"], probe.last["alpha"]
        recs.append(rec)
        if alphas is None:
            assert ph["alpha"] == probe.last["alpha"], f"iteration {t}: alpha gpu {ph['alpha']} vs oracle {probe.last['alpha']}"
        if drift is not None:
            for k in ("x", "y", "z", "wp", "wc", "g", "h"):
                tol = drift_tol(drift, t + 1, k, factor)
                rec[k + "_tol"] = tol
                assert rec[k] <= tol, f"iteration {t}: B:{k} rel err {rec[k]:.3e} > {tol:.3e} (oracle drift {drift[t + 1].get(k):.3e})"
            # d = sigma max(0, 1 - g/h) x: a relative error e of g/h becomes the absolute
            # error sigma |x| (g/h) e in d (cancellation in 1 - g/h), with e bounded by the g, h
            # bounds above plus a few ulps of the division; d^(y) = P d, d^(z) = C d inherit it
            L = probe.last
            x_prev = probe.x - L["alpha"] * L["d"]
            with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
                ratio = np.where(L["h"] > 0, L["g"] / np.where(L["h"] > 0, L["h"], 1.0), 0.0)
            e = 1e-12 + drift_tol(drift, t + 1, "g", factor) + drift_tol(drift, t + 1, "h", factor)
            allow = e * probe.sigma * np.abs(x_prev) * np.minimum(np.abs(ratio), 2.0)
            for k, al in (("d", allow), ("dy", probe.lp.P @ allow), ("dz", probe.lp.C @ allow)):
                tol = drift_tol(drift, t + 1, k, factor)
                ex = excess(ph[k], L[k], tol * np.abs(L[k]) + al)
                assert ex <= 0, f"iteration {t}: B:{k} beyond max({tol:.2e} rel, cancellation allowance) by {ex:.3e}"
        else:
            for k in ("x", "y", "z"):
                assert rec[k] <= RTOL, f"iteration {t}: B:{k} rel err {rec[k]:.3e}"
            assert rec["wp_excess"] <= 0 and rec["wc_excess"] <= 0, f"iteration {t}: B:w beyond propagated bound {rec}"
        if strict_derived:   # standard step (alpha = 1) trajectories are well conditioned
            L = probe.last
            for k in ("wp", "wc", "g", "h"):
                assert rec[k] <= RTOL, f"iteration {t}: B:{k} rel err {rec[k]:.3e}"
            x_prev = probe.x - L["alpha"] * L["d"]
            with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
                ratio = np.where(L["h"] > 0, L["g"] / np.where(L["h"] > 0, L["h"], 1.0), 0.0)
            # 1 - g/h cancellation: a few ulps of g/h become absolute error sigma x (ulps)
            b = 1e-12 * probe.sigma * np.abs(x_prev) * np.minimum(np.abs(ratio), 2.0)
            for k, allow in (("d", b), ("dy", probe.lp.P @ b), ("dz", probe.lp.C @ b)):
                ex = excess(ph[k], L[k], RTOL * np.abs(L[k]) + allow)
                assert ex <= 0, f"iteration {t}: B:{k} beyond bound by {ex:.3e}"
        st = new
    return recs
