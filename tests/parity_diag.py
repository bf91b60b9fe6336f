"""Diagnostic (run on the GPU box, not a test): lockstep GPU vs oracle per kind, printing the
per-iteration trajectory errors and the first point where the search decisions differ."""
import json
import sys

import numpy as np

import graphgen as gg
import oracle as O
from gpu_common import Gpu, lockstep, phase_parity, solver_for, trajectory_errors

EPS = {"bmatch": 0.1, "match": 0.1, "vcover": 0.05, "domset": 0.05, "densest": 0.1}
CASES = {
    "bmatch": gg.config_graph("c1"),
    "match": gg.rmat(10, 8, seed=4),
    "vcover": gg.erdos_renyi(2000, 16000, seed=5),
    "domset": gg.rmat(11, 16, seed=6),
    "densest": gg.rmat(10, 16, seed=7),
}


def run(kind, G, iters=3000):
    s, d = G.numpy()
    r = O.solve(kind, s, d, G.n_vertices, eps=EPS[kind], max_iter=2000)
    feas = [p[0] for p in r.probes if p[1] == O.FEASIBLE]
    B = feas[-1] if feas else r.bound
    probe = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), EPS[kind], max_iter=iters)
    S = solver_for(kind, G)
    S.set_record(True)
    S.probe_begin(B, EPS[kind])
    gpu = Gpu(S)
    st = gpu.state()
    worst = {}
    first_div = None
    phase_fail = None
    for t in range(iters):
        so = probe.step()
        sg = S.step(0.0)
        if so != sg:
            first_div = first_div or (t, f"status {so} vs {sg}")
            break
        if so != O.RUNNING:
            break
        ph = gpu.phase()
        new = gpu.state()
        if phase_fail is None:
            try:
                phase_parity(probe.lp, probe.eta, probe.sigma, EPS[kind], st, ph, new, None)
            except AssertionError as e:
                phase_fail = (t, str(e))
        rec = trajectory_errors(probe, new, ph, probe.eta)
        for k, v in rec.items():
            worst[k] = max(worst.get(k, -1e300), v)
        if ph["alpha"] != probe.last["alpha"] and first_div is None:
            first_div = (t, f"alpha gpu {ph['alpha']} oracle {probe.last['alpha']}", {k: rec[k] for k in ("x", "y", "z", "wp", "wc")})
            break
        st = new
    print(json.dumps(dict(kind=kind, B=B, t=probe.t, status=probe.status, first_div=first_div,
                          phase_fail=phase_fail, worst=worst), default=str))
    sys.stdout.flush()


if __name__ == "__main__":
    kinds = sys.argv[1:] or list(CASES)
    for k in kinds:
        run(k, CASES[k])
