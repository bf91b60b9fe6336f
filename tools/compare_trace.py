"""Lockstep GPU vs oracle probe on a named instance (tests/instances.py or a CASES entry): prints
the first iteration where the accepted step sizes differ and whether the GPU's step equals Alg. 3
replayed by the oracle on the GPU's own cached vectors (a replay bug) or not (a divergence)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from gpu_common import Gpu, solver_for  # noqa: E402
from instances import EPS, WELL_CONDITIONED  # noqa: E402


def main(name, iters=5000):
    kind, mk = WELL_CONDITIONED[name]
    G = mk()
    s, d = G.numpy()
    eps = EPS[kind]
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=5000)
    S = solver_for(kind, G)
    for B, status, t, _ in r.probes:
        S.set_record(True)
        S.probe_begin(B, eps)
        p = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), eps)
        gpu = Gpu(S)
        for it in range(iters):
            before = gpu.state()
            so = p.step()
            sg = S.step(0.0)
            if so != "running" or sg != "running":
                print(f"B={B:.6g}: oracle {so} gpu {sg} at t={it} (oracle probe t={t})")
                break
            a = S.scalars()["alpha_last"]
            if a != p.last["alpha"]:
                ph = gpu.phase()
                sc = before["sc"]
                si = O.SearchInputs(before["y"], ph["dy"], before["z"], ph["dz"], p.eta, sc["sP"], sc["SP"], sc["sC"],
                                    sc["SC"], before["wp"], before["wc"])
                ref = O.binsearch(si, eps).alpha
                print(f"B={B:.6g} t={it}: alpha gpu {a} oracle {p.last['alpha']} oracle-on-gpu-state {ref}")
                return
    print("no difference")


if __name__ == "__main__":
    main(sys.argv[1])
