#!/usr/bin/env python
"""Run-to-run spread of the GPU full solve on densest-bu310 (tests/instances.py): the fast path's
fp64 reductions (red.global.add) land in a different order every run, the fixed-order engine
(deterministic=1) does not.  Prints iteration counts of N solves per engine; oracle count beside."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
from instances import WELL_CONDITIONED, EPS, MAX_ITER
from gpu_common import solver_for

N = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for name in sys.argv[2:] or ["densest-bu310"]:
    kind, mk = WELL_CONDITIONED[name]
    G = mk(); s, d = G.numpy()
    r = O.solve(kind, s, d, G.n_vertices, eps=EPS[kind], max_iter=MAX_ITER)
    for det in (0, 1):
        its, objs = [], []
        for _ in range(N):
            S = solver_for(kind, G, deterministic=det)
            S.solve(EPS[kind], MAX_ITER); st = S.stats()
            its.append(st["iters_total"]); objs.append(st["objective"]); S.close()
        print(f"{name} deterministic={det}: iterations {its} (oracle {r.iters_total}; "
              f"off by {[round(100 * (i - r.iters_total) / r.iters_total, 2) for i in its]} %) "
              f"objective spread {max(objs) - min(objs):.3g} (oracle {r.objective:.12g}, gpu {objs[0]:.12g})", flush=True)
