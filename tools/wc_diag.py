"""Where does the searched c4-recipe lockstep (R-MAT scale 18) first exceed 1e-10 in w_c?  Prints,
per iteration, the worst element of w_c and z: GPU vs oracle values, z, d^(z), alpha."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle as O  # noqa: E402
from gpu_common import Gpu, solver_for  # noqa: E402
from test_scale_parity import _bound  # noqa: E402

cfg, sd = sys.argv[1], int(sys.argv[2])
kind = {"c4": "densest", "c5": "bmatch"}[cfg]
eps = 0.1
G = gg.config_graph(cfg, scale_down=sd, seed=1, device="cuda")
s, d = G.numpy()
B = _bound(kind, G, s, d, eps)
p = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), eps)
S = solver_for(kind, G)
S.set_record(True)
S.probe_begin(B, eps)
gpu = Gpu(S)
for t in range(8):
    p.step()
    S.step(0.0)
    st, ph = gpu.state(), gpu.phase()
    for k, ref in (("z", p.z), ("wc", p.v / p.SC), ("x", p.x)):
        a = st[k]
        r = np.abs(a - ref) / np.maximum(np.abs(ref), 1e-300)
        i = int(np.argmax(r))
        extra = ""
        if k in ("z", "wc"):
            extra = f" z={p.z[i]:.17g} dz={p.last['dz'][i]:.6g} sC={p.sC:.17g} gpu_z={st['z'][i]:.17g}"
        print(f"t={t} alpha gpu {ph['alpha']} or {p.last['alpha']} {k}: max rel {r[i]:.3e} at {i} gpu {a[i]:.17g} ora {ref[i]:.17g}{extra}", flush=True)
