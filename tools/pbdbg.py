import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import graphgen as gg
from paper_2307_03307_b200 import Solver
import oracle as O
G = gg.bipartite_zipf(1024, 1024, 16384, seed=2)
s, d = G.numpy()
for pb in ("0", "1"):
    os.environ["MWU_PB"] = pb
    S = Solver.graph("bmatch", G.src.cuda(), G.dst.cuda(), G.n_vertices, G.n_left)
    S.set_record(True)
    S.probe_begin(500.0, 0.1)
    lp = O.graph_lp("bmatch", s, d, G.n_vertices, 500.0)
    for t in range(4):
        wp = S.vec("wp").cpu().numpy()
        S.step(0.0)
        g = S.vec("g").cpu().numpy()
        gref = lp.P.T @ wp
        print(pb, t, "g err", np.max(np.abs(g - gref) / np.maximum(np.abs(gref), 1e-300)), g[:3], gref[:3], S.scalars()["alpha_last"])
