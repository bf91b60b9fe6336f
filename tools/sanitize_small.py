#!/usr/bin/env python
"""Small solves of every graph kind and a CSR instance (fast and fixed-order paths), for
compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
from paper_2307_03307_b200 import Solver, MIXED
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_common import csr_tuple, lp_mats

for det in (0, 1):
    for kind, G in (("densest", gg.rmat(9, 8, seed=3)), ("bmatch", gg.bipartite_uniform(60, 70, 900, seed=2)),
                    ("match", gg.rmat(9, 8, seed=4)), ("vcover", gg.erdos_renyi(700, 3000, seed=5)),
                    ("domset", gg.rmat(9, 8, seed=6))):
        S = Solver.graph(kind, G.src.cuda(), G.dst.cuda(), G.n_vertices, G.n_left if kind == "bmatch" else 0,
                         deterministic=det)
        out = S.solve(0.1, 60)
        x = S.x()
        print(kind, det, out, S.stats()["objective"], float(x.sum()))
lp = gg.random_planted_lp(200, 120, 90, 0.03, seed=5)
P, C = lp_mats(lp)
S = Solver.csr(MIXED, lp.n, P=csr_tuple(P), C=csr_tuple(C))
print("csr", S.solve(0.1, 100))
torch.cuda.synchronize()
print("sanitize run done")
