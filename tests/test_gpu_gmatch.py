"""Generalized matching l <= M x <= u on the GPU: the CSR of
P = diag(1/u) M and C = diag(1/l) M built on device bit-exact against the oracle's matrices, the
lockstep per-iteration checks of the mixed engine, and a full (single-probe) solve against the
oracle on an App. A.2-shaped instance (users l = 3, u = 5; items u = 200)."""
import numpy as np
import pytest
import torch

import graphgen as gg
import oracle as O
from gpu_common import lockstep, self_drift

pytestmark = pytest.mark.gpu


def _solver(g, lb, ub, **kw):
    from paper_2307_03307_b200 import Solver
    return Solver.gmatch(g.src.cuda(), g.dst.cuda(), g.n_vertices, lb.cuda(), ub.cuda(), **kw)


@pytest.mark.parametrize("seed", [1, 2])
def test_gmatch_structure_bit_exact(cuda_ok, seed):
    g, lb, ub = gg.gmatch_instance(300, 120, seed=seed)
    s, d = g.numpy()
    P, C = O.gmatch_matrices(s, d, g.n_vertices, lb.numpy(), ub.numpy())
    P2, _ = O.drop_empty_rows(P)
    S = _solver(g, lb, ub)
    assert np.array_equal(S.structure("p_rowptr").numpy(), P2.indptr)
    assert np.array_equal(S.structure("p_colidx").numpy(), P2.indices)
    assert np.array_equal(S.structure("c_rowptr").numpy(), C.indptr)
    assert np.array_equal(S.structure("c_colidx").numpy(), C.indices)


def test_gmatch_lockstep(cuda_ok):
    g, lb, ub = gg.gmatch_instance(400, 150, seed=3)
    s, d = g.numpy()
    lp = O.gmatch_lp(s, d, g.n_vertices, lb.numpy(), ub.numpy())
    S = _solver(g, lb, ub)
    lockstep(S, O.Probe(lp, 0.1), 1.0, 0.1, 50, alphas=[1.0] * 50, strict_derived=True)
    S2 = _solver(g, lb, ub)
    lockstep(S2, O.Probe(lp, 0.1), 1.0, 0.1, 50, alphas=None, drift=self_drift(lp, 0.1, None, 50))


@pytest.mark.parametrize("seed", [4, 5])
def test_gmatch_solve(cuda_ok, seed):
    g, lb, ub = gg.gmatch_instance(500, 200, seed=seed)
    s, d = g.numpy()
    P, C = O.gmatch_matrices(s, d, g.n_vertices, lb.numpy(), ub.numpy())
    r = O.solve("mixed", P=P, C=C, eps=0.1)
    S = _solver(g, lb, ub)
    out = S.solve(0.1)
    st = S.stats()
    print(f"gmatch seed {seed}: {out} iterations {st['iters_total']} (oracle {r.iters_total}) certificate "
          f"{st['certificate']:.6f} (oracle {r.certificate:.6f})")
    assert out == r.outcome == "feasible"
    assert abs(st["iters_total"] - r.iters_total) <= max(1, 0.02 * r.iters_total)
    x = S.x().cpu().numpy()
    M = O.incidence_M(s, d, g.n_vertices)
    lbn, ubn = lb.numpy(), ub.numpy()
    assert np.all(M @ x >= lbn - 1e-9)                                   # C x_out >= 1 (Q15)
    assert np.all(M @ x <= ubn * st["certificate"] * (1 + 1e-9))        # P x_out <= rho


def test_gmatch_infeasible_and_errors(cuda_ok):
    from paper_2307_03307_b200 import MwuError
    g = gg.star_graph(3)                         # center needs 2, each leaf edge at most 0.5
    lb = torch.tensor([2.0, 0.0, 0.0, 0.0], dtype=torch.float64)
    ub = torch.tensor([5.0, 0.5, 0.5, 0.5], dtype=torch.float64)
    S = _solver(g, lb, ub)
    assert S.solve(0.1) == "infeasible"
    with pytest.raises(MwuError, match="lb <= ub"):
        _solver(g, torch.tensor([2.0, 0, 0, 0], dtype=torch.float64), torch.tensor([1.0, 1, 1, 1], dtype=torch.float64))
