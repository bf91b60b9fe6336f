"""Oracle self-drift table: for every parity case, the oracle rerun from x0 scaled
by 1 +- 2^-52 and the largest relative difference of x, y, z and w_c after iteration t, for the
searched trajectory (Alg. 3 on both) and the standard step (alpha = 1).  CPU only (oracle)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from gpu_common import self_drift  # noqa: E402
from test_gpu_parity import EPS, CASES, _graph, _oracle_probe_bound  # noqa: E402


def main():
    out = []
    for kind, i in CASES:
        G = _graph(kind, i)
        s, d = G.numpy()
        B, _ = _oracle_probe_bound(kind, G)
        lp = O.graph_lp(kind, s, d, G.n_vertices, B)
        row = {"case": f"{kind}-{i}", "n": lp.n}
        for mode, al in (("search", None), ("alpha1", [1.0] * 50)):
            dr = self_drift(lp, EPS[kind], al, 50)
            split = next((t for t, r in enumerate(dr) if r["split"]), None)
            last = [r for r in dr if not r["split"]]
            row[mode] = {"iters": len(dr) - 1, "split_at": split,
                         "x@t": {t: dr[t]["x"] for t in (10, 20, 30, 40, 50) if t < len(dr) and not dr[t]["split"]},
                         "max_state": max(max(r["x"], r["y"], r["z"]) for r in last),
                         "max_wc": max(r["wc"] for r in last)}
        out.append(row)
        print(json.dumps(row), flush=True)
    return out


if __name__ == "__main__":
    main()
