"""Step-size strategy study — the analog of the paper's Table 3
on a synthetic random geometric graph with 2^18 vertices (rgg-18 itself is not in the container):
for each graph LP, one probe at the bound the full solve settles on, run with the standard step
alpha = 1 (Std, Alg. 1), Alg. 3's binary search (Bin) and Newton's method (Nwt), eps = 0.1 as in
Table 3.  Reports MWU iterations, step-size evaluations per MWU iteration (and HBM passes), and
device time; writes a markdown table.   python tools/step_study.py [--scale 18] [--out FILE]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=18)
    ap.add_argument("--eps", type=float, default=0.1)
    ap.add_argument("--std-max-iter", type=int, default=200000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import graphgen as gg
    from paper_2307_03307_b200 import Solver
    base = gg.rgg(a.scale, seed=1)
    rows = []
    for kind in ("match", "bmatch", "domset", "vcover", "densest"):
        G = gg.biadjacency(base) if kind == "bmatch" else base
        src, dst = G.src.cuda(), G.dst.cuda()
        nl = G.n_left if kind == "bmatch" else 0
        S = Solver.graph(kind, src, dst, G.n_vertices, nl)
        S.solve(a.eps)
        st = S.stats()
        B = st["bound"]
        row = {"kind": kind, "graph": G.name, "edges": G.n_edges, "bound": B, "solve_iters": st["iters_total"]}
        for rule in ("standard", "binary", "newton"):
            T = Solver.graph(kind, src, dst, G.n_vertices, nl, step_rule=rule,
                             max_iter=a.std_max_iter if rule == "standard" else 5000)
            T.probe_begin(B, a.eps)
            out = T.run_probe()
            sc = T.scalars()
            ts = T.stats()
            row[rule] = {"outcome": out, "iters": int(sc["t"]), "evals_per_iter": sc["evals"] / max(1, sc["t"]),
                         "passes_per_iter": sc["passes"] / max(1, sc["t"]), "ms": ts["t_loop_ms"]}
            del T
        rows.append(row)
        print(json.dumps(row), flush=True)
        del S
        torch.cuda.empty_cache()
    lines = [f"Step-size strategies on rgg-{a.scale} (synthetic, {base.n_edges:,} edges), eps = {a.eps}, one probe at "
             "the full solve's final bound, one B200 (Table 3 analog, P:1586-1595)", "",
             "| problem | bound | # MWU iters Std | Bin | Nwt | evals/iter Bin | Nwt | passes/iter Bin | Nwt | ms Std | Bin | Nwt |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        s, b, n = r["standard"], r["binary"], r["newton"]
        lines.append(f"| {r['kind']} | {r['bound']:.6g} | {s['iters']} ({s['outcome']}) | {b['iters']} | {n['iters']} | "
                     f"{b['evals_per_iter']:.2f} | {n['evals_per_iter']:.2f} | {b['passes_per_iter']:.2f} | "
                     f"{n['passes_per_iter']:.2f} | {s['ms']:.1f} | {b['ms']:.2f} | {n['ms']:.2f} |")
    text = "\n".join(lines)
    print(text)
    if a.out:
        open(a.out, "w").write(text + "\n")


if __name__ == "__main__":
    main()
