"""Per-iteration PCG time, one-CTA-per-system solver (SG_PCG_SMALL=1) vs the multi-kernel path
(SG_PCG_SMALL=0), on single trained-GNN heat2d systems of growing size.  Diagnostic only.

    python profiles/small_probe.py
"""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2510_27517_b200 as P
import paper_2510_27517_b200.pcg as PC
m = P.load_checkpoint("tests/golden/trained_heat16.spaignn")
for nx in (16, 32, 48, 64, 90):
    A, meta = P.gen_poisson2d(nx, nx, coeff_seed=3)
    G = P.forward(m, P.build_graph(A, meta)).G
    b = P.gen_rhs(meta, 5)
    out = []
    for flag in ("1", "0"):
        os.environ["SG_PCG_SMALL"] = flag
        for h in (PC._HANDLES or {}).values(): h.close()
        PC._HANDLES = None
        M = P.build_learned_spai(G, m.config.epsilon)
        ts = []
        for _ in range(3):
            r = P.pcg_solve(A, b, M, P.SolveConfig(rtol=1e-8, track_history=False))
            ts.append(r.t_cg_total_ns / 1e3 / max(r.k, 1))
        out.append((flag, r.k, round(min(ts), 2)))
    print(nx, nx * nx, out, flush=True)
