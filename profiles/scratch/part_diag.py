"""Diagnostic: residual-history divergence of the partitioned solve vs the whole-system solve."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2510_27517_b200 as P
from paper_2510_27517_b200 import rowpart as RP
m = P.load_checkpoint("tests/golden/trained_heat16.spaignn")
for (nx, ny, parts, period) in [(96, 40, 2, 11), (96, 40, 2, 10**9), (96, 40, 1, 11), (1024, 24, 4, 11), (1024, 24, 4, 10**9)]:
    A, meta = P.gen_poisson2d(nx, ny, coeff_seed=4)
    b = P.gen_rhs(meta, 17)
    cfg = P.SolveConfig(rtol=1e-9, residual_refresh_period=period)
    G = P.forward(m, P.build_graph(A, meta)).G
    ref = P.pcg_solve(A, b, P.build_learned_spai(G, m.config.epsilon), cfg)
    sol = RP.PartitionedSolver(A, meta, m, parts)
    rep = sol.solve(b, cfg)
    h1, h0 = np.asarray(rep.residual_history), np.asarray(ref.residual_history)
    k = min(len(h1), len(h0))
    d = np.abs(h1[:k] - h0[:k]) / np.abs(h0[:k])
    first = int(np.argmax(d > 1e-13)) if np.any(d > 1e-13) else -1
    print(json.dumps({"case": [nx, ny, parts, period], "k": [rep.k, ref.k], "first_gt_1e-13": first,
                      "d": [float(x) for x in d[:40]]}))
