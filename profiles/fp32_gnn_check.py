# CPU: how far a plain fp32 numpy evaluation of the reference GNN forward is from fp64 (trained vs random-init).
import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import spaigraph_ref as O
from paper_2510_27517_b200.gnn import load_checkpoint
params = load_checkpoint(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests', 'golden', 'trained_heat16.spaignn')).params_flat()
for case in ("trained", "random"):
    offs, cols, vals, coeff = O.gen_poisson2d(64, 64, 5 if case == "trained" else None)
    n = 64*64
    node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d" if case=="trained" else "poisson2d", (64,64), coeff)
    mlps = O.unflatten(params, O.init_params(3)) if case=="trained" else O.init_params(3, seed=0)
    g64 = O.gnn_forward_restructured(mlps, node, offs, cols, ef, 4)
    m32 = [[(W.astype(np.float32), b.astype(np.float32)) for W, b in m] for m in mlps]
    g32 = O.gnn_forward_restructured(m32, node.astype(np.float32), offs, cols, ef.astype(np.float32), 4)
    scale = np.maximum(np.abs(g64), 1e-3*np.abs(g64).max())
    print(case, "fp32 numpy err", np.max(np.abs(g32 - g64)/scale), "max|G|", np.abs(g64).max(), "median |G|", np.median(np.abs(g64)))
