"""Wall time of each stage of the C1 drop-in path (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2510_27517_b200 as P
A, meta = P.gen_poisson2d(64, 64)
model = P.init_model(P.GnnConfig(d_node=3, seed=0))
b = P.gen_rhs(meta, 10**6)
cfg = P.SolveConfig(rtol=1e-6)
for rep in range(3):
    t = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = P.build_graph(A, meta); torch.cuda.synchronize(); t['graph'] = time.perf_counter() - t0; t0 = time.perf_counter()
    G = P.forward(model, g).G; torch.cuda.synchronize(); t['forward'] = time.perf_counter() - t0; t0 = time.perf_counter()
    M = P.build_learned_spai(G, model.config.epsilon); torch.cuda.synchronize(); t['spai'] = time.perf_counter() - t0; t0 = time.perf_counter()
    r = P.pcg_solve(A, b, M, cfg); torch.cuda.synchronize(); t['pcg'] = time.perf_counter() - t0
    print({k: round(v * 1000, 2) for k, v in t.items()}, r.k, round(r.t_cg_total_ns / 1e6, 2), round(r.t_apply_total_ns / 1e6, 2))
