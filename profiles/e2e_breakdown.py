"""Where the end-to-end (host buffers in, host x out) time of one C2 step goes.

    python profiles/e2e_breakdown.py [--systems 128] [--nx 256]

Builds the same reference-typed pinned host systems as bench.py's e2e leg, then times (CUDA
synchronised, wall clock) each stage of `solve_batch`: upload (from_host), graph build, GNN
factor, PCG, x download.  Diagnostic only; not a bench number.
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--systems", type=int, default=128)
    p.add_argument("--nx", type=int, default=256)
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    import torch
    from paper_2510_27517_b200 import _lib
    from paper_2510_27517_b200.batch import SystemBatch, BatchSolver
    from paper_2510_27517_b200.datasets import ProblemMeta
    from paper_2510_27517_b200.gnn import load_checkpoint
    from paper_2510_27517_b200.pcg import SolveConfig
    from paper_2510_27517_b200.dist import local_systems

    _lib.lib()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    model = load_checkpoint(os.path.join(root, "tests", "golden", "trained_heat16.spaignn"))
    cfg = SolveConfig(rtol=1e-6, track_history=False)
    S, n1 = a.systems, a.nx * a.nx
    ids, rhs = local_systems(S, 0, 1)
    batch = SystemBatch.heat2d(a.nx, a.nx, ids, rhs)

    def pinned(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h.numpy()

    offs_h, cols_h = pinned(batch.a.offs.to(torch.int64)), pinned(batch.a.cols.to(torch.int64))
    vals_h, b_h, coeff_h = pinned(batch.a.vals), pinned(batch.b), pinned(batch.coeff)

    class HostCsr:
        def __init__(self, n, o, c, v):
            self.n_rows = self.n_cols = n
            self.row_offsets, self.col_indices, self.values = o, c, v

    As, bs, metas = [], [], []
    loc_offs = torch.empty(S * (n1 + 1), dtype=torch.int64, pin_memory=True).numpy()
    loc_cols = torch.empty(len(cols_h), dtype=torch.int64, pin_memory=True).numpy()
    for k in range(S):
        r0, r1 = int(batch.row_start[k]), int(batch.row_start[k + 1])
        e0, e1 = int(batch.nnz_start[k]), int(batch.nnz_start[k + 1])
        o_k = loc_offs[k * (n1 + 1):(k + 1) * (n1 + 1)]
        np.subtract(offs_h[r0:r1 + 1], e0, out=o_k)
        c_k = loc_cols[e0:e1]
        np.subtract(cols_h[e0:e1], r0, out=c_k)
        As.append(HostCsr(r1 - r0, o_k, c_k, vals_h[e0:e1]))
        bs.append(b_h[r0:r1])
        metas.append(ProblemMeta(family="heat2d", n=r1 - r0, grid=(a.nx, a.nx), coeff=coeff_h[r0:r1],
                                 coeff_seed=ids[k]))
    up = SystemBatch.from_host(As, bs, metas)
    solver = BatchSolver(up, model)
    solver.step(cfg)

    def t(f):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        return r, 1000.0 * (time.perf_counter() - t0)

    for rep in range(a.reps):
        _, t_up = t(lambda: SystemBatch.from_host(As, bs, metas, into=solver.batch))
        _, t_graph = t(solver.build_graph)
        _, t_fac = t(solver.build_factor)
        _, t_pcg = t(lambda: solver.solve(cfg))
        _, t_dn = t(lambda: solver.x.cpu().numpy())
        print(f"rep {rep}: upload {t_up:.1f} ms  graph {t_graph:.1f}  factor {t_fac:.1f}  pcg {t_pcg:.1f}  "
              f"download {t_dn:.1f}  total {t_up + t_graph + t_fac + t_pcg + t_dn:.1f}", flush=True)


if __name__ == "__main__":
    main()
