"""TEST/BASELINE INFRASTRUCTURE ONLY — times the CPU restatement of the reference path.

Used by bench.py's `cpu_baseline` leg and by `bench.py --impl reference` (the reference package
is pure Python and cannot travel to the GPU box, so its restatement `oracle.spaigraph_ref`
stands in for it; the restatement is tape-free and therefore FASTER than the reference's own
`forward`, which makes this a conservative baseline).  One worker process per core, one BLAS
thread each, one system per worker — the reference CLI's own parallelism (cli.py:314-317).
"""
from __future__ import annotations

import os
import time


def solve_one(args):
    """Full hot path for one heat2d system on the CPU: graph -> GNN -> PCG.  Returns
    (seconds for the timed part, k, converged).  Input synthesis is not timed."""
    nx, seed, params, rtol = args
    import numpy as np

    from oracle import spaigraph_ref as O
    offs, cols, vals, coeff = O.gen_poisson2d(nx, nx, seed)
    n = nx * nx
    b = O.gen_rhs(n, seed + 10**6)
    mlps = O.unflatten(np.asarray(params), O.init_params(3))
    t0 = time.perf_counter()
    node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d", (nx, nx), coeff)
    g = O.gnn_forward(mlps, node, offs, cols, ef, 4)
    _, k, conv, _ = O.pcg_solve(offs, cols, vals, b, lambda r: O.learned_apply(n, offs, cols, g, 1e-4, r),
                                rtol=rtol)
    return time.perf_counter() - t0, int(k), bool(conv)


def run_pool(nx, seeds, params, rtol, workers):
    """Solve `seeds` with `workers` processes; returns (wall seconds, per-system results)."""
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        pool.map(_noop, range(workers))  # start-up outside the timed region
        t0 = time.perf_counter()
        res = pool.map(solve_one, [(nx, s, list(params), rtol) for s in seeds])
        wall = time.perf_counter() - t0
    return wall, res


def _noop(_):
    import numpy  # noqa: F401

    from oracle import spaigraph_ref  # noqa: F401
    return 0
