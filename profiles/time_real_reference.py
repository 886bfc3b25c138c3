"""Time the REAL reference package (`spaigraph`, /root/reference/pkg/src) on one C2 system.

The reference is pure Python and cannot travel to the GPU box, so bench.py's CPU arms time the
oracle restatement (oracle/spaigraph_ref.py, tape-free => faster).  This script, run in the build
container where the reference is importable, times the reference's own public path on one
heat2d 256x256 system (seed 0, trained weights, rtol 1e-6) -- build_graph -> forward ->
build_learned_spai -> pcg_solve -- next to the oracle port on the same system and the same
host, so the port-to-reference ratio can be applied to the port's numbers measured on the GPU
box ("extrapolated").  Output: one JSON line (committed as profiles/r03_reference_real_c2.json).

    OPENBLAS_NUM_THREADS=<cores> python profiles/time_real_reference.py
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    import numpy as np

    import spaigraph as S
    from oracle import spaigraph_ref as O
    ckpt = os.path.join(ROOT, "tests", "golden", "trained_heat16.spaignn")
    nx, seed, rtol = 256, 0, 1e-6
    A, meta = S.gen_poisson2d(nx, nx, coeff_seed=seed) if "coeff_seed" in S.gen_poisson2d.__code__.co_varnames \
        else S.gen_poisson2d(nx, nx, seed)
    b = S.gen_rhs(meta, seed + 10**6)
    model = S.load_checkpoint(ckpt)
    t = {}
    t0 = time.perf_counter()
    g = S.build_graph(A, meta)
    t["build_graph"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    fr = S.forward(model, g)
    t["forward"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    M = S.build_learned_spai(fr.G, model.config.epsilon)
    t["build_learned_spai"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rep = S.pcg_solve(A, b, M, S.SolveConfig(rtol=rtol))
    t["pcg_solve"] = time.perf_counter() - t0
    ref_total = sum(t.values())
    # the oracle port on the same system (what bench.py times on the GPU box)
    offs, cols, vals, coeff = O.gen_poisson2d(nx, nx, seed)
    n = nx * nx
    mlps = O.unflatten(np.asarray(model.params_flat()), O.init_params(3))
    t0 = time.perf_counter()
    node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d", (nx, nx), coeff)
    gg = O.gnn_forward(mlps, node, offs, cols, ef, 4)
    _, k_port, _, _ = O.pcg_solve(offs, cols, vals, b, lambda r: O.learned_apply(n, offs, cols, gg, 1e-4, r),
                                  rtol=rtol)
    port_total = time.perf_counter() - t0
    out = {"what": "real reference (spaigraph) vs oracle port, one C2 system (heat2d 256x256 seed 0, trained "
                   "weights, rtol 1e-6), same host, same process",
           "reference_s": t, "reference_total_s": ref_total, "reference_k": int(rep.k),
           "reference_converged": bool(rep.converged), "port_total_s": port_total, "port_k": int(k_port),
           "port_over_reference_speed": ref_total / port_total,
           "host": {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
                    "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"), "python": platform.python_version(),
                    "numpy": np.__version__, "processor": platform.processor() or platform.machine()}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
