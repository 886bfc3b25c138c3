#!/usr/bin/env python
"""Single-system configurations of BASELINE.json (configs[0], [2], [4]) through the public API.

    python bench_configs.py --config c1     # 64x64 Poisson, random-init GNN (d_node=3, seed 0), rtol 1e-6
    python bench_configs.py --config c3     # 128^3 Poisson (n = 2.1M), algebraic features, random-init (d_node=2)
    python bench_configs.py --config c5     # 2048^2 Poisson (n = 4.2M), trained weights, + SAI loss fwd/bwd

One JSON line per run.  A step = build_graph -> forward -> build_learned_spai (G^T) ->
pcg_solve, with A generated on the device beforehand (inputs resident).  The PCG iteration
kernels are sampled by the in-graph event nodes (same method as bench.py) and reported against
the survey's per-iteration byte formula and MEASURED_PEAKS.json.  bench.py (config C2) is the
driver's headline; this script records the other configurations.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1", choices=["c1", "c3", "c4", "c5"])
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=1)
    p.add_argument("--max-iters", type=int, default=None)
    p.add_argument("--cpu", action="store_true", help="also time the CPU restatement (c1 only)")
    p.add_argument("--parts", type=int, default=0,
                   help="c5: solve through the row partition with this many partitions on this GPU (group mode)")
    a = p.parse_args()

    import torch

    import paper_2510_27517_b200 as P
    from paper_2510_27517_b200 import _lib

    _lib.lib()
    dev = torch.device("cuda", 0)
    if a.config == "c1":
        A, meta = P.gen_poisson2d(64, 64)
        model = P.init_model(P.GnnConfig(d_node=3, seed=0))
        b = P.gen_rhs(meta, 10**6)
        desc = "C1: 2D Poisson 64x64 (n=4096), random-init GNN-SPAI (d_node=3, seed 0), PCG rtol 1e-6"
    elif a.config == "c3":
        A, meta = P.gen_poisson3d(128, 128, 128)
        model = P.init_model(P.GnnConfig(d_node=2, seed=0))
        b = P.gen_rhs(meta, 10**6)
        desc = "C3: 3D Poisson 7-point 128^3 (n=2,097,152), algebraic features, random-init GNN (d_node=2), PCG rtol 1e-6"
    elif a.config == "c4":
        from paper_2510_27517_b200.sparse import pad_to_pattern, pattern_square
        t0 = time.perf_counter()
        A = P.rand_spd_sparse(10**6, np.random.default_rng(0), extra_per_row=10)
        t_gen = time.perf_counter() - t0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Pq = pattern_square(A)
        Ap = pad_to_pattern(A, Pq)
        torch.cuda.synchronize()
        t_pat = time.perf_counter() - t0
        meta = None
        model = P.init_model(P.GnnConfig(d_node=2, seed=0))
        b = P.gen_rhs(A.n_rows, 10**6)
        desc = (f"C4: rand_spd_sparse(n=1e6, extra_per_row=10) (nnz {A.nnz}), G on the A^2 pattern (nnz {Pq.nnz}), "
                f"graph on A padded to it, random-init GNN (d_node=2), PCG rtol 1e-6 (generation {t_gen:.1f} s host+GPU, "
                f"A^2 pattern + padding {1000 * t_pat:.0f} ms GPU)")
    else:
        A, meta = P.gen_poisson2d(2048, 2048)
        model = P.load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_heat16.spaignn"))
        b = P.gen_rhs(meta, 10**6)
        desc = "C5: 2D Poisson 2048x2048 (n=4,194,304), trained GNN-SPAI, PCG rtol 1e-6, + SAI loss fwd/bwd"
    cfg = P.SolveConfig(rtol=1e-6, max_iters=a.max_iters)
    b_dev = torch.as_tensor(b, device=dev)
    w_dev = torch.as_tensor(np.random.default_rng(0).standard_normal(A.n_rows), device=dev)

    if a.parts:
        return run_parts(a, P, A, meta, model, b)

    def step(profile=False):
        g = P.build_graph(Ap if a.config == "c4" else A, meta if a.config not in ("c3", "c4") else None)
        G = P.forward(model, g).G
        M = P.build_learned_spai(G, model.config.epsilon)
        if profile:
            from paper_2510_27517_b200.pcg import _handle_for
            h = _handle_for(A, M, "learned")
            h.set_profile(True)
            h.stats(reset=True)
        rep = P.pcg_solve(A, b_dev, M, cfg)
        loss = None
        if a.config == "c5":
            loss, grad = P.sai_loss_and_grad(A, G, model.config.epsilon, w_dev)
        return rep, M, loss

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    import bench as B
    clocks = B.ClockSampler(dev.index or 0)
    times, reps = [], []
    for s in range(a.steps):
        t0 = time.perf_counter()
        rep, M, loss = step(profile=(s == a.steps - 1))
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        reps.append(rep)
    clk = clocks.stop()
    from paper_2510_27517_b200.pcg import _handle_for
    h = _handle_for(A, M, "learned")
    kernels, chunks, prof = h.stats()
    n, nnz = A.n_rows, A.nnz
    nnz_g = Ap.nnz if a.config == "c4" else nnz  # G (and G^T) live on the A^2 pattern for C4
    # SURVEY.md §8(d) B_iter (fp64 values, int32 indices): A once, G^T and G once each, vectors
    it_bytes = (12 * nnz + 4 * (n + 1)) + 2 * (12 * nnz_g + 4 * (n + 1)) + 112 * n
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    per_k = {}
    roof = None
    if prof[4] > 0 and prof[5]:  # DIA kernels: the algorithmic bytes of the layout they run (bench.py)
        peak_b, peak_src = B.hbm_peak()
        strip = a.config == "c5"
        roof = B.pcg_roofline(prof, n, nnz, peak_b, peak_src, K23_SW="k_iter23_s5" if strip else "k_iter23_sw",
                              K1_SW="k_iter1_s5p" if strip else "k_iter1_sw", units_note="one system",
                              which="c5" if strip else "none")
        if roof:
            per_k = {name.split(" ")[0]: v for name, v in roof["per_kernel"].items()}
    elif prof[4] > 0:  # CSR (C4): SURVEY §8(d) bytes, G on its own (A^2) pattern
        csr = 12 * nnz + 4 * (n + 1)
        csr_g = 12 * nnz_g + 4 * (n + 1)
        if prof[7]:  # K2 + K3 fused (t stays on chip)
            per_sys = {"k_iter1": csr + 32 * n, "k_iter23": csr_g + 56 * n}
        else:
            per_sys = {"k_iter1": csr + 32 * n, "k_iter2": csr_g + 56 * n, "k_iter3": csr_g + 24 * n}
        for (name, by), ms in zip(per_sys.items(), prof[:3]):
            avg = ms / prof[4]
            per_k[name] = {"avg_ms": avg, "gbs": by / (avg * 1e-3) / 1e9, "frac": by / (avg * 1e-3) / 1e9 / peak}
    rep = reps[-1]
    ms = 1000 * float(np.median(times))
    out = {"config": a.config, "workload": desc, "metric": "PCG solves/sec (GNN build+solve)",
           "value": 1000.0 / ms, "unit": "solves/s", "ms_per_solve": ms, "k": rep.k, "converged": rep.converged,
           "max_iters": a.max_iters,
           "pcg_ms": (rep.t_cg_total_ns + rep.t_apply_total_ns) / 1e6,
           "pcg_us_per_iteration": (rep.t_cg_total_ns + rep.t_apply_total_ns) / 1e3 / max(rep.k, 1),
           "pcg_time_split_ns": {"t_cg_total_ns": int(rep.t_cg_total_ns), "t_apply_total_ns": int(rep.t_apply_total_ns)},
           "iteration_gbs_survey_bytes": it_bytes * rep.k / ((rep.t_cg_total_ns + rep.t_apply_total_ns) * 1e-9) / 1e9,
           "storage": f"DIA ({int(prof[5])} diagonals)" if prof[5] else "CSR", "per_kernel": per_k,
           "peak_gbs": peak, "n": n, "nnz": nnz, "nnz_G": nnz_g, "clocks": clk}
    if roof:
        out["roofline"] = {k: v for k, v in roof.items() if k != "per_kernel"}
    if loss is not None:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            P.sai_loss_and_grad(A, reps and P.forward(model, P.build_graph(A, meta)).G, model.config.epsilon, w_dev)
        torch.cuda.synchronize()
        out["loss"] = loss
        out["loss_fwd_bwd_ms_incl_forward"] = 1000 * (time.perf_counter() - t0) / 3
    if a.cpu and a.config == "c1":
        from oracle import spaigraph_ref as O
        offs, cols, vals, coeff = O.gen_poisson2d(64, 64)
        t0 = time.perf_counter()
        node, _, ef, _ = O.graph_features(4096, offs, cols, vals, "poisson2d", (64, 64), coeff)
        g = O.gnn_forward(O.init_params(3, seed=0), node, offs, cols, ef, 4)
        _, k_ref, _, _ = O.pcg_solve(offs, cols, vals, b, lambda r: O.learned_apply(4096, offs, cols, g, 1e-4, r),
                                     rtol=1e-6)
        out["cpu_baseline"] = {"value": 1.0 / (time.perf_counter() - t0), "unit": "solves/s", "cores": 1,
                               "kind": "port", "k": k_ref}
    print(json.dumps(out), flush=True)


def run_parts(a, P, A, meta, model, b):
    """C5 through the row partition in group mode (the P-rank emulation on one GPU): setup
    (per-partition GNN blocks, extended systems, handle) and solve timed separately."""
    import torch

    from paper_2510_27517_b200.rowpart import PartitionedSolver
    cfg = P.SolveConfig(rtol=1e-6, max_iters=a.max_iters)
    for _ in range(max(a.warmup, 1)):
        PartitionedSolver(A, meta, model, a.parts).solve(b, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = PartitionedSolver(A, meta, model, a.parts)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    sol.handle.set_profile(True)
    sol.solve(b, cfg)
    sol.handle.stats(reset=True)
    times = []
    for _ in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = sol.solve(b, cfg)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    _, _, prof = sol.handle.stats()
    per = {}
    if prof[4] > 0:
        per = {"k_iter1_ms": prof[0] / prof[4], "k_iter23_ms": prof[1] / prof[4]}
    ms = 1000 * float(np.median(times))
    ext_rows = int(sol.row_start[-1])
    print(json.dumps({"config": "c5", "parts": a.parts, "mode": "group (one handle, one GPU)",
                      "k": rep.k, "converged": rep.converged, "solve_ms": ms, "setup_ms": 1000 * t_setup,
                      "us_per_iteration": 1000 * ms / max(rep.k, 1), "extended_rows": ext_rows,
                      "ghost_overhead": ext_rows / A.n_rows - 1.0, "per_kernel": per}), flush=True)


if __name__ == "__main__":
    main()
