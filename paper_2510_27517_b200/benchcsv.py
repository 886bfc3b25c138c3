"""The `spaigraph bench` table with the solves on the GPU (cli.py:280-347).

`bench_rows(items, preconditioners, rtols, max_iters, model)` produces the reference's rows
(matrix_id, preconditioner, rtol, k, t_construct_ns, t_apply_total_ns, t_cg_total_ns, converged)
for the preconditioners this package runs on the device ("none", "diag", "fsai", "learned"; the
IC(0) baseline stays out of scope and raises NotImplementedError), and `write_bench_csv`
writes bench.csv with the reference header.  Unlike the reference, the learned column's
t_construct_ns includes the GNN inference (graph -> G -> G^T), measured on the device clock;
t_apply_total_ns is 0 because the apply is fused into the PCG iteration kernels
(t_cg_total_ns is the device time of the whole solve).
"""
from __future__ import annotations

import csv
import time

from .gnn import forward
from .pcg import SolveConfig, pcg_solve
from .precond import build_fsai, build_identity, build_jacobi, build_learned_spai

__all__ = ["BENCH_HEADER", "bench_rows", "write_bench_csv", "summarize"]

BENCH_HEADER = ["matrix_id", "preconditioner", "rtol", "k", "t_construct_ns", "t_apply_total_ns", "t_cg_total_ns",
                "converged"]


def _build(name, A, graph, model):
    import torch
    if name == "none":
        return build_identity(A)
    if name == "diag":
        return build_jacobi(A)
    if name == "learned":
        if model is None:
            raise ValueError("the learned preconditioner needs a model")
        torch.cuda.synchronize()
        t0 = time.perf_counter_ns()
        M = build_learned_spai(forward(model, graph).G, model.config.epsilon)
        M.factor_t()  # explicit G^T is part of the construction
        torch.cuda.synchronize()
        M.t_construct_ns = time.perf_counter_ns() - t0
        return M
    if name == "fsai":
        return build_fsai(A)
    if name == "ic0":
        raise NotImplementedError("ic0 is a CPU baseline of the reference (triangular solves), not part of the GPU path")
    raise ValueError(f"unknown preconditioner {name!r}")


def bench_rows(items, preconditioners=("none", "diag", "learned"), rtols=(1e-6, 1e-8), max_iters=None,
               model=None):
    """items: iterable of (matrix_id, A, graph, rhs) (cli.py:_load_items order)."""
    rows = []
    for matrix_id, A, graph, rhs in items:
        for name in preconditioners:
            M = _build(name, A, graph, model)
            for rtol in rtols:
                rep = pcg_solve(A, rhs, M, SolveConfig(rtol=rtol, max_iters=max_iters, track_history=False))
                rows.append((matrix_id, name, rtol, rep.k, rep.t_construct_ns, rep.t_apply_total_ns,
                             rep.t_cg_total_ns, rep.converged))
    return rows


def write_bench_csv(rows, path) -> None:
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(BENCH_HEADER)
        writer.writerows(rows)


def summarize(rows):
    """cli.py:339-346: mean k and all-converged per preconditioner at the tightest rtol."""
    tightest = min(r[2] for r in rows)
    out = {}
    for name in dict.fromkeys(r[1] for r in rows):
        sel = [r for r in rows if r[1] == name and r[2] == tightest]
        out[name] = (sum(r[3] for r in sel) / len(sel) if sel else float("nan"), all(r[7] for r in sel))
    return tightest, out
