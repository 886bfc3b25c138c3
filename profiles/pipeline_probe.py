"""Probe: does running the GNN of one half-batch concurrently with the PCG of the other help?

    python profiles/pipeline_probe.py [--systems 128] [--steps 3]

Two BatchSolvers of S/2 systems on two streams; per step: PCG(A) (host polls stream A) while
GNN(B) runs on stream B, then PCG(B) while GNN(A) runs.  Prints ms per step (all S systems)
for the serial path and for the overlapped one.  Diagnostic only.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--systems", type=int, default=128)
    p.add_argument("--steps", type=int, default=3)
    a = p.parse_args()
    import torch
    from paper_2510_27517_b200 import _lib
    from paper_2510_27517_b200.batch import BatchSolver, SystemBatch
    from paper_2510_27517_b200.dist import local_systems
    from paper_2510_27517_b200.gnn import load_checkpoint
    from paper_2510_27517_b200.pcg import SolveConfig

    _lib.lib()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    model = load_checkpoint(os.path.join(root, "tests", "golden", "trained_heat16.spaignn"))
    cfg = SolveConfig(rtol=1e-6, track_history=False)
    S = a.systems
    ids, rhs = local_systems(S, 0, 1)
    full = BatchSolver(SystemBatch.heat2d(256, 256, ids, rhs), model)
    h = S // 2
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(sa):
        A = BatchSolver(SystemBatch.heat2d(256, 256, ids[:h], rhs[:h]), model)
    with torch.cuda.stream(sb):
        B = BatchSolver(SystemBatch.heat2d(256, 256, ids[h:], rhs[h:]), model)
    torch.cuda.synchronize()

    def gnn(sv, st):
        with torch.cuda.stream(st):
            sv.build_graph()
            sv.build_factor()

    def pcg(sv, st):
        with torch.cuda.stream(st):
            return sv.solve(cfg)

    # warm-up both paths
    full.step(cfg)
    for sv, st in ((A, sa), (B, sb)):
        gnn(sv, st)
        pcg(sv, st)
    torch.cuda.synchronize()

    t0 = time.perf_counter()
    for _ in range(a.steps):
        full.step(cfg)
    torch.cuda.synchronize()
    serial = 1000 * (time.perf_counter() - t0) / a.steps

    gnn(A, sa)
    gnn(B, sb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ks = []
    for _ in range(a.steps):
        ra = pcg(A, sa)
        gnn(A, sa)
        rb = pcg(B, sb)
        gnn(B, sb)
        ks.append([r.k for r in ra] + [r.k for r in rb])
    torch.cuda.synchronize()
    over = 1000 * (time.perf_counter() - t0) / a.steps
    print(f"serial {serial:.1f} ms/step ({S / serial * 1000:.1f} solves/s); overlapped halves {over:.1f} ms/step "
          f"({S / over * 1000:.1f} solves/s); k mean {sum(ks[-1]) / len(ks[-1]):.1f}", flush=True)


if __name__ == "__main__":
    main()
