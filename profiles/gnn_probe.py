"""Time the GNN factor build (forward + G^T gather) of the C2 batch with CUDA events.

    python profiles/gnn_probe.py [--lib path/to/libspaigraph_b200.so] [--systems 128] [--reps 5]

Used to compare kernel variants built into separate libraries (diagnostic only; not a bench
number).  Prints ms per build_factor and the G checksum so variants can be checked for
bit-identical output.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--lib", default=None)
    p.add_argument("--systems", type=int, default=128)
    p.add_argument("--reps", type=int, default=5)
    a = p.parse_args()
    from paper_2510_27517_b200 import _lib
    if a.lib:
        _lib.LIB_PATH = os.path.abspath(a.lib)
    import torch
    from paper_2510_27517_b200.batch import BatchSolver, SystemBatch
    from paper_2510_27517_b200.dist import local_systems
    from paper_2510_27517_b200.gnn import load_checkpoint

    _lib.lib()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    model = load_checkpoint(os.path.join(root, "tests", "golden", "trained_heat16.spaignn"))
    ids, rhs = local_systems(a.systems, 0, 1)
    sv = BatchSolver(SystemBatch.heat2d(256, 256, ids, rhs), model)
    sv.build_graph()
    sv.build_factor()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(a.reps):
        e0.record()
        sv.build_factor()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    g = sv.g.double()
    print(f"lib={_lib.LIB_PATH} build_factor ms: min {min(ts):.2f} med {sorted(ts)[len(ts) // 2]:.2f} "
          f"checksum {float(g.sum()):.17g} {float(g.abs().sum()):.17g}", flush=True)


if __name__ == "__main__":
    main()
