"""Golden fixtures from the REAL reference (run in the build container, where /root/reference
exists; the outputs are committed, the GPU box never reads the reference):

* golden_bench.csv -- `spaigraph bench` (cli.py:280-347) on a generated heat2d 16x16 dataset
  (cmd_generate, 10 matrices, seed 0), the test split (4:1, split seed 0), preconditioners none /
  diag / fsai / learned (learned: the committed trained fixture), rtols 1e-2 .. 1e-8.  IC(0) is a
  CPU baseline out of the GPU path's scope, so it is not requested.
* golden_heat8.mtx / golden_heat8_sym.mtx -- write_matrix_market (sparse.py:268-275) of
  gen_poisson2d(8, 6, coeff_seed=3), and the same matrix in symmetric storage (lower triangle,
  read back through the reference's expansion, sparse.py:253-263).
* golden_heat8.graph.bin -- write_graph_bin (graphfeat.py:108-123) of build_graph(A, meta).
* golden_formats.npz -- the reference readers' arrays of all three files.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bench_format_golden.py
"""
from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")


def bench_csv():
    from spaigraph import cli
    tmp = tempfile.mkdtemp()
    try:
        cfg = {"seed": 0, "out": tmp, "threads": 1,
               "generate": {"family": "heat2d", "count": 10, "nx": 16, "ny": 16},
               "bench": {"family": "heat2d", "count": 10, "use_test_split": True, "split_ratio": [4, 1],
                         "split_seed": 0, "preconditioners": ["none", "diag", "fsai", "learned"],
                         "rtols": [1e-2, 1e-4, 1e-6, 1e-8],
                         "checkpoint": os.path.join(HERE, "trained_heat16.spaignn"), "max_iters": None,
                         "workers": 1}}
        path = os.path.join(tmp, "cfg.json")
        with open(path, "w") as fh:
            json.dump(cfg, fh)
        assert cli.main(["generate", "--config", path]) == 0
        assert cli.main(["bench", "--config", path]) == 0
        shutil.copy(os.path.join(tmp, "bench.csv"), os.path.join(HERE, "golden_bench.csv"))
    finally:
        shutil.rmtree(tmp)


def formats():
    from spaigraph.datasets import gen_poisson2d
    from spaigraph.graphfeat import build_graph, read_graph_bin, write_graph_bin
    from spaigraph.sparse import read_matrix_market, write_matrix_market
    A, meta = gen_poisson2d(8, 6, coeff_seed=3)
    mtx = os.path.join(HERE, "golden_heat8.mtx")
    write_matrix_market(A, mtx)
    rows = A.row_expand()
    low = A.col_indices <= rows
    sym = os.path.join(HERE, "golden_heat8_sym.mtx")
    with open(sym, "w", encoding="ascii") as fh:
        fh.write("%%MatrixMarket matrix coordinate real symmetric\n% lower triangle\n")
        fh.write(f"{A.n_rows} {A.n_cols} {int(low.sum())}\n")
        for r, c, v in zip(rows[low], A.col_indices[low], A.values[low]):
            fh.write(f"{r + 1} {c + 1} {v:.16e}\n")
    g = build_graph(A, meta)
    gb = os.path.join(HERE, "golden_heat8.graph.bin")
    write_graph_bin(g, gb)
    A1, A2, g1 = read_matrix_market(mtx), read_matrix_market(sym), read_graph_bin(gb)
    np.savez(os.path.join(HERE, "golden_formats.npz"),
             a_offs=A.row_offsets, a_cols=A.col_indices, a_vals=A.values,
             m_offs=A1.row_offsets, m_cols=A1.col_indices, m_vals=A1.values,
             s_offs=A2.row_offsets, s_cols=A2.col_indices, s_vals=A2.values,
             g_node=g1.node_features, g_edge=g1.edge_features, g_list=g1.edge_list, g_norm=g1.norm_A,
             coeff=meta.coeff)


if __name__ == "__main__":
    bench_csv()
    formats()
    print("ok")
