"""CPU: on-disk formats written by this package are byte-identical to the reference's own
writers: Matrix Market (sparse.py:268-275) and SPGRAPH\\x01 graph.bin
(graphfeat.py:108-123).  The golden files come from the real reference
(tests/golden/make_bench_format_golden.py); the readers are checked on the GPU
(tests/test_gpu_formats.py)."""
import os
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def _golden():
    return np.load(os.path.join(GOLD, "golden_formats.npz"))


def test_write_matrix_market_matches_reference_bytes(tmp_path):
    from paper_2510_27517_b200.sparse import write_matrix_market
    g = _golden()
    offs, cols, vals = g["a_offs"], g["a_cols"], g["a_vals"]
    n = len(offs) - 1
    A = SimpleNamespace(n_rows=n, n_cols=n, nnz=len(cols), col_indices=cols, values=vals,
                        row_expand=lambda: np.repeat(np.arange(n, dtype=np.int64), np.diff(offs)))
    out = tmp_path / "a.mtx"
    write_matrix_market(A, out)
    assert out.read_bytes() == open(os.path.join(GOLD, "golden_heat8.mtx"), "rb").read()


def test_write_graph_bin_matches_reference_bytes(tmp_path):
    from paper_2510_27517_b200.graphfeat import write_graph_bin
    g = _golden()
    graph = SimpleNamespace(n_nodes=g["g_node"].shape[0], n_edges=g["g_list"].shape[0],
                            d_node=g["g_node"].shape[1], d_edge=g["g_edge"].shape[1], norm_A=float(g["g_norm"]),
                            node_features=g["g_node"], edge_features=g["g_edge"], edge_list=g["g_list"])
    out = tmp_path / "g.bin"
    write_graph_bin(graph, out)
    assert out.read_bytes() == open(os.path.join(GOLD, "golden_heat8.graph.bin"), "rb").read()


def test_golden_bench_csv_schema():
    import csv
    from paper_2510_27517_b200.benchcsv import BENCH_HEADER
    rows = list(csv.reader(open(os.path.join(GOLD, "golden_bench.csv"))))
    assert rows[0] == BENCH_HEADER
    assert len(rows) == 1 + 2 * 4 * 4  # 2 test matrices x 4 preconditioners x 4 rtols
