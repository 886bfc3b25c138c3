"""Golden vectors for gen_synthetic (datasets.py:148-193) from the REAL reference (test
infrastructure; runs only in the build container, where /root/reference exists).

    python tests/golden/make_synthetic_golden.py   # writes tests/golden/golden_synthetic.npz

Cases: the reference tests' own calls (test_datasets.py:87, 93, 100) plus n = 1, a dense P
(density 1.0) and a mid-size sparse one.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from spaigraph.datasets import gen_synthetic  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [(50, 0.05, 2), (10, 0.0, 0), (1024, 3e-4, 7), (1, 1.0, 3), (30, 1.0, 4), (400, 0.01, 5)]


def main():
    out = {"cases": np.array(CASES, dtype=np.float64)}
    for t, (n, dens, seed) in enumerate(CASES):
        A, meta = gen_synthetic(n, dens, seed)
        out[f"s{t}_offs"] = A.row_offsets
        out[f"s{t}_cols"] = A.col_indices
        out[f"s{t}_vals"] = A.values
        out[f"s{t}_result_density"] = meta.result_density
        print(n, dens, seed, "nnz", A.nnz)
    np.savez_compressed(os.path.join(HERE, "golden_synthetic.npz"), **out)


if __name__ == "__main__":
    main()
