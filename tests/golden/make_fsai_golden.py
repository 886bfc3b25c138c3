"""Golden vectors for the FSAI baseline from the REFERENCE package.

Runs in the build container only (needs /root/reference): build_fsai (precond.py:262-305) on a
heat2d 12x12 system and a random sparse SPD matrix; the factor values, the fallback count and
pcg_solve's k / history length with that preconditioner.  Writes tests/golden/golden_fsai.npz.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from spaigraph.datasets import gen_poisson2d, gen_rhs  # noqa: E402
from spaigraph.pcg import SolveConfig, pcg_solve  # noqa: E402
from spaigraph.precond import build_fsai  # noqa: E402


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    out = {}
    A, meta = gen_poisson2d(12, 12, coeff_seed=4)
    b = gen_rhs(meta, 7)
    for tag, M_, b_ in (("heat", A, b),):
        P = build_fsai(M_)
        out[tag + "_offs"], out[tag + "_cols"], out[tag + "_vals"] = M_.row_offsets, M_.col_indices, M_.values
        out[tag + "_lvals"] = P.g_lower.values
        out[tag + "_fallbacks"] = np.int64(P.fallback_rows)
        out[tag + "_b"] = b_
        rep = pcg_solve(M_, b_, P, SolveConfig(rtol=1e-8))
        out[tag + "_k"] = np.int64(rep.k)
        out[tag + "_x"] = rep.x
    np.savez_compressed(os.path.join(here, "golden_fsai.npz"), **out)
    print({k: (int(v) if np.ndim(v) == 0 else np.shape(v)) for k, v in out.items()})


if __name__ == "__main__":
    main()
