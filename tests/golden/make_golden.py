"""Generate golden vectors by running the REFERENCE package (test infrastructure).

Runs only in the build container, where /root/reference exists.  Every array in the .npz
files below is an output of the reference `spaigraph` (pkg/src/spaigraph) on seeded inputs;
tests/test_oracle.py pins the oracle restatement to them on the CPU and the `-m gpu` tests pin
the CUDA path to them on a B200 (the GPU box has no /root/reference, so the fixtures travel).

    python tests/golden/make_golden.py          # rewrites tests/golden/golden_*.npz

Cases:
  c1      gen_poisson2d(64,64); build_graph; random-init GnnConfig(d_node=3, seed=0) forward;
          b = gen_rhs(meta, 10**6); pcg_solve(rtol=1e-6) -> k, history, x;
          sai_loss(w=default_rng(0).standard_normal(n)) and its tape gradient w.r.t. G values.
  heat    gen_poisson2d(16,16,coeff_seed=3) with the trained fixture (trained_heat16.spaignn),
          b = gen_rhs(meta, 3 + 10**6), rtol 1e-8 and 1e-6.
  sparse  rand_sparse_spd / rand_sparse (reference tests/conftest.py) -> from_coo, transpose,
          spmv, spmv_transpose, norms, is_symmetric, algebraic graph features, small-GNN G
          (hidden 6, 2 layers, tanh and relu), learned apply, loss + gradient for 3 norm kinds.
  pcg     identity / jacobi / learned solves on small systems incl. delta termination,
          max_iters exhaustion, refresh periods, zero rhs.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from conftest import rand_sparse, rand_sparse_spd  # noqa: E402  (reference test helpers)
from spaigraph.autodiff import Tape  # noqa: E402
from spaigraph.datasets import gen_poisson2d, gen_rhs  # noqa: E402
from spaigraph.gnn import GnnConfig, forward, init_model, load_checkpoint  # noqa: E402
from spaigraph.graphfeat import build_graph  # noqa: E402
from spaigraph.pcg import SolveConfig, pcg_solve  # noqa: E402
from spaigraph.precond import build_identity, build_jacobi, build_learned_spai  # noqa: E402
from spaigraph.sparse import SparseMatrix, mean_abs_nonzero_norm, spmv, spmv_transpose  # noqa: E402
from spaigraph.training import NORM_KINDS, matrix_norm, sai_loss, sai_loss_on_tape  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def csr(prefix, A, out):
    out[prefix + "_n_rows"] = A.n_rows
    out[prefix + "_n_cols"] = A.n_cols
    out[prefix + "_offs"] = A.row_offsets
    out[prefix + "_cols"] = A.col_indices
    out[prefix + "_vals"] = A.values


def loss_grad(A, G, eps, w, kind):
    tape = Tape()
    gv = tape.leaf(G.values)
    loss = sai_loss_on_tape(tape, A, gv, G.pattern, eps, w, kind)
    tape.backward(loss)
    return float(loss.value), gv.grad.copy()


def case_c1():
    out = {}
    A, meta = gen_poisson2d(64, 64)
    g = build_graph(A, meta)
    csr("A", A, out)
    out["norm_A"] = g.norm_A
    out["node_features"] = g.node_features
    model = init_model(GnnConfig(d_node=3, seed=0))
    out["params"] = model.params_flat()
    G = forward(model, g).G
    out["G_vals"] = G.values
    b = gen_rhs(meta, 10**6)
    out["b"] = b
    rep = pcg_solve(A, b, build_learned_spai(G, model.config.epsilon), SolveConfig(rtol=1e-6))
    out["k"], out["converged"] = rep.k, rep.converged
    out["history"] = np.asarray(rep.residual_history)
    out["x"] = rep.x
    w = np.random.default_rng(0).standard_normal(A.n_rows)
    out["w"] = w
    out["loss"], out["grad"] = loss_grad(A, G, model.config.epsilon, w, "mean_abs_nonzero")
    np.savez_compressed(os.path.join(HERE, "golden_c1.npz"), **out)
    print("c1 k", rep.k, "loss", out["loss"])


def case_heat():
    out = {}
    model = load_checkpoint(os.path.join(HERE, "trained_heat16.spaignn"))
    out["params"] = model.params_flat()
    for nx, seed in ((16, 3), (32, 7)):
        A, meta = gen_poisson2d(nx, nx, coeff_seed=seed)
        g = build_graph(A, meta)
        p = f"h{nx}"
        csr(p + "A", A, out)
        out[p + "coeff"] = meta.coeff
        out[p + "node_features"] = g.node_features
        out[p + "norm_A"] = g.norm_A
        G = forward(model, g).G
        out[p + "G_vals"] = G.values
        b = gen_rhs(meta, seed + 10**6)
        out[p + "b"] = b
        M = build_learned_spai(G, model.config.epsilon)
        for rtol, tag in ((1e-8, "r8"), (1e-6, "r6")):
            rep = pcg_solve(A, b, M, SolveConfig(rtol=rtol))
            out[p + "k_" + tag] = rep.k
            out[p + "hist_" + tag] = np.asarray(rep.residual_history)
            out[p + "x_" + tag] = rep.x
    np.savez_compressed(os.path.join(HERE, "golden_heat.npz"), **out)
    print("heat", {k: int(v) for k, v in out.items() if "k_" in k})


def case_sparse():
    out = {}
    rng = np.random.default_rng(2024)
    # COO -> CSR with shuffled triplets (from_coo sorts), incl. an explicit zero and empty rows
    R = rand_sparse(40, 30, rng, density=0.15)
    rows, cols, vals = R.row_expand(), R.col_indices, R.values.copy()
    vals[3] = 0.0
    perm = rng.permutation(len(rows))
    out["trip_rows"], out["trip_cols"], out["trip_vals"] = rows[perm], cols[perm], vals[perm]
    B = SparseMatrix.from_coo(40, 30, rows[perm], cols[perm], vals[perm])
    csr("coo", B, out)
    T = B.transpose()
    csr("cooT", T, out)
    x30, x40 = rng.standard_normal(30), rng.standard_normal(40)
    out["x30"], out["x40"] = x30, x40
    out["coo_spmv"] = spmv(B, x30)
    out["coo_spmvT"] = spmv_transpose(B, x40)
    out["coo_norm"] = mean_abs_nonzero_norm(B)
    # long rows (exercise numpy's pairwise order: 8-accumulator blocks and the >128 split)
    L = rand_sparse(12, 700, rng, density=0.6)
    csr("long", L, out)
    out["x700"] = rng.standard_normal(700)
    out["long_spmv"] = spmv(L, out["x700"])
    # SPD systems with a symmetric pattern
    for tag, n in (("s15", 15), ("s60", 60), ("s300", 300)):
        A = rand_sparse_spd(n, rng)
        csr(tag, A, out)
        g = build_graph(A)
        out[tag + "_node_features"] = g.node_features
        out[tag + "_norm_A"] = g.norm_A
        for kind in NORM_KINDS:
            out[tag + "_mnorm_" + kind] = matrix_norm(A, kind)
        Gr = A.with_values(rng.standard_normal(A.nnz))
        out[tag + "_Grand"] = Gr.values
        r = rng.standard_normal(n)
        out[tag + "_r"] = r
        out[tag + "_apply"] = build_learned_spai(Gr, 2e-3).apply(r)
        out[tag + "_spmv"] = spmv(A, r)
        out[tag + "_spmvT"] = spmv_transpose(Gr, r)
        w = rng.standard_normal(n)
        out[tag + "_w"] = w
        for kind in NORM_KINDS:
            lv, gr = loss_grad(A, Gr, 1e-3, w, kind)
            out[tag + "_loss_" + kind] = lv
            out[tag + "_grad_" + kind] = gr
        for act in ("relu", "tanh"):
            cfg = GnnConfig(n_layers=2, hidden_dim=6, d_node=2, seed=5, activation=act)
            m = init_model(cfg)
            out[tag + "_small_params_" + act] = m.params_flat()
            out[tag + "_small_G_" + act] = forward(m, g).G.values
        m24 = init_model(GnnConfig(d_node=2, seed=1))
        out[tag + "_g24_params"] = m24.params_flat()
        out[tag + "_g24_G"] = forward(m24, g).G.values
    # non-symmetric pattern (build_graph must reject)
    out["asym_offs"] = np.array([0, 2, 3]); out["asym_cols"] = np.array([0, 1, 1])
    np.savez_compressed(os.path.join(HERE, "golden_sparse.npz"), **out)
    print("sparse done")


def case_pcg():
    out = {}
    rng = np.random.default_rng(77)
    cases = []
    A = rand_sparse_spd(60, rng)
    b = rng.standard_normal(60)
    cases.append(("id_true", A, b, "identity", SolveConfig(rtol=1e-8)))
    cases.append(("jac_true", A, b, "jacobi", SolveConfig(rtol=1e-8)))
    cases.append(("jac_delta", A, b, "jacobi", SolveConfig(rtol=1e-10, termination="delta")))
    cases.append(("id_max3", A, b, "identity", SolveConfig(max_iters=3)))
    cases.append(("id_p7", A, b, "identity", SolveConfig(rtol=1e-10, residual_refresh_period=7)))
    cases.append(("zero_rhs", A, np.zeros(60), "identity", SolveConfig()))
    Gr = A.with_values(rng.standard_normal(A.nnz) * 0.3)
    cases.append(("learn_true", A, b, ("learned", Gr, 1e-3), SolveConfig(rtol=1e-8)))
    cases.append(("learn_p3", A, b, ("learned", Gr, 1e-3), SolveConfig(rtol=1e-9, residual_refresh_period=3)))
    cases.append(("learn_delta", A, b, ("learned", Gr, 1e-3), SolveConfig(rtol=1e-9, termination="delta")))
    csr("A", A, out)
    out["b"] = b
    out["Gr"] = Gr.values
    names = []
    for name, A_, b_, pre, cfg in cases:
        if pre == "identity":
            M = build_identity(A_)
        elif pre == "jacobi":
            M = build_jacobi(A_)
        else:
            M = build_learned_spai(pre[1], pre[2])
        rep = pcg_solve(A_, b_, M, cfg)
        out[name + "_k"] = rep.k
        out[name + "_conv"] = rep.converged
        out[name + "_x"] = rep.x
        out[name + "_hist"] = np.asarray(rep.residual_history)
        names.append(name)
    np.savez_compressed(os.path.join(HERE, "golden_pcg.npz"), **out)
    print("pcg", {n: int(out[n + "_k"]) for n in names})


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "sparse", "pcg", "heat"]
    for w in which:
        globals()["case_" + w]()
