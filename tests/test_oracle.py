"""CPU: pin the oracle restatement (oracle/spaigraph_ref.py) to the reference's golden vectors.

The fixtures were produced by the reference itself (tests/golden/make_golden.py).  Integer and
pattern outputs must be bit-identical; SpMV / transpose-SpMV / apply / norms / features are
bit-identical too (same numpy order); GNN outputs are tolerance-checked (BLAS order differs).
"""
import math

import numpy as np
import pytest

from oracle import spaigraph_ref as O


def _csr(g, p):
    return int(g[p + "_n_rows"]), int(g[p + "_n_cols"]), g[p + "_offs"], g[p + "_cols"], g[p + "_vals"]


def test_from_coo_and_transpose_bit_exact(g_sparse):
    g = g_sparse
    offs, cols, vals = O.csr_from_coo(40, 30, g["trip_rows"], g["trip_cols"], g["trip_vals"])
    assert np.array_equal(offs, g["coo_offs"]) and np.array_equal(cols, g["coo_cols"])
    assert np.array_equal(vals, g["coo_vals"])
    ot, ct, vt, perm = O.transpose(40, 30, offs, cols, vals)
    assert np.array_equal(ot, g["cooT_offs"]) and np.array_equal(ct, g["cooT_cols"])
    assert np.array_equal(vt, g["cooT_vals"]) and np.array_equal(vals[perm], vt)


def test_from_coo_rejects_duplicates_and_range():
    with pytest.raises(ValueError, match="duplicate"):
        O.csr_from_coo(2, 2, [0, 0], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError):
        O.csr_from_coo(2, 2, [0], [2], [1.0])
    with pytest.raises(ValueError):
        O.csr_from_coo(2, 2, [-1], [0], [1.0])


def test_spmv_family_bit_exact(g_sparse):
    g = g_sparse
    _, nc, offs, cols, vals = _csr(g, "coo")
    assert np.array_equal(O.spmv(offs, cols, vals, g["x30"]), g["coo_spmv"])
    assert np.array_equal(O.spmv_transpose(nc, offs, cols, vals, g["x40"]), g["coo_spmvT"])
    _, _, lo, lc, lv = _csr(g, "long")
    assert np.array_equal(O.spmv(lo, lc, lv, g["x700"]), g["long_spmv"])
    assert O.mean_abs_nonzero_norm(vals) == g["coo_norm"]
    for tag in ("s15", "s60", "s300"):
        n, _, offs, cols, vals = _csr(g, tag)
        r = g[tag + "_r"]
        assert np.array_equal(O.spmv(offs, cols, vals, r), g[tag + "_spmv"])
        assert np.array_equal(O.spmv_transpose(n, offs, cols, g[tag + "_Grand"], r), g[tag + "_spmvT"])
        assert np.array_equal(O.learned_apply(n, offs, cols, g[tag + "_Grand"], 2e-3, r), g[tag + "_apply"])
        for kind in ("mean_abs_nonzero", "frobenius", "entrywise_l1"):
            assert O.matrix_norm(vals, kind) == g[tag + "_mnorm_" + kind]


def test_reduceat_order_emulation_matches_numpy():
    """The scalar order the GPU parity kernels implement == np.add.reduceat, bitwise."""
    rng = np.random.default_rng(5)
    for m in list(range(1, 40)) + [64, 127, 128, 129, 130, 200, 257, 300, 513, 1000]:
        v = rng.standard_normal(m) * np.exp(rng.uniform(-20, 20, m))
        assert O.reduceat_order_sum(v) == np.add.reduceat(v, [0])[0], m


def test_features_bit_exact(g_sparse, g_c1):
    g = g_sparse
    for tag in ("s15", "s60", "s300"):
        n, _, offs, cols, vals = _csr(g, tag)
        node, el, ef, norm = O.graph_features(n, offs, cols, vals)
        assert norm == g[tag + "_norm_A"]
        assert np.array_equal(node, g[tag + "_node_features"])
        assert np.array_equal(ef[:, 0], vals / norm)
    c = g_c1
    n, _, offs, cols, vals = _csr(c, "A")
    node, _, _, norm = O.graph_features(n, offs, cols, vals, "poisson2d", (64, 64), np.ones(n))
    assert norm == c["norm_A"] == 6792.0886075949365
    assert np.array_equal(node, c["node_features"])
    with pytest.raises(ValueError):
        O.graph_features(2, g["asym_offs"], g["asym_cols"], np.ones(3))


def test_generators_bit_exact(g_c1, g_heat):
    offs, cols, vals, _ = O.gen_poisson2d(64, 64)
    assert np.array_equal(offs, g_c1["A_offs"]) and np.array_equal(cols, g_c1["A_cols"])
    assert np.array_equal(vals, g_c1["A_vals"])
    for nx, seed in ((16, 3), (32, 7)):
        p = f"h{nx}A"
        offs, cols, vals, coeff = O.gen_poisson2d(nx, nx, seed)
        assert np.array_equal(offs, g_heat[p + "_offs"]) and np.array_equal(vals, g_heat[p + "_vals"])
        assert np.array_equal(coeff, g_heat[f"h{nx}coeff"])
    assert np.array_equal(O.gen_rhs(4096, 10**6), g_c1["b"])


def test_poisson3d_generator_entrywise():
    nx, ny, nz = 3, 4, 2
    offs, cols, vals = O.gen_poisson3d(nx, ny, nz)
    ih = [float((m + 1) ** 2) for m in (nx, ny, nz)]
    dense = np.zeros((24, 24))
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                i = ix + nx * (iy + ny * iz)
                dense[i, i] = (2 * ih[0] + 2 * ih[1]) + 2 * ih[2]
                for (jx, jy, jz), h in (((ix - 1, iy, iz), ih[0]), ((ix + 1, iy, iz), ih[0]),
                                        ((ix, iy - 1, iz), ih[1]), ((ix, iy + 1, iz), ih[1]),
                                        ((ix, iy, iz - 1), ih[2]), ((ix, iy, iz + 1), ih[2])):
                    if 0 <= jx < nx and 0 <= jy < ny and 0 <= jz < nz:
                        dense[i, jx + nx * (jy + ny * jz)] = -h
    got = np.zeros((24, 24))
    got[O.row_expand(offs), cols] = vals
    assert np.array_equal(got, dense)
    assert len(cols) == np.count_nonzero(dense)


def _rel_floor(a, b):
    scale = np.maximum(np.abs(b), 1e-3 * np.max(np.abs(b)))
    return float(np.max(np.abs(a - b) / scale))


def test_gnn_forward_both_forms_match_reference(g_sparse, g_c1):
    g = g_sparse
    for tag in ("s15", "s60", "s300"):
        n, _, offs, cols, vals = _csr(g, tag)
        node, _, ef, _ = O.graph_features(n, offs, cols, vals)
        for act in ("relu", "tanh"):
            tmpl = O.init_params(2, n_layers=2, hidden=6, seed=5)
            mlps = O.unflatten(g[tag + "_small_params_" + act], tmpl)
            want = g[tag + "_small_G_" + act]
            assert _rel_floor(O.gnn_forward(mlps, node, offs, cols, ef, 2, act), want) < 1e-12
            assert _rel_floor(O.gnn_forward_restructured(mlps, node, offs, cols, ef, 2, act), want) < 1e-12
        mlps = O.unflatten(g[tag + "_g24_params"], O.init_params(2, seed=1))
        assert _rel_floor(O.gnn_forward_restructured(mlps, node, offs, cols, ef, 4), g[tag + "_g24_G"]) < 1e-12
    c = g_c1
    n, _, offs, cols, vals = _csr(c, "A")
    node, _, ef, _ = O.graph_features(n, offs, cols, vals, "poisson2d", (64, 64), np.ones(n))
    mlps = O.init_params(3, seed=0)
    assert np.array_equal(O.params_flat(mlps), c["params"])  # weights bit-identical
    G = O.gnn_forward_restructured(mlps, node, offs, cols, ef, 4)
    assert _rel_floor(G, c["G_vals"]) < 1e-12
    assert math.fsum(c["G_vals"]) == 73340.91107527948


def test_pcg_oracle_matches_reference(g_pcg):
    g = g_pcg
    n = int(g["A_n_rows"])
    offs, cols, vals, b = g["A_offs"], g["A_cols"], g["A_vals"], g["b"]
    diag = O.diagonal(n, offs, cols, vals)
    applies = {
        "id": lambda r: r.copy(),
        "jac": lambda r: r * (1.0 / diag),
        "learn": lambda r: O.learned_apply(n, offs, cols, g["Gr"], 1e-3, r),
    }
    from spaigraph_cases import PCG_CASES
    for name, (pre, kw) in PCG_CASES.items():
        bb = np.zeros(n) if name == "zero_rhs" else b
        x, k, conv, hist = O.pcg_solve(offs, cols, vals, bb, applies[pre], **kw)
        assert k == int(g[name + "_k"]), name
        assert conv == bool(g[name + "_conv"]), name
        assert np.array_equal(x, g[name + "_x"]), name
        assert np.array_equal(np.asarray(hist), g[name + "_hist"]), name


def test_pcg_c1_iteration_count(g_c1):
    """Config 1: k = 6601; oracle is bitwise the reference loop."""
    c = g_c1
    offs, cols, vals = c["A_offs"], c["A_cols"], c["A_vals"]
    n = len(offs) - 1
    x, k, conv, hist = O.pcg_solve(offs, cols, vals, c["b"],
                                   lambda r: O.learned_apply(n, offs, cols, c["G_vals"], 1e-4, r), rtol=1e-6)
    assert k == int(c["k"]) == 6601 and conv
    assert np.array_equal(x, c["x"])


def test_loss_and_gradient(g_sparse, g_c1):
    g = g_sparse
    for tag in ("s15", "s60", "s300"):
        n, _, offs, cols, vals = _csr(g, tag)
        for kind in ("mean_abs_nonzero", "frobenius", "entrywise_l1"):
            loss, grad = O.sai_loss(n, offs, cols, vals, offs, cols, g[tag + "_Grand"], 1e-3,
                                    g[tag + "_w"], kind, with_grad=True)
            assert loss == g[tag + "_loss_" + kind]
            assert np.array_equal(grad, g[tag + "_grad_" + kind])
    c = g_c1
    n, _, offs, cols, vals = _csr(c, "A")
    loss, grad = O.sai_loss(n, offs, cols, vals, offs, cols, c["G_vals"], 1e-4, c["w"], with_grad=True)
    assert loss == c["loss"] == 104128219.23691551
    assert np.array_equal(grad, c["grad"])


def test_pattern_square_restatement_brute_force():
    """the scipy structural restatement equals a dense boolean product."""
    rng = np.random.default_rng(9)
    offs, cols, vals = O.rand_spd_sparse(60, rng, extra_per_row=3)
    po, pc = O.pattern_square(60, offs, cols)
    B = np.zeros((60, 60), dtype=bool)
    B[O.row_expand(offs), cols] = True
    want = (B.astype(int) @ B.astype(int)) > 0
    got = np.zeros((60, 60), dtype=bool)
    got[O.row_expand(po), pc] = True
    assert np.array_equal(got, want)
    pv = O.pad_to_pattern(offs, cols, vals, po, pc)
    dense = np.zeros((60, 60))
    dense[O.row_expand(po), pc] = pv
    ref = np.zeros((60, 60))
    ref[O.row_expand(offs), cols] = vals
    assert np.array_equal(dense, ref) and len(pv) == len(pc)


def test_coefficient_stencil_formula_regenerates_reference_A(g_heat):
    """The per-row formula of the coefficient-stencil K1 (pcg.cu `stencil5`: faces 0.5*(a_i+a_j),
    a wall face keeps a_i, off-diagonal -face*(n+1)^2, diagonal (w+e)*(nx+1)^2 + (s+n)*(ny+1)^2,
    presence from the row's pattern) reproduces the reference's gen_poisson2d A bit for bit on its
    golden heat2d systems (datasets.py:87-145; tests/golden/golden_heat.npz)."""
    for tag, nx in (("h16", 16), ("h32", 32)):
        offs, cols, vals = g_heat[tag + "A_offs"], g_heat[tag + "A_cols"], g_heat[tag + "A_vals"]
        a = [float(v) for v in g_heat[tag + "coeff"]]
        ihx2 = ihy2 = float((nx + 1) ** 2)
        for i in range(len(offs) - 1):
            row = {int(c): float(v) for c, v in zip(cols[offs[i]:offs[i + 1]], vals[offs[i]:offs[i + 1]])}
            face = {j: (0.5 * (a[i] + a[j]) if j in row else a[i]) for j in (i - nx, i - 1, i + 1, i + nx)}
            want = {i - nx: -(face[i - nx] * ihy2), i - 1: -(face[i - 1] * ihx2), i + 1: -(face[i + 1] * ihx2),
                    i + nx: -(face[i + nx] * ihy2),
                    i: (face[i - 1] + face[i + 1]) * ihx2 + (face[i - nx] + face[i + nx]) * ihy2}
            for j, v in row.items():
                assert np.float64(v).tobytes() == np.float64(want[j]).tobytes(), (tag, i, j)


def test_gen_synthetic_oracle_matches_reference_golden():
    """datasets.py:148-193 (A = P·Pᵀ + εI): the oracle's restatement equals the reference's output
    bit for bit on the reference tests' own calls and the edge cases (n = 1, density 0 and 1)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_synthetic.npz"))
    for t, (n, dens, seed) in enumerate(g["cases"]):
        offs, cols, vals = O.gen_synthetic(int(n), float(dens), int(seed))
        assert np.array_equal(offs, g[f"s{t}_offs"]) and np.array_equal(cols, g[f"s{t}_cols"])
        assert np.array_equal(vals, g[f"s{t}_vals"])
        assert len(cols) / (n * n) == float(g[f"s{t}_result_density"])
