"""GPU: the drop-in boundary of `pcg_solve` for ANY `Preconditioner` (precond.py:42-59,
pcg.py:131-233) and the handle's re-planning when a pattern changes behind its pointers.

Ports the reference's own contract tests (pkg/tests/test_pcg.py:50-57, 163-177: a subclass whose
`apply` counts its calls must be applied 1 + k times, refresh iterations included) and checks that
the generic path (a user `apply` every iteration) and the fused solver agree."""
import os

import numpy as np
import pytest

from oracle import spaigraph_ref as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_27517_b200 as P  # noqa: E402
from paper_2510_27517_b200.precond import IdentityPreconditioner, JacobiPreconditioner, Preconditioner  # noqa: E402

CKPT = os.path.join(os.path.dirname(__file__), "golden", "trained_heat16.spaignn")


def laplacian5(nx, ny):
    """4 / -1 five-point Laplacian on an nx-by-ny grid, entry by entry (independent of the
    package generators)."""
    rows, cols, vals = [], [], []
    for iy in range(ny):
        for ix in range(nx):
            i = iy * nx + ix
            rows.append(i), cols.append(i), vals.append(4.0)
            for jx, jy in ((ix - 1, iy), (ix + 1, iy), (ix, iy - 1), (ix, iy + 1)):
                if 0 <= jx < nx and 0 <= jy < ny:
                    rows.append(i), cols.append(jy * nx + jx), vals.append(-1.0)
    return P.SparseMatrix.from_coo(nx * ny, nx * ny, rows, cols, vals)


class CountingIdentity(IdentityPreconditioner):
    def __init__(self, n):
        super().__init__(n)
        self.calls = 0

    def apply(self, r):
        self.calls += 1
        return super().apply(r)


class DampedJacobi(JacobiPreconditioner):
    """Overrides apply: the fused solver must NOT substitute plain Jacobi for it."""

    def apply(self, r):
        return 0.5 * np.asarray(r) * self.inv_diag


class NumpyScaledIdentity(Preconditioner):
    """A user preconditioner written against numpy only (the reference contract)."""

    variant = "user"

    def __init__(self, n, c):
        super().__init__(n)
        self.c = c
        self.seen = []

    def apply(self, r):
        assert isinstance(r, np.ndarray) and r.dtype == np.float64
        self.seen.append(len(r))
        return self.c * r


def test_preconditioner_applied_every_iteration_including_refresh():
    """pkg/tests/test_pcg.py:163-177 against the drop-in."""
    A = laplacian5(12, 12)
    n = 144
    b = np.ones(n)
    M = CountingIdentity(n)
    rep = P.pcg_solve(A, b, M, P.SolveConfig(rtol=1e-8, residual_refresh_period=10))
    assert rep.converged
    assert rep.k > 10
    assert M.calls == 1 + rep.k
    M2 = CountingIdentity(n)
    rep2 = P.pcg_solve(A, b, M2, P.SolveConfig(rtol=1e-8, residual_refresh_period=10**9))
    assert M2.calls == 1 + rep2.k
    assert rep.t_apply_total_ns > 0 and rep.t_cg_total_ns > 0


def test_generic_path_matches_fused_and_oracle():
    """The generic path (counting subclass) and the fused identity solver follow the same
    reference recurrence: same k, x and history to rounding of the dot products; both equal the
    oracle's pcg_solve (numpy) k."""
    A = laplacian5(20, 17)
    n = A.n_rows
    b = np.random.default_rng(5).standard_normal(n)
    cfg = P.SolveConfig(rtol=1e-9, residual_refresh_period=7)
    gen = P.pcg_solve(A, b, CountingIdentity(n), cfg)
    fused = P.pcg_solve(A, b, P.build_identity(A), cfg)
    _, k_ref, conv_ref, hist_ref = O.pcg_solve(A.row_offsets, A.col_indices, A.values, b, lambda r: r.copy(),
                                               rtol=1e-9, period=7)
    assert gen.converged and fused.converged and conv_ref
    assert abs(gen.k - fused.k) <= 1 and abs(gen.k - k_ref) <= max(1, 0.02 * k_ref)
    m = min(len(gen.residual_history), len(hist_ref))
    np.testing.assert_allclose(gen.residual_history[:m], hist_ref[:m], rtol=1e-8, atol=1e-14)
    np.testing.assert_allclose(gen.x, fused.x, rtol=0, atol=1e-10 * np.max(np.abs(fused.x)))


def test_subclass_overriding_apply_is_not_fused():
    A = laplacian5(15, 15)
    n = A.n_rows
    b = np.random.default_rng(2).standard_normal(n)
    J = P.build_jacobi(A)
    damped = DampedJacobi(1.0 / np.diag(O_dense(A)), 0)
    cfg = P.SolveConfig(rtol=1e-10)
    r_j = P.pcg_solve(A, b, J, cfg)
    r_d = P.pcg_solve(A, b, damped, cfg)
    # 0.5 M^{-1}: the Krylov space is the same; x agrees, but the run went through damped.apply
    assert r_d.converged and r_j.converged
    np.testing.assert_allclose(r_d.x, r_j.x, rtol=0, atol=1e-8 * np.max(np.abs(r_j.x)))
    user = NumpyScaledIdentity(n, 3.0)
    r_u = P.pcg_solve(A, b, user, cfg)
    assert r_u.converged and len(user.seen) == 1 + r_u.k


def O_dense(A):
    d = np.zeros((A.n_rows, A.n_cols))
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_offsets))
    d[rows, A.col_indices] = A.values
    return d


def test_generic_path_not_spd_and_dimension_errors():
    A = P.SparseMatrix.from_dense(np.diag([1.0, -1.0]))
    with pytest.raises(P.NotSpdError):
        P.pcg_solve(A, np.array([1.0, 1.0]), CountingIdentity(2))
    with pytest.raises(ValueError):
        P.pcg_solve(laplacian5(3, 3), np.ones(9), CountingIdentity(8))


@pytest.mark.parametrize("nx", [40, 96, 200])
def test_fused_learned_reports_apply_time(nx):
    """t_apply of the fused learned apply: timed inside the one-launch solvers (40^2: one CTA,
    96^2: a cluster) and from the in-graph event samples on the multi-kernel path (200^2)."""
    m = P.load_checkpoint(CKPT)
    A, meta = P.gen_poisson2d(nx, nx, coeff_seed=4)
    G = P.forward(m, P.build_graph(A, meta)).G
    rep = P.pcg_solve(A, P.gen_rhs(meta, 9), P.build_learned_spai(G, m.config.epsilon), P.SolveConfig(rtol=1e-8))
    assert rep.converged and rep.t_apply_total_ns > 0 and rep.t_cg_total_ns > 0


# --------------------------------------------------------------------------- stale handle re-plan
def _oracle_solve(nx, ny, seed, mlps, rtol):
    offs, cols, vals, coeff = O.gen_poisson2d(nx, ny, seed)
    n = nx * ny
    node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d", (nx, ny), coeff)
    g = O.gnn_forward_restructured(mlps, node, offs, cols, ef, 4)
    b = O.gen_rhs(n, seed + 10**6)
    x, k, conv, _ = O.pcg_solve(offs, cols, vals, b, lambda r: O.learned_apply(n, offs, cols, g, 1e-4, r), rtol=rtol)
    return (offs, cols, vals), b, x, k, conv


def test_solve_batch_pattern_change_with_equal_sizes_is_replanned():
    """512x128 grids followed by 128x512 grids have the same n and nnz, so the
    batch cache refills the SAME device CSR buffers in place.  The PCG handle must notice the new
    pattern (its diagonal set changes from +-512 to +-128) and re-plan; each batch is checked
    against the oracle."""
    from paper_2510_27517_b200 import batch as B
    m = P.load_checkpoint(CKPT)
    mlps = O.unflatten(m.params_flat(), O.init_params(3))
    rtol = 1e-6
    cfg = P.SolveConfig(rtol=rtol)
    B._SOLVERS.clear()
    for nx, ny in ((512, 128), (128, 512)):
        A, meta = P.gen_poisson2d(nx, ny, coeff_seed=3)
        b = P.gen_rhs(meta, 3 + 10**6)
        (rep,) = P.solve_batch([A], [b], m, metas=[meta], cfg=cfg)
        (offs, cols, vals), b_ref, x_ref, k_ref, conv_ref = _oracle_solve(nx, ny, 3, mlps, rtol)
        assert np.array_equal(b, b_ref)
        assert rep.converged and conv_ref
        assert abs(rep.k - k_ref) <= max(1, 0.02 * k_ref), (nx, ny, rep.k, k_ref)
        true_rel = np.linalg.norm(b - O.spmv(offs, cols, vals, rep.x)) / np.linalg.norm(b)
        assert true_rel <= rtol
        assert np.linalg.norm(rep.x - x_ref) <= 1e-6 * np.linalg.norm(x_ref)
    (solver,) = B._SOLVERS.values()
    assert solver.handle.rebuilds() == 1


def test_pcg_solve_same_pointers_new_pattern_replanned():
    """The same through pcg_solve's handle cache: two systems with equal n / nnz whose device
    index buffers land at the same addresses after the first matrix is freed."""
    m = P.load_checkpoint(CKPT)
    out = []
    for nx, ny in ((96, 40), (40, 96)):
        A, meta = P.gen_poisson2d(nx, ny, coeff_seed=1)
        G = P.forward(m, P.build_graph(A, meta)).G
        b = P.gen_rhs(meta, 7)
        rep = P.pcg_solve(A, b, P.build_learned_spai(G, m.config.epsilon), P.SolveConfig(rtol=1e-8))
        rel = np.linalg.norm(b - P.spmv(A, rep.x)) / np.linalg.norm(b)
        assert rep.converged and rel <= 1e-8
        out.append(rep.k)
        del A, G
