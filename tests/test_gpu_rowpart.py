"""GPU: ONE system row-partitioned (BASELINE configs[4]) in group mode --
the P partitions are systems of one sg_pcg handle on this GPU, running the multi-GPU design's
kernels, in-kernel s-halo pushes and partition-ordered reductions.  Checked
against pcg_solve on the whole system (k within +-2%, the residual history, the true residual)
and the per-partition GNN blocks against the global G."""
import os

import numpy as np
import pytest

from oracle import spaigraph_ref as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_27517_b200 as P  # noqa: E402
from paper_2510_27517_b200 import rowpart as RP  # noqa: E402

CKPT = os.path.join(os.path.dirname(__file__), "golden", "trained_heat16.spaignn")


def _whole(A, meta, m, b, cfg):
    G = P.forward(m, P.build_graph(A, meta)).G
    return G, P.pcg_solve(A, b, P.build_learned_spai(G, m.config.epsilon), cfg)


@pytest.mark.parametrize("grid,parts,fused", [((96, 40), 1, 1), ((96, 40), 2, 1), ((96, 40), 4, 1), ((1024, 24), 4, 1),
                                              ((784, 20), 2, 1), ((700, 18), 3, 0)])
def test_partitioned_solve_matches_whole_system(grid, parts, fused):
    """(96, 40): 1-D sliding-window kernels (half-bandwidth 96); (1024, 24), (784, 20): the 2-D
    strip kernels (W > 512; 784 leaves a partial strip); (700, 18): the unfused tile kernels
    (W not a multiple of 16)."""
    m = P.load_checkpoint(CKPT)
    nx, ny = grid
    A, meta = P.gen_poisson2d(nx, ny, coeff_seed=4)
    b = P.gen_rhs(meta, 17)
    cfg = P.SolveConfig(rtol=1e-9, residual_refresh_period=11)
    _, ref = _whole(A, meta, m, b, cfg)
    sol = RP.PartitionedSolver(A, meta, m, parts)
    rep = sol.solve(b, cfg)
    assert rep.converged and ref.converged
    assert abs(rep.k - ref.k) <= max(1, 0.02 * ref.k), (rep.k, ref.k)
    # partials are grouped per partition: the histories start equal to rounding (1e-16) and the
    # Krylov recurrence amplifies that slowly; a wrong ghost value would show at once
    np.testing.assert_allclose(rep.residual_history[:25], ref.residual_history[:25], rtol=1e-11)
    o, c, v = A.row_offsets, A.col_indices, A.values
    assert np.linalg.norm(b - O.spmv(o, c, v, rep.x)) / np.linalg.norm(b) <= 1e-9
    assert sol.handle.stats()[2][7] == float(fused)


def test_partition_factors_equal_global_g():
    """Each partition's G (GNN on its own block: global norm from exact per-partition
    accumulators, global grid coordinates, receptive-field margin) equals the global G rows."""
    m = P.load_checkpoint(CKPT)
    A, meta = P.gen_poisson2d(64, 50, coeff_seed=7)
    G = P.forward(m, P.build_graph(A, meta)).G
    g = G.values
    o, c = A.row_offsets, A.col_indices
    sol = RP.PartitionedSolver(A, meta, m, 3)
    for f in sol.factors:
        e0, e1 = f.ext
        fo, fc, fg = f.offs.cpu().numpy(), f.cols.cpu().numpy(), f.g_vals.cpu().numpy()
        fa = f.a_vals.cpu().numpy()
        for i in range(e0, e1):
            li = i - e0
            keep = (c[o[i]:o[i + 1]] >= e0) & (c[o[i]:o[i + 1]] < e1)
            assert np.array_equal(fc[fo[li]:fo[li + 1]] + e0, c[o[i]:o[i + 1]][keep])
            assert np.array_equal(fa[fo[li]:fo[li + 1]], A.values[o[i]:o[i + 1]][keep])
            ref = g[o[i]:o[i + 1]][keep]
            np.testing.assert_allclose(fg[fo[li]:fo[li + 1]], ref, rtol=1e-13, atol=1e-13 * np.max(np.abs(g)))


def test_partition_norm_is_exact():
    """norm_A from per-partition exact accumulators added as integers == fsum over all values."""
    for parts in (1, 2, 3, 5):
        A, meta = P.gen_poisson2d(37, 41, coeff_seed=parts)
        pl = RP.plan_row_partition(A.row_offsets, A.col_indices, A.n_rows, parts, 4, unit=1)
        nrm = RP.global_norm(A.device(), pl).item()
        assert nrm == O.mean_abs_nonzero_norm(A.values)


def test_c5_four_partitions():
    """The north-star shape: 2048 x 2048 Poisson, 4 partitions of 512 lines (strip kernels)."""
    m = P.load_checkpoint(CKPT)
    A, meta = P.gen_poisson2d(2048, 2048)
    b = P.gen_rhs(meta, 10**6)
    cfg = P.SolveConfig(rtol=1e-6)
    _, ref = _whole(A, meta, m, b, cfg)
    sol = RP.PartitionedSolver(A, meta, m, 4)
    rep = sol.solve(b, cfg)
    assert rep.converged and abs(rep.k - ref.k) <= max(1, 0.02 * ref.k), (rep.k, ref.k)
    np.testing.assert_allclose(rep.residual_history[:50], ref.residual_history[:50], rtol=1e-9)
    o, c, v = A.row_offsets, A.col_indices, A.values
    assert np.linalg.norm(b - O.spmv(o, c, v, rep.x)) / np.linalg.norm(b) <= 1e-6


@pytest.mark.parametrize("parts", [1, 3])
def test_partitioned_sai_loss_and_grad(parts):
    """Loss forward + backward on the row partition == the whole-system loss (1e-13) and its
    dL/dg on every owned entry (1e-12)."""
    m = P.load_checkpoint(CKPT)
    A, meta = P.gen_poisson2d(60, 45, coeff_seed=2)
    G = P.forward(m, P.build_graph(A, meta)).G
    w = np.random.default_rng(0).standard_normal(A.n_rows)
    loss_ref, grad_ref = P.sai_loss_and_grad(A, G, m.config.epsilon, w)
    sol = RP.PartitionedSolver(A, meta, m, parts)
    loss, grads = sol.sai_loss_and_grad(w)
    assert abs(loss - loss_ref) <= 1e-13 * abs(loss_ref)
    o = A.row_offsets
    scale = np.max(np.abs(grad_ref))
    for f, gp in zip(sol.factors, grads):
        fo = f.offs.cpu().numpy()
        gp = gp.cpu().numpy()
        lo, hi = f.own[0] - f.ext[0], f.own[1] - f.ext[0]
        ours = gp[fo[lo]:fo[hi]]
        ref = grad_ref[o[f.own[0]]:o[f.own[1]]]
        np.testing.assert_allclose(ours, ref, rtol=1e-12, atol=1e-12 * scale)


def test_peer_mode_single_rank_runs_the_peer_reduction_path():
    """Peer mode with one rank: the kernels take the peer branch of part_fin (epoch, parity
    double buffer, system-scope release / acquire flags -- here on the rank's own block), the
    exported IPC blob is consumed by sg_pcg_set_peers; the result equals pcg_solve's.  (More
    ranks need more GPUs: their schedule runs on 2 gloo ranks in tests/test_rowpart_cpu.py.)"""
    m = P.load_checkpoint(CKPT)
    A, meta = P.gen_poisson2d(96, 40, coeff_seed=4)
    b = P.gen_rhs(meta, 17)
    cfg = P.SolveConfig(rtol=1e-9, residual_refresh_period=11)
    _, ref = _whole(A, meta, m, b, cfg)
    sol = RP.PeerPartitionSolver(A, meta, m, rank=0, world=1)
    rep = sol.solve(b, cfg)
    rep2 = sol.solve(b, cfg)  # epochs keep counting across solves
    assert rep.converged and rep.k == ref.k and rep2.k == rep.k
    np.testing.assert_allclose(rep.residual_history[:25], ref.residual_history[:25], rtol=1e-12)
    np.testing.assert_array_equal(rep.x, rep2.x)
