"""Batches of independent systems on one GPU.

The reference solves one system per call (cli.py:293-317 loops over matrices, optionally in a
thread pool).  Here a batch of systems lives block-diagonally in one set of CSR arrays
(global row / column indices), so that ONE GNN pass and ONE device-resident PCG loop serve the
whole batch: per-system norms and features, one fused GNN forward over the union graph, one
G^T gather, and the batched PCG (`sg_pcg_*`) in which every system keeps its own scalars,
convergence test and history and stops independently.  Multi-GPU data parallelism shards the
systems over ranks with no collective in the data path (see `shard_range`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .datasets import heat_coeff
from .gnn import GnnModel, forward_device
from .pcg import PcgHandle, SolveConfig, report_from
from .sparse import DeviceCsr, SparseMatrix

__all__ = ["SystemBatch", "BatchSolver", "solve_batch", "shard_range"]


def shard_range(n_items: int, rank: int, world: int):
    """Contiguous, balanced split of n_items over `world` ranks: [lo, hi) of `rank`."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class SystemBatch:
    """Block-diagonal device storage of independent square systems.

    Fields: `a` (DeviceCsr over all rows), `row_start` / `nnz_start` (n_systems+1 host int64
    boundaries), `b` (device rhs), per-system PDE metadata (`grids`, `coeff` device array
    aligned with rows, `coeff_mean`) or None for algebraic features.
    """

    def __init__(self, a: DeviceCsr, row_start, nnz_start, b, grids=None, coeff=None, coeff_mean=None):
        self.a = a
        self.row_start = np.asarray(row_start, dtype=np.int64)
        self.nnz_start = np.asarray(nnz_start, dtype=np.int64)
        self.b = b
        self.grids, self.coeff, self.coeff_mean = grids, coeff, coeff_mean

    @property
    def n_systems(self) -> int:
        return len(self.row_start) - 1

    @property
    def d_node(self) -> int:
        return 3 if self.grids is not None else 2

    # -------------------------------------------------------------------- construction
    @staticmethod
    def heat2d(nx: int, ny: int, coeff_seeds, rhs_seeds) -> "SystemBatch":
        """gen_poisson2d(nx, ny, coeff_seed=s) + gen_rhs(meta, r) for every (s, r), built in place on
        the GPU (host: only the PCG64 draws of the coefficient fields and right-hand sides)."""
        import torch
        S = len(coeff_seeds)
        n1, nnz1 = nx * ny, 5 * nx * ny - 2 * nx - 2 * ny
        offs = L.empty(S * n1 + 1, torch.int32)
        cols = L.empty(S * nnz1, torch.int32)
        vals = L.empty(S * nnz1, torch.float64)
        coeff_h = np.concatenate([heat_coeff(nx, ny, s) for s in coeff_seeds])
        coeff = L.to_device(coeff_h, torch.float64)
        b_h = np.concatenate([_rhs(n1, r) for r in rhs_seeds])
        b = L.to_device(b_h, torch.float64)
        for k in range(S):
            L.check(L.lib().sg_gen_poisson2d(nx, ny, C.c_void_p(coeff.data_ptr() + 8 * k * n1), k * n1, k * nnz1,
                                             L.ptr(offs), L.ptr(cols), L.ptr(vals), L.stream_ptr()))
        a = DeviceCsr(S * n1, S * n1, offs, cols, vals)
        means = [float(coeff_h[k * n1:(k + 1) * n1].mean()) for k in range(S)]
        return SystemBatch(a, np.arange(S + 1) * n1, np.arange(S + 1) * nnz1, b, [(nx, ny)] * S, coeff, means)

    @staticmethod
    def from_host(As, bs, metas=None, into: "SystemBatch | None" = None) -> "SystemBatch":
        """Upload reference-typed host systems (int64 CSR, f64 values, host rhs) into one batch.

        `into`: reuse the device buffers of an existing batch with identical sizes.
        """
        import torch
        S = len(As)
        rows = [int(A.n_rows) for A in As]
        nnzs = [int(len(A.col_indices)) for A in As]
        row_start = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
        nnz_start = np.concatenate([[0], np.cumsum(nnzs)]).astype(np.int64)
        n, nnz = int(row_start[-1]), int(nnz_start[-1])
        if n + 1 > 2**31 - 1 or nnz > 2**31 - 1:
            raise ValueError("batch too large for int32 device indices")
        pde = metas is not None and all(getattr(m, "family", None) in ("poisson2d", "heat2d") for m in metas)
        reuse = (into is not None and np.array_equal(into.row_start, row_start)
                 and np.array_equal(into.nnz_start, nnz_start) and getattr(into, "_stage", None) is not None)
        if reuse:
            offs, cols, vals, b = into.a.offs, into.a.cols, into.a.vals, into.b
            coeff = into.coeff if pde else None
            so, sc, seg_o, seg_c = into._stage
        else:
            offs, cols = L.empty(n + 1, torch.int32), L.empty(nnz, torch.int32)
            vals, b = L.empty(nnz, torch.float64), L.empty(n, torch.float64)
            coeff = L.empty(n, torch.float64) if pde else None
            so, sc = L.empty(n, torch.int64), L.empty(nnz, torch.int64)
            # per-segment tables for the batched narrowing: (start, bound, shift)
            seg_o = (L.to_device(row_start, torch.int64), L.to_device(np.asarray(nnzs) + 1, torch.int64),
                     L.to_device(nnz_start[:-1], torch.int64))
            seg_c = (L.to_device(nnz_start, torch.int64), L.to_device(np.asarray(rows), torch.int64),
                     L.to_device(row_start[:-1], torch.int64))
        lib = L.lib()
        # H2D: one async copy per host array (asynchronous when the host array is pinned)
        for k, A in enumerate(As):
            r0, e0 = int(row_start[k]), int(nnz_start[k])
            if A.n_rows != A.n_cols:
                raise ValueError("systems must be square")
            o = np.asarray(A.row_offsets)
            if o.dtype != np.int64 or len(o) != rows[k] + 1:
                o = np.ascontiguousarray(o, dtype=np.int64)
                if len(o) != rows[k] + 1:
                    raise ValueError("row_offsets must have length n_rows + 1")
            so[r0:r0 + rows[k]].copy_(torch.from_numpy(o[:-1]), non_blocking=True)
            sc[e0:e0 + nnzs[k]].copy_(torch.from_numpy(np.ascontiguousarray(A.col_indices, dtype=np.int64)),
                                      non_blocking=True)
            vals[e0:e0 + nnzs[k]].copy_(torch.from_numpy(np.ascontiguousarray(A.values, dtype=np.float64)),
                                        non_blocking=True)
            b[r0:r0 + rows[k]].copy_(torch.from_numpy(np.ascontiguousarray(bs[k], dtype=np.float64)),
                                     non_blocking=True)
            if pde:
                coeff[r0:r0 + rows[k]].copy_(torch.from_numpy(np.ascontiguousarray(metas[k].coeff, dtype=np.float64)),
                                             non_blocking=True)
        # int64 -> int32 with per-system range checks and block-diagonal shifts: two launches
        L.call_ws(lib.sg_narrow_index_segments, L.ptr(so), L.ptr(offs), n, L.ptr(seg_o[0]), L.ptr(seg_o[1]),
                  L.ptr(seg_o[2]), S, what="narrow offsets")
        L.call_ws(lib.sg_narrow_index_segments, L.ptr(sc), L.ptr(cols), nnz, L.ptr(seg_c[0]), L.ptr(seg_c[1]),
                  L.ptr(seg_c[2]), S, what="narrow columns")
        offs[n:n + 1].fill_(nnz)
        L.call_ws(lib.sg_csr_validate, n, n, nnz, L.ptr(offs), L.ptr(cols), what="validate batch")
        grids = [tuple(m.grid) for m in metas] if pde else None
        means = [float(np.asarray(m.coeff, dtype=np.float64).mean()) for m in metas] if pde else None
        if reuse:
            # same device buffers refilled in place: keep the object (and its cached row index,
            # transpose permutation and any PCG handle built on it); the pattern may differ, so
            # recompute the pattern-derived caches in place
            into.a.refresh_pattern()
            into.grids, into.coeff, into.coeff_mean = grids, coeff, means
            return into
        a = DeviceCsr(n, n, offs, cols, vals)
        out = SystemBatch(a, row_start, nnz_start, b, grids, coeff, means)
        out._stage = (so, sc, seg_o, seg_c)
        return out


def _rhs(n, seed):
    b = np.random.default_rng(seed).standard_normal(n)
    return b / np.linalg.norm(b)


class BatchSolver:
    """GNN build + PCG solve for a SystemBatch (device buffers and CUDA graphs reused per step)."""

    def __init__(self, batch: SystemBatch, model: GnnModel):
        import torch
        self.batch, self.model = batch, model
        a = batch.a
        S = batch.n_systems
        self.norms = L.empty(S, torch.float64)
        self.node = L.empty(a.n_rows * batch.d_node, torch.float64)
        self.edge = L.empty(a.nnz, torch.float64)
        self.gt_vals = L.empty(a.nnz, torch.float64)
        self.x = L.empty(a.n_rows, torch.float64)
        self._norm_ws = None
        self.g = L.empty(a.nnz, torch.float64)  # G values; fixed buffer so the PCG handle is reused
        self.handle = None

    def _meta_device(self):
        """Per-system metadata on device (row / nnz boundaries, grids, coefficient means)."""
        import torch
        bt = self.batch
        key = (id(bt), tuple(bt.coeff_mean or ()), tuple(bt.grids or ()))
        if getattr(self, "_meta_key", None) != key:
            self._row_start_d = L.to_device(bt.row_start, torch.int64)
            self._nnz_start_d = L.to_device(bt.nnz_start, torch.int64)
            if bt.grids is not None:
                self._nx_d = L.to_device(np.array([g[0] for g in bt.grids], dtype=np.int64), torch.int64)
                self._ny_d = L.to_device(np.array([g[1] for g in bt.grids], dtype=np.int64), torch.int64)
                self._cmean_d = L.to_device(np.asarray(bt.coeff_mean, dtype=np.float64), torch.float64)
            self._meta_key = key
        return self._row_start_d, self._nnz_start_d

    def build_graph(self):
        """Exact per-system norms + features (graphfeat.py:63-105) for the whole batch: two
        launches (segmented exact sum, batched features), independent of the batch size."""
        bt, a, lib = self.batch, self.batch.a, L.lib()
        rs, ns = self._meta_device()
        max_len = int(np.max(np.diff(bt.nnz_start)))
        if self._norm_ws is None or self._norm_ws[2] != (bt.n_systems, max_len):
            buf, nb = L.workspace(lib.sg_matrix_norm_batched, None, None, bt.n_systems, max_len, 0, None)
            self._norm_ws = (buf, nb, (bt.n_systems, max_len))
        ws, wsb, _ = self._norm_ws
        sp = L.stream_ptr()
        L.check(lib.sg_matrix_norm_batched(L.ptr(a.vals), L.ptr(ns), bt.n_systems, max_len, 0, L.ptr(self.norms),
                                           L.ptr(ws), C.byref(wsb), sp))
        if bt.grids is not None:
            L.check(lib.sg_graph_features_batched(L.ptr(rs), bt.n_systems, a.n_rows, L.ptr(a.offs), L.ptr(a.cols),
                                                  L.ptr(a.vals), L.ptr(self.norms), 1, L.ptr(self._nx_d),
                                                  L.ptr(self._ny_d), L.ptr(bt.coeff), L.ptr(self._cmean_d),
                                                  L.ptr(self.node), L.ptr(self.edge), sp))
        else:
            L.check(lib.sg_graph_features_batched(L.ptr(rs), bt.n_systems, a.n_rows, L.ptr(a.offs), L.ptr(a.cols),
                                                  L.ptr(a.vals), L.ptr(self.norms), 0, None, None, None, None,
                                                  L.ptr(self.node), L.ptr(self.edge), sp))

    def build_factor(self):
        """G = GNN(graph) on the union graph; explicit G^T values via the transpose permutation."""
        a = self.batch.a
        forward_device(self.model, a, self.node, self.edge, self.batch.d_node, out=self.g)
        _, _, perm = a.transpose_pattern()
        L.check(L.lib().sg_gather_f64(L.ptr(self.g), L.ptr(perm), L.ptr(self.gt_vals), a.nnz, L.stream_ptr()))

    def solve(self, cfg: SolveConfig):
        a = self.batch.a
        ot, ct, _ = a.transpose_pattern()
        if self.handle is None or self.handle.a is not a:
            g_dev = a.with_values(self.g)
            gt_dev = DeviceCsr(a.n_cols, a.n_rows, ot, ct, self.gt_vals)
            self.handle = PcgHandle(a, self.batch.row_start, L.PRECOND_LEARNED, g_dev, gt_dev, None,
                                    self.model.config.epsilon)
        return self.handle.solve(self.batch.b, self.x, cfg)

    def step(self, cfg: SolveConfig):
        """One full pass of the hot path for every system: graph -> G -> G^T -> PCG."""
        self.build_graph()
        self.build_factor()
        return self.solve(cfg)

    def reports(self, results, cfg: SolveConfig, x_host=None):
        out = []
        for k, res in enumerate(results):
            hist = self.handle.history(k, int(res.hist_len)) if cfg.track_history else None
            xk = None if x_host is None else x_host[self.batch.row_start[k]:self.batch.row_start[k + 1]]
            out.append(report_from(res, xk, hist, 0, self.handle.last_elapsed_ns))
        return out


_SOLVERS: dict = {}


def solve_batch(As, bs, model: GnnModel, metas=None, cfg: SolveConfig | None = None, history: bool = False):
    """Public batched entry: host systems in, host solutions out (the e2e path).

    Equivalent, system by system, to
        G = forward(model, build_graph(A, meta)).G
        pcg_solve(A, b, build_learned_spai(G, model.config.epsilon), cfg)
    Returns a list of SolveReport (x as numpy).  Device buffers, the transpose permutation and
    the PCG graphs are cached per batch shape, so repeated calls only move data and compute.
    """
    cfg = cfg or SolveConfig()
    key = (tuple(int(A.n_rows) for A in As), tuple(int(len(A.col_indices)) for A in As), id(model))
    cached = _SOLVERS.get(key)
    batch = SystemBatch.from_host(As, bs, metas, into=cached.batch if cached else None)
    if cached is None or cached.batch.a.offs is not batch.a.offs:
        cached = BatchSolver(batch, model)
        _SOLVERS.clear()
        _SOLVERS[key] = cached
    else:
        cached.batch = batch
    results = cached.step(cfg)
    x_host = cached.x.cpu().numpy()
    return cached.reports(results, cfg if history else SolveConfig(**{**cfg.__dict__, "track_history": False}),
                          x_host)
