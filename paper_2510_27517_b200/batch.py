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
import os

import numpy as np

from . import _lib as L
from .datasets import heat_coeff
from .gnn import GnnModel, forward_device
from .pcg import PcgHandle, SolveConfig, report_from
from .sparse import DeviceCsr, SparseMatrix

__all__ = ["SystemBatch", "HostUpload", "BatchSolver", "solve_batch", "solve_batch_stream", "shard_range"]


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
        self._upload = None  # HostUpload staging area when built from host arrays

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
        stage = into._upload if (into is not None and getattr(into, "_upload", None) is not None
                                 and into._upload.fits(As, metas)) else HostUpload(As, metas)
        stage.upload(As, bs, metas)
        return stage.finalize(into)


def _host_runs(arrays, dtype):
    """Group consecutive host arrays that are adjacent in memory (views of one buffer, e.g. one
    pinned allocation): yields (first, last + 1, contiguous numpy view of the run)."""
    import ctypes
    S, k = len(arrays), 0
    while k < S:
        a0 = np.ascontiguousarray(arrays[k], dtype=dtype)
        end, j = a0.ctypes.data + a0.nbytes, k + 1
        while j < S:
            aj = arrays[j]
            if not (isinstance(aj, np.ndarray) and aj.dtype == dtype and aj.flags.c_contiguous
                    and aj.ctypes.data == end):
                break
            end += aj.nbytes
            j += 1
        if j == k + 1 or a0.nbytes == 0:
            yield k, k + 1, a0
            k += 1
            continue
        nbytes = end - a0.ctypes.data
        buf = (ctypes.c_char * nbytes).from_address(a0.ctypes.data)
        yield k, j, np.frombuffer(buf, dtype=dtype)
        k = j


class HostUpload:
    """Device staging area for one host batch: the raw H2D targets (int64 indices, values, rhs,
    coefficients).  `upload` only enqueues copies (on the current stream; asynchronous for
    pinned host memory) and records an event; `finalize` turns the staged arrays into the
    working int32 batch.  Two of these let the next batch travel over PCIe while the current one
    is solved (`solve_batch_stream`)."""

    def __init__(self, As, metas=None):
        import torch
        self.rows = [int(A.n_rows) for A in As]
        self.nnzs = [int(len(A.col_indices)) for A in As]
        self.row_start = np.concatenate([[0], np.cumsum(self.rows)]).astype(np.int64)
        self.nnz_start = np.concatenate([[0], np.cumsum(self.nnzs)]).astype(np.int64)
        n, nnz = int(self.row_start[-1]), int(self.nnz_start[-1])
        if n + 1 > 2**31 - 1 or nnz > 2**31 - 1:
            raise ValueError("batch too large for int32 device indices")
        self.n, self.nnz = n, nnz
        self.pde = _is_pde(metas)
        self.so, self.sc = L.empty(n, torch.int64), L.empty(nnz, torch.int64)
        self.vals, self.b = L.empty(nnz, torch.float64), L.empty(n, torch.float64)
        self.coeff = L.empty(n, torch.float64) if self.pde else None
        # per-segment tables for the batched narrowing: (start, bound, shift)
        self.seg_o = (L.to_device(self.row_start, torch.int64), L.to_device(np.asarray(self.nnzs) + 1, torch.int64),
                      L.to_device(self.nnz_start[:-1], torch.int64))
        self.seg_c = (L.to_device(self.nnz_start, torch.int64), L.to_device(np.asarray(self.rows), torch.int64),
                      L.to_device(self.row_start[:-1], torch.int64))
        self.ready = torch.cuda.Event()
        self.consumed = None
        self._hold = None
        self.grids = self.means = None

    def fits(self, As, metas=None) -> bool:
        return (len(As) == len(self.rows) and all(int(A.n_rows) == r for A, r in zip(As, self.rows))
                and all(int(len(A.col_indices)) == e for A, e in zip(As, self.nnzs)) and _is_pde(metas) == self.pde)

    def upload(self, As, bs, metas=None):
        import torch
        if not self.fits(As, metas):
            raise ValueError("batch shape differs from this staging area")
        rows, r_st, e_st = self.rows, self.row_start, self.nnz_start
        offs = []
        for k, A in enumerate(As):
            if A.n_rows != A.n_cols:
                raise ValueError("systems must be square")
            o = np.asarray(A.row_offsets)
            if o.dtype != np.int64 or len(o) != rows[k] + 1:
                o = np.ascontiguousarray(o, dtype=np.int64)
                if len(o) != rows[k] + 1:
                    raise ValueError("row_offsets must have length n_rows + 1")
            offs.append(o)
            if len(bs[k]) != rows[k]:
                raise ValueError(f"dimension mismatch: matrix is {rows[k]}, rhs is {len(bs[k])}")
            if len(A.values) != self.nnzs[k]:
                raise ValueError("values and col_indices differ in length")

        def put(dst, arrays, starts, dtype):
            for k0, k1, h in _host_runs(arrays, dtype):
                if h.size:
                    dst[int(starts[k0]):int(starts[k0]) + h.size].copy_(torch.from_numpy(h), non_blocking=True)

        # row offsets without their last entry (adjacent systems' offset arrays are not adjacent)
        for k, o in enumerate(offs):
            if rows[k]:
                self.so[int(r_st[k]):int(r_st[k + 1])].copy_(torch.from_numpy(o[:-1]), non_blocking=True)
        put(self.sc, [A.col_indices for A in As], e_st, np.int64)
        put(self.vals, [A.values for A in As], e_st, np.float64)
        put(self.b, list(bs), r_st, np.float64)
        if self.pde:
            put(self.coeff, [m.coeff for m in metas], r_st, np.float64)
            self.grids = [tuple(m.grid) for m in metas]
            self.means = [float(np.asarray(m.coeff, dtype=np.float64).mean()) for m in metas]
        else:
            self.grids = self.means = None
        self._hold = (As, bs, metas)  # host arrays stay alive until the copies are consumed
        self.ready.record()

    def finalize(self, into: "SystemBatch | None" = None) -> "SystemBatch":
        """Staged arrays -> the working batch (int32 indices with per-system range checks and
        block-diagonal shifts, validation, values / rhs / coefficients), on the current stream."""
        import torch
        cur = torch.cuda.current_stream()
        cur.wait_event(self.ready)
        n, nnz, S = self.n, self.nnz, len(self.rows)
        reuse = (into is not None and np.array_equal(into.row_start, self.row_start)
                 and np.array_equal(into.nnz_start, self.nnz_start) and (into.coeff is not None) == self.pde)
        if reuse:
            offs, cols, vals, b, coeff = into.a.offs, into.a.cols, into.a.vals, into.b, into.coeff
        else:
            offs, cols = L.empty(n + 1, torch.int32), L.empty(nnz, torch.int32)
            vals, b = L.empty(nnz, torch.float64), L.empty(n, torch.float64)
            coeff = L.empty(n, torch.float64) if self.pde else None
        lib = L.lib()
        L.call_ws(lib.sg_narrow_index_segments, L.ptr(self.so), L.ptr(offs), n, L.ptr(self.seg_o[0]),
                  L.ptr(self.seg_o[1]), L.ptr(self.seg_o[2]), S, what="narrow offsets")
        L.call_ws(lib.sg_narrow_index_segments, L.ptr(self.sc), L.ptr(cols), nnz, L.ptr(self.seg_c[0]),
                  L.ptr(self.seg_c[1]), L.ptr(self.seg_c[2]), S, what="narrow columns")
        offs[n:n + 1].fill_(nnz)
        L.call_ws(lib.sg_csr_validate, n, n, nnz, L.ptr(offs), L.ptr(cols), what="validate batch")
        vals.copy_(self.vals)
        b.copy_(self.b)
        if self.pde:
            coeff.copy_(self.coeff)
        self.consumed = torch.cuda.Event()
        self.consumed.record(cur)
        self._hold = None
        if reuse:
            # same device buffers refilled in place: keep the object (and its cached row index,
            # transpose permutation and any PCG handle built on it); the pattern may differ, so
            # recompute the pattern-derived caches in place
            into.a.refresh_pattern()
            into.grids, into.coeff_mean = self.grids, self.means
            into._upload = self
            return into
        out = SystemBatch(DeviceCsr(n, n, offs, cols, vals), self.row_start, self.nnz_start, b, self.grids,
                          coeff, self.means)
        out._upload = self
        return out


def _is_pde(metas) -> bool:
    return metas is not None and len(metas) > 0 and all(getattr(m, "family", None) in ("poisson2d", "heat2d")
                                                        for m in metas)


def _rhs(n, seed):
    b = np.random.default_rng(seed).standard_normal(n)
    return b / np.linalg.norm(b)


class BatchSolver:
    """GNN build + PCG solve for a SystemBatch (device buffers and CUDA graphs reused per step)."""

    def __init__(self, batch: SystemBatch, model: GnnModel, edge_precision: str | None = None):
        import torch
        self.batch, self.model = batch, model
        # GNN edge pass arithmetic (gnn.forward_device): "fp64" DMMA (default) or "tf32x3" on
        # tcgen05 -- SG_GNN_EDGE=tf32x3 selects it without code changes (the C2 configuration of
        # SURVEY.md §8(d) allows an fp32 GNN with the fp64 PCG)
        self.edge_precision = edge_precision or os.environ.get("SG_GNN_EDGE", "fp64")
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
        forward_device(self.model, a, self.node, self.edge, self.batch.d_node, out=self.g,
                       edge_precision=self.edge_precision)
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
        self._stencil()
        return self.handle.solve(self.batch.b, self.x, cfg)

    def _stencil(self):
        """gen_poisson2d batches (one grid shape, coefficients on device): K1 regenerates A from
        the coefficients (the solver verifies A bitwise at every solve and falls back to A's
        stored diagonals on any mismatch).  SG_PCG_STENCIL=0 turns it off.  C2: K1 94.6 -> 87.4 us."""
        bt = self.batch
        grids = set(bt.grids or ())
        if bt.coeff is None or len(grids) != 1 or os.environ.get("SG_PCG_STENCIL", "1") == "0":
            return
        nx, ny = grids.pop()
        self.handle.set_stencil(bt.coeff, nx, ny)

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


def _pinned(n: int):
    import torch
    return torch.empty(n, dtype=torch.float64, pin_memory=True)


def solve_batch(As, bs, model: GnnModel, metas=None, cfg: SolveConfig | None = None, history: bool = False):
    """Public batched entry: host systems in, host solutions out (the e2e path).

    Equivalent, system by system, to
        G = forward(model, build_graph(A, meta)).G
        pcg_solve(A, b, build_learned_spai(G, model.config.epsilon), cfg)
    Returns a list of SolveReport (x as numpy, owned by the caller).  Device buffers, the
    transpose permutation and the PCG graphs are cached per batch shape, so repeated calls only
    move data and compute.  For a stream of batches see `solve_batch_stream`, which overlaps the
    next batch's upload with the current solve.
    """
    cfg = cfg or SolveConfig()
    key = (tuple(int(A.n_rows) for A in As), tuple(int(len(A.col_indices)) for A in As), id(model))
    cached = _SOLVERS.get(key)
    batch = SystemBatch.from_host(As, bs, metas, into=cached.batch if cached else None)
    if cached is None or cached.batch.a.offs is not batch.a.offs:
        cached = BatchSolver(batch, model)
        cached._x_pinned = _pinned(batch.a.n_rows)
        _SOLVERS.clear()
        _SOLVERS[key] = cached
    else:
        cached.batch = batch
    results = cached.step(cfg)
    cached._x_pinned.copy_(cached.x, non_blocking=True)  # D2H into page-locked memory
    import torch
    torch.cuda.current_stream().synchronize()
    x_host = cached._x_pinned.numpy().copy()
    return cached.reports(results, cfg if history else SolveConfig(**{**cfg.__dict__, "track_history": False}),
                          x_host)


def solve_batch_stream(batches, model: GnnModel, cfg: SolveConfig | None = None, depth: int = 2):
    """Pipelined `solve_batch` over an iterable of (As, bs, metas) host batches; yields one list of
    SolveReport per batch, in order.

    While batch i is solved, batch i+1's host arrays are copied to a second device staging area
    on a separate stream (enqueued once batch i's GNN is in flight), so PCIe traffic overlaps the
    GPU work.  Each batch's x arrays are views of a page-locked host ring of `depth` slots: they
    stay valid until `depth` further batches have been yielded (copy them to keep them longer).
    Host arrays of a batch must stay unmodified until its results are yielded.  Solver state
    (device buffers, PCG graphs, staging areas, the ring) is cached per batch shape like
    `solve_batch`'s.
    """
    import torch
    cfg = cfg or SolveConfig()
    rep_cfg = SolveConfig(**{**cfg.__dict__, "track_history": False})
    it = iter(batches)
    cur = next(it, None)
    if cur is None:
        return
    state = {"solver": None}

    def key_of(item):
        As = item[0]
        return (tuple(int(A.n_rows) for A in As), tuple(int(len(A.col_indices)) for A in As), id(model))

    def stream_state(solver):
        if getattr(solver, "_stream", None) is None:
            solver._stream = {"copy": torch.cuda.Stream(device=L.device()), "stages": [None, None], "ring": None}
        return solver._stream

    def start(ss, slot, item):
        As, bs, metas = item
        st = ss["stages"][slot]
        if st is None or not st.fits(As, metas):
            st = ss["stages"][slot] = HostUpload(As, metas)
        if st.consumed is not None:
            ss["copy"].wait_event(st.consumed)
        with torch.cuda.stream(ss["copy"]):
            st.upload(As, bs, metas)

    # the first batch: solver from the shape cache, upload on its copy stream
    cached = _SOLVERS.get(key_of(cur))
    pending = None
    if cached is not None:
        ss = stream_state(cached)
        start(ss, 0, cur)
        pending = (cached, ss, 0)
    slot, i = 0, 0
    while cur is not None:
        if pending is None:  # new shape: build the batch (and solver) synchronously
            batch = SystemBatch.from_host(*cur)
            solver = BatchSolver(batch, model)
            _SOLVERS.clear()
            _SOLVERS[key_of(cur)] = solver
            ss = stream_state(solver)
            slot = 0
        else:
            solver, ss, slot = pending
            batch = ss["stages"][slot].finalize(solver.batch)
            if batch is not solver.batch:
                solver.batch = batch
        if ss["ring"] is None or len(ss["ring"]) != max(depth, 1) or ss["ring"][0].numel() != batch.a.n_rows:
            ss["ring"] = [_pinned(batch.a.n_rows) for _ in range(max(depth, 1))]
        solver.build_graph()
        solver.build_factor()
        nxt = next(it, None)
        pending = None
        if nxt is not None and key_of(nxt) == key_of(cur):  # next upload rides under this GNN + PCG
            start(ss, 1 - slot, nxt)
            pending = (solver, ss, 1 - slot)
        results = solver.solve(cfg)
        xh = ss["ring"][i % len(ss["ring"])]
        xh.copy_(solver.x, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        yield solver.reports(results, rep_cfg, xh.numpy())
        cur, i = nxt, i + 1
