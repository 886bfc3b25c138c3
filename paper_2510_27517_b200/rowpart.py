"""Row-partitioned PCG for ONE large system (BASELINE configs[4] / C5).

Two implementations:

* **Banded systems, device-resident** (the product path): `plan_row_partition`
  splits the rows into contiguous blocks (whole grid lines); partition p holds an EXTENDED local
  system = owned rows +- 3 half-bandwidths of ghost rows, and its G rows come from the GNN run on
  its own block of rows plus the receptive field (global features: exact norm from per-partition
  accumulators, global grid coordinates) -- no communication.  The PCG kernels (fused
  sliding-window / strip kernels included) run over the whole extended system; only owned rows
  enter the dot products and write s, and the kernel that computes s also stores the first /
  last owned rows into the neighbours' ghost rows.  With 3 ghost layers d, q, r and x stay exact
  where they are read (tests/test_rowpart_cpu.py::test_ghost_scheme_reproduces_global_pcg), so
  per iteration the only communication is that one s halo and the two scalar reductions.
  `PartitionedSolver` runs P partitions as the systems of ONE handle on one GPU (group mode: the
  tested emulation of P ranks); `PeerPartitionSolver` runs one partition per rank / GPU (peer
  mode: CUDA-IPC-mapped neighbour memory over NVLink, flag-synchronised reductions).
* **Any pattern, host-driven** (`DistPcg`, `solve_rowpart`): a general halo plan (the owned
  rows' off-rank columns, grouped by owner), local SpMVs through the C-ABI kernels and
  torch.distributed collectives per dot product -- pcg.py:131-233 verbatim with one host round
  trip per scalar; covered by 2-rank gloo tests with a numpy backend.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .batch import shard_range
from .pcg import NotSpdError

__all__ = ["HaloPlan", "build_plan", "hop_closure", "local_transpose_rows", "DistPcg", "solve_rowpart",
           "RowPartition", "plan_row_partition", "PartitionedSolver", "solve_partitioned", "PeerPartitionSolver",
           "partition_factor", "global_norm", "row_block", "exchange_blobs"]


def hop_closure(offs, cols, seeds: np.ndarray, hops: int) -> np.ndarray:
    """Sorted set of nodes within `hops` graph hops of `seeds` (CSR adjacency)."""
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    cur = np.unique(np.asarray(seeds, dtype=np.int64))
    seen = cur
    for _ in range(hops):
        starts, ends = offs[cur], offs[cur + 1]
        lens = ends - starts
        if lens.sum() == 0:
            break
        idx = np.repeat(starts - np.cumsum(np.concatenate([[0], lens[:-1]])), lens) + np.arange(lens.sum())
        nb = np.unique(cols[idx])
        new = np.setdiff1d(nb, seen, assume_unique=True)
        if len(new) == 0:
            break
        seen = np.union1d(seen, new)
        cur = new
    return seen


@dataclass
class HaloPlan:
    n: int
    rank: int
    world: int
    bounds: np.ndarray                 # world+1 row boundaries
    r0: int
    r1: int
    halo: np.ndarray                   # global indices of halo entries, grouped by owner (ascending)
    recv_counts: list                  # per source rank
    send_idx: list = field(default_factory=list)  # per destination rank: LOCAL owned indices to send

    @property
    def n_own(self) -> int:
        return self.r1 - self.r0

    @property
    def n_ext(self) -> int:
        return self.n_own + len(self.halo)

    def ext_index(self, g: np.ndarray) -> np.ndarray:
        """Global column -> extended local index (owned first, then halo)."""
        g = np.asarray(g, dtype=np.int64)
        out = np.empty(len(g), dtype=np.int64)
        own = (g >= self.r0) & (g < self.r1)
        out[own] = g[own] - self.r0
        pos = np.searchsorted(self._halo_sorted, g[~own])
        out[~own] = self.n_own + self._halo_perm[pos]
        return out

    def finalize(self):
        order = np.argsort(self.halo, kind="stable")
        self._halo_sorted = self.halo[order]
        self._halo_perm = order
        return self


def build_plan(offs, cols, n: int, rank: int, world: int, exchange) -> HaloPlan:
    """Halo plan for the owned rows.  `exchange(list_of_index_arrays_per_rank) -> list received`
    performs the all_to_all of variable-length int64 arrays (torch.distributed in production,
    a direct shuffle in single-process tests)."""
    bounds = np.array([shard_range(n, p, world)[0] for p in range(world)] + [n], dtype=np.int64)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    needed = np.unique(cols[offs[r0]:offs[r1]])
    needed = needed[(needed < r0) | (needed >= r1)]
    owner = np.searchsorted(bounds, needed, side="right") - 1
    per_src = [needed[owner == p] for p in range(world)]
    halo = np.concatenate(per_src) if per_src else np.zeros(0, np.int64)
    asked = exchange(per_src)  # what every rank needs FROM me
    plan = HaloPlan(n, rank, world, bounds, r0, r1, halo, [len(x) for x in per_src],
                    [np.asarray(a, dtype=np.int64) - r0 for a in asked])
    return plan.finalize()


def local_rows(offs, cols, vals, plan: HaloPlan):
    """Owned rows of a global CSR with columns in extended local indexing (storage order kept,
    so per-row summation orders are the reference's)."""
    offs = np.asarray(offs, dtype=np.int64)
    lo, hi = offs[plan.r0], offs[plan.r1]
    lo_offs = offs[plan.r0:plan.r1 + 1] - lo
    return lo_offs, plan.ext_index(np.asarray(cols)[lo:hi]), np.asarray(vals)[lo:hi]


def local_transpose_rows(offs, cols, vals, plan: HaloPlan):
    """Owned rows of G^T (row i holds G(j, i) for stored (j, i), ascending j = np.add.at order),
    columns in extended local indexing.  Needs G's rows for owned + halo nodes, i.e. the
    global arrays restricted to those rows are sufficient."""
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals)
    rows_needed = np.union1d(np.arange(plan.r0, plan.r1), plan.halo)
    starts, ends = offs[rows_needed], offs[rows_needed + 1]
    lens = ends - starts
    idx = np.repeat(starts - np.cumsum(np.concatenate([[0], lens[:-1]])), lens) + np.arange(lens.sum())
    src_row = np.repeat(rows_needed, lens)
    dst = cols[idx]
    keep = (dst >= plan.r0) & (dst < plan.r1)
    src_row, dst, v = src_row[keep], dst[keep], vals[idx][keep]
    order = np.lexsort((src_row, dst))
    src_row, dst, v = src_row[order], dst[order], v[order]
    t_offs = np.zeros(plan.n_own + 1, dtype=np.int64)
    np.add.at(t_offs, dst - plan.r0 + 1, 1)
    np.cumsum(t_offs, out=t_offs)
    return t_offs, plan.ext_index(src_row), v


class DistPcg:
    """pcg.py:131-233 over a row partition.  ops: backend of local kernels; comm: collectives.

    comm must provide allreduce_sum(np.ndarray) -> np.ndarray and
    halo(x_ext, plan) -> None (fills x_ext[n_own:] from the owners).
    """

    def __init__(self, plan: HaloPlan, ops, comm, a_loc, g_loc, gt_loc, epsilon: float):
        self.plan, self.ops, self.comm = plan, ops, comm
        ops.n_own = plan.n_own
        self.A, self.G, self.Gt = (ops.matrix(*m) for m in (a_loc, g_loc, gt_loc))
        self.eps = float(epsilon)

    def _apply(self, r, t, s):
        """s = G (G^T r) + eps r on the owned rows (precond.py:143-145); r, t extended."""
        o = self.ops
        self.comm.halo(r, self.plan)
        o.spmv_seq(self.Gt, r, t)
        self.comm.halo(t, self.plan)
        o.spmv(self.G, t, s)
        o.axpby(s, s, r, self.eps, 0)  # s + eps * r

    def _dot(self, x, y):
        return self.ops.dot(x, y)

    def solve(self, b_own, rtol=1e-8, max_iters=None, period=50, termination="true_residual",
              track_history=True):
        o, plan, comm = self.ops, self.plan, self.comm
        n_glob = plan.n
        max_iters = 20 * n_glob if max_iters is None else max_iters
        use_true = termination == "true_residual"
        vec = lambda: o.zeros(plan.n_ext)  # noqa: E731
        b, x, r, d, q, s, t, tmp = (vec() for _ in range(8))
        o.copy_own(b, b_own)
        norm_b = math.sqrt(comm.allreduce_sum(np.array([o.dot(b, b)]))[0])
        if norm_b == 0.0:
            return o.own(x), 0, True, ([0.0] if track_history else None)
        o.copy(r, b)  # r = b - A*0
        self._apply(r, t, d)
        delta, rr = comm.allreduce_sum(np.array([o.dot(r, d), o.dot(r, r)]))
        if delta < 0.0:
            raise NotSpdError("preconditioner is not positive definite", 0, delta)
        delta0 = delta
        history = [math.sqrt(rr) / norm_b]
        i, converged = 0, False
        while i < max_iters:
            if not use_true and delta <= rtol ** 2 * delta0:
                break
            comm.halo(d, plan)
            o.spmv(self.A, d, q)
            dq = comm.allreduce_sum(np.array([o.dot(d, q)]))[0]
            if dq <= 0.0:
                raise NotSpdError("matrix is not positive definite along search direction", i, dq)
            alpha = delta / dq
            o.axpby(x, x, d, alpha, 0)
            refreshed = i > 0 and i % period == 0
            if refreshed:
                comm.halo(x, plan)
                o.spmv(self.A, x, tmp)
                o.axpby(r, b, tmp, 1.0, 1)
            else:
                o.axpby(r, r, q, alpha, 1)
            self._apply(r, t, s)
            delta_old = delta
            delta, rr = comm.allreduce_sum(np.array([o.dot(r, s), o.dot(r, r)]))
            if delta < 0.0:
                raise NotSpdError("preconditioner is not positive definite", i, delta)
            o.axpby(d, s, d, delta / delta_old, 0)
            i += 1
            rel = math.sqrt(rr) / norm_b
            history.append(rel)
            if use_true and rel <= rtol:
                if refreshed:
                    converged = True
                    break
                comm.halo(x, plan)
                o.spmv(self.A, x, tmp)
                o.axpby(tmp, b, tmp, 1.0, 1)
                rel_f = math.sqrt(comm.allreduce_sum(np.array([o.dot(tmp, tmp)]))[0]) / norm_b
                history[-1] = rel_f
                if rel_f <= rtol:
                    converged = True
                    break
                o.copy(r, tmp)
        if not use_true and not converged:
            comm.halo(x, plan)
            o.spmv(self.A, x, tmp)
            o.axpby(tmp, b, tmp, 1.0, 1)
            converged = math.sqrt(comm.allreduce_sum(np.array([o.dot(tmp, tmp)]))[0]) / norm_b <= rtol
        return o.own(x), i, converged, (history if track_history else None)


class CudaOps:
    """Local kernels on the GPU through the C-ABI (numpy-order SpMV, exact axpby, dot)."""

    def __init__(self):
        import torch
        from . import _lib as L
        self.L, self.torch = L, torch
        self._dot_ws = None

    def matrix(self, offs, cols, vals):
        L, torch = self.L, self.torch
        o = L.to_device(np.asarray(offs, np.int64).astype(np.int32), torch.int32)
        c = L.to_device(np.asarray(cols, np.int64).astype(np.int32), torch.int32)
        v = L.to_device(np.asarray(vals, np.float64), torch.float64)
        return (len(offs) - 1, o, c, v)

    def zeros(self, n):
        return self.L.zeros(n, self.torch.float64)

    def copy_own(self, dst, src):
        dst[: len(src)].copy_(self.torch.as_tensor(src, device=dst.device))

    def copy(self, dst, src):
        dst.copy_(src)

    def own(self, x):
        return x[: self.n_own].cpu().numpy()

    def spmv(self, M, x, y):
        n, o, c, v = M
        self.L.check(self.L.lib().sg_spmv(n, self.L.ptr(o), self.L.ptr(c), self.L.ptr(v), self.L.ptr(x),
                                          self.L.ptr(y), self.L.stream_ptr()))

    def spmv_seq(self, M, x, y):
        n, o, c, v = M
        self.L.check(self.L.lib().sg_spmv_seq(n, self.L.ptr(o), self.L.ptr(c), self.L.ptr(v), self.L.ptr(x),
                                              self.L.ptr(y), self.L.stream_ptr()))

    def axpby(self, out, a, b, c, mode):
        n = self.n_own
        self.L.check(self.L.lib().sg_axpby(self.L.ptr(out), self.L.ptr(a), self.L.ptr(b), float(c), n, mode,
                                           self.L.stream_ptr()))

    def dot(self, x, y):
        L, torch = self.L, self.torch
        n = self.n_own
        if self._dot_ws is None:
            self._dot_ws = (L.workspace(L.lib().sg_dot, None, None, n, None), L.empty(1, torch.float64))
        (ws, wsb), out = self._dot_ws
        L.check(L.lib().sg_dot(L.ptr(x), L.ptr(y), n, L.ptr(out), L.ptr(ws), C_byref(wsb), L.stream_ptr()))
        return float(out.item())


def C_byref(x):
    import ctypes
    return ctypes.byref(x)


class TorchComm:
    """Collectives over torch.distributed (NCCL on GPUs, gloo on CPU); a single process without
    a process group behaves as world_size 1."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.device = torch, dist, device
        self.single = not (dist.is_available() and dist.is_initialized())

    def allreduce_sum(self, arr):
        if self.single:
            return np.asarray(arr, dtype=np.float64)
        t = self.torch.as_tensor(np.asarray(arr, dtype=np.float64), device=self.device)
        self.dist.all_reduce(t)
        return t.cpu().numpy()

    def exchange_lists(self, per_rank):
        """all_to_all of variable-length int64 arrays via all_gather_object (setup only)."""
        if self.single:
            return [np.asarray(a, dtype=np.int64) for a in per_rank]
        world = self.dist.get_world_size()
        gathered = [None] * world
        self.dist.all_gather_object(gathered, [np.asarray(a, np.int64).tolist() for a in per_rank])
        me = self.dist.get_rank()
        return [np.asarray(gathered[p][me], dtype=np.int64) for p in range(world)]

    def halo(self, x_ext, plan: HaloPlan):
        if self.single:
            return
        torch, dist = self.torch, self.dist
        ops = []
        send_bufs = []
        for p in range(plan.world):
            idx = plan.send_idx[p] if p < len(plan.send_idx) else np.zeros(0, np.int64)
            if p != plan.rank and len(idx):
                buf = x_ext[torch.as_tensor(idx, device=x_ext.device)].contiguous()
                send_bufs.append(buf)
                ops.append(dist.P2POp(dist.isend, buf, p))
        off = plan.n_own
        recv = []
        for p in range(plan.world):
            cnt = plan.recv_counts[p]
            if p != plan.rank and cnt:
                buf = torch.empty(cnt, dtype=x_ext.dtype, device=x_ext.device)
                recv.append((off, buf))
                ops.append(dist.P2POp(dist.irecv, buf, p))
            off += cnt
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for o_, buf in recv:
            x_ext[o_:o_ + len(buf)].copy_(buf)


def solve_rowpart(A, meta, model, b, rtol=1e-8, max_iters=None, period=50, termination="true_residual",
                  rank=None, world=None, comm=None):
    """Full hot path for one system on a row partition: global features, receptive-field
    subgraph GNN (no communication), local G / G^T rows, distributed PCG.  Returns the owned
    slice of x, k, converged, history, and the plan.  Every rank holds the global A (input)."""
    import torch
    import torch.distributed as dist

    from . import _lib as L
    from .gnn import forward_device
    from .graphfeat import build_graph
    from .sparse import DeviceCsr
    if comm is None:
        comm = TorchComm(L.device())
    if rank is None:
        rank = dist.get_rank() if not comm.single else 0
        world = dist.get_world_size() if not comm.single else 1
    n = A.n_rows
    offs, cols, vals = A.row_offsets, A.col_indices, A.values
    gr = build_graph(A, meta)
    node = gr.node_features
    edge = gr.edge_features[:, 0]
    plan = build_plan(offs, cols, n, rank, world, comm.exchange_lists)
    R = hop_closure(offs, cols, np.arange(plan.r0, plan.r1), model.config.n_layers + 2)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(offs))
    in_r = np.zeros(n, dtype=bool)
    in_r[R] = True
    keep = in_r[rows] & in_r[cols]
    remap = -np.ones(n, dtype=np.int64)
    remap[R] = np.arange(len(R))
    sub_offs = np.zeros(len(R) + 1, dtype=np.int64)
    np.add.at(sub_offs, remap[rows[keep]] + 1, 1)
    np.cumsum(sub_offs, out=sub_offs)
    sub = DeviceCsr(len(R), len(R), L.to_device(sub_offs.astype(np.int32), torch.int32),
                    L.to_device(remap[cols[keep]].astype(np.int32), torch.int32),
                    L.to_device(vals[keep], torch.float64))
    g_sub = forward_device(model, sub, L.to_device(np.ascontiguousarray(node[R]).ravel(), torch.float64),
                           L.to_device(edge[keep], torch.float64), gr.d_node).cpu().numpy()
    g = np.full(len(vals), np.nan)
    g[np.flatnonzero(keep)] = g_sub  # exact for rows within one hop of the owned rows
    pcg = DistPcg(plan, CudaOps(), comm, local_rows(offs, cols, vals, plan), local_rows(offs, cols, g, plan),
                  local_transpose_rows(offs, cols, g, plan), model.config.epsilon)
    b = np.asarray(b, dtype=np.float64)
    x_own, k, conv, hist = pcg.solve(b[plan.r0:plan.r1], rtol=rtol, max_iters=max_iters, period=period,
                                     termination=termination)
    return x_own, k, conv, hist, plan


# ------------------------------------------------------------------------------------------------
# Device-resident row partition of a BANDED system (the C5 grid split into blocks of lines)
# ------------------------------------------------------------------------------------------------
GHOST_LAYERS = 3  # ghost depth in half-bandwidths: s is exchanged, d, q, r, x stay exact


@dataclass
class RowPartition:
    """Contiguous row split of one banded system into `parts` partitions.

    own[p]  = [lo, hi)   owned rows (global), multiples of `unit` (a grid line for stencils)
    ext[p]  = own +- GHOST_LAYERS * hb, clipped: the partition's extended local system
    gnn[p]  = ext +- (n_layers + 2) * hb, clipped: the rows whose GNN inputs make G exact on ext
              (receptive field)
    """

    n: int
    parts: int
    hb: int          # half-bandwidth max |col - row|
    unit: int        # owned-block granularity
    own: list
    ext: list
    gnn: list

    @property
    def ghost_lo(self):
        return [o[0] - e[0] for o, e in zip(self.own, self.ext)]

    @property
    def ghost_hi(self):
        return [e[1] - o[1] for o, e in zip(self.own, self.ext)]


def plan_row_partition(offs, cols, n: int, parts: int, n_layers: int, unit: int | None = None) -> RowPartition:
    """Balanced split of n rows (in units of `unit` rows; default: the half-bandwidth when it
    divides n, i.e. grid lines of a 5-point / 7-point stencil) with the ghost and receptive-field
    extents above.  Every partition must own at least its neighbours' ghost depth."""
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(offs))
    hb = int(np.max(np.abs(cols - rows))) if len(cols) else 0
    hb = max(hb, 1)
    if unit is None:
        unit = hb if n % hb == 0 else 1
    if n % unit:
        raise ValueError(f"{n} rows are not a whole number of {unit}-row units")
    nu = n // unit
    if parts < 1 or parts > nu:
        raise ValueError(f"cannot split {nu} units into {parts} partitions")
    own = []
    for p in range(parts):
        a, b = shard_range(nu, p, parts)
        own.append((a * unit, b * unit))
    g = GHOST_LAYERS * hb
    r = (n_layers + 2) * hb
    ext = [(max(0, lo - g), min(n, hi + g)) for lo, hi in own]
    gnn = [(max(0, e0 - r), min(n, e1 + r)) for e0, e1 in ext]
    for p, (lo, hi) in enumerate(own):
        need = max(g if p > 0 else 0, g if p < parts - 1 else 0)
        if parts > 1 and hi - lo < need:
            raise ValueError(f"partition {p} owns {hi - lo} rows, fewer than the ghost depth {need}")
    return RowPartition(n, parts, hb, unit, own, ext, gnn)


def row_block(offs, cols, r0, r1, c0, c1, col_base=0, entry_base=0, out=None):
    """Rows [r0, r1) of a device CSR restricted to columns [c0, c1) (sg_csr_row_block).
    Returns (offs, cols, src) int32 device tensors (src = source entry of every kept entry), or
    fills `out` = (offs_view, cols_view, src_view) and returns the entry count."""
    import ctypes

    import torch

    from . import _lib as L
    lib = L.lib()
    nnz = ctypes.c_int64(0)
    buf, wsb = L.workspace(lib.sg_csr_row_block, None, None, r0, r1, c0, c1, col_base, entry_base, None, None,
                           None, None)
    L.check(lib.sg_csr_row_block(L.ptr(offs), L.ptr(cols), r0, r1, c0, c1, col_base, entry_base, None, None, None,
                                 ctypes.byref(nnz), L.ptr(buf), ctypes.byref(wsb), L.stream_ptr()), "row block")
    m = int(nnz.value)
    if out is None:
        out = (L.empty(r1 - r0 + 1, torch.int32), L.empty(m, torch.int32), L.empty(m, torch.int32))
        ret = out
    else:
        ret = m
    o, c, sidx = out
    L.check(lib.sg_csr_row_block(L.ptr(offs), L.ptr(cols), r0, r1, c0, c1, col_base, entry_base, L.ptr(o),
                                 L.ptr(c[:m]), L.ptr(sidx[:m]), None, L.ptr(buf), ctypes.byref(wsb),
                                 L.stream_ptr()), "row block")
    return ret


def _gather(vals, idx):
    import torch

    from . import _lib as L
    out = L.empty(idx.shape[0], torch.float64)
    L.check(L.lib().sg_gather_f64(L.ptr(vals), L.ptr(idx), L.ptr(out), idx.shape[0], L.stream_ptr()))
    return out


def norm_accumulator(vals_dev, kind: int = 0):
    """Transferable exact-sum accumulator of |v| (sg_norm_accum): int64 device tensor."""
    import ctypes

    import torch

    from . import _lib as L
    lib = L.lib()
    acc = L.empty(lib.sg_norm_acc_size(), torch.int64)
    buf, wsb = L.workspace(lib.sg_norm_accum, None, 0, kind, None)
    L.check(lib.sg_norm_accum(L.ptr(vals_dev), int(vals_dev.shape[0]), kind, L.ptr(acc), L.ptr(buf),
                              ctypes.byref(wsb), L.stream_ptr()), "norm accumulate")
    return acc


def norm_from_accumulator(acc_dev, count: int, kind: int = 0):
    import torch

    from . import _lib as L
    out = L.empty(1, torch.float64)
    L.check(L.lib().sg_norm_from_acc(L.ptr(acc_dev), int(count), kind, L.ptr(out), L.stream_ptr()), "norm")
    return out


@dataclass
class PartitionFactor:
    """One partition's extended local system on its device: A and G rows [e0, e1) with columns
    clipped to [e0, e1) (local indices), the pattern shared."""

    p: int
    own: tuple
    ext: tuple
    offs: object
    cols: object
    a_vals: object
    g_vals: object


def partition_factor(part: RowPartition, p: int, A_dev, meta, model, norm_dev, coeff_mean=None, src_row0=0):
    """What rank p does before its solve, with no communication: cut its GNN block out of A
    (its own rows plus the receptive field), compute the block's features with the GLOBAL
    norm / grid coordinates / coefficient mean, run the GNN on the block, and keep A's and G's
    rows of the extended system.  A_dev: a device CSR holding (at least) the block's rows, with
    GLOBAL column indices, its row 0 being global row `src_row0` -- the whole matrix in the
    single-GPU emulation, the rank's own row slab on the peer path."""
    import torch

    from . import _lib as L
    from .gnn import forward_device
    from .sparse import DeviceCsr
    b0, b1 = part.gnn[p]
    e0, e1 = part.ext[p]
    bo, bc, bsrc = row_block(A_dev.offs, A_dev.cols, b0 - src_row0, b1 - src_row0, b0, b1)
    bv = _gather(A_dev.vals, bsrc)
    blk = DeviceCsr(b1 - b0, b1 - b0, bo, bc, bv)
    family = getattr(meta, "family", None)
    pde = family in ("poisson2d", "heat2d")
    d_node = 3 if pde else 2
    node = L.empty((b1 - b0) * d_node, torch.float64)
    edge = L.empty(blk.nnz, torch.float64)
    if pde:
        nx, ny = meta.grid
        coeff = np.asarray(meta.coeff, dtype=np.float64)
        cmean = float(coeff.mean()) if coeff_mean is None else coeff_mean
        cblk = L.to_device(np.ascontiguousarray(coeff[b0:b1]), torch.float64)
        L.check(L.lib().sg_graph_features_block(b1 - b0, b0, part.n, L.ptr(bo), L.ptr(bc), L.ptr(bv), L.ptr(norm_dev),
                                                1, int(nx), int(ny), L.ptr(cblk), cmean, L.ptr(node), L.ptr(edge),
                                                L.stream_ptr()), "block features")
    else:
        L.check(L.lib().sg_graph_features_block(b1 - b0, b0, part.n, L.ptr(bo), L.ptr(bc), L.ptr(bv), L.ptr(norm_dev),
                                                0, 0, 0, None, 1.0, L.ptr(node), L.ptr(edge), L.stream_ptr()),
                "block features")
    gb = forward_device(model, blk, node, edge, d_node)
    eo, ec, esrc = row_block(bo, bc, e0 - b0, e1 - b0, e0 - b0, e1 - b0)
    return PartitionFactor(p, part.own[p], part.ext[p], eo, ec, _gather(bv, esrc), _gather(gb, esrc))


def global_norm(A_dev, part: RowPartition, allreduce=None, parts=None, src_row0=0, nnz_total=None):
    """norm_A = fsum|A| / nnz from per-partition exact accumulators over the OWNED rows' values:
    each partition (rank) accumulates its own entries, the accumulators are added as integers
    (`allreduce`: torch.distributed all_reduce of the int64 tensor on the peer path; a plain sum
    of every partition's accumulator in the emulation), one rounding -- bit-identical to the
    reference's math.fsum over all entries (sparse.py:204-213)."""
    offs = A_dev.offs
    accs = []
    for p in (range(part.parts) if parts is None else parts):
        lo, hi = part.own[p]
        e_lo, e_hi = int(offs[lo - src_row0].item()), int(offs[hi - src_row0].item())
        accs.append(norm_accumulator(A_dev.vals[e_lo:e_hi]))
    acc = accs[0].clone()
    for a in accs[1:]:
        acc += a
    if allreduce is not None:
        allreduce(acc)
    return norm_from_accumulator(acc, A_dev.nnz if nnz_total is None else nnz_total)


class PartitionedSolver:
    """The row-partitioned hot path of ONE system in group mode: the partitions are the systems
    of one sg_pcg handle (sg_pcg_set_partition) on one GPU -- the emulation of `parts` ranks
    that runs the exact kernels, halo pushes and ordered reductions of the multi-GPU design,
    with every kernel covering all partitions.  `solve` returns a SolveReport for the whole
    system (x assembled from the owned rows)."""

    def __init__(self, A, meta, model, parts: int, unit: int | None = None):
        import torch

        from . import _lib as L
        from .sparse import DeviceCsr
        self.A, self.meta, self.model = A, meta, model
        a = A.device()
        n = A.n_rows
        self.part = plan_row_partition(A.row_offsets, A.col_indices, n, parts, model.config.n_layers, unit)
        norm = global_norm(a, self.part)
        self.factors = [partition_factor(self.part, p, a, meta, model, norm) for p in range(parts)]
        sizes = [f.ext[1] - f.ext[0] for f in self.factors]
        nnzs = [int(f.cols.shape[0]) for f in self.factors]
        self.row_start = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.nnz_start = np.concatenate([[0], np.cumsum(nnzs)]).astype(np.int64)
        N, E = int(self.row_start[-1]), int(self.nnz_start[-1])
        offs, cols = L.empty(N + 1, torch.int32), L.empty(E, torch.int32)
        av, gv = L.empty(E, torch.float64), L.empty(E, torch.float64)
        self._ws_bufs = []
        for p, f in enumerate(self.factors):  # block-diagonal union of the extended systems
            r0, e0 = int(self.row_start[p]), int(self.nnz_start[p])
            L.check(L.lib().sg_csr_row_block(L.ptr(f.offs), L.ptr(f.cols), 0, sizes[p], 0, sizes[p], r0, e0,
                                             L.ptr(offs[r0:]), L.ptr(cols[e0:]), None, None,
                                             *self._ws(f, sizes[p]), L.stream_ptr()), "union")
            av[e0:e0 + nnzs[p]].copy_(f.a_vals)
            gv[e0:e0 + nnzs[p]].copy_(f.g_vals)
        self.a_union = DeviceCsr(N, N, offs, cols, av)
        self.g_union = self.a_union.with_values(gv)
        self.gt_union = self.g_union.transpose()
        from .pcg import PcgHandle
        self.handle = PcgHandle(self.a_union, self.row_start, L.PRECOND_LEARNED, self.g_union, self.gt_union, None,
                                model.config.epsilon)
        lo = np.array([f.own[0] - f.ext[0] for f in self.factors], dtype=np.int64)
        hi = np.array([f.own[1] - f.ext[0] for f in self.factors], dtype=np.int64)
        import ctypes
        L.check(L.lib().sg_pcg_set_partition(self.handle._h, lo.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                             hi.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))), "set_partition")

    def _ws(self, f, nr):
        """Workspace of one sg_csr_row_block call (kept alive on the solver: the call is
        asynchronous)."""
        import ctypes

        from . import _lib as L
        buf, wsb = L.workspace(L.lib().sg_csr_row_block, None, None, 0, nr, 0, nr, 0, 0, None, None, None, None)
        self._ws_bufs.append(buf)
        return L.ptr(buf), ctypes.byref(wsb)

    def solve(self, b, cfg=None):
        import torch

        from . import _lib as L
        from .pcg import SolveConfig, report_from
        cfg = cfg or SolveConfig()
        b = np.asarray(b, dtype=np.float64)
        b_ext = np.concatenate([b[f.ext[0]:f.ext[1]] for f in self.factors])
        bd = L.to_device(b_ext, torch.float64)
        xd = L.empty(len(b_ext), torch.float64)
        res = self.handle.solve(bd, xd, cfg)
        xh = xd.cpu().numpy()
        x = np.concatenate([xh[int(self.row_start[p]) + f.own[0] - f.ext[0]:int(self.row_start[p]) + f.own[1] - f.ext[0]]
                            for p, f in enumerate(self.factors)])
        hist = self.handle.history(0, int(res[0].hist_len)) if cfg.track_history else None
        assert all(r.k == res[0].k and r.converged == res[0].converged for r in res), "partitions diverged"
        return report_from(res[0], x, hist, 0, self.handle.last_elapsed_ns)


    def sai_loss_and_grad(self, w, epsilon: float | None = None, norm_kind: str = "mean_abs_nonzero"):
        """The SAI loss ||(A (G G^T + eps I) w)/||A|| - w||^2 and dL/dg (training.py:57-94, the
        tape backward autodiff.py:203-239, 265-303) on the row partition: every partition
        evaluates its extended system; the one halo is z (neighbours' owned rows into the ghost
        rows, here a device copy between the partitions' buffers), the norm and loss partials add
        in partition order.  Returns (loss, [dL/dg of each partition's extended G, exact on the
        entries of its owned rows])."""
        import ctypes

        import torch

        from . import _lib as L
        from .training import NORM_KINDS
        lib = L.lib()
        kind = NORM_KINDS.index(norm_kind)
        eps = self.model.config.epsilon if epsilon is None else float(epsilon)
        w = np.asarray(w, dtype=np.float64)
        P_ = len(self.factors)
        mats = []
        for f in self.factors:
            ne = f.ext[1] - f.ext[0]
            from .sparse import DeviceCsr
            a = DeviceCsr(ne, ne, f.offs, f.cols, f.a_vals)
            g = a.with_values(f.g_vals)
            mats.append((a, a.transpose(), g, g.transpose()))
        parts = L.empty(2 * P_, torch.float64)
        for p, f in enumerate(self.factors):
            a = mats[p][0]
            lo, hi = f.own[0] - f.ext[0], f.own[1] - f.ext[0]
            e_lo, e_hi = int(a.offs[lo].item()), int(a.offs[hi].item())
            L.call_ws(lib.sg_loss_norm_partial, L.ptr(a.vals[e_lo:e_hi]), e_hi - e_lo, kind, L.ptr(parts[2 * p:]),
                      what="loss norm partial")
        norm3 = L.empty(3, torch.float64)
        nnz_total = int(self.A.nnz)
        L.check(lib.sg_loss_norm_combine(L.ptr(parts), P_, nnz_total, kind, L.ptr(norm3), L.stream_ptr()))
        ts, zs, ws_ = [], [], []
        lparts = L.empty(2 * P_, torch.float64)
        for p, f in enumerate(self.factors):
            a, _, g, gt = mats[p]
            ne = a.n_rows
            wd = L.to_device(np.ascontiguousarray(w[f.ext[0]:f.ext[1]]), torch.float64)
            t, z = L.empty(ne, torch.float64), L.empty(ne, torch.float64)
            L.call_ws(lib.sg_sai_loss_part_fwd, ne, L.ptr(a.offs), L.ptr(a.cols), L.ptr(a.vals), L.ptr(g.offs),
                      L.ptr(g.cols), L.ptr(g.vals), L.ptr(gt.offs), L.ptr(gt.cols), L.ptr(gt.vals), eps, L.ptr(wd),
                      L.ptr(norm3), f.own[0] - f.ext[0], f.own[1] - f.ext[0], L.ptr(t), L.ptr(z),
                      L.ptr(lparts[2 * p:]), what="partitioned loss forward")
            ts.append(t), zs.append(z), ws_.append(wd)
        for p, f in enumerate(self.factors):  # the z halo: neighbours' owned rows -> my ghost rows
            for q in (p - 1, p + 1):
                if 0 <= q < P_:
                    fq = self.factors[q]
                    r0, r1 = max(f.ext[0], fq.own[0]), min(f.ext[1], fq.own[1])
                    if r0 < r1:
                        zs[p][r0 - f.ext[0]:r1 - f.ext[0]].copy_(zs[q][r0 - fq.ext[0]:r1 - fq.ext[0]])
        loss = ctypes.c_double(0.0)
        L.check(lib.sg_loss_sum_parts(L.ptr(lparts), P_, ctypes.byref(loss), L.stream_ptr()))
        grads = []
        for p, f in enumerate(self.factors):
            a, at, g, gt = mats[p]
            grad = L.zeros(g.nnz, torch.float64)
            L.call_ws(lib.sg_sai_loss_part_bwd, a.n_rows, L.ptr(at.offs), L.ptr(at.cols), L.ptr(at.vals),
                      L.ptr(gt.offs), L.ptr(gt.cols), L.ptr(gt.vals), L.ptr(g.offs), L.ptr(g.rows()), L.ptr(g.cols),
                      L.ptr(ws_[p]), L.ptr(ts[p]), L.ptr(zs[p]), L.ptr(norm3), f.own[0] - f.ext[0],
                      f.own[1] - f.ext[0], L.ptr(grad), what="partitioned loss backward")
            grads.append(grad)
        return float(loss.value), grads


def solve_partitioned(A, meta, model, b, parts: int, cfg=None):
    """GNN build + PCG of one system split into `parts` row partitions on this GPU (group
    mode).  Same result as pcg_solve on the whole system up to the order of the dot-product
    partial sums."""
    return PartitionedSolver(A, meta, model, parts).solve(b, cfg)


# ------------------------------------------------------------------------------------------------
# Peer mode: one partition per rank, one process per GPU (the multi-GPU path of BASELINE configs[4])
# ------------------------------------------------------------------------------------------------
def exchange_blobs(blob: bytes, group=None) -> list:
    """all_gather of one opaque byte string per rank (setup only; gloo or NCCL)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return out


def host_row_slab(A, r0: int, r1: int):
    """Rows [r0, r1) of a host CSR (reference int64 arrays) uploaded as a device CSR with GLOBAL
    column indices: the only part of A a rank ever moves to its GPU."""
    import torch

    from . import _lib as L
    from .sparse import DeviceCsr
    offs = np.asarray(A.row_offsets, dtype=np.int64)
    lo, hi = int(offs[r0]), int(offs[r1])
    o = L.to_device((offs[r0:r1 + 1] - lo).astype(np.int32), torch.int32)
    c = L.to_device(np.asarray(A.col_indices[lo:hi], dtype=np.int64).astype(np.int32), torch.int32)
    v = L.to_device(np.ascontiguousarray(A.values[lo:hi], dtype=np.float64), torch.float64)
    return DeviceCsr(r1 - r0, A.n_cols, o, c, v)


class PeerPartitionSolver:
    """Rank `rank` of `world` (torch.distributed initialised, one process per GPU): the rank's
    partition as a one-system sg_pcg handle in peer mode (sg_pcg_peer_export / sg_pcg_set_peers:
    s halos stored into the neighbours' ghost rows over NVLink by the kernels, reductions by peer
    stores + system-scope flags).  Setup communicates twice: the exact norm accumulator
    (integer all-reduce) and the peer blobs (all_gather); the solve communicates only inside the
    kernels.  Every rank returns the same k / history and its own slice of x."""

    def __init__(self, A, meta, model, rank: int | None = None, world: int | None = None, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib as L
        from .pcg import PcgHandle
        from .sparse import DeviceCsr
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        n = A.n_rows
        self.part = part = plan_row_partition(A.row_offsets, A.col_indices, n, self.world, model.config.n_layers)
        b0, b1 = part.gnn[self.rank]
        slab = host_row_slab(A, b0, b1)

        def allreduce(acc):
            if self.world > 1:
                t = acc.cpu() if dist.get_backend(group) == "gloo" else acc
                dist.all_reduce(t, group=group)
                acc.copy_(t)

        norm = global_norm(slab, part, allreduce, parts=[self.rank], src_row0=b0, nnz_total=len(A.col_indices))
        f = self.factor = partition_factor(part, self.rank, slab, meta, model, norm, src_row0=b0)
        ne = f.ext[1] - f.ext[0]
        a = DeviceCsr(ne, ne, f.offs, f.cols, f.a_vals)
        g = a.with_values(f.g_vals)
        self._mats = (a, g, g.transpose())
        self.handle = PcgHandle(a, np.array([0, ne]), L.PRECOND_LEARNED, g, self._mats[2], None,
                                model.config.epsilon)
        lib = L.lib()
        blob = (ctypes.c_ubyte * lib.sg_pcg_peer_info_size())()
        own_lo, own_hi = f.own[0] - f.ext[0], f.own[1] - f.ext[0]
        L.check(lib.sg_pcg_peer_export(self.handle._h, own_lo, own_hi, self.world, blob), "peer export")
        blobs = exchange_blobs(bytes(blob), group) if self.world > 1 else [bytes(blob)]
        allb = (ctypes.c_ubyte * (len(blob) * self.world)).from_buffer_copy(b"".join(blobs))
        L.check(lib.sg_pcg_set_peers(self.handle._h, self.rank, self.world, allb), "set peers")

    def solve(self, b, cfg=None):
        import torch

        from . import _lib as L
        from .pcg import SolveConfig, report_from
        cfg = cfg or SolveConfig()
        f = self.factor
        bd = L.to_device(np.ascontiguousarray(np.asarray(b, dtype=np.float64)[f.ext[0]:f.ext[1]]), torch.float64)
        xd = L.empty(f.ext[1] - f.ext[0], torch.float64)
        (res,) = self.handle.solve(bd, xd, cfg)
        x = xd[f.own[0] - f.ext[0]:f.own[1] - f.ext[0]].cpu().numpy()
        hist = self.handle.history(0, int(res.hist_len)) if cfg.track_history else None
        return report_from(res, x, hist, 0, self.handle.last_elapsed_ns)
