"""Row-partitioned PCG for ONE large system across ranks.

Rank p owns the contiguous rows [r0, r1) (balanced split).  Everything a rank needs is built
once from the global CSR pattern:

* halo plan — the columns of the owned rows that other ranks own, grouped by owner; the owners
  learn which of their values to send (one all_to_all of index lists).  Local vectors are
  "extended": [owned | halo from rank 0 | halo from rank 1 | ...];
* the GNN factor: a rank runs the forward pass on the (L+2)-hop induced subgraph of its rows with
  globally computed features (G's rows within one hop of the owned rows are then
  exact), so the GNN needs no communication at all; G^T's owned rows are assembled locally from
  G's rows of the owned + 1-hop halo nodes;
* per PCG iteration: 3 halo exchanges (d', r', t) and 2 all-reduces (d'.q; [r'.s, ||r'||^2]),
  plus one halo exchange + SpMV on refresh / fresh-residual iterations.

The control flow is pcg.py:131-233 verbatim, driven from the host (scalars are all-reduced and
read back every iteration).  Local products and updates go through an `ops` backend: `CudaOps`
(the C-ABI kernels; numpy summation orders, bit-exact per row) on GPUs with NCCL, or a numpy
backend in the CPU tests with gloo.  The fused, device-resident multi-rank loop (peer-memory
halos inside the iteration kernels) is the next step; this module fixes the partitioning, the
communication schedule and their tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .batch import shard_range
from .pcg import NotSpdError

__all__ = ["HaloPlan", "build_plan", "hop_closure", "local_transpose_rows", "DistPcg", "BandPart", "band_partition",
           "band_local", "solve_rowpart_device"]


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
# Device-resident row partition (banded matrices, e.g. the C5 grid split into blocks of lines)
# ------------------------------------------------------------------------------------------------
@dataclass
class BandPart:
    """Rank `rank`'s extended local system for a contiguous row split of a banded matrix:
    owned rows [r0, r1) plus `ghost_lo` / `ghost_hi` ghost rows (the neighbours' boundary rows;
    ghost width = the half-bandwidth, clipped at the matrix ends)."""

    n: int
    rank: int
    world: int
    r0: int
    r1: int
    ghost_lo: int
    ghost_hi: int

    @property
    def e0(self):
        return self.r0 - self.ghost_lo

    @property
    def e1(self):
        return self.r1 + self.ghost_hi

    @property
    def left(self):
        return self.rank - 1 if self.rank > 0 else -1

    @property
    def right(self):
        return self.rank + 1 if self.rank < self.world - 1 else -1


def band_partition(offs, cols, n: int, rank: int, world: int) -> BandPart:
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(offs))
    hb = int(np.max(np.abs(cols - rows))) if len(cols) else 0
    r0, r1 = shard_range(n, rank, world)
    gl = min(hb, r0) if rank > 0 else 0
    gh = min(hb, n - r1) if rank < world - 1 else 0
    for p in range(world):  # every owned block must be at least one band wide
        a, b = shard_range(n, p, world)
        if world > 1 and b - a < hb:
            raise ValueError(f"rank {p} owns {b - a} rows, fewer than the half-bandwidth {hb}")
    return BandPart(n, rank, world, r0, r1, gl, gh)


def band_local(offs, cols, vals, part: BandPart):
    """Rows [e0, e1) of a CSR matrix with columns shifted to the extended local index space;
    entries whose column falls outside it (only possible in the outermost ghost rows) dropped."""
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    lo, hi = offs[part.e0], offs[part.e1]
    c = cols[lo:hi]
    v = vals[lo:hi]
    r = np.repeat(np.arange(part.e0, part.e1), np.diff(offs[part.e0:part.e1 + 1]))
    keep = (c >= part.e0) & (c < part.e1)
    lo_offs = np.zeros(part.e1 - part.e0 + 1, dtype=np.int64)
    np.add.at(lo_offs, r[keep] - part.e0 + 1, 1)
    np.cumsum(lo_offs, out=lo_offs)
    return lo_offs, c[keep] - part.e0, v[keep]


def _nccl_comm(rank: int, world: int):
    """One NCCL communicator for the solve: the unique id travels over torch.distributed when a
    process group exists (a 1-rank communicator otherwise)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from . import _lib as L
    uid = (ctypes.c_ubyte * 128)()
    if rank == 0:
        L.check(L.lib().sg_nccl_unique_id(ctypes.cast(uid, ctypes.c_void_p)), "nccl unique id")
    if world > 1:
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8,
                         device=L.device() if dist.get_backend() == "nccl" else "cpu")
        dist.broadcast(t, 0)
        uid = (ctypes.c_ubyte * 128)(*t.cpu().tolist())
    comm = ctypes.c_void_p()
    L.check(L.lib().sg_nccl_comm_init(ctypes.byref(comm), ctypes.cast(uid, ctypes.c_void_p), world, rank),
            "nccl comm init")
    return comm


def solve_rowpart_device(A, meta, model, b, rtol=1e-8, max_iters=None, period=50, termination="true_residual",
                         rank=None, world=None):
    """The hot path for one banded system split by rows across ranks, with the PCG loop on the
    device: every rank builds its extended local system (owned rows + ghost rows), runs the GNN
    on the receptive field of those rows (no communication: features are global),
    and solves with sg_pcg in row-partitioned mode — halo exchanges and scalar all-reduces are
    NCCL operations inside the captured iteration graphs.  Returns (x_own, k, converged,
    history, part)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from . import _lib as L
    from .gnn import forward_device
    from .graphfeat import build_graph
    from .pcg import SolveConfig, report_from
    from .sparse import DeviceCsr
    if rank is None:
        init = dist.is_available() and dist.is_initialized()
        rank = dist.get_rank() if init else 0
        world = dist.get_world_size() if init else 1
    n = A.n_rows
    offs, cols, vals = A.row_offsets, A.col_indices, A.values
    part = band_partition(offs, cols, n, rank, world)
    gr = build_graph(A, meta)
    node, edge = gr.node_features, gr.edge_features[:, 0]
    # GNN on the (L+2)-hop receptive field of the extended rows: their G rows are exact
    R = hop_closure(offs, cols, np.arange(part.e0, part.e1), model.config.n_layers + 2)
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
    g = np.zeros(len(vals))
    g[np.flatnonzero(keep)] = g_sub
    ao, ac, av = band_local(offs, cols, vals, part)
    _, _, gv = band_local(offs, cols, g, part)
    ne = part.e1 - part.e0
    a_dev = DeviceCsr(ne, ne, L.to_device(ao.astype(np.int32), torch.int32), L.to_device(ac.astype(np.int32), torch.int32),
                      L.to_device(av, torch.float64))
    g_dev = a_dev.with_values(L.to_device(gv, torch.float64))
    gt_dev = g_dev.transpose()
    h = ctypes.c_void_p()
    L.check(L.lib().sg_pcg_create_part(ctypes.byref(h), ne, part.ghost_lo, part.ghost_lo + (part.r1 - part.r0),
                                       L.ptr(a_dev.offs), L.ptr(a_dev.cols), L.ptr(a_dev.vals), L.PRECOND_LEARNED,
                                       L.ptr(g_dev.offs), L.ptr(g_dev.cols), L.ptr(g_dev.vals), L.ptr(gt_dev.offs),
                                       L.ptr(gt_dev.cols), L.ptr(gt_dev.vals), None, float(model.config.epsilon),
                                       L.stream_ptr()), "pcg_create_part")
    comm = _nccl_comm(rank, world)
    try:
        L.check(L.lib().sg_pcg_set_comm(h, comm, part.left, part.right, part.ghost_lo, part.ghost_hi), "set_comm")
        cfg = SolveConfig(rtol=rtol, max_iters=max_iters, residual_refresh_period=period, termination=termination)
        b_ext = np.zeros(ne)
        b_ext[part.ghost_lo:part.ghost_lo + part.r1 - part.r0] = np.asarray(b, dtype=np.float64)[part.r0:part.r1]
        bd = L.to_device(b_ext, torch.float64)
        xd = L.empty(ne, torch.float64)
        res = (L.SolveResultC * 1)()
        ns = ctypes.c_int64(0)
        L.check(L.lib().sg_pcg_solve(h, L.ptr(bd), L.ptr(xd), ctypes.byref(cfg.to_c()), res, ctypes.byref(ns),
                                     L.stream_ptr()), "pcg_solve (row partition)")
        hist = np.empty(max(int(res[0].hist_len), 0))
        if len(hist):
            L.check(L.lib().sg_pcg_history(h, 0, hist.ctypes.data_as(ctypes.c_void_p), len(hist)))
        x_own = xd[part.ghost_lo:part.ghost_lo + part.r1 - part.r0].cpu().numpy()
        rep = report_from(res[0], x_own, hist.tolist(), 0, int(ns.value))
    finally:
        L.lib().sg_pcg_destroy(h)
        L.lib().sg_nccl_comm_destroy(comm)
    return rep.x, rep.k, rep.converged, rep.residual_history, part
