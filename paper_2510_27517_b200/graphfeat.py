"""Matrix -> feature graph, drop-in for `spaigraph.graphfeat` (graphfeat.py:63-105).

`build_graph` computes the features on the GPU: the exact (fsum-identical) mean-abs norm,
edge features vals/norm, and node features (PDE [x, y, a/mean(a)] or algebraic
[rowsum/n/norm, diag/norm]) — bit-identical to the reference.  The returned `MatrixGraph`
keeps device tensors; the host arrays of the reference dataclass are materialised on access.
"""
from __future__ import annotations

import struct

import numpy as np

from . import _lib as L
from .sparse import SparseMatrix, norm_device

__all__ = ["MatrixGraph", "build_graph", "write_graph_bin", "read_graph_bin"]

_MAGIC = b"SPGRAPH\x01"


class MatrixGraph:
    """Feature arrays aligned with a matrix's CSR enumeration (graphfeat.py:24-60).

    Device fields: `matrix` (the DeviceCsr the graph was built from, whose pattern is the edge
    list), `node_dev` [n x d_node], `edge_dev` [nnz] (d_edge == 1), `norm_dev` (scalar).
    """

    def __init__(self, n_nodes, node_features=None, edge_list=None, edge_features=None, norm_A=None,
                 *, matrix=None, node_dev=None, edge_dev=None, norm_dev=None):
        import torch
        self.n_nodes = int(n_nodes)
        if matrix is None:  # constructed from host arrays, as the reference dataclass
            node_features = np.ascontiguousarray(node_features, dtype=np.float64)
            edge_list = np.ascontiguousarray(edge_list, dtype=np.int64)
            edge_features = np.ascontiguousarray(edge_features, dtype=np.float64)
            if node_features.ndim != 2 or node_features.shape[0] != self.n_nodes:
                raise ValueError("node_features must be (n_nodes, d_node)")
            if edge_list.ndim != 2 or edge_list.shape[1] != 2:
                raise ValueError("edge_list must be (n_edges, 2)")
            if edge_features.ndim != 2 or edge_features.shape[0] != edge_list.shape[0]:
                raise ValueError("edge_features must be (n_edges, d_edge)")
            rows = edge_list[:, 0]
            if np.any(rows[1:] < rows[:-1]):
                raise ValueError("edge list is not in CSR order")
            offs = np.zeros(self.n_nodes + 1, dtype=np.int64)
            np.add.at(offs, rows + 1, 1)
            np.cumsum(offs, out=offs)
            # values are irrelevant for the graph; the pattern is validated on device
            matrix = SparseMatrix(self.n_nodes, self.n_nodes, offs, edge_list[:, 1],
                                  np.zeros(len(rows))).device()
            node_dev = L.to_device(node_features.ravel(), torch.float64)
            edge_dev = L.to_device(edge_features.ravel(), torch.float64)
            self._d_edge = edge_features.shape[1]
            self._node_h, self._edge_h = node_features, edge_features
            self._norm_h = float(norm_A)
            norm_dev = L.to_device(np.array([self._norm_h]), torch.float64)
        else:
            self._d_edge = 1
            self._node_h = self._edge_h = None
            self._norm_h = None
        self.matrix = matrix
        self.node_dev, self.edge_dev, self.norm_dev = node_dev, edge_dev, norm_dev
        self._d_node = int(node_dev.shape[0] // max(self.n_nodes, 1)) if self.n_nodes else 0
        if node_features is not None:
            self._d_node = node_features.shape[1]

    @property
    def n_edges(self) -> int:
        return self.matrix.nnz

    @property
    def d_node(self) -> int:
        return self._d_node

    @property
    def d_edge(self) -> int:
        return self._d_edge

    @property
    def norm_A(self) -> float:
        if self._norm_h is None:
            self._norm_h = float(self.norm_dev.item())
        return self._norm_h

    @property
    def node_features(self) -> np.ndarray:
        if self._node_h is None:
            self._node_h = self.node_dev.cpu().numpy().reshape(self.n_nodes, self._d_node)
        return self._node_h

    @property
    def edge_features(self) -> np.ndarray:
        if self._edge_h is None:
            self._edge_h = self.edge_dev.cpu().numpy().reshape(-1, self._d_edge)
        return self._edge_h

    @property
    def edge_list(self) -> np.ndarray:
        rows = self.matrix.rows().cpu().numpy().astype(np.int64)
        return np.stack([rows, self.matrix.cols.cpu().numpy().astype(np.int64)], axis=1)


def _coeff_mean(coeff: np.ndarray) -> float:
    # graphfeat.py:99 `coeff.mean()`: numpy's pairwise sum / n over the host coefficient field.
    return float(coeff.mean())


def build_graph(A: SparseMatrix, meta=None) -> MatrixGraph:
    """graphfeat.py:63-105 on the GPU (bit-identical features)."""
    import torch
    if A.n_rows != A.n_cols:
        raise ValueError("graph requires a square matrix")
    if not A.pattern.is_symmetric():
        raise ValueError("graph requires a symmetric sparsity pattern")
    n = A.n_rows
    if A.nnz == 0:
        raise ValueError("norm of a matrix with no stored entries")
    d = A.device()
    norm = norm_device(d.vals, d.nnz, 0)
    family = getattr(meta, "family", None)
    edge = L.empty(d.nnz, torch.float64)
    if family in ("poisson2d", "heat2d"):
        grid = meta.grid
        coeff = np.asarray(meta.coeff, dtype=np.float64)
        if grid is None or int(np.prod(grid)) != n:
            raise ValueError("meta grid does not match matrix size")
        if len(coeff) != n:
            raise ValueError("meta coefficient field does not match matrix size")
        nx, ny = grid
        coeff_d = getattr(meta, "coeff_dev", None)
        if coeff_d is None:
            coeff_d = L.to_device(coeff, torch.float64)
        node = L.empty(n * 3, torch.float64)
        L.check(L.lib().sg_graph_features(n, 0, L.ptr(d.offs), L.ptr(d.cols), L.ptr(d.vals), L.ptr(norm), 1,
                                          int(nx), int(ny), L.ptr(coeff_d), _coeff_mean(coeff),
                                          L.ptr(node), L.ptr(edge), L.stream_ptr()))
    else:
        if family is not None and family != "synthetic":
            raise ValueError(f"unknown problem family {family!r}")
        node = L.empty(n * 2, torch.float64)
        L.check(L.lib().sg_graph_features(n, 0, L.ptr(d.offs), L.ptr(d.cols), L.ptr(d.vals), L.ptr(norm), 0,
                                          0, 0, None, 1.0, L.ptr(node), L.ptr(edge), L.stream_ptr()))
    g = MatrixGraph(n, matrix=d, node_dev=node, edge_dev=edge, norm_dev=norm)
    g._d_node = 3 if family in ("poisson2d", "heat2d") else 2
    return g


def write_graph_bin(graph: MatrixGraph, path):
    """graphfeat.py:108-123."""
    header = struct.pack("<4Qd", graph.n_nodes, graph.n_edges, graph.d_node, graph.d_edge, graph.norm_A)
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(header)
        fh.write(np.ascontiguousarray(graph.node_features, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(graph.edge_features, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(graph.edge_list, dtype="<i8").tobytes())


def read_graph_bin(path) -> MatrixGraph:
    """graphfeat.py:126-146."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[: len(_MAGIC)] != _MAGIC:
        raise ValueError(f"not a graph container: {path}")
    off = len(_MAGIC)
    n_nodes, n_edges, d_node, d_edge, norm = struct.unpack_from("<4Qd", blob, off)
    off += struct.calcsize("<4Qd")

    def take(count, dtype):
        nonlocal off
        arr = np.frombuffer(blob, dtype=dtype, count=count, offset=off)
        off += arr.nbytes
        return arr

    node = take(n_nodes * d_node, "<f8").reshape(n_nodes, d_node)
    edge = take(n_edges * d_edge, "<f8").reshape(n_edges, d_edge)
    el = take(n_edges * 2, "<i8").reshape(n_edges, 2)
    if off != len(blob):
        raise ValueError("trailing bytes in graph container")
    return MatrixGraph(int(n_nodes), node, el, edge, float(norm))
