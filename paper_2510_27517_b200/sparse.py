"""CSR storage and the SpMV kernels, drop-in for `spaigraph.sparse` (sparse.py).

`SparseMatrix` keeps the reference's immutable-CSR contract (int64 offsets/indices, f64 values
as numpy arrays on the host side; explicit zeros are pattern-significant), and additionally a
device copy (int32 indices, f64 values, padded for vector loads) that every compute path uses.
Structure validation, COO->CSR, transpose, symmetry and the products run as CUDA kernels from
libspaigraph_b200.so; numpy is only used to hand arrays across the boundary.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

__all__ = ["SparseMatrix", "SparsityPattern", "DeviceCsr", "spmv", "spmv_transpose",
           "mean_abs_nonzero_norm", "read_matrix_market", "write_matrix_market"]

INT32_MAX = 2**31 - 1


class DeviceCsr:
    """Device view: int32 row offsets / column indices (shared between matrices with the same
    pattern) and f64 values.  Plain container; tensors are padded by 16 bytes."""

    __slots__ = ("n_rows", "n_cols", "nnz", "offs", "cols", "vals", "_rows", "_t")

    def __init__(self, n_rows, n_cols, offs, cols, vals):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.nnz = int(cols.shape[0])
        self.offs, self.cols, self.vals = offs, cols, vals
        self._rows = None
        self._t = None  # (offs_t, cols_t, perm) cache

    def rows(self):
        """Row index of every stored entry (sparse.py:64-66), computed once on device."""
        if self._rows is None:
            import torch
            r = L.empty(self.nnz, torch.int32)
            L.check(L.lib().sg_row_expand(self.n_rows, L.ptr(self.offs), L.ptr(r), L.stream_ptr()))
            self._rows = r
        return self._rows

    def transpose_pattern(self):
        """(offs_t, cols_t, perm) with values_t = values[perm] (sparse.py:129-136)."""
        if self._t is None:
            import torch
            self._t = (L.empty(self.n_cols + 1, torch.int32), L.empty(self.nnz, torch.int32),
                       L.empty(self.nnz, torch.int32))
            self._compute_transpose()
        return self._t

    def _compute_transpose(self):
        ot, ct, perm = self._t
        L.call_ws(L.lib().sg_csr_transpose, self.n_rows, self.n_cols, self.nnz, L.ptr(self.offs),
                  L.ptr(self.cols), L.ptr(ot), L.ptr(ct), L.ptr(perm), what="transpose")

    def refresh_pattern(self):
        """Recompute the pattern-derived caches IN PLACE after the index arrays were refilled
        (keeps every pointer a captured PCG handle holds valid)."""
        if self._rows is not None:
            L.check(L.lib().sg_row_expand(self.n_rows, L.ptr(self.offs), L.ptr(self._rows), L.stream_ptr()))
        if self._t is not None:
            self._compute_transpose()

    def with_values(self, vals):
        d = DeviceCsr(self.n_rows, self.n_cols, self.offs, self.cols, vals)
        d._rows, d._t = self._rows, self._t
        return d

    def transpose(self):
        """Explicit transpose: pattern of A^T plus gathered values (bit-exact vs sparse.py:129)."""
        import torch
        ot, ct, perm = self.transpose_pattern()
        vt = L.empty(self.nnz, torch.float64)
        L.check(L.lib().sg_gather_f64(L.ptr(self.vals), L.ptr(perm), L.ptr(vt), self.nnz, L.stream_ptr()))
        return DeviceCsr(self.n_cols, self.n_rows, ot, ct, vt)


def _upload_index(a, lo, hi):
    """Reference int64 index array -> padded int32 device tensor (range-checked on device)."""
    import torch
    a = np.ascontiguousarray(a, dtype=np.int64)
    if len(a) and (len(a) > INT32_MAX):
        raise ValueError("array too long for int32 device indices")
    src = L.to_device(a, torch.int64)
    out = L.empty(len(a), torch.int32)
    if len(a):
        L.call_ws(L.lib().sg_narrow_index, L.ptr(src), L.ptr(out), len(a), int(lo), int(hi), 0,
                  what="narrow")
    return out


def _validate_device(n_rows, n_cols, offs, cols):
    L.call_ws(L.lib().sg_csr_validate, n_rows, n_cols, int(cols.shape[0]), L.ptr(offs), L.ptr(cols),
              what="validate")


class SparsityPattern:
    """CSR structure without values (sparse.py:46-78)."""

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, *, _dev=None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self._offs_h = None if row_offsets is None else np.ascontiguousarray(row_offsets, dtype=np.int64)
        self._cols_h = None if col_indices is None else np.ascontiguousarray(col_indices, dtype=np.int64)
        self._dev = _dev  # (offs, cols) int32 device tensors
        if _dev is None:
            if self._offs_h.ndim != 1 or len(self._offs_h) != self.n_rows + 1:
                raise ValueError("row_offsets must have length n_rows + 1")
            self.device()  # uploads + validates on the GPU

    @property
    def row_offsets(self):
        if self._offs_h is None:
            self._offs_h = self._dev[0].cpu().numpy().astype(np.int64)
        return self._offs_h

    @property
    def col_indices(self):
        if self._cols_h is None:
            self._cols_h = self._dev[1].cpu().numpy().astype(np.int64)
        return self._cols_h

    @property
    def nnz(self) -> int:
        return int(self._dev[1].shape[0]) if self._dev is not None else len(self._cols_h)

    def device(self):
        if self._dev is None:
            if self.n_rows + 1 > INT32_MAX or len(self._cols_h) > INT32_MAX:
                raise ValueError("pattern too large for int32 device indices")
            nnz = len(self._cols_h)
            offs = _upload_index(self._offs_h, -(2**31), 2**31)
            cols = _upload_index(self._cols_h, -(2**31), 2**31)
            _validate_device(self.n_rows, self.n_cols, offs, cols)
            self._dev = (offs, cols)
        return self._dev

    def row_expand(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_offsets))

    def is_symmetric(self) -> bool:
        """sparse.py:68-78, evaluated on device (every (i,j) has a stored (j,i))."""
        if self.n_rows != self.n_cols:
            return False
        offs, cols = self.device()
        res = C.c_int32(0)
        L.call_ws(L.lib().sg_pattern_is_symmetric, self.n_rows, self.nnz, L.ptr(offs), L.ptr(cols),
                  C.byref(res), what="is_symmetric")
        return bool(res.value)


class SparseMatrix:
    """Immutable CSR matrix with 64-bit float values (sparse.py:81-172)."""

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values, *, _dev: DeviceCsr | None = None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self._dev = _dev
        if _dev is None:
            offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
            cols = np.ascontiguousarray(col_indices, dtype=np.int64)
            vals = np.ascontiguousarray(values, dtype=np.float64)
            if offs.ndim != 1 or len(offs) != self.n_rows + 1:
                raise ValueError("row_offsets must have length n_rows + 1")
            if len(vals) != len(cols):
                raise ValueError("values and col_indices must have equal length")
            self._offs_h, self._cols_h, self._vals_h = offs, cols, vals
            self.device()
        else:
            self._offs_h = self._cols_h = self._vals_h = None

    # --- construction -------------------------------------------------------------------
    @staticmethod
    def from_device(dev: DeviceCsr) -> "SparseMatrix":
        return SparseMatrix(dev.n_rows, dev.n_cols, None, None, None, _dev=dev)

    @staticmethod
    def from_coo(n_rows: int, n_cols: int, rows, cols, vals) -> "SparseMatrix":
        """sparse.py:138-158 on device: stable radix sort by (row, col), duplicates rejected."""
        import torch
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        if not (len(rows) == len(cols) == len(vals)):
            raise ValueError("coordinate arrays must have equal length")
        nnz = len(rows)
        d_r, d_c, d_v = L.to_device(rows, torch.int64), L.to_device(cols, torch.int64), L.to_device(vals, torch.float64)
        offs = L.empty(n_rows + 1, torch.int32)
        oc = L.empty(nnz, torch.int32)
        ov = L.empty(nnz, torch.float64)
        dup = (C.c_int64 * 2)()
        L.call_ws(L.lib().sg_csr_from_coo, n_rows, n_cols, nnz, L.ptr(d_r), L.ptr(d_c), L.ptr(d_v),
                  L.ptr(offs), L.ptr(oc), L.ptr(ov), dup, what="from_coo")
        return SparseMatrix.from_device(DeviceCsr(n_rows, n_cols, offs, oc, ov))

    @staticmethod
    def from_dense(dense, keep=None) -> "SparseMatrix":
        dense = np.asarray(dense, dtype=np.float64)
        if keep is None:
            keep = dense != 0.0
        r, c = np.nonzero(keep)
        return SparseMatrix.from_coo(dense.shape[0], dense.shape[1], r, c, dense[r, c])

    @staticmethod
    def identity(n: int) -> "SparseMatrix":
        idx = np.arange(n, dtype=np.int64)
        return SparseMatrix(n, n, np.arange(n + 1, dtype=np.int64), idx, np.ones(n))

    # --- device / host views ---------------------------------------------------------------
    def device(self) -> DeviceCsr:
        if self._dev is None:
            import torch
            if self.n_rows + 1 > INT32_MAX or len(self._cols_h) > INT32_MAX:
                raise ValueError("matrix too large for int32 device indices")
            offs = _upload_index(self._offs_h, -(2**31), 2**31)
            cols = _upload_index(self._cols_h, -(2**31), 2**31)
            _validate_device(self.n_rows, self.n_cols, offs, cols)
            vals = L.to_device(self._vals_h, torch.float64)
            self._dev = DeviceCsr(self.n_rows, self.n_cols, offs, cols, vals)
        return self._dev

    @property
    def row_offsets(self) -> np.ndarray:
        if self._offs_h is None:
            self._offs_h = self._dev.offs.cpu().numpy().astype(np.int64)
        return self._offs_h

    @property
    def col_indices(self) -> np.ndarray:
        if self._cols_h is None:
            self._cols_h = self._dev.cols.cpu().numpy().astype(np.int64)
        return self._cols_h

    @property
    def values(self) -> np.ndarray:
        if self._vals_h is None:
            self._vals_h = self._dev.vals.cpu().numpy()
        return self._vals_h

    @property
    def nnz(self) -> int:
        return self._dev.nnz if self._dev is not None else len(self._vals_h)

    @property
    def pattern(self) -> SparsityPattern:
        d = self.device()
        return SparsityPattern(self.n_rows, self.n_cols, self._offs_h, self._cols_h, _dev=(d.offs, d.cols))

    def row_expand(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_offsets))

    def with_values(self, values) -> "SparseMatrix":
        """Same pattern, new values (positional); shares the device index arrays."""
        import torch
        d = self.device()
        if isinstance(values, torch.Tensor):
            v = values.to(dtype=torch.float64)
        else:
            v = np.ascontiguousarray(values, dtype=np.float64)
            if len(v) != d.nnz:
                raise ValueError("values and col_indices must have equal length")
            v = L.to_device(v, torch.float64)
        if v.shape[0] != d.nnz:
            raise ValueError("values and col_indices must have equal length")
        m = SparseMatrix.from_device(d.with_values(v))
        m._offs_h, m._cols_h = self._offs_h, self._cols_h
        return m

    def diagonal(self) -> np.ndarray:
        if self.n_rows != self.n_cols:
            raise ValueError("diagonal of a non-square matrix")
        return self.diagonal_device()[0].cpu().numpy()

    def diagonal_device(self):
        import torch
        d = self.device()
        diag = L.empty(self.n_rows, torch.float64)
        present = L.empty(self.n_rows, torch.int32)
        L.check(L.lib().sg_csr_diagonal(self.n_rows, L.ptr(d.offs), L.ptr(d.cols), L.ptr(d.vals),
                                        L.ptr(diag), L.ptr(present), L.stream_ptr()))
        return diag, present

    def transpose(self) -> "SparseMatrix":
        return SparseMatrix.from_device(self.device().transpose())

    def __repr__(self):
        return f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz}, device=cuda)"


def _as_dev_vector(x, n, what="vector"):
    import torch
    if isinstance(x, torch.Tensor):
        if x.shape[0] != n:
            raise ValueError(f"dimension mismatch: {what} has length {x.shape[0]}, expected {n}")
        return x.to(device=L.device(), dtype=torch.float64).contiguous(), True
    x = np.asarray(x, dtype=np.float64)
    if len(x) != n:
        raise ValueError(f"dimension mismatch: {what} has length {len(x)}, expected {n}")
    return L.to_device(x, torch.float64), False


def spmv(A: SparseMatrix, x):
    """y = A x (sparse.py:186-191), numpy reduceat summation order, bit-identical."""
    import torch
    n = x.shape[0] if isinstance(x, torch.Tensor) else len(np.asarray(x))
    if A.n_cols != n:
        raise ValueError(f"dimension mismatch: matrix has {A.n_cols} columns, vector has {n}")
    d = A.device()
    xd, was_t = _as_dev_vector(x, A.n_cols)
    y = L.empty(A.n_rows, torch.float64)
    # long rows (C4's G on the A^2 pattern): a warp per row, same order
    fn = L.lib().sg_spmv_warp if d.nnz >= 32 * A.n_rows else L.lib().sg_spmv
    L.check(fn(A.n_rows, L.ptr(d.offs), L.ptr(d.cols), L.ptr(d.vals), L.ptr(xd), L.ptr(y), L.stream_ptr()))
    return y if was_t else y.cpu().numpy()


def spmv_transpose(A: SparseMatrix, x):
    """y = A^T x (sparse.py:194-201) over the explicit transpose; np.add.at order, bit-identical."""
    import torch
    n = x.shape[0] if isinstance(x, torch.Tensor) else len(np.asarray(x))
    if A.n_rows != n:
        raise ValueError(f"dimension mismatch: matrix has {A.n_rows} rows, vector has {n}")
    t = A.device().transpose()
    xd, was_t = _as_dev_vector(x, A.n_rows)
    y = L.empty(A.n_cols, torch.float64)
    L.check(L.lib().sg_spmv_seq(t.n_rows, L.ptr(t.offs), L.ptr(t.cols), L.ptr(t.vals), L.ptr(xd), L.ptr(y),
                                L.stream_ptr()))
    return y if was_t else y.cpu().numpy()


def pattern_square(A: SparseMatrix) -> SparsityPattern:
    """pattern(|A| |A|) on the GPU (SURVEY.md §8(a) a5, config C4's G pattern)."""
    import torch
    if A.n_rows != A.n_cols:
        raise ValueError("pattern square requires a square matrix")
    d = A.device()
    n = A.n_rows
    offs = L.empty(n + 1, torch.int32)
    nnz = C.c_int64(0)
    buf, wsb = L.workspace(L.lib().sg_pattern_square, n, L.ptr(d.offs), L.ptr(d.cols), L.ptr(offs), None,
                           C.byref(nnz))
    L.check(L.lib().sg_pattern_square(n, L.ptr(d.offs), L.ptr(d.cols), L.ptr(offs), None, C.byref(nnz),
                                      L.ptr(buf), C.byref(wsb), L.stream_ptr()), "pattern_square")
    cols = L.empty(int(nnz.value), torch.int32)
    L.check(L.lib().sg_pattern_square(n, L.ptr(d.offs), L.ptr(d.cols), L.ptr(offs), L.ptr(cols), C.byref(nnz),
                                      L.ptr(buf), C.byref(wsb), L.stream_ptr()), "pattern_square")
    return SparsityPattern(n, n, None, None, _dev=(offs, cols))


def pad_to_pattern(A: SparseMatrix, pattern: SparsityPattern) -> SparseMatrix:
    """A's values on a superset pattern with explicit zeros elsewhere (pattern-significant)."""
    import torch
    if (pattern.n_rows, pattern.n_cols) != (A.n_rows, A.n_cols):
        raise ValueError("pattern shape does not match the matrix")
    d = A.device()
    po, pc = pattern.device()
    out = L.empty(int(pc.shape[0]), torch.float64)
    L.call_ws(L.lib().sg_csr_pad_to_pattern, A.n_rows, L.ptr(d.offs), L.ptr(d.cols), L.ptr(d.vals), L.ptr(po),
              L.ptr(pc), L.ptr(out), what="pad_to_pattern")
    return SparseMatrix.from_device(DeviceCsr(A.n_rows, A.n_cols, po, pc, out))


def norm_device(vals, nnz: int, kind: int):
    """Device scalar: exact-sum matrix norm (kind 0 mean-abs, 1 frobenius, 2 entrywise l1)."""
    import torch
    out = L.empty(1, torch.float64)
    L.call_ws(L.lib().sg_matrix_norm, L.ptr(vals), int(nnz), int(kind), L.ptr(out), what="norm")
    return out


def mean_abs_nonzero_norm(A: SparseMatrix) -> float:
    """sparse.py:204-213: fsum(|v|)/nnz, correctly rounded (bit-identical) on device."""
    if A.nnz == 0:
        raise ValueError("norm of a matrix with no stored entries")
    return float(norm_device(A.device().vals, A.nnz, 0).item())


def read_matrix_market(path) -> SparseMatrix:
    """sparse.py:216-265 (host text parsing; the COO->CSR build runs on device)."""
    with open(path, "r", encoding="ascii") as fh:
        header = fh.readline()
        parts = header.strip().split()
        if (len(parts) != 5 or parts[0] != "%%MatrixMarket" or parts[1].lower() != "matrix"
                or parts[2].lower() != "coordinate" or parts[3].lower() != "real"
                or parts[4].lower() not in ("general", "symmetric")):
            raise ValueError(f"malformed Matrix Market header: {header.strip()!r}")
        symmetric = parts[4].lower() == "symmetric"
        line = fh.readline()
        while line.startswith("%"):
            line = fh.readline()
        try:
            n_rows, n_cols, nnz = (int(t) for t in line.split())
        except Exception as exc:
            raise ValueError(f"malformed size line: {line.strip()!r}") from exc
        body = np.loadtxt(fh, dtype=np.float64, ndmin=2, max_rows=nnz) if nnz else np.zeros((0, 3))
    if body.shape != (nnz, 3):
        raise ValueError("malformed entry lines")
    rows = body[:, 0].astype(np.int64) - 1
    cols = body[:, 1].astype(np.int64) - 1
    vals = body[:, 2].copy()
    if nnz > 0 and (rows.min() < 0 or rows.max() >= n_rows or cols.min() < 0 or cols.max() >= n_cols):
        raise ValueError("entry index out of range")
    if symmetric:
        if n_rows != n_cols:
            raise ValueError("symmetric header on a non-square matrix")
        if np.any(cols > rows):
            raise ValueError("symmetric file stores an upper-triangular entry")
        off = cols < rows
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    return SparseMatrix.from_coo(n_rows, n_cols, rows, cols, vals)


def write_matrix_market(A: SparseMatrix, path) -> None:
    """sparse.py:268-275."""
    rows = A.row_expand()
    with open(path, "w", encoding="ascii") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{A.n_rows} {A.n_cols} {A.nnz}\n")
        for r, c, v in zip(rows, A.col_indices, A.values):
            fh.write(f"{r + 1} {c + 1} {v:.16e}\n")
