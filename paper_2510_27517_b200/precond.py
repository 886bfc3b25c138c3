"""Preconditioners behind the reference's apply contract (precond.py:42-145, 148-164, 308-312).

`LearnedSpaiPreconditioner` (M^{-1} = G G^T + eps I) is the hot path: it owns the explicit
transpose G^T on device (same pattern as G for the symmetric patterns the GNN emits; values
gathered through a permutation computed once), and `apply` runs two bit-exact SpMV kernels.
Inside `pcg_solve` the apply is fused into the iteration kernels instead.  Identity and Jacobi
are supported by the same fused solver (comparison baselines).
"""
from __future__ import annotations

import time
from abc import ABC, abstractmethod

import numpy as np

from . import _lib as L
from .sparse import SparseMatrix, _as_dev_vector

__all__ = ["Preconditioner", "IdentityPreconditioner", "JacobiPreconditioner",
           "LearnedSpaiPreconditioner", "build_identity", "build_jacobi", "build_learned_spai",
           "PRECONDITIONER_NAMES"]

PRECONDITIONER_NAMES = ("none", "diag", "ic0", "fsai", "learned")


class Preconditioner(ABC):
    """SPD linear operator approximating the inverse of the system matrix (precond.py:42-59)."""

    variant: str = "abstract"
    kind: int = -1

    def __init__(self, n: int, t_construct_ns: int = 0):
        self.n = n
        self.t_construct_ns = t_construct_ns

    @abstractmethod
    def apply(self, r):
        """s = M^{-1} r."""

    def _check_dim(self, r):
        import torch
        n = r.shape[0] if isinstance(r, torch.Tensor) else len(np.asarray(r))
        if n != self.n:
            raise ValueError(f"dimension mismatch: operator is {self.n}, vector is {n}")
        return _as_dev_vector(r, self.n)


class IdentityPreconditioner(Preconditioner):
    variant = "none"
    kind = L.PRECOND_IDENTITY

    def apply(self, r):
        rd, was_t = self._check_dim(r)
        return rd.clone() if was_t else rd.cpu().numpy()


class JacobiPreconditioner(Preconditioner):
    variant = "diag"
    kind = L.PRECOND_JACOBI

    def __init__(self, inv_diag, t_construct_ns: int = 0):
        import torch
        inv_diag = np.asarray(inv_diag, dtype=np.float64)
        super().__init__(len(inv_diag), t_construct_ns)
        self.inv_diag = inv_diag
        self.inv_diag_dev = L.to_device(inv_diag, torch.float64)

    def apply(self, r):
        rd, was_t = self._check_dim(r)
        out = rd * self.inv_diag_dev  # elementwise r * inv_diag, as precond.py:79
        return out if was_t else out.cpu().numpy()


class LearnedSpaiPreconditioner(Preconditioner):
    """M^{-1} = G G^T + eps I (precond.py:123-145)."""

    variant = "learned"
    kind = L.PRECOND_LEARNED

    def __init__(self, factor: SparseMatrix, epsilon: float, t_construct_ns: int = 0):
        if epsilon < 0.0:
            raise ValueError("epsilon must be nonnegative")
        super().__init__(factor.n_rows, t_construct_ns)
        if factor.n_rows != factor.n_cols:
            raise ValueError("factor must be square")
        self.factor = factor
        self.epsilon = float(epsilon)
        self._gt = None

    def factor_t(self):
        """Explicit G^T on device (built once)."""
        if self._gt is None:
            self._gt = self.factor.device().transpose()
        return self._gt

    def apply(self, r):
        import torch
        rd, was_t = self._check_dim(r)
        g, gt = self.factor.device(), self.factor_t()
        t = L.empty(self.n, torch.float64)
        s = L.empty(self.n, torch.float64)
        L.check(L.lib().sg_learned_apply(self.n, L.ptr(g.offs), L.ptr(g.cols), L.ptr(g.vals), L.ptr(gt.offs),
                                         L.ptr(gt.cols), L.ptr(gt.vals), self.epsilon, L.ptr(rd), L.ptr(t),
                                         L.ptr(s), L.stream_ptr()))
        return s if was_t else s.cpu().numpy()


def build_identity(A: SparseMatrix) -> IdentityPreconditioner:
    return IdentityPreconditioner(A.n_rows)


def build_jacobi(A: SparseMatrix) -> JacobiPreconditioner:
    """precond.py:152-164: diagonal extracted on device; requires a present, positive diagonal."""
    t0 = time.perf_counter_ns()
    diag_d, present_d = A.diagonal_device()
    d = diag_d.cpu().numpy()
    present = present_d.cpu().numpy().astype(bool)
    if not present.all():
        raise ValueError(f"missing diagonal entry at row {int(np.flatnonzero(~present)[0])}")
    if np.any(d <= 0.0):
        raise ValueError(f"nonpositive diagonal entry at row {int(np.flatnonzero(d <= 0.0)[0])}")
    return JacobiPreconditioner(1.0 / d, t_construct_ns=time.perf_counter_ns() - t0)


def build_learned_spai(factor: SparseMatrix, epsilon: float) -> LearnedSpaiPreconditioner:
    """precond.py:308-312.  Unlike the reference, construction includes building G^T."""
    t0 = time.perf_counter_ns()
    pre = LearnedSpaiPreconditioner(factor, epsilon)
    pre.factor_t()
    pre.t_construct_ns = time.perf_counter_ns() - t0
    return pre


class FsaiPreconditioner(Preconditioner):
    """precond.py:103-120: lower-triangular factor G with G A G^T ~= I; M^{-1} = G^T (G r)."""

    variant = "fsai"
    kind = L.PRECOND_LEARNED  # the fused PCG runs it as a factored M with F = G^T and eps = 0

    def __init__(self, g_lower: SparseMatrix, fallback_rows: int, t_construct_ns: int = 0):
        super().__init__(g_lower.n_rows, t_construct_ns)
        self.g_lower = g_lower
        self.fallback_rows = int(fallback_rows)
        self._ft = None

    def factor_pair(self):
        """(F, F^T) = (G^T, G) as device CSR for the fused PCG kernels."""
        if self._ft is None:
            gl = self.g_lower.device()
            self._ft = (gl.transpose(), gl)
        return self._ft

    def apply(self, r):
        from .sparse import spmv, spmv_transpose
        rd, was_t = self._check_dim(r)
        out = spmv_transpose(self.g_lower, spmv(self.g_lower, rd))
        return out if was_t else out.cpu().numpy()


def build_fsai(A: SparseMatrix) -> FsaiPreconditioner:
    """precond.py:262-305 with the per-row dense solves on the GPU (sg_fsai_build)."""
    import ctypes as C

    import torch
    t0 = time.perf_counter_ns()
    if A.n_rows != A.n_cols:
        raise ValueError("matrix must be square")
    offs, cols = np.asarray(A.row_offsets), np.asarray(A.col_indices)
    rows = np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(offs))
    low = cols <= rows
    l_offs = np.zeros(A.n_rows + 1, dtype=np.int64)
    np.add.at(l_offs, rows[low] + 1, 1)
    np.cumsum(l_offs, out=l_offs)
    l_cols = cols[low]
    last = l_offs[1:] - 1
    bad = np.flatnonzero((np.diff(l_offs) == 0) | (l_cols[np.maximum(last, 0)] != np.arange(A.n_rows)))
    if len(bad):
        raise ValueError(f"missing diagonal entry in row {int(bad[0])}")
    diag_d, _ = A.diagonal_device()
    if bool((diag_d <= 0.0).any()):
        raise ValueError("FSAI requires a positive diagonal")
    a = A.device()
    lo_d = L.to_device(l_offs.astype(np.int32), torch.int32)
    lc_d = L.to_device(l_cols.astype(np.int32), torch.int32)
    lv_d = L.empty(len(l_cols), torch.float64)
    fb = C.c_int64(0)
    L.check(L.lib().sg_fsai_build(A.n_rows, L.ptr(a.offs), L.ptr(a.cols), L.ptr(a.vals), L.ptr(lo_d), L.ptr(lc_d),
                                  L.ptr(lv_d), C.byref(fb), L.stream_ptr()), "fsai_build")
    from .sparse import DeviceCsr
    g_lower = SparseMatrix.from_device(DeviceCsr(A.n_rows, A.n_cols, lo_d, lc_d, lv_d))
    return FsaiPreconditioner(g_lower, fb.value, t_construct_ns=time.perf_counter_ns() - t0)
