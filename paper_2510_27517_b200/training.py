"""Scale-invariant SAI loss on the GPU, drop-in for `spaigraph.training.sai_loss` (training.py:41-94).

`sai_loss` returns ||(A (G G^T + eps I) w)/||A|| - w||^2; `sai_loss_and_grad` additionally
returns dL/dg for every stored entry of G — the gradient the reference obtains by recording
the loss on its tape and calling `Tape.backward` (autodiff.py:203-239, 265-303), in the same
rounding order.  The training loop itself (AdamW, GNN backward) is SURVEY.md §8(f) "next".
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib as L
from .sparse import SparseMatrix, _as_dev_vector, norm_device

__all__ = ["NORM_KINDS", "matrix_norm", "sai_loss", "sai_loss_and_grad"]

NORM_KINDS = ("mean_abs_nonzero", "frobenius", "entrywise_l1")


def matrix_norm(A: SparseMatrix, kind: str = "mean_abs_nonzero") -> float:
    """training.py:44-54 (exact summation on device, bit-identical to math.fsum)."""
    if A.nnz == 0:
        raise ValueError("norm of a matrix with no stored entries")
    if kind not in NORM_KINDS:
        raise ValueError(f"unknown norm kind {kind!r}, expected one of {NORM_KINDS}")
    return float(norm_device(A.device().vals, A.nnz, NORM_KINDS.index(kind)).item())


def _loss(A: SparseMatrix, G: SparseMatrix, epsilon: float, w, norm_kind: str, with_grad: bool):
    import torch
    if norm_kind not in NORM_KINDS:
        raise ValueError(f"unknown norm kind {norm_kind!r}, expected one of {NORM_KINDS}")
    n = A.n_rows
    wn = w.shape[0] if isinstance(w, torch.Tensor) else len(np.asarray(w))
    if wn != n:
        raise ValueError(f"probe vector has length {wn}, matrix is {n}")
    if A.nnz == 0:
        raise ValueError("matrix norm is zero")
    wd, was_t = _as_dev_vector(w, n, "probe vector")
    a, g = A.device(), G.device()
    at, gt = a.transpose(), g.transpose()
    grad = L.empty(g.nnz, torch.float64) if with_grad else None
    loss = C.c_double(0.0)
    args = (n, L.ptr(a.offs), L.ptr(a.cols), L.ptr(a.vals), L.ptr(at.offs), L.ptr(at.cols), L.ptr(at.vals),
            L.ptr(g.offs), L.ptr(g.cols), L.ptr(g.vals), L.ptr(gt.offs), L.ptr(gt.cols), L.ptr(gt.vals),
            L.ptr(g.rows()), float(epsilon), L.ptr(wd), NORM_KINDS.index(norm_kind), C.byref(loss), L.ptr(grad))
    L.call_ws(L.lib().sg_sai_loss, *args, what="sai_loss")
    if not with_grad:
        return float(loss.value)
    return float(loss.value), (grad if was_t else grad.cpu().numpy())


def sai_loss(A: SparseMatrix, G: SparseMatrix, epsilon: float, w, norm_kind: str = "mean_abs_nonzero") -> float:
    """training.py:84-94."""
    return _loss(A, G, epsilon, w, norm_kind, False)


def sai_loss_and_grad(A: SparseMatrix, G: SparseMatrix, epsilon: float, w,
                      norm_kind: str = "mean_abs_nonzero"):
    """(loss, dL/dg) == sai_loss_on_tape(...) + Tape.backward(...) w.r.t. a leaf holding G.values."""
    return _loss(A, G, epsilon, w, norm_kind, True)


def hutchinson_frobenius_estimate(A: SparseMatrix, m_apply, n_samples: int, seed: int = 0) -> float:
    """training.py:97-113 with the products on device (m_apply: numpy -> numpy)."""
    from .sparse import spmv
    if n_samples < 1:
        raise ValueError("need at least one sample")
    rng = np.random.default_rng(seed)
    samples = []
    for _ in range(n_samples):
        w = rng.standard_normal(A.n_rows)
        z = spmv(A, m_apply(w)) - w
        samples.append(float(z @ z))
    return math.fsum(samples) / n_samples
