"""Scale-invariant SAI loss on the GPU, drop-in for `spaigraph.training.sai_loss` (training.py:41-94).

`sai_loss` returns ||(A (G G^T + eps I) w)/||A|| - w||^2; `sai_loss_and_grad` additionally
returns dL/dg for every stored entry of G — the gradient the reference obtains by recording
the loss on its tape and calling `Tape.backward` (autodiff.py:203-239, 265-303), in the same
rounding order.  The GNN training step follows: training forward, backward
through the restructured GNN, AdamW and `train` (training.py:242-314) with every step on the GPU.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib as L
from .sparse import SparseMatrix, _as_dev_vector, norm_device

__all__ = ["NORM_KINDS", "matrix_norm", "sai_loss", "sai_loss_and_grad", "gnn_train_forward", "gnn_backward",
           "matrix_loss_and_grad", "union_graph", "batch_loss_and_grad", "TrainConfig", "TrainItem", "TrainLog", "TrainingDivergedError", "AdamWDevice",
           "train"]

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


# ------------------------------------------------------------------------------------------------
# GNN training step on the GPU: training forward with every intermediate,
# backward through the restructured GNN, AdamW, and the reference train() loop.
# ------------------------------------------------------------------------------------------------
class _Views:
    """Offsets of every (W, b) of the model inside its flat parameter vector (params_flat order,
    gnn.py:130-136): mlp k -> [(W offset, d_in, d_out, b offset), ...]."""

    def __init__(self, model):
        self.mlps = []
        pos = 0
        for m in model.mlps():
            ent = []
            for W, b in m.weights:
                din, dout = W.shape
                ent.append((pos, din, dout, pos + din * dout))
                pos += din * dout + dout
            self.mlps.append(ent)
        self.n = pos


class _Dev:
    """Device primitive calls (sg_dense_affine & co.) with pointer arithmetic on flat tensors."""

    def __init__(self):
        self.lib = L.lib()
        self._ws = None

    @staticmethod
    def p(t, off=0):
        return C.c_void_p(0 if t is None else t.data_ptr() + 8 * off)

    def affine(self, N, din, dout, x, ldi, W, woff, ldw, out, ldo, b=None, boff=0, add=None, relu=False,
               trans=False):
        L.check(self.lib.sg_dense_affine(N, din, dout, self.p(x), ldi, self.p(W, woff), ldw, 1 if trans else 0,
                                         self.p(b, boff) if b is not None else None,
                                         self.p(add) if add is not None else None, self.p(out), ldo,
                                         1 if relu else 0, L.stream_ptr()), "dense_affine")

    def add_into(self, dst, src):
        """dst = dst + 1.0 * src (sg_axpby)."""
        L.check(self.lib.sg_axpby(self.p(dst), self.p(dst), self.p(src), 1.0, dst.numel(), 0, L.stream_ptr()))

    def relu_grad(self, pre, src, dst):
        L.check(self.lib.sg_relu_grad(pre.numel(), self.p(pre), self.p(src), self.p(dst), L.stream_ptr()))

    def seg(self, n, d, offs, perm, src, dst, acc=False):
        L.check(self.lib.sg_segment_sum(n, d, self.p(offs), self.p(perm) if perm is not None else None,
                                        self.p(src), self.p(dst), 1 if acc else 0, L.stream_ptr()))

    def outer(self, N, da, db, A, lda, B, ldb, out, ooff, acc=True):
        import torch
        need = C.c_size_t(0)
        L.check(self.lib.sg_outer_sum(N, da, db, None, lda, None, ldb, None, 0, None, C.byref(need), None))
        if self._ws is None or self._ws.numel() * 8 < need.value:
            self._ws = L.empty(need.value // 8 + 64, torch.float64)
        L.check(self.lib.sg_outer_sum(N, da, db, self.p(A) if A is not None else None, lda, self.p(B), ldb,
                                      self.p(out, ooff), 1 if acc else 0, self.p(self._ws), C.byref(need),
                                      L.stream_ptr()), "outer_sum")

    def edge_pre(self, E, d, rows, cols, P, Q, ef, crow, crow_off, H, b, boff, pre):
        L.check(self.lib.sg_edge_pre(E, d, self.p(rows), self.p(cols), self.p(P), self.p(Q),
                                     self.p(ef) if ef is not None else None,
                                     self.p(crow, crow_off) if crow is not None else None,
                                     self.p(H) if H is not None else None,
                                     self.p(b, boff) if b is not None else None, self.p(pre),
                                     L.stream_ptr()), "edge_pre")


def _check_trainable(cfg):
    if cfg.mlp_hidden_layers != 1 or cfg.message_uses_hidden_edge or cfg.activation != "relu" or cfg.d_edge != 1:
        raise NotImplementedError("GPU training supports the reference default model (one hidden layer per MLP, "
                                  "relu, d_edge = 1, message_uses_hidden_edge = False)")


def gnn_train_forward(model, graph):
    """The GNN forward (gnn.py:208-253 in the restructured form) keeping every intermediate the
    backward needs.  Returns a dict; `g` is the [nnz] output (equal to `forward` within 1e-12)."""
    import torch
    cfg = model.config
    _check_trainable(cfg)
    dv, V = _Dev(), _Views(model)
    W = model.params_device()
    mat = graph.matrix
    n, E, d, Lc = mat.n_rows, mat.nnz, cfg.hidden_dim, cfg.n_layers
    rows, cols = mat.rows(), mat.cols
    ef = graph.edge_dev
    f64 = torch.float64
    z = lambda *s: torch.empty(*s, dtype=f64, device=L.device())  # noqa: E731
    st = {"n": n, "E": E, "d": d}
    # node encoder: a0 = V W1 + b1, X0 = relu(a0) W2 + b2
    (w1, din, _, b1), (w2, _, _, b2) = V.mlps[0]
    st["a0"] = a0 = z(n, d)
    dv.affine(n, din, d, graph.node_dev, din, W, w1, d, a0, d, W, b1)
    r0 = z(n, d)
    dv.relu_grad(a0, a0, r0)
    X = z(n, d)
    dv.affine(n, d, d, r0, d, W, w2, d, X, d, W, b2)
    st["X"] = [X]
    st["pre_m"], st["S"], st["m"], st["am"] = [], [], [], []
    deg = L.to_device(np.diff(mat.offs[:n + 1].cpu().numpy().astype(np.int64)).astype(np.float64), f64)
    st["deg"] = deg
    for t in range(Lc):
        fm, fv = V.mlps[2 + 3 * t], V.mlps[3 + 3 * t]
        (m1, _, _, mb1), (m2, _, _, mb2) = fm
        Pm, Qm = z(n, d), z(n, d)
        dv.affine(n, d, d, X, d, W, m1, d, Pm, d)
        dv.affine(n, d, d, X, d, W, m1 + d * d, d, Qm, d)
        pre = z(E, d)
        dv.edge_pre(E, d, rows, cols, Pm, Qm, ef, W, m1 + 2 * d * d, None, W, mb1, pre)
        zz = z(E, d)
        dv.relu_grad(pre, pre, zz)
        S = z(n, d)
        dv.seg(n, d, mat.offs, None, zz, S)
        m = z(n, d)
        dv.affine(n, d, d, S, d, W, m2, d, m, d)
        dv.affine(n, 1, d, deg, 1, W, mb2, d, m, d, add=m)  # m = S W2 + deg b2
        (v1, _, _, vb1), (v2, _, _, vb2) = fv
        am = z(n, d)
        dv.affine(n, d, d, m, d, W, v1, d, am, d, W, vb1)
        zm = z(n, d)
        dv.relu_grad(am, am, zm)
        Xn = z(n, d)
        dv.affine(n, d, d, zm, d, W, v2, d, Xn, d, W, vb2, add=X)
        st["pre_m"].append(pre); st["S"].append(S); st["m"].append(m); st["am"].append(am)
        X = Xn
        st["X"].append(X)
    # edge path
    (e1, _, _, eb1), (e2, _, _, eb2) = V.mlps[1]
    ae = z(E, d)
    dv.affine(E, 1, d, ef, 1, W, e1, d, ae, d, W, eb1)
    re = z(E, d)
    dv.relu_grad(ae, ae, re)
    h = z(E, d)
    dv.affine(E, d, d, re, d, W, e2, d, h, d, W, eb2)
    st["ae"], st["h"], st["pre_f"] = ae, [h], []
    for t in range(Lc):
        fe = V.mlps[4 + 3 * t]
        (f1, _, _, fb1), (f2, _, _, fb2) = fe
        Xt = st["X"][t + 1]
        Pf, Qf, Hw = z(n, d), z(n, d), z(E, d)
        dv.affine(n, d, d, Xt, d, W, f1, d, Pf, d)
        dv.affine(n, d, d, Xt, d, W, f1 + d * d, d, Qf, d)
        dv.affine(E, d, d, h, d, W, f1 + 2 * d * d, d, Hw, d)
        pre = z(E, d)
        dv.edge_pre(E, d, rows, cols, Pf, Qf, None, None, 0, Hw, W, fb1, pre)
        rf = z(E, d)
        dv.relu_grad(pre, pre, rf)
        hn = z(E, d)
        dv.affine(E, d, d, rf, d, W, f2, d, hn, d, W, fb2, add=h)
        st["pre_f"].append(pre)
        h = hn
        st["h"].append(h)
    (d1, _, _, db1), (d2, _, _, db2) = V.mlps[-1]
    ad = z(E, d)
    dv.affine(E, d, d, h, d, W, d1, d, ad, d, W, db1)
    rd = z(E, d)
    dv.relu_grad(ad, ad, rd)
    g = z(E)
    dv.affine(E, d, 1, rd, d, W, d2, 1, g, 1, W, db2)
    st["ad"], st["g"] = ad, g
    return st


def gnn_backward(model, graph, st, dg):
    """dL/dθ (params_flat order) from dL/dg through the restructured GNN (reverse of
    gnn_train_forward).  Column (gather-by-j) sums run over the transposed pattern in ascending
    source row, i.e. the tape's np.add.at order."""
    import torch
    cfg = model.config
    dv, V = _Dev(), _Views(model)
    W = model.params_device()
    mat = graph.matrix
    n, E, d, Lc = st["n"], st["E"], st["d"], cfg.n_layers
    rows, cols = mat.rows(), mat.cols
    offs_t, _, perm = mat.transpose_pattern()
    ef = graph.edge_dev
    f64 = torch.float64
    z = lambda *s: torch.empty(*s, dtype=f64, device=L.device())  # noqa: E731
    grad = torch.zeros(V.n + 2, dtype=f64, device=L.device())[:V.n]
    dg = dg if isinstance(dg, torch.Tensor) else L.to_device(np.asarray(dg, dtype=np.float64), f64)
    dg = dg[:E].reshape(E, 1)
    # decoder
    (d1, _, _, db1), (d2, _, _, db2) = V.mlps[-1]
    ad = st["ad"]
    rd = z(E, d)
    dv.relu_grad(ad, ad, rd)
    dv.outer(E, d, 1, rd, d, dg, 1, grad, d2)           # dW2 = relu(ad)^T dg
    dv.outer(E, 1, 1, None, 1, dg, 1, grad, db2)        # db2 = sum dg
    dz = z(E, d)
    dv.affine(E, 1, d, dg, 1, W, d2, 1, dz, d, trans=True)  # dg W2^T
    dv.relu_grad(ad, dz, dz)
    hL = st["h"][-1]
    dv.outer(E, d, d, hL, d, dz, d, grad, d1)
    dv.outer(E, 1, d, None, 1, dz, d, grad, db1)
    dh = z(E, d)
    dv.affine(E, d, d, dz, d, W, d1, d, dh, d, trans=True)
    dX = [z(n, d).zero_() for _ in range(Lc + 1)]
    zero_n = z(n, d).zero_()
    # edge layers, reverse
    for t in reversed(range(Lc)):
        fe = V.mlps[4 + 3 * t]
        (f1, _, _, fb1), (f2, _, _, fb2) = fe
        pre, h_t, Xt = st["pre_f"][t], st["h"][t], st["X"][t + 1]
        rf = z(E, d)
        dv.relu_grad(pre, pre, rf)
        dv.outer(E, d, d, rf, d, dh, d, grad, f2)
        dv.outer(E, 1, d, None, 1, dh, d, grad, fb2)
        dp = z(E, d)
        dv.affine(E, d, d, dh, d, W, f2, d, dp, d, trans=True)
        dv.relu_grad(pre, dp, dp)
        dv.outer(E, d, d, h_t, d, dp, d, grad, f1 + 2 * d * d)
        dv.outer(E, 1, d, None, 1, dp, d, grad, fb1)
        dPf, dQf = z(n, d), z(n, d)
        dv.seg(n, d, mat.offs, None, dp, dPf)
        dv.seg(n, d, offs_t, perm, dp, dQf)
        dv.outer(n, d, d, Xt, d, dPf, d, grad, f1)
        dv.outer(n, d, d, Xt, d, dQf, d, grad, f1 + d * d)
        dv.affine(n, d, d, dPf, d, W, f1, d, dX[t + 1], d, trans=True, add=dX[t + 1])
        dv.affine(n, d, d, dQf, d, W, f1 + d * d, d, dX[t + 1], d, trans=True, add=dX[t + 1])
        dhn = z(E, d)
        dv.affine(E, d, d, dp, d, W, f1 + 2 * d * d, d, dhn, d, trans=True, add=dh)
        dh = dhn
    # edge encoder
    (e1, _, _, eb1), (e2, _, _, eb2) = V.mlps[1]
    ae = st["ae"]
    re = z(E, d)
    dv.relu_grad(ae, ae, re)
    dv.outer(E, d, d, re, d, dh, d, grad, e2)
    dv.outer(E, 1, d, None, 1, dh, d, grad, eb2)
    da = z(E, d)
    dv.affine(E, d, d, dh, d, W, e2, d, da, d, trans=True)
    dv.relu_grad(ae, da, da)
    dv.outer(E, 1, d, ef.reshape(E, 1), 1, da, d, grad, e1)
    dv.outer(E, 1, d, None, 1, da, d, grad, eb1)
    # node layers, reverse
    deg = st["deg"]
    for t in reversed(range(Lc)):
        fm, fv = V.mlps[2 + 3 * t], V.mlps[3 + 3 * t]
        (m1, _, _, mb1), (m2, _, _, mb2) = fm
        (v1, _, _, vb1), (v2, _, _, vb2) = fv
        dXn, Xt = dX[t + 1], st["X"][t]
        pre, S, m, am = st["pre_m"][t], st["S"][t], st["m"][t], st["am"][t]
        dv.add_into(dX[t], dXn)                                # residual
        zm = z(n, d)
        dv.relu_grad(am, am, zm)
        dv.outer(n, d, d, zm, d, dXn, d, grad, v2)
        dv.outer(n, 1, d, None, 1, dXn, d, grad, vb2)
        dam = z(n, d)
        dv.affine(n, d, d, dXn, d, W, v2, d, dam, d, trans=True)
        dv.relu_grad(am, dam, dam)
        dv.outer(n, d, d, m, d, dam, d, grad, v1)
        dv.outer(n, 1, d, None, 1, dam, d, grad, vb1)
        dm = z(n, d)
        dv.affine(n, d, d, dam, d, W, v1, d, dm, d, trans=True)
        dv.outer(n, d, d, S, d, dm, d, grad, m2)
        dv.outer(n, 1, d, deg, 1, dm, d, grad, mb2)            # m = S W2 + deg b2
        dS = z(n, d)
        dv.affine(n, d, d, dm, d, W, m2, d, dS, d, trans=True)
        # dpre_e = dS[row_e] * [pre_e > 0]
        dpre = z(E, d)
        dv.edge_pre(E, d, rows, cols, dS, zero_n, None, None, 0, None, None, 0, dpre)
        dv.relu_grad(pre, dpre, dpre)
        dv.outer(E, 1, d, None, 1, dpre, d, grad, mb1)
        dv.outer(E, 1, d, ef.reshape(E, 1), 1, dpre, d, grad, m1 + 2 * d * d)  # edge-feature row c
        dP, dQ = z(n, d), z(n, d)
        dv.seg(n, d, mat.offs, None, dpre, dP)
        dv.seg(n, d, offs_t, perm, dpre, dQ)
        dv.outer(n, d, d, Xt, d, dP, d, grad, m1)
        dv.outer(n, d, d, Xt, d, dQ, d, grad, m1 + d * d)
        dv.affine(n, d, d, dP, d, W, m1, d, dX[t], d, trans=True, add=dX[t])
        dv.affine(n, d, d, dQ, d, W, m1 + d * d, d, dX[t], d, trans=True, add=dX[t])
    # node encoder
    (w1, din, _, b1), (w2, _, _, b2) = V.mlps[0]
    a0 = st["a0"]
    r0 = z(n, d)
    dv.relu_grad(a0, a0, r0)
    dv.outer(n, d, d, r0, d, dX[0], d, grad, w2)
    dv.outer(n, 1, d, None, 1, dX[0], d, grad, b2)
    da0 = z(n, d)
    dv.affine(n, d, d, dX[0], d, W, w2, d, da0, d, trans=True)
    dv.relu_grad(a0, da0, da0)
    dv.outer(n, din, d, graph.node_dev.reshape(n, din), din, da0, d, grad, w1)
    dv.outer(n, 1, d, None, 1, da0, d, grad, b1)
    return grad


def matrix_loss_and_grad(model, A: SparseMatrix, graph, rng, n_samples: int = 1,
                         norm_kind: str = "mean_abs_nonzero"):
    """training.py:_matrix_loss_and_grad on the GPU: forward, the mean SAI loss over
    `n_samples` fresh Hutchinson probes drawn from `rng` (same draws as the reference), and
    dL/dθ (device tensor, params_flat order)."""
    st = gnn_train_forward(model, graph)
    mat = graph.matrix
    G = SparseMatrix.from_device(mat.with_values(st["g"]))
    losses, dg = [], None
    for _ in range(n_samples):
        w = rng.standard_normal(A.n_rows)
        loss, g = _loss(A, G, model.config.epsilon, w, norm_kind, True)
        losses.append(loss)
        import torch
        gd = g if isinstance(g, torch.Tensor) else L.to_device(g, torch.float64)
        dg = gd if dg is None else dg + gd
    total = losses[0]
    for lv in losses[1:]:
        total = total + lv
    mean_loss = total * (1.0 / n_samples)
    if n_samples > 1:
        dg = dg * (1.0 / n_samples)
    return mean_loss, gnn_backward(model, graph, st, dg)


def union_graph(graphs):
    """Block-diagonal union of MatrixGraphs (one GNN pass for a whole minibatch)."""
    import torch
    from .graphfeat import MatrixGraph
    from .sparse import DeviceCsr
    offs_parts, cols_parts, node_parts, edge_parts = [], [], [], []
    n0 = e0 = 0
    for g in graphs:
        m = g.matrix
        offs_parts.append(m.offs[:m.n_rows].to(torch.int64) + e0)
        cols_parts.append(m.cols[:m.nnz].to(torch.int64) + n0)
        node_parts.append(g.node_dev[:m.n_rows * g.d_node])
        edge_parts.append(g.edge_dev[:m.nnz])
        n0 += m.n_rows
        e0 += m.nnz
    dev = L.device()
    offs = torch.cat(offs_parts + [torch.tensor([e0], dtype=torch.int64, device=dev)]).to(torch.int32)
    cols = torch.cat(cols_parts).to(torch.int32)
    mat = DeviceCsr(n0, n0, offs, cols, torch.zeros(e0, dtype=torch.float64, device=dev))
    return MatrixGraph(n0, matrix=mat, node_dev=torch.cat(node_parts), edge_dev=torch.cat(edge_parts),
                       norm_dev=None)


def batch_loss_and_grad(model, items, rng, n_samples: int = 1, norm_kind: str = "mean_abs_nonzero"):
    """The minibatch's losses and the SUM of their gradients with ONE training forward and ONE
    backward over the union graph (probes drawn per matrix in batch order, as the reference)."""
    import torch
    ug = union_graph([it.graph for it in items])
    st = gnn_train_forward(model, ug)
    g_all = st["g"]
    losses, dgs = [], []
    e0 = 0
    for it in items:
        mat = it.graph.matrix
        G = SparseMatrix.from_device(mat.with_values(g_all[e0:e0 + mat.nnz].contiguous()))
        ls, dg = [], None
        for _ in range(n_samples):
            w = rng.standard_normal(it.A.n_rows)
            loss, g = _loss(it.A, G, model.config.epsilon, w, norm_kind, True)
            ls.append(loss)
            gd = g if isinstance(g, torch.Tensor) else L.to_device(g, torch.float64)
            dg = gd if dg is None else dg + gd
        total = ls[0]
        for lv in ls[1:]:
            total = total + lv
        losses.append(total * (1.0 / n_samples))
        dgs.append(dg * (1.0 / n_samples) if n_samples > 1 else dg)
        e0 += mat.nnz
    return losses, gnn_backward(model, ug, st, torch.cat(dgs))


# ------------------------------------------------------------------------------------------------
# training.py:150-314 — TrainConfig / TrainItem / AdamW / train() with the step on the GPU
# ------------------------------------------------------------------------------------------------
from dataclasses import dataclass, field  # noqa: E402


@dataclass(frozen=True)
class TrainConfig:
    """training.py:150-171."""

    epochs: int = 500
    batch_size: int = 4
    lr: float = 1e-3
    weight_decay: float = 1e-2
    lr_decay: float = 0.99
    hutchinson_samples_per_matrix: int = 1
    seed: int = 0
    norm_kind: str = "mean_abs_nonzero"
    val_every: int = 50
    checkpoint_every: int = 0

    def __post_init__(self):
        if min(self.epochs, self.batch_size, self.hutchinson_samples_per_matrix) < 1:
            raise ValueError("epochs, batch size, and sample counts must be positive")
        if self.lr <= 0 or self.weight_decay < 0:
            raise ValueError("lr must be positive and weight decay nonnegative")
        if not 0.0 < self.lr_decay <= 1.0:
            raise ValueError("lr_decay must lie in (0, 1]")
        if self.norm_kind not in NORM_KINDS:
            raise ValueError(f"unknown norm kind {self.norm_kind!r}")


@dataclass
class TrainItem:
    """training.py:174-178."""

    A: SparseMatrix
    graph: object
    b: np.ndarray | None = None


class TrainingDivergedError(RuntimeError):
    """training.py:181-189."""

    def __init__(self, epoch: int, loss: float, checkpoint_path):
        msg = f"non-finite loss {loss} at epoch {epoch}"
        if checkpoint_path is not None:
            msg += f"; last good parameters saved to {checkpoint_path}"
        super().__init__(msg)
        self.epoch = epoch
        self.loss = loss


@dataclass
class TrainLog:
    """training.py:192-197: rows of (epoch, mean_loss, lr, wallclock_s, val_mean_k)."""

    rows: list = field(default_factory=list)

    def losses(self):
        return np.array([r[1] for r in self.rows])


class AdamWDevice:
    """adamw_step (training.py:126-147) on device: parameters and both moments stay resident."""

    def __init__(self, params_dev, beta1=0.9, beta2=0.999, eps=1e-8):
        import torch
        n = params_dev.numel()
        self.p = params_dev
        self.m = torch.zeros(n, dtype=torch.float64, device=params_dev.device)
        self.v = torch.zeros(n, dtype=torch.float64, device=params_dev.device)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps

    def step(self, grad_sum, t: int, lr: float, weight_decay: float, batch_len: int):
        L.check(L.lib().sg_adamw(self.p.numel(), L.ptr(self.p), L.ptr(grad_sum), L.ptr(self.m), L.ptr(self.v),
                                 float(lr), float(weight_decay), self.beta1, self.beta2, self.eps, int(t),
                                 float(batch_len), L.stream_ptr()), "adamw")


def _validation_mean_k(model, val_items) -> float:
    """training.py:229-239 (learned SPAI + PCG on the GPU)."""
    from .gnn import forward
    from .pcg import SolveConfig, pcg_solve
    from .precond import build_learned_spai
    ks = []
    cfg = SolveConfig(rtol=1e-8)
    for item in val_items:
        G = forward(model, item.graph).G
        b = item.b if item.b is not None else np.ones(item.A.n_rows) / math.sqrt(item.A.n_rows)
        ks.append(pcg_solve(item.A, b, build_learned_spai(G, model.config.epsilon), cfg).k)
    return float(np.mean(ks))


def train(model, train_items, cfg: TrainConfig, val_items=(), log_path=None, checkpoint_path=None,
          batched: bool = False) -> TrainLog:
    """training.py:242-314 with forward, loss, backward and AdamW on the GPU.  Same seeded
    shuffles and probes (one host PCG64 stream), same batch averaging, lr decay, divergence
    handling, CSV log and checkpoints.  batched=True runs each minibatch as ONE union graph
    (one forward, one backward; the gradient sum is then reduced in a different order than the
    reference's per-matrix accumulation, so trajectories agree to rounding, not bit for bit)."""
    import csv
    import time
    import torch
    from .gnn import save_checkpoint
    train_items = list(train_items)
    if not train_items:
        raise ValueError("empty training set")
    rng = np.random.default_rng(cfg.seed)
    params = L.to_device(model.params_flat(), torch.float64).clone()
    opt = AdamWDevice(params)
    lr = cfg.lr
    t = 0
    log = TrainLog()
    fh = writer = None
    if log_path is not None:
        fh = open(log_path, "w", newline="")
        writer = csv.writer(fh)
        writer.writerow(["epoch", "mean_loss", "lr", "wallclock_s", "val_mean_k"])
    t0 = time.perf_counter()
    last_good = model.params_flat().copy()
    grad_sum = torch.zeros_like(params)
    try:
        for epoch in range(1, cfg.epochs + 1):
            order = rng.permutation(len(train_items))
            epoch_losses = []
            for start in range(0, len(order), cfg.batch_size):
                batch = order[start:start + cfg.batch_size]
                grad_sum.zero_()

                def diverged(loss_val):
                    if checkpoint_path is not None:
                        model.set_params_flat(last_good)
                        save_checkpoint(model, checkpoint_path)
                    raise TrainingDivergedError(epoch, loss_val, checkpoint_path)

                if batched:
                    losses, grad = batch_loss_and_grad(model, [train_items[i] for i in batch], rng,
                                                       cfg.hutchinson_samples_per_matrix, cfg.norm_kind)
                    for loss_val in losses:
                        if not math.isfinite(loss_val):
                            diverged(loss_val)
                        epoch_losses.append(loss_val)
                    L.check(L.lib().sg_axpby(L.ptr(grad_sum), L.ptr(grad_sum), L.ptr(grad), 1.0, grad.numel(), 0,
                                             L.stream_ptr()))
                else:
                    for idx in batch:
                        item = train_items[idx]
                        loss_val, grad = matrix_loss_and_grad(model, item.A, item.graph, rng,
                                                              cfg.hutchinson_samples_per_matrix, cfg.norm_kind)
                        if not math.isfinite(loss_val):
                            diverged(loss_val)
                        epoch_losses.append(loss_val)
                        L.check(L.lib().sg_axpby(L.ptr(grad_sum), L.ptr(grad_sum), L.ptr(grad), 1.0,
                                                 grad.numel(), 0, L.stream_ptr()))
                t += 1
                opt.step(grad_sum, t, lr, cfg.weight_decay, len(batch))
                model.set_params_flat(params.cpu().numpy())
            val_k = ""
            if val_items and cfg.val_every > 0 and (epoch % cfg.val_every == 0 or epoch == cfg.epochs):
                val_k = _validation_mean_k(model, val_items)
            row = (epoch, float(np.mean(epoch_losses)), lr, time.perf_counter() - t0, val_k)
            log.rows.append(row)
            if writer is not None:
                writer.writerow(row)
                fh.flush()
            if checkpoint_path is not None and cfg.checkpoint_every > 0 and epoch % cfg.checkpoint_every == 0:
                save_checkpoint(model, checkpoint_path)
            last_good = model.params_flat().copy()
            lr *= cfg.lr_decay
    finally:
        if fh is not None:
            fh.close()
    if checkpoint_path is not None:
        save_checkpoint(model, checkpoint_path)
    return log
