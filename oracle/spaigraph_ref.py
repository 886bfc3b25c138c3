"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference `spaigraph` hot path.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/spaigraph/).  The restatement works on plain arrays (CSR triples),
not on the reference dataclasses, and never records a tape, so it runs at sizes the
reference `forward()` cannot.

Pinned against the reference itself: see tests/golden/make_golden.py (generator, runs the
reference in the build container) and tests/test_oracle.py (checks).  Not importable from the
product package.
"""
from __future__ import annotations

import math

import numpy as np

# ----------------------------------------------------------------------------------------------
# L1 sparse core  (sparse.py)
# ----------------------------------------------------------------------------------------------


class StructureError(ValueError):
    pass


def validate_csr(n_rows, n_cols, offs, cols):
    """sparse.py:27-43 (_validate_structure)."""
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if offs.ndim != 1 or len(offs) != n_rows + 1:
        raise StructureError("row_offsets must have length n_rows + 1")
    if offs[0] != 0:
        raise StructureError("row_offsets[0] must be 0")
    if offs[-1] != len(cols):
        raise StructureError("row_offsets[-1] must equal nnz")
    if np.any(np.diff(offs) < 0):
        raise StructureError("row_offsets must be nondecreasing")
    if len(cols):
        if cols.min() < 0 or cols.max() >= n_cols:
            raise StructureError("column index out of range")
        same = np.repeat(np.arange(n_rows), np.diff(offs))
        interior = np.flatnonzero(same[1:] == same[:-1])
        if np.any(cols[interior + 1] <= cols[interior]):
            raise StructureError("col_indices must be strictly increasing within each row")


def row_expand(offs):
    """sparse.py:64-66."""
    offs = np.asarray(offs, dtype=np.int64)
    return np.repeat(np.arange(len(offs) - 1, dtype=np.int64), np.diff(offs))


def csr_from_coo(n_rows, n_cols, rows, cols, vals):
    """sparse.py:138-158 (SparseMatrix.from_coo): lexsort (row, col), reject duplicates."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if not (len(rows) == len(cols) == len(vals)):
        raise StructureError("coordinate arrays must have equal length")
    if len(rows) and (rows.min() < 0 or rows.max() >= n_rows):
        raise StructureError("row index out of range")
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if len(rows) > 1:
        dup = (rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])
        if np.any(dup):
            k = int(np.flatnonzero(dup)[0])
            raise StructureError(f"duplicate entry at ({rows[k]}, {cols[k]})")
    offs = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(offs, rows + 1, 1)
    np.cumsum(offs, out=offs)
    validate_csr(n_rows, n_cols, offs, cols)
    return offs, cols, vals


def transpose(n_rows, n_cols, offs, cols, vals):
    """sparse.py:129-136.  Also returns perm with vals_t == vals[perm]."""
    rows = row_expand(offs)
    cols = np.asarray(cols, dtype=np.int64)
    order = np.lexsort((rows, cols))
    offs_t = np.zeros(n_cols + 1, dtype=np.int64)
    np.add.at(offs_t, cols[order] + 1, 1)
    np.cumsum(offs_t, out=offs_t)
    return offs_t, rows[order], np.asarray(vals)[order], order


def is_symmetric_pattern(n_rows, n_cols, offs, cols):
    """sparse.py:68-78."""
    if n_rows != n_cols:
        return False
    rows = row_expand(offs)
    cols = np.asarray(cols, dtype=np.int64)
    fwd = np.lexsort((cols, rows))
    bwd = np.lexsort((rows, cols))
    return bool(np.array_equal(rows[fwd], cols[bwd]) and np.array_equal(cols[fwd], rows[bwd]))


def segment_sums(contrib, offs):
    """sparse.py:175-183 (_segment_sums: np.add.reduceat over nonempty rows).

    The output is float64 even for longdouble contributions (the reference assigns into a
    float64 array), so autodiff.py:288's row sums are rounded to double.
    """
    offs = np.asarray(offs, dtype=np.int64)
    n = len(offs) - 1
    out = np.zeros((n,) + contrib.shape[1:], dtype=np.float64)
    starts = offs[:-1]
    nonempty = offs[1:] > starts
    if np.any(nonempty):
        out[nonempty] = np.add.reduceat(contrib, starts[nonempty], axis=0)
    return out


def _pairwise(v, lo, n):
    """numpy's pairwise_sum (umath loops_utils) for n elements of v starting at lo."""
    if n < 8:
        s = 0.0
        for i in range(n):
            s = s + v[lo + i]
        return s
    if n <= 128:
        r = [v[lo + j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = r[j] + v[lo + i + j]
            i += 8
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            s = s + v[lo + i]
            i += 1
        return s
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(v, lo, n2) + _pairwise(v, lo + n2, n - n2)


def reduceat_order_sum(v):
    """Scalar emulation of np.add.reduceat on one segment: v[0] + pairwise(v[1:]).

    SURVEY.md A.3 (numpy 2.3.5).  This is the order the GPU parity SpMV implements
    (paper_2510_27517_b200/csrc/spmv.cuh:row_sum_numpy); tests pin it against numpy.
    """
    v = [float(t) for t in v]
    if not v:
        return 0.0
    return v[0] + _pairwise(v, 1, len(v) - 1)


def spmv(offs, cols, vals, x):
    """sparse.py:186-191: reduceat of vals * x[cols] (product rounded, then summed)."""
    x = np.asarray(x, dtype=np.float64)
    return segment_sums(np.asarray(vals) * x[np.asarray(cols)], offs)


def spmv_transpose(n_cols, offs, cols, vals, x):
    """sparse.py:194-201: np.add.at in storage order, starting from 0.0."""
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros(n_cols)
    np.add.at(y, np.asarray(cols), np.asarray(vals) * x[row_expand(offs)])
    return y


def spmv_transpose_explicit(n_cols, offs_t, cols_t, vals_t, x):
    """sparse.py:194-201 evaluated over an explicit transpose (offs_t, cols_t, vals_t from
    `transpose`): np.add.at visits entries in storage order, so y_j accumulates its products in
    ascending original row order starting from 0.0 -- exactly a left-to-right sum along row j of
    the transpose.  Vectorised over rows one position at a time (each step is the same single
    rounding per element), bit-identical to `spmv_transpose` and much faster at C5 size."""
    offs_t = np.asarray(offs_t, dtype=np.int64)
    x = np.asarray(x, dtype=np.float64)
    lens = np.diff(offs_t)
    y = np.zeros(n_cols)
    for p in range(int(lens.max()) if len(lens) else 0):
        rows = np.flatnonzero(lens > p)
        k = offs_t[rows] + p
        y[rows] = y[rows] + np.asarray(vals_t)[k] * x[np.asarray(cols_t)[k]]
    return y


def mean_abs_nonzero_norm(vals):
    """sparse.py:204-213: fsum(|v|)/nnz, correctly rounded sum."""
    vals = np.asarray(vals, dtype=np.float64)
    if len(vals) == 0:
        raise StructureError("norm of a matrix with no stored entries")
    return math.fsum(np.abs(vals)) / len(vals)


def matrix_norm(vals, kind="mean_abs_nonzero"):
    """training.py:44-54."""
    vals = np.asarray(vals, dtype=np.float64)
    if len(vals) == 0:
        raise StructureError("norm of a matrix with no stored entries")
    if kind == "mean_abs_nonzero":
        return mean_abs_nonzero_norm(vals)
    if kind == "frobenius":
        return math.sqrt(math.fsum((vals * vals).tolist()))
    if kind == "entrywise_l1":
        return math.fsum(np.abs(vals).tolist())
    raise ValueError(kind)


def diagonal(n, offs, cols, vals):
    """sparse.py:119-127."""
    d = np.zeros(n)
    rows = row_expand(offs)
    mask = rows == np.asarray(cols)
    d[rows[mask]] = np.asarray(vals)[mask]
    return d


def pattern_square(n, offs, cols):
    """SURVEY.md §8(a) a5 (no reference function; the paper lists two-hop patterns as future
    work): the STRUCTURAL pattern of |A| |A| — (i, j) is stored iff some k has
    (i, k) and (k, j) stored.  Restated with scipy on an all-ones copy (no cancellation),
    sorted indices."""
    import scipy.sparse as sp
    offs = np.asarray(offs, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    B = sp.csr_matrix((np.ones(len(cols)), cols, offs), shape=(n, n))
    P = (B @ B).tocsr()
    P.sort_indices()
    return P.indptr.astype(np.int64), P.indices.astype(np.int64)


def pad_to_pattern(offs, cols, vals, p_offs, p_cols):
    """A's values scattered onto a superset pattern, explicit zeros elsewhere."""
    n = len(offs) - 1
    out = np.zeros(len(p_cols))
    rows = row_expand(offs)
    prow = row_expand(p_offs)
    key_p = prow * n + np.asarray(p_cols)
    key_a = rows * n + np.asarray(cols)
    pos = np.searchsorted(key_p, key_a)
    assert np.array_equal(key_p[pos], key_a), "pattern does not contain A"
    out[pos] = vals
    return out


# ----------------------------------------------------------------------------------------------
# L6 generators  (datasets.py) + the new 3-D generator of SURVEY.md §8(d) C3
# ----------------------------------------------------------------------------------------------

COEFF_LO, COEFF_HI = 1e-4, 5e-4


def poisson2d_coeff(nx, ny, coeff_seed):
    """datasets.py:100-106."""
    n = nx * ny
    if coeff_seed is None:
        return np.ones(n)
    rng = np.random.default_rng(coeff_seed)
    return np.exp(rng.uniform(math.log(COEFF_LO), math.log(COEFF_HI), size=n))


def gen_poisson2d(nx, ny, coeff_seed=None):
    """datasets.py:87-145.  Returns (offs, cols, vals, coeff)."""
    n = nx * ny
    coeff = poisson2d_coeff(nx, ny, coeff_seed)
    a = coeff.reshape(ny, nx)
    ihx2, ihy2 = float((nx + 1) ** 2), float((ny + 1) ** 2)
    west = a.copy(); west[:, 1:] = 0.5 * (a[:, 1:] + a[:, :-1])
    east = a.copy(); east[:, :-1] = 0.5 * (a[:, :-1] + a[:, 1:])
    south = a.copy(); south[1:, :] = 0.5 * (a[1:, :] + a[:-1, :])
    north = a.copy(); north[:-1, :] = 0.5 * (a[:-1, :] + a[1:, :])
    diag = (west + east) * ihx2 + (south + north) * ihy2
    idx = np.arange(n).reshape(ny, nx)
    rows = [idx.ravel(), idx[:, 1:].ravel(), idx[:, :-1].ravel(), idx[1:, :].ravel(), idx[:-1, :].ravel()]
    cols = [idx.ravel(), idx[:, :-1].ravel(), idx[:, 1:].ravel(), idx[:-1, :].ravel(), idx[1:, :].ravel()]
    vals = [diag.ravel(), (-west[:, 1:] * ihx2).ravel(), (-east[:, :-1] * ihx2).ravel(),
            (-south[1:, :] * ihy2).ravel(), (-north[:-1, :] * ihy2).ravel()]
    offs, c, v = csr_from_coo(n, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    return offs, c, v, coeff


def gen_poisson3d(nx, ny, nz):
    """NEW: 7-point -Laplace on the unit cube, Dirichlet walls.

    diag = 2(1/hx^2 + 1/hy^2 + 1/hz^2) evaluated as ((2*ihx2 + 2*ihy2) + 2*ihz2); off-diagonals
    -1/h^2; h = 1/(n+1); idx = ix + nx*(iy + ny*iz).  No reference generator exists, so this
    definition is the pin (tests/test_oracle.py checks it against an entry-by-entry build).
    """
    n = nx * ny * nz
    ihx2, ihy2, ihz2 = float((nx + 1) ** 2), float((ny + 1) ** 2), float((nz + 1) ** 2)
    diag_v = (2.0 * ihx2 + 2.0 * ihy2) + 2.0 * ihz2
    idx = np.arange(n).reshape(nz, ny, nx)
    rows = [idx.ravel()]
    cols = [idx.ravel()]
    vals = [np.full(n, diag_v)]
    for axis, ih in ((2, ihx2), (1, ihy2), (0, ihz2)):
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[axis] = slice(1, None)
        hi[axis] = slice(None, -1)
        a, b = idx[tuple(lo)].ravel(), idx[tuple(hi)].ravel()
        rows += [a, b]
        cols += [b, a]
        vals += [np.full(len(a), -ih), np.full(len(b), -ih)]
    offs, c, v = csr_from_coo(n, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    return offs, c, v


def gen_rhs(n, seed):
    """datasets.py:209-212."""
    b = np.random.default_rng(seed).standard_normal(n)
    return b / np.linalg.norm(b)


def rand_spd_sparse(n, rng, extra_per_row=3):
    """verify.py:39-61 (config-4 generator)."""
    entries = {}
    for _ in range(extra_per_row * n):
        i = int(rng.integers(n))
        j = int(rng.integers(n))
        if i == j:
            continue
        v = float(rng.uniform(-1.0, 1.0))
        entries[(i, j)] = v
        entries[(j, i)] = v
    row_abs = np.zeros(n)
    for (i, _), v in entries.items():
        row_abs[i] += abs(v)
    for i in range(n):
        entries[(i, i)] = row_abs[i] + 1.0 + float(rng.uniform(0.0, 1.0))
    keys = sorted(entries)
    return csr_from_coo(n, n, np.array([k[0] for k in keys]), np.array([k[1] for k in keys]),
                        np.array([entries[k] for k in keys]))


SYNTHETIC_EPS = 1e-4  # datasets.py:42


def gen_synthetic(n, density, seed):
    """datasets.py:148-193: A = P·Pᵀ + εI.  Small cases only (dictionary accumulation per column
    group in ascending column order, as the reference does)."""
    rng = np.random.default_rng(seed)
    nnz_p = int(round(density * n * n))
    flat = rng.choice(n * n, size=nnz_p, replace=False)
    pr, pc, pv = flat // n, flat % n, rng.standard_normal(nnz_p)
    order = np.lexsort((pr, pc))
    pr, pc, pv = pr[order], pc[order], pv[order]
    acc = {}
    start = 0
    while start < nnz_p:
        stop = start
        while stop < nnz_p and pc[stop] == pc[start]:
            stop += 1
        for p in range(start, stop):
            for q in range(start, stop):
                key = (int(pr[p]), int(pr[q]))
                acc[key] = acc.get(key, 0.0) + float(pv[p]) * float(pv[q])
        start = stop
    for i in range(n):
        acc[(i, i)] = acc.get((i, i), 0.0) + SYNTHETIC_EPS
    keys = sorted(acc)
    return csr_from_coo(n, n, np.array([k[0] for k in keys], dtype=np.int64),
                        np.array([k[1] for k in keys], dtype=np.int64), np.array([acc[k] for k in keys]))


# ----------------------------------------------------------------------------------------------
# L3 graph features  (graphfeat.py)
# ----------------------------------------------------------------------------------------------


def graph_features(n, offs, cols, vals, family=None, grid=None, coeff=None):
    """graphfeat.py:63-105.  Returns (node_features, edge_list, edge_features, norm_A)."""
    if not is_symmetric_pattern(n, n, offs, cols):
        raise StructureError("graph requires a symmetric sparsity pattern")
    vals = np.asarray(vals, dtype=np.float64)
    norm = mean_abs_nonzero_norm(vals)
    rows = row_expand(offs)
    edge_list = np.stack([rows, np.asarray(cols, dtype=np.int64)], axis=1)
    edge_features = (vals / norm)[:, None]
    if family in ("poisson2d", "heat2d"):
        nx, ny = grid
        coeff = np.asarray(coeff, dtype=np.float64)
        idx = np.arange(n)
        ix, iy = idx % nx, idx // nx
        hx, hy = 1.0 / (nx + 1), 1.0 / (ny + 1)
        node = np.stack([(ix + 1) * hx, (iy + 1) * hy, coeff / coeff.mean()], axis=1)
    else:
        rs = segment_sums(vals, offs)
        node = np.stack([rs / n / norm, diagonal(n, offs, cols, vals) / norm], axis=1)
    return node, edge_list, edge_features, norm


# ----------------------------------------------------------------------------------------------
# L3 GNN  (gnn.py) — weights and a tape-free forward
# ----------------------------------------------------------------------------------------------


def init_params(d_node, d_edge=1, n_layers=4, hidden=24, mlp_hidden_layers=1, seed=0,
                message_uses_hidden_edge=False):
    """gnn.py:98-106, 152-172: Glorot-uniform W, zero b, declaration order.

    Returns a list of MLPs; each MLP is a list of (W, b) with W shaped (d_in, d_out).
    Order: e_n, e_e, (f_m, f_v, f_e) x n_layers, decoder.
    """
    rng = np.random.default_rng(seed)

    def dims(di, do):
        return [di] + [hidden] * mlp_hidden_layers + [do]

    def mlp(ds):
        out = []
        for a, b in zip(ds[:-1], ds[1:]):
            bound = np.sqrt(6.0 / (a + b))
            out.append((rng.uniform(-bound, bound, size=(a, b)), np.zeros(b)))
        return out

    d = hidden
    me = d if message_uses_hidden_edge else d_edge
    mlps = [mlp(dims(d_node, d)), mlp(dims(d_edge, d))]
    for _ in range(n_layers):
        mlps += [mlp(dims(2 * d + me, d)), mlp(dims(d, d)), mlp(dims(3 * d, d))]
    mlps.append(mlp(dims(d, 1)))
    return mlps


def params_flat(mlps):
    """gnn.py:130-136."""
    return np.concatenate([np.concatenate([W.ravel(), b]) for m in mlps for W, b in m])


def unflatten(flat, template):
    """gnn.py:138-149 (set_params_flat)."""
    out, pos = [], 0
    for m in template:
        mm = []
        for W, b in m:
            Wn = flat[pos:pos + W.size].reshape(W.shape); pos += W.size
            bn = flat[pos:pos + b.size]; pos += b.size
            mm.append((Wn, bn))
        out.append(mm)
    assert pos == len(flat)
    return out


def _mlp(m, x, act):
    """gnn.py:198-205 (_apply_mlp): affine, activation between layers, linear output."""
    h = x
    for k, (W, b) in enumerate(m):
        h = h @ W + b
        if k < len(m) - 1:
            h = np.maximum(h, 0.0) if act == "relu" else np.tanh(h)
    return h


def gnn_forward(mlps, node_features, offs, cols, edge_features, n_layers, act="relu"):
    """gnn.py:208-253 without the tape: same ops in the same order (gather/concat/matmul)."""
    offs = np.asarray(offs, dtype=np.int64)
    rows = row_expand(offs)
    cols = np.asarray(cols, dtype=np.int64)
    it = iter(mlps)
    e_n, e_e = next(it), next(it)
    layers = [(next(it), next(it), next(it)) for _ in range(n_layers)]
    dec = next(it)
    X = _mlp(e_n, node_features, act)
    H = _mlp(e_e, edge_features, act)
    for f_m, f_v, f_e in layers:
        msg = _mlp(f_m, np.concatenate([X[rows], X[cols], edge_features], axis=1), act)
        X = X + _mlp(f_v, segment_sums(msg, offs), act)
        H = H + _mlp(f_e, np.concatenate([X[rows], X[cols], H], axis=1), act)
    return _mlp(dec, H, act)[:, 0].copy()


def gnn_forward_restructured(mlps, node_features, offs, cols, edge_features, n_layers, act="relu"):
    """the algebraically identical form the CUDA kernels implement.

    Node path never reads H; the message MLP's first layer is split across the concat
    (P = X W1[:d], Q = X W1[d:2d]) and its linear second layer is applied after the segment
    sum.  Only valid for mlp_hidden_layers == 1 and message_uses_hidden_edge == False.
    """
    offs = np.asarray(offs, dtype=np.int64)
    rows = row_expand(offs)
    cols = np.asarray(cols, dtype=np.int64)
    deg = np.diff(offs).astype(np.float64)[:, None]
    actf = (lambda v: np.maximum(v, 0.0)) if act == "relu" else np.tanh
    it = iter(mlps)
    e_n, e_e = next(it), next(it)
    layers = [(next(it), next(it), next(it)) for _ in range(n_layers)]
    dec = next(it)
    d = e_n[-1][0].shape[1]
    X = _mlp(e_n, node_features, act)
    Xs = []
    for (f_m, f_v, f_e) in layers:
        (W1, b1), (W2, b2) = f_m
        P, Q, c = X @ W1[:d], X @ W1[d:2 * d], W1[2 * d:]
        S = segment_sums(actf(P[rows] + Q[cols] + edge_features @ c + b1), offs)
        m = S @ W2 + deg * b2
        X = X + _mlp(f_v, m, act)
        Xs.append(X)
    h = _mlp(e_e, edge_features, act)
    for X_t, (_, _, f_e) in zip(Xs, layers):
        (W1, b1), (W2, b2) = f_e
        pre = (X_t @ W1[:d])[rows] + (X_t @ W1[d:2 * d])[cols] + h @ W1[2 * d:] + b1
        h = h + actf(pre) @ W2 + b2
    return _mlp(dec, h, act)[:, 0].copy()


# ----------------------------------------------------------------------------------------------
# L4 preconditioner + PCG  (precond.py, pcg.py)
# ----------------------------------------------------------------------------------------------


def learned_apply(n, offs, cols, gvals, eps, r):
    """precond.py:143-145: spmv(G, spmv_transpose(G, r)) + eps * r."""
    return spmv(offs, cols, gvals, spmv_transpose(n, offs, cols, gvals, r)) + eps * r


class OracleNotSpd(RuntimeError):
    """pcg.py:38-44."""

    def __init__(self, message, iteration, value):
        super().__init__(f"{message} (iteration {iteration}, value {value:.6e})")
        self.iteration = iteration
        self.value = value


def pcg_solve(offs, cols, avals, b, apply, rtol=1e-8, max_iters=None, period=50,
              track_history=True, termination="true_residual"):
    """pcg.py:131-233, control flow restated line for line.

    Returns (x, k, converged, history).  `apply` is the preconditioner (r -> s).
    """
    b = np.asarray(b, dtype=np.float64)
    n = len(b)
    max_iters = 20 * n if max_iters is None else max_iters
    use_true = termination == "true_residual"
    norm_b = float(np.linalg.norm(b))
    x = np.zeros(n)
    if norm_b == 0.0:
        return x, 0, True, ([0.0] if track_history else None)
    r = b - spmv(offs, cols, avals, x)
    d = apply(r)
    delta_new = float(r @ d)
    if delta_new < 0.0:
        raise OracleNotSpd("preconditioner is not positive definite", 0, delta_new)
    delta_0 = delta_new
    history = [float(np.linalg.norm(r)) / norm_b]
    i = 0
    converged = False
    while i < max_iters:
        if not use_true and delta_new <= rtol ** 2 * delta_0:
            break
        q = spmv(offs, cols, avals, d)
        dq = float(d @ q)
        if dq <= 0.0:
            raise OracleNotSpd("matrix is not positive definite along search direction", i, dq)
        alpha = delta_new / dq
        x = x + alpha * d
        refreshed = i > 0 and i % period == 0
        r = b - spmv(offs, cols, avals, x) if refreshed else r - alpha * q
        s = apply(r)
        delta_old = delta_new
        delta_new = float(r @ s)
        if delta_new < 0.0:
            raise OracleNotSpd("preconditioner is not positive definite", i, delta_new)
        d = s + (delta_new / delta_old) * d
        i += 1
        rel = float(np.linalg.norm(r)) / norm_b
        history.append(rel)
        if use_true and rel <= rtol:
            if refreshed:
                converged = True
                break
            r_fresh = b - spmv(offs, cols, avals, x)
            rel_fresh = float(np.linalg.norm(r_fresh)) / norm_b
            history[-1] = rel_fresh
            if rel_fresh <= rtol:
                converged = True
                break
            r = r_fresh
    if not use_true and not converged:
        converged = float(np.linalg.norm(b - spmv(offs, cols, avals, x))) / norm_b <= rtol
    return x, i, converged, (history if track_history else None)


# ----------------------------------------------------------------------------------------------
# L5 SAI loss  (training.py:57-94, autodiff.py:190-239, 265-303)
# ----------------------------------------------------------------------------------------------


def sai_loss(n, a_offs, a_cols, a_vals, g_offs, g_cols, g_vals, eps, w, norm_kind="mean_abs_nonzero",
             with_grad=False):
    """Forward (A side in np.longdouble, as autodiff.py:275-290) and, optionally, dL/dg.

    The gradient follows the tape's backward closures in order (autodiff.py:210-218,
    231-237, 294-300): du = add.at(A^T (2 inv_norm z64)), v = G^T du (add.at),
    dg = du[row]*t[col] + w[row]*v[col].
    """
    w = np.asarray(w, dtype=np.float64)
    a_vals = np.asarray(a_vals, dtype=np.float64)
    t = spmv_transpose(n, g_offs, g_cols, g_vals, w)
    u = spmv(g_offs, g_cols, g_vals, t) + eps * w
    vals_ld = a_vals.astype(np.longdouble)
    abs_ld = np.abs(vals_ld)
    if norm_kind == "mean_abs_nonzero":
        norm_ld = abs_ld.sum() / len(a_vals)
    elif norm_kind == "frobenius":
        norm_ld = np.sqrt((vals_ld * vals_ld).sum())
    elif norm_kind == "entrywise_l1":
        norm_ld = abs_ld.sum()
    else:
        raise ValueError(norm_kind)
    u_ld = u.astype(np.longdouble)
    y_ld = segment_sums(vals_ld * u_ld[np.asarray(a_cols)], a_offs)
    z_ld = y_ld / norm_ld - w.astype(np.longdouble)
    loss = float(np.float64((z_ld * z_ld).sum()))
    if not with_grad:
        return loss
    z64 = z_ld.astype(np.float64)
    inv_norm = float(np.longdouble(1.0) / norm_ld)
    dz = (2.0 * 1.0 * inv_norm) * z64
    du = spmv_transpose(n, a_offs, a_cols, a_vals, dz)
    g_rows = row_expand(g_offs)
    g_cols = np.asarray(g_cols, dtype=np.int64)
    grad = du[g_rows] * t[g_cols]
    v = spmv_transpose(n, g_offs, g_cols, g_vals, du)
    grad = grad + w[g_rows] * v[g_cols]
    return loss, grad
