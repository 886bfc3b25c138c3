"""Problem generators, drop-in for `spaigraph.datasets` (datasets.py:45-212) plus the 3-D and
random-SPD generators of SURVEY.md §8(d).

The coefficient field of "heat2d" is drawn on the host with numpy's PCG64 (the reference's RNG
stream, datasets.py:104-105); the matrix itself is emitted on the GPU in CSR order by a stencil
kernel (bit-identical values, no sort).  `gen_rhs` is the reference's host RNG draw.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .sparse import DeviceCsr, SparseMatrix

__all__ = ["ProblemMeta", "gen_poisson2d", "gen_poisson3d", "gen_rhs", "make_split", "rand_spd_sparse",
           "COEFF_LO", "COEFF_HI"]

COEFF_LO = 1e-4
COEFF_HI = 5e-4


@dataclass(frozen=True, eq=False)
class ProblemMeta:
    """datasets.py:45-84 (+ an optional device copy of the coefficient field)."""

    family: str
    n: int
    grid: tuple | None = None
    coeff: np.ndarray | None = None
    coeff_seed: int | None = None
    gen_seed: int | None = None
    density: float | None = None
    result_density: float | None = None
    epsilon_reg: float | None = None
    coeff_dev: object = None

    def to_dict(self) -> dict:
        return {"family": self.family, "n": self.n, "grid": list(self.grid) if self.grid is not None else None,
                "coeff": self.coeff.tolist() if self.coeff is not None else None, "coeff_seed": self.coeff_seed,
                "gen_seed": self.gen_seed, "density": self.density, "result_density": self.result_density,
                "epsilon_reg": self.epsilon_reg}


def heat_coeff(nx: int, ny: int, coeff_seed):
    """datasets.py:100-106: ones, or log-uniform in [1e-4, 5e-4] from PCG64(coeff_seed)."""
    if coeff_seed is None:
        return np.ones(nx * ny)
    rng = np.random.default_rng(coeff_seed)
    return np.exp(rng.uniform(math.log(COEFF_LO), math.log(COEFF_HI), size=nx * ny))


def poisson2d_device(nx: int, ny: int, coeff_dev) -> DeviceCsr:
    import torch
    n = nx * ny
    nnz = 5 * n - 2 * nx - 2 * ny
    offs = L.empty(n + 1, torch.int32)
    cols = L.empty(nnz, torch.int32)
    vals = L.empty(nnz, torch.float64)
    L.check(L.lib().sg_gen_poisson2d(nx, ny, L.ptr(coeff_dev), 0, 0, L.ptr(offs), L.ptr(cols), L.ptr(vals),
                                     L.stream_ptr()))
    return DeviceCsr(n, n, offs, cols, vals)


def gen_poisson2d(nx: int, ny: int, coeff_seed: int | None = None):
    """datasets.py:87-145 (matrix built on the GPU)."""
    import torch
    if nx < 1 or ny < 1:
        raise ValueError("grid dimensions must be positive")
    coeff = heat_coeff(nx, ny, coeff_seed)
    coeff_dev = L.to_device(coeff, torch.float64)
    A = SparseMatrix.from_device(poisson2d_device(nx, ny, coeff_dev))
    # the generator's node field: pcg_solve lets its streamed K1 regenerate A from it (8 instead
    # of 24 B per row), after verifying A against it bitwise at every solve (sg_pcg_set_stencil)
    A._stencil = (coeff_dev, nx, ny)
    family = "poisson2d" if coeff_seed is None else "heat2d"
    meta = ProblemMeta(family=family, n=nx * ny, grid=(nx, ny), coeff=coeff, coeff_seed=coeff_seed,
                       coeff_dev=coeff_dev)
    return A, meta


def gen_poisson3d(nx: int, ny: int, nz: int):
    """7-point -Laplace on the unit cube (no reference generator).

    Returned meta has family "synthetic" so build_graph uses the 2-d algebraic features.
    """
    import torch
    if nx < 1 or ny < 1 or nz < 1:
        raise ValueError("grid dimensions must be positive")
    n = nx * ny * nz
    nnz = 7 * n - 2 * ny * nz - 2 * nx * nz - 2 * nx * ny
    offs = L.empty(n + 1, torch.int32)
    cols = L.empty(nnz, torch.int32)
    vals = L.empty(nnz, torch.float64)
    L.check(L.lib().sg_gen_poisson3d(nx, ny, nz, L.ptr(offs), L.ptr(cols), L.ptr(vals), L.stream_ptr()))
    A = SparseMatrix.from_device(DeviceCsr(n, n, offs, cols, vals))
    return A, ProblemMeta(family="synthetic", n=n)


def gen_rhs(meta, seed: int) -> np.ndarray:
    """datasets.py:209-212."""
    n = meta.n if hasattr(meta, "n") else int(meta)
    b = np.random.default_rng(seed).standard_normal(n)
    return b / np.linalg.norm(b)


def make_split(dataset, ratio: tuple = (4, 1), seed: int = 0):
    """datasets.py:196-206."""
    items = list(dataset)
    tr, te = ratio
    if tr < 1 or te < 1:
        raise ValueError("split ratio parts must be positive")
    perm = np.random.default_rng(seed).permutation(len(items))
    n_test = len(items) * te // (tr + te)
    return [items[i] for i in perm[n_test:]], [items[i] for i in perm[:n_test]]


SYNTHETIC_EPS = 1e-4  # datasets.py:42


def gen_synthetic(n: int, density: float, seed: int):
    """datasets.py:148-193: A = P·Pᵀ + εI, P uniformly random sparse standard-normal.

    The draws are the reference's (host PCG64: ``choice`` without replacement, then
    ``standard_normal``); everything after them runs on the device: P's rows and its transpose by
    the radix-sort COO→CSR / transpose kernels, the Gram pattern by the warp symbolic product
    (``sg_gram_pattern``), and the values by ``sg_gram_values``, which merges rows i and j of P in
    ascending column order -- the order the reference's dictionary accumulation visits P's column
    groups in -- so every entry is bit-identical.
    """
    import ctypes as C

    import torch
    if n < 1:
        raise ValueError("matrix size must be positive")
    if not 0.0 <= density <= 1.0:
        raise ValueError("density must lie in [0, 1]")
    rng = np.random.default_rng(seed)
    nnz_p = int(round(density * n * n))
    flat = rng.choice(n * n, size=nnz_p, replace=False)
    p_vals = rng.standard_normal(nnz_p)
    P = SparseMatrix.from_coo(n, n, flat // n, flat % n, p_vals).device()
    ot, ct, _ = P.transpose_pattern()
    offs = L.empty(n + 1, torch.int32)
    nnz = C.c_int64(0)
    lib = L.lib()
    buf, wsb = L.workspace(lib.sg_gram_pattern, n, L.ptr(P.offs), L.ptr(P.cols), L.ptr(ot), L.ptr(ct),
                           L.ptr(offs), None, C.byref(nnz))
    L.check(lib.sg_gram_pattern(n, L.ptr(P.offs), L.ptr(P.cols), L.ptr(ot), L.ptr(ct), L.ptr(offs), None,
                                C.byref(nnz), L.ptr(buf), C.byref(wsb), L.stream_ptr()), "gen_synthetic")
    cols = L.empty(int(nnz.value), torch.int32)
    L.check(lib.sg_gram_pattern(n, L.ptr(P.offs), L.ptr(P.cols), L.ptr(ot), L.ptr(ct), L.ptr(offs),
                                L.ptr(cols), C.byref(nnz), L.ptr(buf), C.byref(wsb), L.stream_ptr()),
            "gen_synthetic")
    vals = L.empty(int(nnz.value), torch.float64)
    L.check(lib.sg_gram_values(n, L.ptr(P.offs), L.ptr(P.cols), L.ptr(P.vals), L.ptr(offs), L.ptr(cols),
                               SYNTHETIC_EPS, L.ptr(vals), L.stream_ptr()), "gen_synthetic")
    A = SparseMatrix.from_device(DeviceCsr(n, n, offs, cols, vals))
    meta = ProblemMeta(family="synthetic", n=n, gen_seed=seed, density=density,
                       result_density=A.nnz / (n * n), epsilon_reg=SYNTHETIC_EPS)
    return A, meta


def rand_spd_sparse(n: int, rng, extra_per_row: int = 3) -> SparseMatrix:
    """verify.py:39-61 (config-4 generator): same PCG64 draw sequence, vectorised bookkeeping.

    The reference draws (i, j, v) one triple at a time; numpy's Generator produces the same
    stream when the scalar calls are kept, so the draws stay scalar and only the dictionary
    bookkeeping is vectorised (last write wins for repeated pairs, as in the dict).
    """
    m = extra_per_row * n
    ii = np.empty(m, dtype=np.int64)
    jj = np.empty(m, dtype=np.int64)
    vv = np.zeros(m)
    keep = np.zeros(m, dtype=bool)
    for t in range(m):
        i = int(rng.integers(n))
        j = int(rng.integers(n))
        ii[t], jj[t] = i, j
        if i == j:
            continue
        vv[t] = float(rng.uniform(-1.0, 1.0))
        keep[t] = True
    # entries[(i,j)] = entries[(j,i)] = v in draw order: later draws overwrite earlier ones
    r = np.concatenate([ii[keep], jj[keep]])
    c = np.concatenate([jj[keep], ii[keep]])
    order = np.concatenate([np.flatnonzero(keep)] * 2)
    v = np.concatenate([vv[keep], vv[keep]])
    key = r * n + c
    # last occurrence (max draw index) per key
    srt = np.lexsort((order, key))
    last = np.ones(len(srt), dtype=bool)
    last[:-1] = key[srt][1:] != key[srt][:-1]
    sel = srt[last]
    r, c, v = r[sel], c[sel], v[sel]
    row_abs = np.zeros(n)
    # reference: for (i, _), v in entries.items(): row_abs[i] += abs(v) (dict insertion order)
    first_ins = np.lexsort((order[srt], key[srt]))
    ins = np.ones(len(srt), dtype=bool)
    ins[1:] = key[srt][1:] != key[srt][:-1]
    ins_order = order[srt][ins]          # first insertion draw of each key
    ins_key = key[srt][ins]
    ins_pos = np.argsort(ins_order, kind="stable")
    del first_ins
    kv = dict(zip(key[sel].tolist(), v.tolist()))
    for kk in ins_key[ins_pos].tolist():
        row_abs[kk // n] += abs(kv[kk])
    diag = np.empty(n)
    for i in range(n):
        diag[i] = row_abs[i] + 1.0 + float(rng.uniform(0.0, 1.0))
    rows = np.concatenate([r, np.arange(n)])
    cols = np.concatenate([c, np.arange(n)])
    vals = np.concatenate([v, diag])
    return SparseMatrix.from_coo(n, n, rows, cols, vals)


def write_rhs_vec(b, path) -> None:
    """datasets.py:221-231: u64 little-endian length header, then f64 little-endian data; written
    to `path.tmp` and renamed (atomic).  Accepts numpy arrays or device tensors."""
    import os
    import struct
    try:
        import torch
        if isinstance(b, torch.Tensor):
            b = b.detach().to("cpu").numpy()
    except ImportError:  # pragma: no cover
        pass
    b = np.asarray(b, dtype=np.float64)
    tmp = str(path) + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(struct.pack("<Q", len(b)))
        fh.write(np.ascontiguousarray(b, dtype="<f8").tobytes())
    os.replace(tmp, str(path))


def read_rhs_vec(path, device: bool = False):
    """datasets.py:234-242 (same header checks and ValueErrors).  device=True reads the payload
    into page-locked memory and returns a device tensor (one asynchronous H2D copy)."""
    import struct
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 8:
        raise ValueError("rhs file too short for its header")
    (n,) = struct.unpack_from("<Q", raw, 0)
    if len(raw) != 8 + 8 * n:
        raise ValueError(f"rhs file length {len(raw)} does not match header count {n}")
    b = np.frombuffer(raw, dtype="<f8", offset=8).astype(np.float64)
    if not device:
        return b
    import torch
    from . import _lib as L
    host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    host.numpy()[:] = b
    out = L.empty(n, torch.float64)
    out.copy_(host, non_blocking=True)
    return out
