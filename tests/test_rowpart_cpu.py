"""CPU: the row-partitioned PCG — halo plan, receptive-field subgraph
GNN, and the distributed solve over 2 gloo ranks — with a numpy stand-in for the local kernels
(the test backend; the product backend is CudaOps).  Compared with the single-process oracle."""
import json
import os
import socket
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import spaigraph_ref as O  # noqa: E402
from paper_2510_27517_b200.rowpart import build_plan, hop_closure, local_rows, local_transpose_rows  # noqa: E402


def _problem(nx=14):
    offs, cols, vals, coeff = O.gen_poisson2d(nx, nx, 5)
    n = nx * nx
    node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d", (nx, nx), coeff)
    mlps = O.init_params(3, seed=2)
    g = O.gnn_forward_restructured(mlps, node, offs, cols, ef, 4)
    return n, offs, cols, vals, node, ef, mlps, g


def _local_exchange(plans_needed):
    """Single-process stand-in for the all_to_all of index lists."""
    world = len(plans_needed)
    return [[plans_needed[p][q] for p in range(world)] for q in range(world)]


def test_halo_plan_and_local_rows():
    n, offs, cols, vals, *_ = _problem()
    world = 3
    needed = []
    for rank in range(world):
        captured = {}

        def ex(per_src, captured=captured):
            captured["per_src"] = per_src
            return [np.zeros(0, np.int64)] * world
        build_plan(offs, cols, n, rank, world, ex)
        needed.append(captured["per_src"])
    asked = _local_exchange(needed)
    x = np.random.default_rng(0).standard_normal(n)
    for rank in range(world):
        plan = build_plan(offs, cols, n, rank, world, lambda per_src, r=rank: asked[r])
        lo, lc, lv = local_rows(offs, cols, vals, plan)
        x_ext = np.concatenate([x[plan.r0:plan.r1], x[plan.halo]])
        # owned rows of A x, bitwise (same per-row order)
        assert np.array_equal(O.spmv(lo, lc, lv, x_ext), O.spmv(offs, cols, vals, x)[plan.r0:plan.r1])
        # send lists are the owners' view of the halo
        for p in range(world):
            assert np.array_equal(np.sort(plan.send_idx[p] + plan.r0), np.sort(needed[p][rank]))


def test_local_transpose_rows_match_global_transpose():
    n, offs, cols, vals, node, ef, mlps, g = _problem()
    world = 2
    needed = []
    for rank in range(world):
        cap = {}
        build_plan(offs, cols, n, rank, world, lambda ps, cap=cap: cap.setdefault("p", ps) and [np.zeros(0, np.int64)] * world)
        needed.append(cap["p"])
    asked = _local_exchange(needed)
    x = np.random.default_rng(1).standard_normal(n)
    full = O.spmv_transpose(n, offs, cols, g, x)
    for rank in range(world):
        plan = build_plan(offs, cols, n, rank, world, lambda ps, r=rank: asked[r])
        to, tc, tv = local_transpose_rows(offs, cols, g, plan)
        x_ext = np.concatenate([x[plan.r0:plan.r1], x[plan.halo]])
        got = np.array([sum_seq(tv[to[i]:to[i + 1]] * x_ext[tc[to[i]:to[i + 1]]]) for i in range(plan.n_own)])
        assert np.array_equal(got, full[plan.r0:plan.r1])


def sum_seq(v):
    s = 0.0
    for t in v:
        s = s + t
    return s


def test_receptive_field_subgraph_gnn_is_exact():
    """G rows within one hop of the owned rows are exact on the (L+2)-hop subgraph."""
    n, offs, cols, vals, node, ef, mlps, g = _problem()
    owned = np.arange(60, 110)
    R = hop_closure(offs, cols, owned, 4 + 2)
    rows = O.row_expand(offs)
    keep = np.isin(rows, R) & np.isin(cols, R)
    remap = -np.ones(n, dtype=np.int64)
    remap[R] = np.arange(len(R))
    sub_rows, sub_cols = remap[rows[keep]], remap[np.asarray(cols)[keep]]
    sub_offs = np.zeros(len(R) + 1, dtype=np.int64)
    np.add.at(sub_offs, sub_rows + 1, 1)
    np.cumsum(sub_offs, out=sub_offs)
    g_sub = O.gnn_forward_restructured(mlps, node[R], sub_offs, sub_cols, ef[keep], 4)
    one_hop = hop_closure(offs, cols, owned, 1)
    # compare every stored entry of the rows in one_hop
    g_full_of_kept = g[keep]
    sel = np.isin(rows[keep], one_hop)
    assert np.max(np.abs(g_sub[sel] - g_full_of_kept[sel])) <= 1e-12 * np.max(np.abs(g))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import numpy as np, torch
import torch.distributed as dist
from oracle import spaigraph_ref as O
from paper_2510_27517_b200.dist import init_from_env
from paper_2510_27517_b200.rowpart import (build_plan, local_rows, local_transpose_rows, DistPcg, TorchComm)

class NumpyOps:   # test backend: numpy stand-ins for the CUDA kernels, same summation orders
    def matrix(self, o, c, v): return (len(o) - 1, np.asarray(o), np.asarray(c), np.asarray(v))
    def zeros(self, n): return torch.zeros(n, dtype=torch.float64)
    def copy_own(self, d, s): d[:len(s)] = torch.as_tensor(s)
    def copy(self, d, s): d.copy_(s)
    def own(self, x): return x[:self.n_own].numpy().copy()
    def spmv(self, M, x, y):
        n, o, c, v = M
        y.numpy()[:n] = O.spmv(o, c, v, x.numpy())
    def spmv_seq(self, M, x, y):
        n, o, c, v = M
        xv, yv = x.numpy(), y.numpy()
        for i in range(n):
            s = 0.0
            for k in range(o[i], o[i + 1]):
                s = s + v[k] * xv[c[k]]
            yv[i] = s
    def axpby(self, out, a, b, c, mode):
        n = self.n_own
        p = c * b.numpy()[:n]
        out.numpy()[:n] = a.numpy()[:n] + p if mode == 0 else a.numpy()[:n] - p
    def dot(self, x, y):
        n = self.n_own
        return float(x.numpy()[:n] @ y.numpy()[:n])

rank, world, _ = init_from_env("gloo")
nx = 14
offs, cols, vals, coeff = O.gen_poisson2d(nx, nx, 5)
n = nx * nx
node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d", (nx, nx), coeff)
g = O.gnn_forward_restructured(O.init_params(3, seed=2), node, offs, cols, ef, 4)
b = O.gen_rhs(n, 77)
comm = TorchComm()
plan = build_plan(offs, cols, n, rank, world, comm.exchange_lists)
pcg = DistPcg(plan, NumpyOps(), comm, local_rows(offs, cols, vals, plan), local_rows(offs, cols, g, plan),
              local_transpose_rows(offs, cols, g, plan), 1e-4)
x_own, k, conv, hist = pcg.solve(b[plan.r0:plan.r1], rtol=1e-8, period=7)
parts = [None] * world
dist.all_gather_object(parts, x_own.tolist())
if rank == 0:
    x = np.concatenate([np.asarray(p) for p in parts])
    xr, kr, cr, hr = O.pcg_solve(offs, cols, vals, b, lambda r: O.learned_apply(n, offs, cols, g, 1e-4, r),
                                 rtol=1e-8, period=7)
    print(json.dumps({{"k": k, "kr": kr, "conv": conv, "cr": cr, "dx": float(np.max(np.abs(x - xr)) / np.max(np.abs(xr))),
                      "res": float(np.linalg.norm(b - O.spmv(offs, cols, vals, x))),
                      "hlen": len(hist), "hrlen": len(hr)}}))
dist.barrier()
dist.destroy_process_group()
"""


def test_distributed_pcg_two_gloo_ranks(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER.format(root=ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300,
                       env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["conv"] and out["cr"]
    assert abs(out["k"] - out["kr"]) <= max(1, round(0.02 * out["kr"]))
    # two valid solutions at rtol 1e-8 differ by ~cond(A) * 1e-8; the residual is the contract
    assert out["res"] <= 1e-8 and out["dx"] < 1e-6
    assert out["hlen"] == out["k"] + 1


def test_row_partition_plan():
    """plan_row_partition: owned blocks tile the rows in whole grid lines, ghosts are 3 half-
    bandwidths (clipped at the ends), the GNN block adds the (L+2)-hop receptive field."""
    from paper_2510_27517_b200.rowpart import GHOST_LAYERS, plan_row_partition
    o, c, v, _ = O.gen_poisson2d(12, 40)
    n = len(o) - 1
    for parts in (1, 2, 3, 4):
        pl = plan_row_partition(o, c, n, parts, n_layers=4)
        assert pl.hb == 12 and pl.unit == 12
        assert pl.own[0][0] == 0 and pl.own[-1][1] == n
        for (a0, a1), (b0, b1) in zip(pl.own[:-1], pl.own[1:]):
            assert a1 == b0 and a1 % 12 == 0
        for p, ((lo, hi), (e0, e1), (g0, g1)) in enumerate(zip(pl.own, pl.ext, pl.gnn)):
            assert e0 == max(0, lo - GHOST_LAYERS * 12) and e1 == min(n, hi + GHOST_LAYERS * 12)
            assert g0 == max(0, e0 - 6 * 12) and g1 == min(n, e1 + 6 * 12)
    import pytest
    with pytest.raises(ValueError):
        plan_row_partition(o, c, n, 20, n_layers=4)  # 2 lines each < 3-line ghosts


def _band(offs, cols, vals, e0, e1):
    """Rows [e0, e1) with columns clipped to [e0, e1), local indices (storage order kept)."""
    rows = np.repeat(np.arange(len(offs) - 1), np.diff(offs))
    sel = (rows >= e0) & (rows < e1) & (cols >= e0) & (cols < e1)
    lo = np.zeros(e1 - e0 + 1, dtype=np.int64)
    np.add.at(lo, rows[sel] - e0 + 1, 1)
    return np.cumsum(lo), cols[sel] - e0, vals[sel]


def test_ghost_scheme_reproduces_global_pcg():
    """The partition design of DESIGN.md §7 in numpy: every vector is computed over each
    partition's WHOLE extended system (3 half-bandwidths of ghost rows, truncated rows at its
    edges), s only on owned rows and then copied into the neighbours' ghost rows, dot products
    over owned rows added in partition order -- exactly the kernels' schedule (K1, fused K2+K3,
    refresh, fresh residual).  Its residual history equals the oracle's global pcg_solve up to
    dot-product rounding, so the redundant ghost computation is exact where it is read."""
    from paper_2510_27517_b200.rowpart import plan_row_partition
    nx, ny = 11, 48
    offs, cols, vals, coeff = O.gen_poisson2d(nx, ny, 3)
    n = nx * ny
    node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d", (nx, ny), coeff)
    from paper_2510_27517_b200.gnn import load_checkpoint
    params = load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_heat16.spaignn")).params_flat()
    g = O.gnn_forward_restructured(O.unflatten(params, O.init_params(3)), node, offs, cols, ef, 4)
    eps = 1e-4
    b = O.gen_rhs(n, 9)
    rtol, period = 1e-10, 7
    _, k_ref, conv_ref, hist_ref = O.pcg_solve(offs, cols, vals, b,
                                               lambda r: O.learned_apply(n, offs, cols, g, eps, r),
                                               rtol=rtol, period=period)
    for parts in (2, 3, 4):
        pl = plan_row_partition(offs, cols, n, parts, n_layers=4)
        P_ = []
        for (lo, hi), (e0, e1) in zip(pl.own, pl.ext):
            ao, ac, av = _band(offs, cols, vals, e0, e1)
            _, _, gv = _band(offs, cols, g, e0, e1)
            P_.append(dict(o=slice(lo - e0, hi - e0), e=(e0, e1), n=e1 - e0, a=(ao, ac, av), g=(ao, ac, gv),
                           b=b[e0:e1].copy()))

        def A(p, x):
            return O.spmv(*p["a"], x)

        def Gt(p, x):
            return O.spmv_transpose(p["n"], *p["g"], x)

        def Gm(p, x):
            return O.spmv(*p["g"], x)

        def dot(u, v):  # owned rows, partition order
            s = 0.0
            for p, a, c in zip(P_, u, v):
                s = s + float(a[p["o"]] @ c[p["o"]])
            return s

        def exchange_s(S):  # owned s -> every other partition's ghost rows
            for q, p in enumerate(P_):
                for r, pr in enumerate(P_):
                    if r == q:
                        continue
                    lo = max(p["e"][0], pr["e"][0] + pr["o"].start)
                    hi = min(p["e"][1], pr["e"][0] + pr["o"].stop)
                    if lo < hi:
                        S[q][lo - p["e"][0]:hi - p["e"][0]] = S[r][lo - pr["e"][0]:hi - pr["e"][0]]

        def apply(r):  # setup2 / K2+K3 / refresh K3: s on owned rows, then the halo push
            S = []
            for p, rp in zip(P_, r):
                s_ = np.zeros(p["n"])
                s_[p["o"]] = (Gm(p, Gt(p, rp)) + eps * rp)[p["o"]]
                S.append(s_)
            exchange_s(S)
            return S

        x = [np.zeros(p["n"]) for p in P_]
        r = [p["b"].copy() for p in P_]
        norm_b = np.sqrt(dot(r, r))
        s = apply(r)
        d = [np.zeros(p["n"]) for p in P_]
        delta = dot(r, s)
        delta0 = delta
        hist = [np.sqrt(dot(r, r)) / norm_b]
        beta, i, fresh, conv = 0.0, 0, False, False
        while i < 20 * n:
            d = [si + beta * di for si, di in zip(s, d)]  # K1
            q = [A(p, di) for p, di in zip(P_, d)]
            if fresh:
                rf = [p["b"] - A(p, xi) for p, xi in zip(P_, x)]
                rel = np.sqrt(dot(rf, rf)) / norm_b
                hist[-1] = rel
                if rel <= rtol:
                    conv = True
                    break
                r, fresh = rf, False
            alpha = delta / dot(d, q)
            x = [xi + alpha * di for xi, di in zip(x, d)]
            refreshed = i > 0 and i % period == 0
            if refreshed:
                r = [p["b"] - A(p, xi) for p, xi in zip(P_, x)]
            else:
                r = [ri - alpha * qi for ri, qi in zip(r, q)]
            s = apply(r)
            delta_old, delta = delta, dot(r, s)
            beta = delta / delta_old
            i += 1
            rel = np.sqrt(dot(r, r)) / norm_b
            hist.append(rel)
            if rel <= rtol:
                if refreshed:
                    conv = True
                    break
                fresh = True
        # a ghost value that were wrong where it is read would break the recurrence at once; the
        # only difference left is the order of the dot products' additions
        assert conv and conv_ref and abs(i - k_ref) <= max(1, 0.02 * k_ref), (parts, i, k_ref)
        np.testing.assert_allclose(hist[:60], hist_ref[:60], rtol=1e-6, atol=1e-9)


PEER_WORKER = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import numpy as np
import torch
import torch.distributed as dist
from oracle import spaigraph_ref as O
from paper_2510_27517_b200.dist import init_from_env
from paper_2510_27517_b200.rowpart import exchange_blobs, plan_row_partition

rank, world, _ = init_from_env("gloo")
nx, ny = 9, 30
offs, cols, vals, coeff = O.gen_poisson2d(nx, ny, 2)
n = nx * ny
node, _, ef, _ = O.graph_features(n, offs, cols, vals, "heat2d", (nx, ny), coeff)
from paper_2510_27517_b200.gnn import load_checkpoint
params = load_checkpoint(os.path.join({root!r}, "tests", "golden", "trained_heat16.spaignn")).params_flat()
g = O.gnn_forward_restructured(O.unflatten(params, O.init_params(3)), node, offs, cols, ef, 4)
b = O.gen_rhs(n, 3)
eps, rtol, period = 1e-4, 1e-8, 9
pl = plan_row_partition(offs, cols, n, world, n_layers=4)
# the peer blobs travel once (sg_pcg_set_peers' input); every rank sees every blob in rank order
blobs = exchange_blobs(("peer-info-%d" % rank).encode())
assert blobs == [("peer-info-%d" % q).encode() for q in range(world)], blobs
(lo, hi), (e0, e1) = pl.own[rank], pl.ext[rank]
rows = np.repeat(np.arange(n), np.diff(offs))
sel = (rows >= e0) & (rows < e1) & (cols >= e0) & (cols < e1)
lo_offs = np.cumsum(np.concatenate([[0], np.bincount(rows[sel] - e0, minlength=e1 - e0)]))
A = (lo_offs, cols[sel] - e0, vals[sel])
G = (lo_offs, cols[sel] - e0, g[sel])
own = slice(lo - e0, hi - e0)
ne = e1 - e0

def dot(u, v):  # partials in rank order: what part_fin (peer mode) adds
    parts = [None] * world
    dist.all_gather_object(parts, float(u[own] @ v[own]))
    s = 0.0
    for p in parts:
        s = s + p
    return s

def push_s(s):  # the kernels' peer stores: owned boundary rows -> neighbours' ghost rows
    reqs = []
    if rank > 0:
        gh = pl.ext[rank - 1][1] - pl.own[rank - 1][1]
        reqs.append(dist.isend(torch.from_numpy(s[own][:gh].copy()), rank - 1))
    if rank < world - 1:
        gl = pl.own[rank + 1][0] - pl.ext[rank + 1][0]
        reqs.append(dist.isend(torch.from_numpy(s[own][len(s[own]) - gl:].copy()), rank + 1))
    if rank > 0:
        buf = torch.empty(lo - e0, dtype=torch.float64)
        dist.recv(buf, rank - 1)
        s[:lo - e0] = buf.numpy()
    if rank < world - 1:
        buf = torch.empty(e1 - hi, dtype=torch.float64)
        dist.recv(buf, rank + 1)
        s[hi - e0:] = buf.numpy()
    for r_ in reqs:
        r_.wait()

def apply(r):
    s = np.zeros(ne)
    s[own] = (O.spmv(*G, O.spmv_transpose(ne, *G, r)) + eps * r)[own]
    push_s(s)
    return s

bl = b[e0:e1].copy()
x, r, d = np.zeros(ne), bl.copy(), np.zeros(ne)
norm_b = np.sqrt(dot(r, r))
s = apply(r)
delta = dot(r, s)
hist = [np.sqrt(dot(r, r)) / norm_b]
beta, i, fresh, conv = 0.0, 0, False, False
while i < 20 * n:
    d = s + beta * d
    q = O.spmv(*A, d)
    if fresh:
        rf = bl - O.spmv(*A, x)
        rel = np.sqrt(dot(rf, rf)) / norm_b
        hist[-1] = rel
        if rel <= rtol:
            conv = True
            break
        r, fresh = rf, False
    alpha = delta / dot(d, q)
    x = x + alpha * d
    refreshed = i > 0 and i % period == 0
    r = bl - O.spmv(*A, x) if refreshed else r - alpha * q
    s = apply(r)
    delta_old, delta = delta, dot(r, s)
    beta = delta / delta_old
    i += 1
    rel = np.sqrt(dot(r, r)) / norm_b
    hist.append(rel)
    if rel <= rtol:
        if refreshed:
            conv = True
            break
        fresh = True
xs = [None] * world
dist.all_gather_object(xs, x[own].tolist())
if rank == 0:
    xg = np.concatenate([np.asarray(p) for p in xs])
    _, kr, cr, hr = O.pcg_solve(offs, cols, vals, b, lambda v: O.learned_apply(n, offs, cols, g, eps, v),
                                rtol=rtol, period=period)
    print(json.dumps({{"k": i, "kr": kr, "conv": conv, "cr": cr, "hist": hist[:40], "hr": hr[:40],
                      "res": float(np.linalg.norm(b - O.spmv(offs, cols, vals, xg)) / np.linalg.norm(b))}}))
dist.barrier()
dist.destroy_process_group()
"""


def test_peer_partition_schedule_two_gloo_ranks(tmp_path):
    """The peer-mode schedule across 2 processes: each rank plans the partition itself, builds
    only its extended system, exchanges its peer blob once, pushes its s boundary rows into the
    neighbour's ghost rows (send/recv standing in for the NVLink peer stores) and adds the
    reduction partials in rank order -- the same result as the oracle's global pcg_solve."""
    script = tmp_path / "peer_worker.py"
    script.write_text(PEER_WORKER.format(root=ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300,
                       env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["conv"] and out["cr"] and abs(out["k"] - out["kr"]) <= max(1, 0.02 * out["kr"])
    np.testing.assert_allclose(out["hist"], out["hr"], rtol=1e-6, atol=1e-10)
    assert out["res"] <= 1e-8
