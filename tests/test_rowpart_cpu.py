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


def test_band_partition_extended_systems():
    """Contiguous row split of a banded matrix (the device-resident row partition): owned blocks
    tile the rows, neighbouring ghost widths agree (what one rank sends is what the other
    receives), and every owned row of the extended local system equals the global row."""
    from oracle import spaigraph_ref as O
    from paper_2510_27517_b200.rowpart import band_local, band_partition
    o, c, v, _ = O.gen_poisson2d(12, 9)
    n = len(o) - 1
    for world in (1, 2, 3):
        parts = [band_partition(o, c, n, r, world) for r in range(world)]
        assert parts[0].r0 == 0 and parts[-1].r1 == n
        for a, b in zip(parts[:-1], parts[1:]):
            assert a.r1 == b.r0 and a.ghost_hi == b.ghost_lo == 12  # half-bandwidth = nx
        for p in parts:
            lo, lc, lv = band_local(o, c, v, p)
            for i in range(p.r0, p.r1):
                li = i - p.e0
                gl = slice(o[i], o[i + 1])
                assert np.array_equal(lc[lo[li]:lo[li + 1]] + p.e0, c[gl])
                assert np.array_equal(lv[lo[li]:lo[li + 1]], v[gl])
