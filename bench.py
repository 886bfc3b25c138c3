#!/usr/bin/env python
"""Benchmark: PCG solves/s for GNN build + solve (BASELINE.json metric) on config C2.

Workload (BASELINE.json configs[1]): variable-coefficient 2-D diffusion
systems (gen_poisson2d(256, 256, coeff_seed=s), heat2d family), 128 systems per GPU (1024 at
8 GPUs, weak scaling), trained GNN weights (tests/golden/trained_heat16.spaignn, produced by the
reference trainer), b_s = gen_rhs(meta, s + 10**6), PCG to rtol 1e-6, fp64 throughout.

One step = the hot path for every local system: build_graph features -> GNN forward -> G and
explicit G^T -> device-resident batched PCG.  `value` times steps on inputs already resident in
HBM (working set ~1.7 GB/GPU > 126 MB L2, so no L2 flush is needed); `e2e` times the public
batched API (`solve_batch`) from host buffers (int64 CSR, f64 values / coefficients / rhs) to
host solutions, copies included.  Multi-GPU: one process per GPU (torchrun), systems sharded by
rank, no collective in the solve; max-over-ranks device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
CKPT = os.path.join(ROOT, "tests", "golden", "trained_heat16.spaignn")
METRIC = "PCG solves/sec (GNN build+solve)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--systems-per-gpu", type=int, default=128)
    p.add_argument("--nx", type=int, default=256)
    p.add_argument("--rtol", type=float, default=1e-6)
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-workers", type=int, default=0)
    return p.parse_args()


def config_block(a, world):
    return {"workload": f"C2: heat2d {a.nx}x{a.nx} (5-point, variable coefficient), "
                        f"{a.systems_per_gpu} systems/GPU, GNN-SPAI (trained weights) + PCG rtol {a.rtol:g}",
            "systems_per_gpu": a.systems_per_gpu, "global_systems": a.systems_per_gpu * world,
            "n_per_system": a.nx * a.nx, "nnz_per_system": 5 * a.nx * a.nx - 4 * a.nx,
            "parallelism": f"dp{world} (systems sharded by rank, no collective in the solve)",
            "cache": "inputs larger than L2 (~1.7 GB working set per GPU vs 126 MB L2); no flush"}


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name).read().splitlines():
            parts = [t.strip() for t in line.split(",")]
            if len(parts) == 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:]))
                except ValueError:
                    pass
        os.unlink(self.f.name)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        sm = sorted(r[0] for r in rows)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def cpu_baseline(a, params, workers, seeds):
    from oracle.cpu_baseline import run_pool
    wall, res = run_pool(a.nx, seeds, params, a.rtol, workers)
    return wall, res


def run_reference(a, rank, world):
    """--impl reference: the reference path's CPU implementation (oracle port) on host cores."""
    if rank != 0:
        return
    from paper_2510_27517_b200.gnn import load_checkpoint
    params = load_checkpoint(CKPT).params_flat()
    workers = a.cpu_workers or min(os.cpu_count() or 1, 16)
    vals = []
    seed = 0
    for step in range(a.warmup + a.steps):
        seeds = list(range(seed, seed + workers))
        seed += workers
        wall, res = cpu_baseline(a, params, workers, seeds)
        if step >= a.warmup:
            vals.append((wall, res))
    walls = [w for w, _ in vals]
    ms = 1000.0 * float(np.mean(walls))
    value = workers / (ms / 1000.0)
    ks = [k for _, res in vals for _, k, _ in res]
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_block(a, world),
           "cpu_baseline": {"value": value, "unit": "solves/s", "cores": workers, "kind": "port",
                            "sample": f"{workers} systems per step ({workers} worker processes x 1 system, "
                                      f"1 BLAS thread each), numpy restatement oracle/spaigraph_ref.py",
                            "mean_k": float(np.mean(ks))},
           "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_ours(a, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_2510_27517_b200 import _lib
    from paper_2510_27517_b200.batch import BatchSolver, SystemBatch, solve_batch, solve_batch_stream
    from paper_2510_27517_b200.datasets import ProblemMeta
    from paper_2510_27517_b200.dist import gather_stats, local_systems, max_over_ranks
    from paper_2510_27517_b200.gnn import load_checkpoint
    from paper_2510_27517_b200.pcg import SolveConfig

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _lib.lib()
    model = load_checkpoint(CKPT)
    cfg = SolveConfig(rtol=a.rtol)
    S = a.systems_per_gpu
    ids, rhs = local_systems(S, rank, world)
    batch = SystemBatch.heat2d(a.nx, a.nx, ids, rhs)
    solver = BatchSolver(batch, model)
    for _ in range(max(a.warmup, 1)):
        res = solver.step(cfg)
    solver.handle.set_profile(True)
    res = solver.step(cfg)  # capture the profiled graphs outside the timed region
    solver.handle.stats(reset=True)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ks = []
    for _ in range(a.steps):
        res = solver.step(cfg)
        ks.append([r.k for r in res])
    e1.record()
    barrier()
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1) / a.steps
    ms = max_over_ranks(ms_local, dev)
    kernels, chunks, prof = solver.handle.stats(reset=True)
    L = model.config.n_layers
    # per step: batched norm (2) + batched features (1) + GNN (encode, L layers, edge pass) +
    # G^T gather (1) + everything the PCG handle launched (DIA conversion, setup, graph nodes)
    gpu_launches = a.steps * (3 + (2 + L) + 1) + kernels
    k_all, conv_all = gather_stats(ks[-1], [r.converged for r in res], dev)

    # ---- roofline of the PCG iteration kernels (sampled live by in-graph event nodes)
    n1 = a.nx * a.nx
    e1n = 5 * n1 - 4 * a.nx
    fused = bool(prof[7])
    K1N = "k_iter1 (q = A d, d = s + beta d, d.q)"
    K2N = "k_iter2 (x, r update, t = G^T r, r.r)"
    K3N = "k_iter3 (s = G t + eps r, r.s)"
    K23N = "k_iter23 (fused: x, r update, t = G^T r on chip, s = G t + eps r, r.r, r.s)"
    # algorithmic bytes per system per launch: CSR matrix bytes
    # (12 B/nnz + 4 B/row) + the vectors each kernel must read / write once
    csr = 12 * e1n + 4 * (n1 + 1)
    per_sys = {K1N: csr + 32 * n1}
    if fused:  # t never leaves the SM: reads x d r q, writes x r s
        per_sys[K23N] = csr + 56 * n1
    else:
        per_sys.update({K2N: csr + 56 * n1, K3N: csr + 24 * n1})
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # bytes the diagonal-major layout physically has to move per row (values incl. padding,
    # 1-byte presence mask, vectors); A read by its lower half when bitwise symmetric, or as
    # one coefficient per row when K1 regenerates it from gen_poisson2d's stencil (a_sym 2)
    nd, a_sym = int(prof[5]), int(prof[6])
    n_low = 1 if a_sym == 2 else (nd // 2 + 1) if a_sym else nd
    phys = {}
    if nd:
        phys = {K1N: (8 * n_low + 1 + 32) * n1}
        if fused:
            phys[K23N] = (8 * nd + 1 + 56) * n1
        else:
            phys.update({K2N: (8 * nd + 1 + 56) * n1, K3N: (8 * nd + 1 + 24) * n1})
    kern = {}
    samples = prof[4]
    if samples > 0:
        avg_active = prof[3] / samples
        for (name, b), t_ms in zip(per_sys.items(), prof[:3]):
            avg_ms = t_ms / samples
            achieved = b * avg_active / (avg_ms * 1e-3) / 1e9
            kern[name] = {"avg_ms": avg_ms, "gbs": achieved, "frac": achieved / peak,
                          "bytes_per_launch": b * avg_active}
            if name in phys:
                pg = phys[name] * avg_active / (avg_ms * 1e-3) / 1e9
                kern[name].update({"physical_bytes_per_launch": phys[name] * avg_active, "physical_gbs": pg,
                                   "physical_frac": pg / peak})
    dom = max(kern, key=lambda k: kern[k]["avg_ms"]) if kern else None
    roofline = None
    if dom:
        traffic = ncu_traffic("k_iter23_sw" if dom == K23N else "k_iter1_sw" if dom == K1N else None)
        roofline = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak,
                    "unit": "GB/s", "frac": kern[dom]["frac"],
                    "traffic": traffic["bytes"] if traffic else None,
                    "traffic_source": traffic["source"] if traffic else None,
                    "achieved_physical": kern[dom].get("physical_gbs"),
                    "frac_physical": kern[dom].get("physical_frac"),
                    "frac_vs_nominal_8tbs": kern[dom]["gbs"] / 8000.0,
                    "frac_physical_vs_nominal_8tbs": (kern[dom].get("physical_gbs") or 0.0) / 8000.0,
                    "bytes_note": "achieved = SURVEY.md §8(d) CSR bytes (12 B/nnz + 4 B/row + vectors); the kernels "
                                  f"run the diagonal-major layout ({nd} diagonals{', A by its lower half' if a_sym else ''}) "
                                  "which moves fewer bytes: physical_* counts those (8 B/diagonal/row + 1 B mask + vectors)",
                    "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)" if peak_src == "measured" else peak_src,
                    "per_kernel": kern, "samples": int(samples), "avg_active_systems": prof[3] / samples}

    # ---- e2e through the public batched API from host buffers
    e2e = None
    if not a.no_e2e:
        As, bs, metas = [], [], []
        a_dev = batch.a

        def pinned(t):  # host copy in page-locked memory (the contract's "pinned host memory")
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h.numpy()

        offs_h = pinned(a_dev.offs.to(torch.int64))
        cols_h = pinned(a_dev.cols.to(torch.int64))
        vals_h = pinned(a_dev.vals)
        b_h = pinned(batch.b)
        coeff_h = pinned(batch.coeff)

        class HostCsr:  # reference-typed host system (int64 CSR, f64 values)
            def __init__(self, n, o, c, v):
                self.n_rows = self.n_cols = n
                self.row_offsets, self.col_indices, self.values = o, c, v

        # per-system reference-typed arrays (local int64 indices) living in pinned memory
        loc_offs = torch.empty(S * (n1 + 1), dtype=torch.int64, pin_memory=True).numpy()
        loc_cols = torch.empty(len(cols_h), dtype=torch.int64, pin_memory=True).numpy()
        for k in range(S):
            r0, r1 = int(batch.row_start[k]), int(batch.row_start[k + 1])
            e0_, e1_ = int(batch.nnz_start[k]), int(batch.nnz_start[k + 1])
            o_k = loc_offs[k * (n1 + 1):(k + 1) * (n1 + 1)]
            np.subtract(offs_h[r0:r1 + 1], e0_, out=o_k)
            c_k = loc_cols[e0_:e1_]
            np.subtract(cols_h[e0_:e1_], r0, out=c_k)
            As.append(HostCsr(r1 - r0, o_k, c_k, vals_h[e0_:e1_]))
            bs.append(b_h[r0:r1])
            metas.append(ProblemMeta(family="heat2d", n=r1 - r0, grid=(a.nx, a.nx), coeff=coeff_h[r0:r1],
                                     coeff_seed=ids[k]))
        h2d = sum(A.row_offsets.nbytes + A.col_indices.nbytes + A.values.nbytes for A in As) + \
            sum(b.nbytes for b in bs) + sum(m.coeff.nbytes for m in metas)
        d2h = sum(b.nbytes for b in bs) + 8 * 2 * S
        reps = solve_batch(As, bs, model, metas, cfg)  # warm-up (allocations, graphs)
        for reps in solve_batch_stream([(As, bs, metas)] * 2, model, cfg):  # staging areas, host ring
            pass
        barrier()
        t0 = time.perf_counter()
        for reps in solve_batch_stream([(As, bs, metas)] * a.e2e_steps, model, cfg):
            pass  # every batch: H2D of all inputs (overlapping the previous solve), solve, D2H of x
        barrier()
        e2e_ms = max_over_ranks(1000.0 * (time.perf_counter() - t0) / a.e2e_steps, dev)
        assert [r.k for r in reps] == ks[-1], "e2e path must reproduce the device path"
        e2e = {"value": world * S / (e2e_ms / 1000.0), "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
               "api": "paper_2510_27517_b200.solve_batch_stream(batches of host int64 CSR, f64 values/coeff/rhs) "
                      "-> host x; the next batch's H2D overlaps the current solve"}

    # ---- CPU baseline (rank 0, N = 1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        workers = a.cpu_workers or min(os.cpu_count() or 1, 16)
        wall, cres = cpu_baseline(a, model.params_flat(), workers, list(range(workers)))
        cpu = {"value": workers / wall, "unit": "solves/s", "cores": workers, "kind": "port",
               "sample": f"{workers} of the same heat2d {a.nx}x{a.nx} systems (seeds 0..{workers - 1}), "
                         f"{workers} processes x 1 BLAS thread, numpy restatement of the reference path "
                         f"(tape-free => faster than the reference forward); wall {wall:.1f} s",
               "k": [k for _, k, _ in cres], "gpu_k_same_systems": [int(x) for x in k_all[:workers]]}

    if rank == 0:
        value = world * S / (ms / 1000.0)
        out = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded heat2d generators, trained weights)",
               "config": config_block(a, world), "e2e": e2e, "gpu_launches": int(gpu_launches),
               "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
               "k": {"mean": float(np.mean(k_all)), "min": int(np.min(k_all)), "max": int(np.max(k_all)),
                     "all_converged": bool(np.all(conv_all == 1))},
               "pcg_graph_launches_per_step": chunks / a.steps}
        print(json.dumps(out), flush=True)


NCU_SUMMARY = (sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_pcg_sw_128sys.txt"))) or
               [os.path.join(ROOT, "profiles", "r01_ncu_full_pcg_sw_128sys.txt")])[-1]  # newest round


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` from the committed ncu --set full
    capture of this workload (one launch, 128-system batch), in bytes; None if absent."""
    if not kernel or not os.path.exists(NCU_SUMMARY):
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for line in open(NCU_SUMMARY):
        if f" {kernel}<" not in line.split("|")[0]:
            continue
        vals = {}
        for cell in line.split("|")[1:]:
            key, _, v = cell.strip().partition("=")
            name, _, unit = key.partition("[")
            vals[name] = float(v) * scale.get(unit.rstrip("]"), float("nan"))
        if "dram__bytes_read.sum" in vals and "dram__bytes_write.sum" in vals:
            return {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                    "source": os.path.relpath(NCU_SUMMARY, ROOT) + " (ncu --set full, one launch)"}
    return None


def main():
    a = parse()
    from paper_2510_27517_b200.dist import init_from_env
    if a.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(a, rank, world)
        return
    rank, world, local = init_from_env()
    run_ours(a, rank, world, local)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
