"""Timeline of the C5 strip kernels from per-CTA %globaltimer stamps (sg_pcg_set_trace).

    python profiles/trace_probe.py [--iters 200]

Solves C5 (2048^2, trained GNN) with max_iters = --iters through the public API with the probe
on, then prints, for the LAST launch of k_iter1_s5p (K1) and k_iter23_s5 (K2+K3): the spread of
CTA entry times, of stream ends, of arrivals, the last CTA's finaliser time, and the gap from
one kernel's finaliser to the next kernel's first CTA entry.  Diagnostic only (the stamps cost a
few instructions per CTA); the timings it reports are not bench numbers.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_27517_b200 as P  # noqa: E402
from paper_2510_27517_b200 import _lib as L  # noqa: E402
from paper_2510_27517_b200.pcg import _handle_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    A, meta = P.gen_poisson2d(2048, 2048)
    model = P.load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_heat16.spaignn"))
    G = P.forward(model, P.build_graph(A, meta)).G
    M = P.build_learned_spai(G, model.config.epsilon)
    b = torch.as_tensor(P.gen_rhs(meta, 10**6), device="cuda")
    cfg = P.SolveConfig(rtol=1e-6, max_iters=a.iters)
    P.pcg_solve(A, b, M, cfg)  # plan the handle
    h = _handle_for(A, M, "learned")
    buf = torch.zeros(2 * 16384, dtype=torch.int64, device="cuda")
    L.check(L.lib().sg_pcg_set_trace(h._h, C.c_void_p(buf.data_ptr())))
    out = {}
    for rep in range(3):
        buf.zero_()
        P.pcg_solve(A, b, M, cfg)
        torch.cuda.synchronize()
        t = buf.cpu().numpy().reshape(2, 2048, 8)
        res = {}
        for kid, name in ((0, "K1 k_iter1_s5p"), (1, "K2+K3 k_iter23_s5")):
            tk = t[kid]
            used = tk[:, 0] > 0
            sm = tk[used][:, 4]
            tk = tk[used][:, :4].astype(np.float64)
            t0 = tk[:, 0].min()
            fin = tk[:, 3][tk[:, 3] > 0]
            # stream time of a CTA vs how many CTAs shared its SM, its strip and its line range
            # (the range table is line-range-major: CTA b = strip b % 8 of line range b // 8)
            dur = tk[:, 1] - tk[:, 0]
            per_sm = np.bincount(sm, minlength=int(sm.max()) + 1)
            load = per_sm[sm]
            by_load = {int(c): [round(float(np.median(dur[load == c])) / 1e3, 2), int((load == c).sum())]
                       for c in np.unique(load)}
            nct = len(dur)
            strip = np.arange(nct) % 8
            by_strip = [round(float(np.median(dur[strip == q])) / 1e3, 2) for q in range(8)]
            die = sm % 2
            by_sm_parity = [round(float(np.median(dur[die == q])) / 1e3, 2) for q in range(2)]
            first_half = sm < 74
            by_sm_half = [round(float(np.median(dur[first_half])) / 1e3, 2), round(float(np.median(dur[~first_half])) / 1e3, 2)]
            pos = np.arange(nct) // 8
            corr_pos = float(np.corrcoef(pos, dur)[0, 1]) if nct > 2 else None
            bidx = np.arange(nct)
            nsm = int(sm.max()) + 1
            by_wave = [round(float(np.median(dur[(bidx >= w * nsm) & (bidx < (w + 1) * nsm)])) / 1e3, 2)
                       for w in range((nct + nsm - 1) // nsm)]
            # order of the CTA on its SM by entry time (0 = first resident)
            rank = np.zeros(nct, dtype=int)
            for q in np.unique(sm):
                ids = np.flatnonzero(sm == q)
                rank[ids[np.argsort(tk[ids, 0], kind="stable")]] = np.arange(len(ids))
            by_rank = [round(float(np.median(dur[rank == q])) / 1e3, 2) for q in range(int(rank.max()) + 1)]
            same_wave_sm = float(np.mean(sm[:nsm] == np.arange(nsm))) if nct >= nsm else None
            res[name] = {"ctas": int(used.sum()),
                         "entry_us": [round((np.percentile(tk[:, 0], q) - t0) / 1e3, 2) for q in (0, 50, 100)],
                         "stream_end_us": [round((np.percentile(tk[:, 1], q) - t0) / 1e3, 2) for q in (0, 50, 100)],
                         "arrive_us": [round((np.percentile(tk[:, 2], q) - t0) / 1e3, 2) for q in (0, 50, 100)],
                         "finaliser_done_us": round((fin.max() - t0) / 1e3, 2) if len(fin) else None,
                         "stream_us_median_by_ctas_on_sm": by_load,
                         "stream_us_median_by_block_wave": by_wave,
                         "stream_us_median_by_order_on_sm": by_rank,
                         "frac_of_first_nsm_ctas_on_sm_equal_block_id": same_wave_sm,
                         "sm_of_blocks_0_10_148_150_296_300": [int(sm[i]) for i in (0, 10, 148, 150, 296, 300) if i < nct],
                         "stream_us_median_by_strip": by_strip,
                         "stream_us_median_by_sm_parity": by_sm_parity,
                         "stream_us_median_sm_lt74_ge74": by_sm_half,
                         "corr_stream_time_vs_range_index_in_strip": round(corr_pos, 3) if corr_pos is not None else None,
                         "stream_us_pct_0_10_50_90_100": [round(float(np.percentile(dur, q)) / 1e3, 2) for q in (0, 10, 50, 90, 100)],
                         "t0": t0, "fin_abs": float(fin.max()) if len(fin) else None}
        k1, k23 = res["K1 k_iter1_s5p"], res["K2+K3 k_iter23_s5"]
        # the last K1 launch precedes the last K2+K3 launch of the solve (same iteration)
        gap = (k23["t0"] - k1["fin_abs"]) / 1e3 if k1["fin_abs"] else None
        for v in res.values():
            v.pop("t0"); v.pop("fin_abs")
        res["gap_K1_finaliser_to_K23_first_entry_us"] = round(gap, 2) if gap is not None else None
        out[f"solve{rep}"] = res
    L.check(L.lib().sg_pcg_set_trace(h._h, None))
    print(json.dumps({"probe": "C5 strip kernel timeline (percentiles 0/50/100 relative to the first CTA entry)",
                      "iters": a.iters, **out}, indent=1))


if __name__ == "__main__":
    main()
