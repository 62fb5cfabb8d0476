"""Per-kernel throughput / roofline numbers outside the headline bench (run on the GPU box).

score_graphs : materialized uint16 graphs streamed from HBM (HBM roofline, 70 B/candidate at V=7)
score_x      : materialized FleetConfig CSR rows (n + m bytes per candidate)
oracle       : c0 exhaustive enumeration (generated candidates)
sweep        : c4 counter-RNG two-pod sweep (generated candidates)
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09781_b200.engine import CloverEngine  # noqa: E402
from paper_2304_09781_b200.profiles import synthetic_profile  # noqa: E402
from paper_2304_09781_b200.search import random_fleets  # noqa: E402
from paper_2304_09781_b200.graph import build_graph  # noqa: E402

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
    if os.path.exists("MEASURED_PEAKS.json") else {"hbm_gbs": 6550.7}


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    eng = CloverEngine(n_max=64)
    prof = synthetic_profile("efficientnet")
    out = []
    # --- score_graphs from HBM: 50M graphs (3.5 GB), n=64
    n = 64
    sc = eng.calibrate(prof, n, 350.0, 0.5)
    base = np.array([build_graph(f, prof).weights for f in random_fleets(eng, prof, n, 5, 4096)], dtype=np.uint16)
    count = 50_000_000
    W = torch.from_numpy(base.view(np.int16)).cuda().view(torch.uint16).repeat(count // 4096 + 1, 1)[:count].contiguous()
    ms = timeit(lambda: eng.score_graphs(W, prof, sc, outputs=False), reps=5)
    bytes_ = count * W.shape[1] * 2
    out.append({"kernel": "score_graphs", "candidates": count, "ms": ms, "candidates_per_s": count / ms * 1e3,
                "GB_per_s": bytes_ / ms / 1e6, "hbm_peak_GBps": PEAKS["hbm_gbs"],
                "frac": bytes_ / ms / 1e6 / PEAKS["hbm_gbs"], "bytes_per_candidate": W.shape[1] * 2})
    del W
    # --- score_x from HBM: 1M FleetConfig CSR rows of an n=64 fleet (xp n B + xv m B + 8 B offset)
    fl = random_fleets(eng, prof, n, 9, 4096, 0)
    reps = 256
    xp1 = np.array([f.partitions for f in fl], dtype=np.uint8)
    xv1 = [np.array(f.assignments, dtype=np.uint8) for f in fl]
    xp = np.tile(xp1, (reps, 1))
    xvs = xv1 * reps
    xv = np.concatenate(xvs)
    off = np.zeros(len(xvs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(x) for x in xvs])
    xp_d, xv_d, off_d = torch.from_numpy(xp).cuda(), torch.from_numpy(xv).cuda(), torch.from_numpy(off).cuda()
    cnt = len(xvs)
    ms = timeit(lambda: eng.score_x(xp_d, xv_d, off_d, n, prof, sc, outputs=False), reps=5)
    bytes_ = xp.nbytes + xv.nbytes + off.nbytes
    out.append({"kernel": "score_x", "candidates": cnt, "ms": ms, "candidates_per_s": cnt / ms * 1e3,
                "GB_per_s": bytes_ / ms / 1e6, "hbm_peak_GBps": PEAKS["hbm_gbs"],
                "frac": bytes_ / ms / 1e6 / PEAKS["hbm_gbs"], "bytes_per_candidate": bytes_ / cnt})
    # --- oracle c0
    sc1 = eng.calibrate(prof, 1, 400.0, 0.5)
    tot = eng.oracle_size(prof)
    ms = timeit(lambda: eng.oracle_search(prof, sc1))
    out.append({"kernel": "oracle", "candidates": tot, "ms": ms, "candidates_per_s": tot / ms * 1e3})
    # --- sweep c4 (two 128-GPU pods)
    pr, pb = synthetic_profile("resnet"), synthetic_profile("bert")
    sr, sb = eng.calibrate(pr, 128, 300.0, 0.5), eng.calibrate(pb, 128, 300.0, 0.5)
    pods = [(pr, sr, 128, 0.5), (pb, sb, 128, 0.5)]
    cnt = 20_000_000
    ms = timeit(lambda: eng.sweep(pods, 0, cnt, 1), reps=3, warm=1)
    out.append({"kernel": "sweep_2pods_n256", "candidates": cnt, "ms": ms, "candidates_per_s": cnt / ms * 1e3,
                "projected_1e9_s": 1e9 / (cnt / ms * 1e3)})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
