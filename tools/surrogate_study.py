"""Design study for the p95 surrogate (CPU only): compare candidate table models of the
fleet p95 with the SPEC's serving simulator (oracle/des.py) on fleets that straddle
L_tail.  Populations: random realizable fleets and biased draws from BASE-like
(large slices, large variants) to random.  Usage: python tools/surrogate_study.py [n] [fleets]
"""

import json
import math
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import des as D  # noqa: E402
from oracle.rng import Stream, derive_seed  # noqa: E402
from oracle.search import feasible_lists, row_kinds  # noqa: E402
from oracle.tables import OracleTables  # noqa: E402
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY  # noqa: E402
from paper_2304_09781_b200.profiles import synthetic_profile  # noqa: E402

FAM = os.environ.get("FAM", "efficientnet")
PROF = synthetic_profile(FAM)
T = OracleTables.from_profile(PROF)
CB = 0.0
SIM = D.sim_input(PROF)


def draw(i, n, p_big, p_top):
    st = Stream(derive_seed(99, i))
    ids = DEFAULT_TOPOLOGY.config_ids
    fl = feasible_lists(T)
    inst = []
    for _g in range(n):
        cid = ids[0] if st.bounded(1000) < p_big * 1000 else ids[st.bounded(len(ids))]
        for k in row_kinds(DEFAULT_TOPOLOGY, cid):
            lst = fl[k]
            v = lst[-1] if st.bounded(1000) < p_top * 1000 else lst[st.bounded(len(lst))]
            inst.append((v - 1) * 5 + k)
    return inst


def des_p95(args):
    inst, R, dur = args
    return D.simulate(inst, SIM, R, dur, 230409781).p95_ms


def models(inst, R):
    E = T.E
    w = np.bincount(np.array(inst), minlength=E).astype(np.float64)
    mean = np.array([SIM.edges[e].mean_ms for e in range(E)])
    lat = np.asarray(T.lat95, dtype=np.float64)
    thr = 1000.0 / mean
    M = (w * thr).sum()
    m = w.sum()
    rho = min(R / M, 0.999)
    fac = 1.0 + rho ** 8 / (m * (1.0 - rho))
    present = w > 0
    out = {"lmax": lat[present].max() * fac}

    def quant(share):
        order = np.argsort(lat, kind="stable")
        tot = share.sum()
        acc = 0.0
        for e in order:
            if share[e] <= 0:
                continue
            acc += share[e]
            if 20.0 * (tot - acc) <= tot:
                return lat[e]
        return lat[order[-1]]
    out["thr_q"] = quant(w * thr) * fac
    out["cnt_q"] = quant(w) * fac
    # DES-like shares: rate_j = 1 / (s_j + W), sum = R (longest-idle-first dispatch)
    if R >= M:
        out["idle_q"] = out["thr_q"]
    else:
        lo, hi = 0.0, 1e6
        for _ in range(80):
            Wm = 0.5 * (lo + hi)
            if (w * 1000.0 / (mean + Wm)).sum() > R:
                lo = Wm
            else:
                hi = Wm
        out["idle_q"] = quant(w / (mean + lo)) * fac
    out["rho"] = R / M
    c = CB
    out["c_q"] = quant(w / (mean + c)) * fac
    W0 = max(m / R * 1000.0 - m / M * 1000.0, 0.0)
    out["w0_q"] = quant(w / (mean + W0)) * fac
    order = np.argsort(lat, kind="stable")[::-1]
    t = 0.0
    kq = None
    for e in order:
        if w[e] <= 0:
            continue
        t += 1000.0 * w[e] / (mean[e] + W0)
        if 20.0 * t > R:
            kq = e
            break
    if kq is None:
        kq = [e for e in order if w[e] > 0][-1]
    out["w0R_q"] = lat[kq] * fac
    # stochastic families: mixture quantile with the same shares (rate_j / R)
    share = 1000.0 * w / (mean + W0) / R
    dist = SIM.edges[0].dist
    sig = SIM.edges[0].sigma
    from math import erfc, log, sqrt, exp
    def surv(e, L):
        if dist == 0:
            return 1.0 if mean[e] > L else 0.0
        if dist == 1:
            return exp(-L / mean[e])
        mu = log(mean[e]) - 0.5 * sig * sig
        return 0.5 * erfc((log(L) - mu) / (sig * sqrt(2.0)))
    if dist == 0:
        out["mix_exact"] = out["w0R_q"]
        out["mix_edge"] = out["w0R_q"]
    else:
        lo, hi = 1e-3, 1e5
        for _ in range(100):
            mid = sqrt(lo * hi)
            t = sum(share[e] * surv(e, mid) for e in range(E) if w[e] > 0)
            if t > 0.05:
                lo = mid
            else:
                hi = mid
        out["mix_exact"] = hi * fac
        # boundary edge + within-edge conditional quantile
        Tprev = 0.0
        val = None
        for e in order:
            if w[e] <= 0:
                continue
            if Tprev + share[e] > 0.05:
                p = 1.0 - (0.05 - Tprev) / share[e]
                if dist == 1:
                    val = mean[e] * (-log(1.0 - p))
                else:
                    from statistics import NormalDist
                    mu = log(mean[e]) - 0.5 * sig * sig
                    val = exp(mu + sig * NormalDist().inv_cdf(p))
                break
            Tprev += share[e]
        if val is None:
            val = lat[order[-1]]
        out["mix_edge"] = val * fac
    return out


def spearman(a, b):
    from scipy.stats import spearmanr
    return float(spearmanr(a, b).statistic)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 160
    dur = float(os.environ.get("DUR", "600"))
    V = T.V
    R = 0.7 * n * 1000.0 / SIM.edges[(V - 1) * 5].mean_ms
    base = [(V - 1) * 5] * n
    pops = []
    for i in range(N):
        p_big = 0.5 + 0.5 * (i % 8) / 8.0
        p_top = 0.5 + 0.5 * ((i // 8) % 5) / 5.0
        pops.append(draw(i, n, p_big, p_top))
    with mp.Pool(8) as pool:
        des = pool.map(des_p95, [(base, R, dur)] + [(f, R, dur) for f in pops])
    lt_des = des[0]
    dP = np.array(des[1:])
    res = {"n": n, "fleets": N, "R": R, "l_tail_des": lt_des, "des_meet": int((dP <= lt_des).sum())}
    global CB
    s_b = SIM.edges[(V - 1) * 5].mean_ms
    CB = s_b * (1.0 - 0.7) / 0.7
    mb = models(base, R)
    ms = [models(f, R) for f in pops]
    for key in ("lmax", "thr_q", "cnt_q", "idle_q", "c_q", "w0_q", "w0R_q", "mix_exact", "mix_edge"):
        L = np.array([x[key] for x in ms])
        s_s = L <= mb[key]
        s_d = dP <= lt_des
        res[key] = {"spearman": spearman(L, dP), "sla_agree": float(np.mean(s_s == s_d)),
                    "surr_meet": int(s_s.sum()), "both": int((s_s & s_d).sum()),
                    "surr_only": int((s_s & ~s_d).sum()), "des_only": int((~s_s & s_d).sum()),
                    "med_rel_err": float(np.median(np.abs(L - dP) / dP)), "l_tail": float(mb[key])}
        under = np.array([x["rho"] for x in ms]) < 0.95
        res[key]["spearman_rho_lt_0.95"] = spearman(L[under], dP[under])
    res["underloaded"] = int(under.sum())
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
