import sys, numpy as np
from oracle.anneal import anneal_chain
from oracle.evaluator import calibrate, base_graph
from oracle.tables import OracleTables
from oracle.feasibility import FeasOracle
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200.profiles import synthetic_profile
eng = CloverEngine(n_max=8)
p = synthetic_profile("efficientnet"); T = OracleTables.from_profile(p); n = 8
feas = FeasOracle(DEFAULT_TOPOLOGY, n)
lams = [i / 10 for i in range(11)]
scs = [calibrate(p, T, n, 400.0, l) for l in lams]
starts = np.repeat(base_graph(7, n)[None, :], len(lams), axis=0)
ap = AnnealParams(max_steps=40)
for cl in (1, 4):
    host = eng.anneal(starts, p, scs, ap, 1234, n=n, cluster=cl, log=True).host()
    for c in range(3):
        out = anneal_chain(starts[c], n, T, scs[c], ap, 1234, c, feas, log=True)
        lg = host["log"][c]
        print("cluster", cl, "chain", c, "evals", host["results"][c]["evals"], out.evals)
        for k, row in enumerate(out.log):
            d = lg[k]
            flag = "" if (d["n_neighbours"] == row["n_neighbours"] and d["h"] == row["h"]) else "  <-- DIFF"
            print(k, d["n_neighbours"], row["n_neighbours"], d["h"], row["h"], d["accepted"], row["accepted"], flag)
