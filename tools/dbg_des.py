import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
from test_gpu_des import random_fleets
from oracle import des
from paper_2304_09781_b200 import sim as S
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
eng = CloverEngine()
p = synthetic_profile('bert'); fl = random_fleets(p, 3, 6, 80); sim = des.sim_input(p)
w = S.Workload(90.0, 60.0, 1237)
refs = [des.simulate(des.fleet_edges(f), sim, 90.0, 60.0, 1237) for f in fl]
for trial in range(3):
    reps = S.simulate_fleets(fl, p, w, engine=eng)
    print('batch', trial, [(r.p95_ms == o.p95_ms, r.mean_latency_ms == o.mean_latency_ms, r.energy_wh_total == o.energy_wh_total) for r, o in zip(reps, refs)])
for c, f in enumerate(fl):
    r = S.simulate_fleets([f], p, w, engine=eng)[0]
    print('single', c, r.p95_ms, refs[c].p95_ms, r.mean_latency_ms, refs[c].mean_latency_ms)
