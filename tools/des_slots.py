"""Time the serving DES with register-resident keys vs the shared-memory group layout
for several fleet sizes (CLV_SIM_SLOTS caps the register slots per lane)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, %r)
from paper_2304_09781_b200 import sim as S
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
from paper_2304_09781_b200.search import base_config, random_fleets
eng = CloverEngine(n_max=64); prof = synthetic_profile("efficientnet")
for n in (2, 4, 8, 16, 64):
    fl = random_fleets(eng, prof, n, 3, 1024, 0)
    e = [S.fleet_instances(f, prof) for f in fl]
    off = np.concatenate([[0], np.cumsum([len(x) for x in e])]).astype(np.int64)
    rate = S.calibrate_arrival_rate(base_config(n, prof), prof, 0.7)
    w = S.Workload(rate, 60.0, 5)
    inst = torch.from_numpy(np.concatenate(e)).cuda(); offd = torch.from_numpy(off).cuda()
    eng.simulate(inst, offd, prof, w, counts=False); torch.cuda.synchronize()
    t0 = time.time(); r = eng.simulate(inst, offd, prof, w, counts=False); torch.cuda.synchronize()
    print("n=%%d kmax=%%d requests=%%d ms=%%.1f" %% (n, int(np.diff(off).max()), r[3], 1000 * (time.time() - t0)))
''' % ROOT
for cap in ("0", "16"):
    print("CLV_SIM_SLOTS=" + cap, flush=True)
    subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, CLV_SIM_SLOTS=cap))
