import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
from paper_2304_09781_b200 import search as S
eng = CloverEngine(n_max=64); prof = synthetic_profile("efficientnet")
sc = eng.calibrate(prof, bench.N_FLEET, bench.CI, bench.LAMBDA)
ap = bench.anneal_params(64)
st = [bench.make_starts(prof, bench.SEED, i * 128, 128, 0.75) for i in range(12)]
for i in range(3): S.anneal_chains(eng, st[i], prof, sc, ap, i, cluster=0)
torch.cuda.synchronize()
ev = torch.cuda.Event(enable_timing=True)
for i in range(3, 8):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    r = S.anneal_chains(eng, st[i], prof, sc, ap, i, cluster=0)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("wall %.3f ms  device(e0..e1) %.3f ms" % ((t1 - t0) * 1e3, e0.elapsed_time(e1)))
# device-only anneal + select
d = torch.from_numpy(st[3].view(np.int16)).cuda().view(torch.uint16)
for i in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); b = eng.anneal(d, prof, sc, ap, 3, cluster=0); e1.record(); torch.cuda.synchronize()
    print("anneal only %.3f ms" % e0.elapsed_time(e1))
