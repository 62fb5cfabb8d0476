"""Host-side profile of the e2e re-plan path (anneal_chains): wall time per re-plan vs device time, cProfile top entries."""
import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
from paper_2304_09781_b200.search import anneal_chains
eng = CloverEngine(n_max=64); prof = synthetic_profile("efficientnet")
sc = eng.calibrate(prof, bench.N_FLEET, bench.CI, bench.LAMBDA)
ap = bench.anneal_params(64)
st = [bench.make_starts(prof, bench.SEED, i * 128, 128, 0.75) for i in range(12)]
for i in range(3): anneal_chains(eng, st[i], prof, sc, ap, i)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(3, 12): anneal_chains(eng, st[i], prof, sc, ap, i)
torch.cuda.synchronize()
print("e2e per re-plan ms", (time.perf_counter() - t0) / 9 * 1000)
# device-only
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
d = torch.from_numpy(st[3].view(np.int16)).cuda().view(torch.uint16)
e0.record(); b = eng.anneal(d, prof, sc, ap, 3); e1.record(); torch.cuda.synchronize()
print("device anneal ms", e0.elapsed_time(e1))
pr = cProfile.Profile(); pr.enable()
for i in range(3, 12): anneal_chains(eng, st[i], prof, sc, ap, i)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
