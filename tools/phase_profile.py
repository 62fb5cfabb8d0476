"""Per-phase cycle profile of the chain kernel (build variant CLV_ANNEAL_VARIANT=9).

Prints the mean cycles per chain step of each phase for the leader CTA and one
other CTA of the cluster, and how often the slice-delta feasibility refresh runs.
Run on the GPU box:  CLV_ANNEAL_VARIANT=9 python tools/phase_profile.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2304_09781_b200 import _native as N  # noqa: E402
from paper_2304_09781_b200.engine import CloverEngine  # noqa: E402
from paper_2304_09781_b200.objective import AnnealParams  # noqa: E402
from paper_2304_09781_b200.profiles import synthetic_profile  # noqa: E402

SLOTS = 20
NAMES = ["prepare", "score", "cta_reduce", "sync1", "leader", "sync2", "apply"]

eng = CloverEngine(n_max=64)
prof = synthetic_profile("efficientnet")
sc = eng.calibrate(prof, bench.N_FLEET, bench.CI, bench.LAMBDA)
st = bench.make_starts(prof, bench.SEED, 0, 128, 0.75)
ap = bench.anneal_params(256)
lib = N.load()
lib.clv_debug_anneal_profile.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
cl = int(os.environ.get("CLV_PROFILE_CLUSTER", "2"))   # the auto size at 128 chains
b = eng.anneal(st, prof, sc, ap, 1, cluster=cl)
torch.cuda.synchronize()
steps = b.host()["results"]["steps"].astype(np.float64)
nb = len(st) * cl
buf = np.zeros(nb * SLOTS, dtype=np.int64)
lib.clv_debug_anneal_profile(buf.ctypes.data, nb * SLOTS)
buf = buf.reshape(len(st), cl, SLOTS)
per_step = lambda x: x.sum() / steps.sum()
lead = {k: int(per_step(buf[:, 0, q])) for q, k in enumerate(NAMES)}
other = {k: int(per_step(buf[:, 1, q])) for q, k in enumerate(NAMES)}
nref = buf[:, 0, 8].sum()
print("cluster %d cycles/step leader CTA: %s\n  rank-1 CTA: %s" % (cl, lead, other))
print("leader: apply_move %d cycles per step" % per_step(buf[:, 0, 9]))
print("prepare: refresh + pair count + scans %d, entry build + singles %d cycles per step"
      % (per_step(buf[:, 0, 10]), per_step(buf[:, 0, 11])))
print("prepare part 1: refresh + present-edge list + pair prefix %d | pair decode + thread scan %d | warp scan %d"
      % (per_step(buf[:, 0, 12]), per_step(buf[:, 0, 13]), per_step(buf[:, 0, 14])))
print("  of which thread 0 until the present-edge list starts (refresh issue / wait) %d" % per_step(buf[:, 0, 15]))
print("feasibility refresh in %.1f%% of steps; prepare cycles per refresh step %d, per other step %d"
      % (100.0 * nref / steps.sum(), buf[:, 0, 7].sum() / max(nref, 1),
         (buf[:, 0, 0].sum() - buf[:, 0, 7].sum()) / max(steps.sum() - nref, 1)))
surv = buf[:, :, 16].sum()
ev = b.host()["results"]["evals"].astype(np.float64).sum()
print("screen: %d double moves scored in full of %d candidates (%.2f%%)" % (surv, ev, 100.0 * surv / ev))
print("  of which singles / unit moves (warm-up): %d" % buf[:, :, 19].sum())
print("leader: record merge %d, decision until apply %d cycles per step" % (per_step(buf[:, 0, 17]), per_step(buf[:, 0, 18])))
