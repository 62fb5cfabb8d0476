"""Per-phase cycle profile of the chain kernel (CLV_ANNEAL_VARIANT=9 build variant): cycles per step by phase."""
import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, torch, time, ctypes, os
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
from paper_2304_09781_b200.objective import AnnealParams
from paper_2304_09781_b200 import _native as N
import bench
eng=CloverEngine(n_max=64); prof=synthetic_profile('efficientnet')
sc=eng.calibrate(prof,64,350.0,0.5)
st=bench.make_starts(eng,prof,bench.SEED,0,128)
ap=AnnealParams(max_steps=64)
lib=N.load(); lib.clv_debug_anneal_profile.argtypes=[ctypes.c_void_p, ctypes.c_size_t]
for cl in (3,):
    b=eng.anneal(st,prof,sc,ap,1,cluster=cl); torch.cuda.synchronize()
    nb=len(st)*cl
    buf=np.zeros(nb*8,dtype=np.int64); lib.clv_debug_anneal_profile(buf.ctypes.data, nb*8)
    buf=buf.reshape(len(st),cl,8)
    names=["prepare","score","cta_reduce","sync1","leader","sync2","apply"]
    lead=buf[:,0,:7].mean(0)/64; other=buf[:,1,:7].mean(0)/64
    nref = -(buf[:,0,6] // 1000000)        # refresh steps are counted in the 'apply' slot (-1e6 each)
    buf[:,:,6] = buf[:,:,6] % 1000000
    print("refresh steps per chain (of 64):", float(nref.mean()), " prepare cycles per refresh step:",
          int(buf[:,0,7].sum() / max(nref.sum(), 1)), " per other step:",
          int((buf[:,0,0].sum() - buf[:,0,7].sum()) / max(64 * len(buf) - nref.sum(), 1)))
    print("cluster",cl,"cycles/step leader:", {k:int(v) for k,v in zip(names,lead)}, "\n  rank1:", {k:int(v) for k,v in zip(names,other)})

