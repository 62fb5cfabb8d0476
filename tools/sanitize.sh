#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on a small chain batch (run on the GPU box)
PY='import sys; sys.path.insert(0,".")
import torch
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
from paper_2304_09781_b200.objective import AnnealParams
import bench
eng=CloverEngine(n_max=64); prof=synthetic_profile("efficientnet")
sc=eng.calibrate(prof,64,350.0,0.5)
st=bench.make_starts(prof,1,0,3,0.75)
for mode in ("best","uniform"):
    b=eng.anneal(st,prof,sc,AnnealParams(max_steps=3, proposal=mode),1,cluster=2)
b=eng.anneal(st,prof,sc,AnnealParams(max_steps=3, proposal="uniform", evaluate="proposal"),1,cluster=3)
b=eng.anneal(st,prof,sc,AnnealParams(max_steps=3, move_set="paper", cooling="multiplicative"),1,cluster=3)
best,_=eng.score_graphs(st,prof,sc)
eng.replan(st,prof,sc,AnnealParams(max_steps=3),1,cluster=0)
pr2=synthetic_profile("resnet"); s2=eng.calibrate(pr2,16,300.0,0.5)
eng.sweep([(pr2,s2,16,0.5),(prof,eng.calibrate(prof,16,300.0,0.5),16,0.5)],0,3000,7)
eng.oracle_search(prof, eng.calibrate(prof,1,400.0,0.5))
import numpy as np
from paper_2304_09781_b200.search import random_fleets
fl=random_fleets(eng,prof,64,9,300,0)
eng.score_fleets(fl,prof,sc)
for f in (fl[:5],):
    xp=np.array([x.partitions for x in f],dtype=np.uint8); xvs=[np.array(x.assignments,dtype=np.uint8) for x in f]
    xvs[3]=xvs[3][:-2]; xp[4,7]=99
    off=np.concatenate([[0],np.cumsum([len(x) for x in xvs])]).astype(np.int64)
    try: eng.score_x(xp,np.concatenate(xvs),off,64,prof,sc)
    except Exception as e: print("expected:", type(e).__name__, e)
torch.cuda.synchronize(); print("ok")'
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -c "$PY" > gpurun_out/sanitize_$tool.txt 2>&1
  tail -4 gpurun_out/sanitize_$tool.txt
done
