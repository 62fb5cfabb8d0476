mkdir -p gpurun_out
for CL in 1 2; do
(timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --cluster $CL > gpurun_out/c${CL}a.log 2>&1 &)
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --cluster $CL > gpurun_out/c${CL}b.log 2>&1
sleep 8
echo "CL=$CL"; grep -c "launch failure" gpurun_out/c${CL}a.log gpurun_out/c${CL}b.log; grep -o '"value": [0-9.e+]*' gpurun_out/c${CL}a.log gpurun_out/c${CL}b.log
done
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
from paper_2304_09781_b200.objective import AnnealParams
import bench
eng=CloverEngine(n_max=64); prof=synthetic_profile('efficientnet')
sc=eng.calibrate(prof,64,350.0,0.5)
st=bench.make_starts(eng,prof,1,0,4)
b=eng.anneal(st,prof,sc,AnnealParams(max_steps=3),1,cluster=2)
torch.cuda.synchronize(); print('ok', b.host()['results']['evals'].sum())
" > gpurun_out/sync.log 2>&1
tail -8 gpurun_out/sync.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2304_09781_b200.engine import CloverEngine
from paper_2304_09781_b200.profiles import synthetic_profile
from paper_2304_09781_b200.objective import AnnealParams
import bench
eng=CloverEngine(n_max=64); prof=synthetic_profile('efficientnet')
sc=eng.calibrate(prof,64,350.0,0.5)
st=bench.make_starts(eng,prof,1,0,2)
b=eng.anneal(st,prof,sc,AnnealParams(max_steps=2),1,cluster=2)
torch.cuda.synchronize(); print('ok', b.host()['results']['evals'].sum())
" > gpurun_out/race.log 2>&1
tail -30 gpurun_out/race.log
