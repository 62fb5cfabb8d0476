#!/bin/bash
# GPU box, one development iteration: -m gpu suite, bench line (with the 16-chain oracle parity leg), phase profile.
TAG=${TAG:-it}
mkdir -p gpurun_out
python -m paper_2304_09781_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 600 python bench.py --no-cpu-replan ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
CLV_ANNEAL_VARIANT=9 timeout 300 python tools/phase_profile.py > gpurun_out/${TAG}_phase.txt 2>&1
tail -4 gpurun_out/${TAG}_gputest.log
python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
print("value %.4g e2e %.4g ms/step %.3f parity %s quality %s" % (d["value"], d["e2e"]["value"], d["ms_per_step"], d["parity"], d["replan_quality"]))
PY
tail -c 400 gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_phase.txt
