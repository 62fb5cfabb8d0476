#!/bin/bash
# GPU box: sanitizer runs, the launch list of the headline bench command and one ncu --set full
# capture of the chain kernel (outputs in gpurun_out/, summarised into profiles/ by the caller).
TAG=${TAG:-final}
mkdir -p gpurun_out
python -m paper_2304_09781_b200.build > /dev/null
bash tools/sanitize.sh > gpurun_out/${TAG}_sanitize.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:anneal -s 3 -c 1 \
    -o gpurun_out/${TAG}_anneal -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full_run.log 2>&1
CLV_ANNEAL_VARIANT=9 timeout 300 python tools/phase_profile.py > gpurun_out/${TAG}_phase.txt 2>&1
cat gpurun_out/${TAG}_sanitize.log; cat gpurun_out/${TAG}_phase.txt; ls -la gpurun_out | grep ${TAG}
