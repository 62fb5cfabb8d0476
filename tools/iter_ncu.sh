#!/bin/bash
# GPU box: iteration (tests + bench + phase profile) and one ncu --set full capture of the chain kernel.
TAG=${TAG:-it}
bash tools/iter.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:anneal -s 3 -c 1 \
    -o gpurun_out/${TAG}_anneal -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full_run.log 2>&1
ls -la gpurun_out | tail -3
