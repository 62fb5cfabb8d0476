#!/bin/bash
# Run on the GPU box: bench line, launch list, one full ncu capture of the chain kernel
# and the per-phase cycle profile.  Outputs land in gpurun_out/ (summarise into profiles/).
# TAG names the outputs (e.g. r02b).
set -x
TAG=${TAG:-prof}
mkdir -p gpurun_out
python -m paper_2304_09781_b200.build
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-replan > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 3000 gpurun_out/${TAG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:anneal -s 3 -c 1 \
    -o gpurun_out/${TAG}_anneal -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full_run.log 2>&1
CLV_ANNEAL_VARIANT=9 timeout 300 python tools/phase_profile.py > gpurun_out/${TAG}_phase_profile.txt 2>&1
cat gpurun_out/${TAG}_phase_profile.txt
ls -la gpurun_out
