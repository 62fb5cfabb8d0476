#!/bin/bash
# GPU box: full -m gpu suite, smoke, default bench line and the 1024-chain c2 line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --chains 1024 --steps 5 --warmup 3 --no-cpu-replan > gpurun_out/bench1024.json 2> gpurun_out/bench1024.err
tail -3 gpurun_out/gputest.log; tail -2 gpurun_out/smoke.log; tail -c 2500 gpurun_out/bench.json; tail -c 1500 gpurun_out/bench1024.json
