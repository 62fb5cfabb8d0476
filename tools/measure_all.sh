#!/bin/bash
# Run on the GPU box: every bench workload + the reference arm; one JSON line each in gpurun_out/all_*.json
mkdir -p gpurun_out
python -m paper_2304_09781_b200.build > /dev/null
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/all_c2.json 2> gpurun_out/all_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/all_ref.json 2> gpurun_out/all_ref.err
for w in c0 c1 c4 des; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/all_$w.json 2> gpurun_out/all_$w.err
done
timeout 900 python bench.py --workload c3 --steps 1 --warmup 0 > gpurun_out/all_c3.json 2> gpurun_out/all_c3.err
timeout 600 python tools/bench_kernels.py > gpurun_out/all_kernels.json 2> gpurun_out/all_kernels.err
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
for f in gpurun_out/all_*.json; do echo "== $f"; tail -c 600 $f; echo; done
