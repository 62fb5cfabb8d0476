#!/bin/bash
# Run on the GPU box: every bench workload + the reference arm; one JSON line each in gpurun_out/${TAG}_*.json
TAG=${TAG:-all}
mkdir -p gpurun_out
python -m paper_2304_09781_b200.build > /dev/null
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | grep "Model name" >> gpurun_out/${TAG}_nproc.txt
for w in ${WORKLOADS:-c0 c1 c4 c3}; do
  if [ $w = c3 ]; then A="--steps 1 --warmup 0"; else A="--steps 5 --warmup 3"; fi
  timeout 1200 python bench.py --workload $w $A > gpurun_out/${TAG}_$w.json 2> gpurun_out/${TAG}_$w.err
done
if [ -n "$WITH_C2" ]; then
  timeout 900 python bench.py > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err
  timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
  timeout 600 python tools/bench_kernels.py > gpurun_out/${TAG}_kernels.json 2> gpurun_out/${TAG}_kernels.err
fi
for f in gpurun_out/${TAG}_*.json; do echo "== $f"; tail -c 1500 $f; echo; done
for f in gpurun_out/${TAG}_*.err; do echo "== $f"; tail -5 $f; done
