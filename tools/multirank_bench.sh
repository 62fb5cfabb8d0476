#!/bin/bash
# GPU box (one device): the N>1 bench path end to end -- 2 ranks on cuda:0 over gloo (NCCL needs one
# device per rank), each workload's JSON line from rank 0.
mkdir -p gpurun_out
python -m paper_2304_09781_b200.build > /dev/null
export CLV_DIST_BACKEND=gloo
for w in c2 c0 c4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
      bench.py --gpus 2 --workload $w --steps 3 --warmup 3 --sweep 100000000 > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "== $w rc=$?"; tail -c 700 gpurun_out/mr_$w.json; tail -3 gpurun_out/mr_$w.err
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/mr_smoke.log 2>&1; tail -2 gpurun_out/mr_smoke.log
