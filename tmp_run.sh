mkdir -p gpurun_out
bash tools/sanitize.sh
(timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2a.log 2>&1 &)
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2b.log 2>&1
sleep 8
grep -c "launch failure" gpurun_out/c2a.log gpurun_out/c2b.log; grep -o '"value": [0-9.e+]*' gpurun_out/c2a.log gpurun_out/c2b.log
CLV_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/mr.log 2>&1
grep metric gpurun_out/mr.log | tail -c 1200
