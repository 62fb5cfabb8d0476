# Interleaved timing of the headline kernel's tuning variants (CLV_ANNEAL_VARIANT) on one GPU.
for r in 1 2; do for v in ${VARIANTS:-0 1 3 4}; do CLV_ANNEAL_VARIANT=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('variant $v', d['value'], round(d['ms_per_step'],4))"; done; done
