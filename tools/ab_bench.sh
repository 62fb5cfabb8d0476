#!/bin/bash
# A/B timing of alternative builds of libclover_b200.so on one GPU, interleaved so clock
# drift hits both arms alike:  tools/ab_bench.sh ROUNDS lib_a.so lib_b.so ... [-- bench args]
# Prints "<lib> value ms_per_step e2e" per run.
rounds=$1; shift
libs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done
[ "$1" = "--" ] && shift
for r in $(seq "$rounds"); do
  for l in "${libs[@]}"; do
    CLV_LIB_PATH=$(realpath "$l") python bench.py --steps 20 --warmup 5 "$@" 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$l', d['value'], round(d['ms_per_step'],4), d['e2e']['value'])"
  done
done
