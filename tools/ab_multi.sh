#!/bin/bash
# A/B/C... of engine builds in several trees (run on the GPU box), alternating: the C3 phases
# (bench.py kernel-only) and the chain-bound timings (tools/ab_small.py).
# usage: TREES=". _ab/head _ab/v1" tools/ab_multi.sh [rounds]
R=${1:-2}
for i in $(seq 1 $R); do
  for tree in ${TREES:-. _ab/head}; do
    (cd $tree && python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-e2e --no-single --no-latency 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tree', round(d['value'],1), {k: round(v,2) for k,v in d['phases_ms_per_step'].items()})")
    (cd $tree && python $OLDPWD/tools/ab_small.py $tree)
  done
done
