#!/bin/bash
# A/B the DAG kernel: bench.py (kernel-only phases) of the working tree vs _ab/head, alternating.
# usage (on the GPU box): tools/ab_bench.sh [rounds]
R=${1:-3}
for i in $(seq 1 $R); do
  for tree in ${TREES:-. _ab/head}; do
    (cd $tree && python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-e2e --no-single --no-latency 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tree', round(d['value'],1), {k: round(v,2) for k,v in d['phases_ms_per_step'].items()})")
  done
done
