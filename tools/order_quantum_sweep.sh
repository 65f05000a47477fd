for q in ${QS:-0 25 50 100 200 400 800}; do
  echo "== Q=$q TAIL=$GPEMU_ORDER_TAIL"
  GPEMU_ORDER_Q=$q ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:chol_dag -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-fit --no-e2e --no-single --no-latency 2>&1 | grep -E "dram__|gpu__time|lts__t_sector_hit"
  for i in 1 2; do GPEMU_ORDER_Q=$q python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-fit --no-e2e --no-single --no-latency | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['phases_ms_per_step']['cholesky'],3))"; done
done
