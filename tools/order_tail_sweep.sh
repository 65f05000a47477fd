# C3 DRAM bytes and time per chol_dag launch vs the ticket-order tail fraction (GPEMU_ORDER_TAIL)
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-fit --no-e2e --no-latency > /dev/null 2>&1 || exit 1
for t in ${TAILS:-0.4 0.5 0.55 0.7}; do
  echo "tail $t"
  GPEMU_ORDER_TAIL=$t ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:chol_dag -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-fit --no-e2e --no-latency 2>&1 | grep -E "dram__|gpu__time|lts__t_sector_hit"
done
for i in 1 2; do for t in ${TAILS:-0.4 0.5 0.55 0.7}; do
  GPEMU_ORDER_TAIL=$t python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-fit --no-e2e --no-latency | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['value'],1), round(d['phases_ms_per_step']['cholesky'],3))"
done; done
