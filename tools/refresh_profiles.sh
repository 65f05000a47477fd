set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python tools/all_configs.py > gpurun_out/configs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-fit --no-cpu-baseline --no-e2e --no-single > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chol_dag_kernel -c 1 -o gpurun_out/chol_dag_c3 python bench.py --steps 1 --warmup 1 --no-fit --no-cpu-baseline --no-e2e --no-single > gpurun_out/ncu_full.log 2>&1
