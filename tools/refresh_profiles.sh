# Round refresh of the committed evidence (run on the GPU box from the repo root):
# the bench line, all BASELINE configs, the batch-size sweep, the ncu launch list of the bench
# command and one full ncu capture of chol_dag (each ncu command after its plain run exited 0).
set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python tools/all_configs.py > gpurun_out/configs.log 2>&1
python tools/batch_sweep.py > gpurun_out/batch_sweep.txt 2>&1
python bench.py --steps 1 --warmup 1 --no-fit --no-cpu-baseline --no-e2e > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-fit --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chol_dag_kernel -c 1 -o gpurun_out/chol_dag_c3 python bench.py --steps 1 --warmup 1 --no-fit --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
