python tools/ab_bitwise.py > gpurun_out/abw.txt 2>&1
python tools/ab_bitwise.py 1000 3 60 >> gpurun_out/abw.txt 2>&1
python tools/ab_bitwise.py 300 2 7 >> gpurun_out/abw.txt 2>&1
for i in 1 2; do python tools/ab_small.py . ; (cd _ab/head && python ../../tools/ab_small.py head); done > gpurun_out/abs.txt 2>&1
bash tools/ab_bench.sh 2 > gpurun_out/ab.txt 2>&1
