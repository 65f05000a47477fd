#!/bin/bash
# One A/B pass of a kernel change against _ab/head (run on the GPU box): bitwise records on two
# shapes, the C3 phases alternated, the chain-bound timings. Output prefix $1 under gpurun_out/.
P=gpurun_out/${1:-ab}
python tools/ab_bitwise.py > ${P}_bw.txt 2>&1
python tools/ab_bitwise.py 1000 3 60 >> ${P}_bw.txt 2>&1
bash tools/ab_bench.sh ${2:-3} > ${P}_ab.txt 2>&1
for i in 1 2; do python tools/ab_small.py . ; (cd _ab/head && python ../../tools/ab_small.py head); done > ${P}_abs.txt 2>&1
cat ${P}_bw.txt ${P}_ab.txt ${P}_abs.txt
