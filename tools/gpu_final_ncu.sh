#!/bin/bash
# ncu --set full of one config-D step's kernels (one launch of each kind after warm-up)
set -x
mkdir -p gpurun_out
O=gpurun_out/final
timeout 1500 ncu --set full --import-source on --clock-control none --launch-skip 190 -c 70 -o ${O}_ncu_D python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > ${O}_ncu_D.log 2>&1; echo "ncu_full=$?" >> ${O}_status_ncu.txt
