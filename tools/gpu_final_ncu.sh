#!/bin/bash
# ncu --set full of one training step's kernels (the 3rd hg_train_step after warm-up) at one workload
#   bash tools/gpu_final_ncu.sh WORKLOAD GRAPHS KERNELS_PER_STEP
set -x
W=$1; G=$2; K=$3
mkdir -p gpurun_out
O=gpurun_out/final_ncu_$W
timeout 600 python bench.py --workload $W --graphs $G --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > ${O}_plain.json 2> ${O}_plain.err; echo "plain=$?" > ${O}_status.txt
timeout 1800 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "hg_train_step/" --launch-skip $((2 * K)) -c $K -o ${O} python bench.py --workload $W --graphs $G --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > ${O}.log 2>&1; echo "ncu=$?" >> ${O}_status.txt
