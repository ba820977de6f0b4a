#!/bin/bash
# ncu of one config's training step (the 3rd hg_train_step after warm-up):
#   bash tools/gpu_final_ncu.sh WORKLOAD GRAPHS KERNELS_PER_STEP lite   every kernel, metric sections only
#   bash tools/gpu_final_ncu.sh WORKLOAD GRAPHS KERNELS_PER_STEP full   --set full + source, top kernels
set -x
W=$1; G=$2; K=$3; MODE=$4
mkdir -p gpurun_out
O=gpurun_out/final_ncu_${W}_${MODE}
timeout 600 python bench.py --workload $W --graphs $G --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > ${O}_plain.json 2> ${O}_plain.err; echo "plain=$?" > ${O}_status.txt
if [ "$MODE" = lite ]; then
  timeout 1800 ncu --section SpeedOfLight --section LaunchStats --section Occupancy --section SchedulerStats \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,smsp__inst_executed.sum \
    --clock-control none --nvtx --nvtx-include "hg_train_step/" --launch-skip $((2 * K)) -c $K -o ${O} \
    python bench.py --workload $W --graphs $G --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > ${O}.log 2>&1
elif [ "$MODE" = fwd ]; then
  timeout 1800 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "hg_train_step/" \
    -k regex:"k_agg_fwd|TUpdC|MnGram" --launch-skip 2 -c 12 -o ${O} \
    python bench.py --workload $W --graphs $G --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > ${O}.log 2>&1
else
  timeout 1800 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "hg_train_step/" \
    -k regex:"k_agg_fwd|k_agg_bwd|TUpdC|MnGram|k_dxda" --launch-skip 10 -c 5 -o ${O} \
    python bench.py --workload $W --graphs $G --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > ${O}.log 2>&1
fi
echo "ncu=$?" >> ${O}_status.txt
ls -la ${O}*
