#!/bin/bash
# Round-end measurement set on one B200 (results under gpurun_out/final_*; copied to profiles/).
set -x
mkdir -p gpurun_out
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > ${O}_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > ${O}_pytest_gpu.log 2>&1; echo "pytest=$?" > ${O}_status.txt
timeout 600 python bench.py > ${O}_bench_B.json 2> ${O}_bench_B.err; echo "benchB=$?" >> ${O}_status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > ${O}_bench_reference.json 2> ${O}_bench_reference.err; echo "ref=$?" >> ${O}_status.txt
for w in D E256 E512; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --graphs 400000 > ${O}_bench_$w.json 2> ${O}_bench_$w.err; echo "bench$w=$?" >> ${O}_status.txt
done
for w in P55 P200 A; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > ${O}_bench_$w.json 2> ${O}_bench_$w.err; echo "bench$w=$?" >> ${O}_status.txt
done
timeout 600 python bench.py --precision tf32 --no-cpu-baseline > ${O}_bench_B_tf32.json 2> ${O}_bench_B_tf32.err; echo "benchBtf32=$?" >> ${O}_status.txt
timeout 600 python bench.py --workload E256 --precision tf32 --steps 20 --warmup 5 --no-cpu-baseline --graphs 400000 > ${O}_bench_E256_tf32.json 2> ${O}_bench_E256_tf32.err; echo "benchE256tf32=$?" >> ${O}_status.txt
timeout 600 python bench.py --workload E512 --precision tf32 --steps 20 --warmup 5 --no-cpu-baseline --graphs 400000 > ${O}_bench_E512_tf32.json 2> ${O}_bench_E512_tf32.err; echo "benchE512tf32=$?" >> ${O}_status.txt
for v in self scalers5 nodehead all; do
  timeout 600 python bench.py --variant $v --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > ${O}_bench_B_$v.json 2> ${O}_bench_B_$v.err; echo "benchB$v=$?" >> ${O}_status.txt
done
timeout 300 python tools/exp/timeline.py --graphs 20000 --B 128 > ${O}_timeline_B.txt 2>&1
timeout 300 python tools/exp/timeline.py --graphs 40000 --B 512 --dataset aisd > ${O}_timeline_D.txt 2>&1
# launch list (cold-cache, serialised) of one config-B step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches_B.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > ${O}_launches_B.log 2>&1; echo "ncu_launch=$?" >> ${O}_status.txt
