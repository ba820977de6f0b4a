set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg --launch-skip 36 -c 12 -o gpurun_out/r16_agg python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r16_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/r16_status.txt
