set -x
mkdir -p gpurun_out
timeout 300 python tools/exp/timeline.py --graphs 20000 --B 128 > gpurun_out/r32_timeline_B.txt 2>&1; echo "tlB=$?" >> gpurun_out/r32_status.txt
timeout 300 python tools/exp/timeline.py --graphs 40000 --B 512 --dataset aisd > gpurun_out/r32_timeline_D.txt 2>&1; echo "tlD=$?" >> gpurun_out/r32_status.txt
for i in 1 2; do
timeout 300 python bench.py --workload B --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r32_benchB_$i.json 2> gpurun_out/r32_benchB_$i.err; echo "benchB=$?" >> gpurun_out/r32_status.txt
done
