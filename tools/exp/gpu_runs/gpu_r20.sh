set -x
mkdir -p gpurun_out
timeout 300 python tools/exp/timeline.py --graphs 20000 --B 128 > gpurun_out/r20_timeline_B.txt 2>&1; echo "tlB=$?" > gpurun_out/r20_status.txt
timeout 300 python tools/exp/timeline.py --graphs 40000 --B 512 --dataset aisd > gpurun_out/r20_timeline_D.txt 2>&1; echo "tlD=$?" >> gpurun_out/r20_status.txt
