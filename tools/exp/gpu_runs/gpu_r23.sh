set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r23_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r23_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r23_benchB.json 2> gpurun_out/r23_benchB.err; echo "benchB=$?" >> gpurun_out/r23_status.txt
timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r23_benchD.json 2> gpurun_out/r23_benchD.err; echo "benchD=$?" >> gpurun_out/r23_status.txt
timeout 300 python tools/exp/timeline.py --graphs 20000 --B 128 > gpurun_out/r23_timeline_B.txt 2>&1; echo "tlB=$?" >> gpurun_out/r23_status.txt
timeout 300 python tools/exp/timeline.py --graphs 40000 --B 512 --dataset aisd > gpurun_out/r23_timeline_D.txt 2>&1; echo "tlD=$?" >> gpurun_out/r23_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --precision tf32 > gpurun_out/r23_benchB_tf32.json 2> gpurun_out/r23_benchB_tf32.err; echo "benchBtf32=$?" >> gpurun_out/r23_status.txt
timeout 400 python bench.py --workload E256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r23_benchE256.json 2> gpurun_out/r23_benchE256.err; echo "benchE256=$?" >> gpurun_out/r23_status.txt
timeout 400 python bench.py --workload E256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 --precision tf32 > gpurun_out/r23_benchE256_tf32.json 2> gpurun_out/r23_benchE256_tf32.err; echo "benchE256tf32=$?" >> gpurun_out/r23_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --variant all > gpurun_out/r23_benchB_all.json 2> gpurun_out/r23_benchB_all.err; echo "benchBall=$?" >> gpurun_out/r23_status.txt
