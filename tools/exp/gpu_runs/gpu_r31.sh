set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r31_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r31_status.txt
timeout 300 python bench.py --workload B --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r31_benchB.json 2> gpurun_out/r31_benchB.err; echo "benchB=$?" >> gpurun_out/r31_status.txt
timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --graphs 300000 > gpurun_out/r31_benchD.json 2> gpurun_out/r31_benchD.err; echo "benchD=$?" >> gpurun_out/r31_status.txt
timeout 300 python tools/exp/timeline.py --graphs 20000 --B 128 > gpurun_out/r31_timeline_B.txt 2>&1; echo "tlB=$?" >> gpurun_out/r31_status.txt
