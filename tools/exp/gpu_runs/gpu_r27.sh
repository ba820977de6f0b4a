set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r27_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r27_status.txt
timeout 300 python bench.py --workload B --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r27_benchB.json 2> gpurun_out/r27_benchB.err; echo "benchB=$?" >> gpurun_out/r27_status.txt
timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r27_benchD.json 2> gpurun_out/r27_benchD.err; echo "benchD=$?" >> gpurun_out/r27_status.txt
timeout 400 python bench.py --workload E256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r27_benchE256.json 2> gpurun_out/r27_benchE256.err; echo "benchE256=$?" >> gpurun_out/r27_status.txt
