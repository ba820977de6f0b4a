set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r17_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r17_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r17_benchB.json 2> gpurun_out/r17_benchB.err; echo "benchB=$?" >> gpurun_out/r17_status.txt
timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r17_benchD.json 2> gpurun_out/r17_benchD.err; echo "benchD=$?" >> gpurun_out/r17_status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg_bwd --launch-skip 18 -c 1 -o gpurun_out/r17_aggbwd python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r17_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/r17_status.txt
