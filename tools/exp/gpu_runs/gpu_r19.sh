set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r19_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r19_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r19_benchB.json 2> gpurun_out/r19_benchB.err; echo "benchB=$?" >> gpurun_out/r19_status.txt
timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r19_benchD.json 2> gpurun_out/r19_benchD.err; echo "benchD=$?" >> gpurun_out/r19_status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg_fwd --launch-skip 18 -c 1 -o gpurun_out/r19_aggfwd python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r19_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/r19_status.txt
