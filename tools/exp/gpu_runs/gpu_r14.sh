set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r14_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r14_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r14_benchB.json 2> gpurun_out/r14_benchB.err; echo "benchB=$?" >> gpurun_out/r14_status.txt
timeout 300 python bench.py --workload D --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r14_benchD.json 2> gpurun_out/r14_benchD.err; rc=$?; echo "benchD=$rc" >> gpurun_out/r14_status.txt
if [ $rc = 0 ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg --launch-skip 36 -c 12 -o gpurun_out/r14_agg python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r14_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/r14_status.txt
fi
