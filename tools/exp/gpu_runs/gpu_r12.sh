set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r12_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r12_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r12_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r12_benchB.json 2> gpurun_out/r12_benchB.err; echo "benchB=$?" >> gpurun_out/r12_status.txt
timeout 300 python bench.py --workload D --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r12_benchD.json 2> gpurun_out/r12_benchD.err; rc=$?; echo "benchD=$rc" >> gpurun_out/r12_status.txt
if [ $rc = 0 ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_agg --launch-skip 36 -c 2 -o gpurun_out/r12_agg python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r12_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/r12_status.txt
fi
