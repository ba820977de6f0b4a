set -x
mkdir -p gpurun_out
cp paper_2207_11333_b200/lib/libhgnn.so /tmp/libhgnn_default.so
for v in default pdl; do
  if [ $v = default ]; then cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so; else cp paper_2207_11333_b200/lib/variants/libhgnn_$v.so paper_2207_11333_b200/lib/libhgnn.so; fi
  if [ $v = pdl ]; then timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange.py -x -q > gpurun_out/r24_pytest_pdl.log 2>&1; echo "pytest_pdl=$?" >> gpurun_out/r24_status.txt; fi
  timeout 300 python bench.py --workload B --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r24_benchB_$v.json 2> gpurun_out/r24_benchB_$v.err; echo "benchB_$v=$?" >> gpurun_out/r24_status.txt
  timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r24_benchD_$v.json 2> gpurun_out/r24_benchD_$v.err; echo "benchD_$v=$?" >> gpurun_out/r24_status.txt
done
cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_degsort --launch-skip 3 -c 1 -o gpurun_out/r24_degsort python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r24_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/r24_status.txt
