set -x
mkdir -p gpurun_out
cp paper_2207_11333_b200/lib/libhgnn.so /tmp/libhgnn_default.so
for i in 1 2; do
for v in default dmx64 dmx128; do
  if [ $v = default ]; then cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so; else cp paper_2207_11333_b200/lib/variants/libhgnn_$v.so paper_2207_11333_b200/lib/libhgnn.so; fi
  timeout 300 python bench.py --workload B --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r47_benchB_${v}_$i.json 2> gpurun_out/r47_benchB_${v}_$i.err; echo "benchB_$v=$?" >> gpurun_out/r47_status.txt
done
done
cp paper_2207_11333_b200/lib/variants/libhgnn_dmx64.so paper_2207_11333_b200/lib/libhgnn.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r47_pytest_dmx64.log 2>&1; echo "pytest64=$?" >> gpurun_out/r47_status.txt
cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so
