set -x
mkdir -p gpurun_out
cp paper_2207_11333_b200/lib/libhgnn.so /tmp/libhgnn_default.so
cp paper_2207_11333_b200/lib/variants/libhgnn_simt.so paper_2207_11333_b200/lib/libhgnn.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r42_pytest_simt.log 2>&1; echo "pytest_simt=$?" > gpurun_out/r42_status.txt
for i in 1 2; do
for v in default simt; do
  if [ $v = default ]; then cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so; else cp paper_2207_11333_b200/lib/variants/libhgnn_$v.so paper_2207_11333_b200/lib/libhgnn.so; fi
  timeout 300 python bench.py --workload B --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r42_benchB_${v}_$i.json 2> gpurun_out/r42_benchB_${v}_$i.err; echo "benchB_$v=$?" >> gpurun_out/r42_status.txt
done
done
cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so
