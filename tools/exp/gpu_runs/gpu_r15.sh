set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r15_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r15_status.txt
timeout 300 python bench.py --workload B --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r15_benchB.json 2> gpurun_out/r15_benchB.err; echo "benchB=$?" >> gpurun_out/r15_status.txt
cp paper_2207_11333_b200/lib/libhgnn.so /tmp/libhgnn_default.so
for v in default r2b3 r3b2 r3b3; do
  if [ $v = default ]; then cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so; else cp paper_2207_11333_b200/lib/variants/libhgnn_$v.so paper_2207_11333_b200/lib/libhgnn.so; fi
  timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r15_benchD_$v.json 2> gpurun_out/r15_benchD_$v.err; echo "benchD_$v=$?" >> gpurun_out/r15_status.txt
done
cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so
