set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r45_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/r45_status.txt
timeout 300 python tools/exp/timeline.py --graphs 20000 --B 128 > gpurun_out/r45_timeline_B.txt 2>&1; echo "tlB=$?" >> gpurun_out/r45_status.txt
cp paper_2207_11333_b200/lib/libhgnn.so /tmp/libhgnn_default.so
for i in 1 2; do
for v in default old; do
  if [ $v = default ]; then cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so; else cp paper_2207_11333_b200/lib/variants/libhgnn_$v.so paper_2207_11333_b200/lib/libhgnn.so; fi
  timeout 300 python bench.py --workload B --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r45_benchB_${v}_$i.json 2> gpurun_out/r45_benchB_${v}_$i.err; echo "benchB_$v=$?" >> gpurun_out/r45_status.txt
  if [ $i = 1 ]; then
  timeout 300 python bench.py --workload D --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r45_benchD_${v}.json 2> gpurun_out/r45_benchD_${v}.err; echo "benchD_$v=$?" >> gpurun_out/r45_status.txt
  fi
done
done
cp /tmp/libhgnn_default.so paper_2207_11333_b200/lib/libhgnn.so
