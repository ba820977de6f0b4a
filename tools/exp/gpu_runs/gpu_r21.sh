set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_tma|k_dxda|k_tmn" --launch-skip 87 -c 29 -o gpurun_out/r21_gemm python bench.py --workload D --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graphs 300000 > gpurun_out/r21_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/r21_status.txt
