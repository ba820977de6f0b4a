#!/bin/bash
# Multi-GPU round-end set: DDP parity tests and weak-scaling bench lines (p2p and NCCL exchange)
#   bash tools/gpu_final_multi.sh N
set -x
N=$1
mkdir -p gpurun_out
O=gpurun_out/final${N}
nvidia-smi topo -m > ${O}_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ddp.py -q > ${O}_pytest_ddp.log 2>&1; echo "pytest=$?" > ${O}_status.txt
for w in B D; do
  g=$([ $w = B ] && echo $((200000 * N)) || echo $((150000 * N)))
  for ex in p2p nccl; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) \
      bench.py --gpus $N --workload $w --graphs $g --steps 30 --warmup 5 --exchange $ex > ${O}_bench_${w}_${ex}.json 2> ${O}_bench_${w}_${ex}.err
    echo "bench_${w}_${ex}=$?" >> ${O}_status.txt
  done
done
timeout 300 python bench.py --workload B --graphs 200000 --steps 30 --warmup 5 --no-cpu-baseline > ${O}_bench_B_1gpu.json 2> ${O}_bench_B_1gpu.err; echo "bench1=$?" >> ${O}_status.txt
timeout 300 python bench.py --workload D --graphs 150000 --steps 30 --warmup 5 --no-cpu-baseline > ${O}_bench_D_1gpu.json 2> ${O}_bench_D_1gpu.err; echo "bench1D=$?" >> ${O}_status.txt
