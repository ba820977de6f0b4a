#!/bin/bash
# Weak-scaling bench lines at 1/2/4 GPUs (one process per GPU, torchrun, NCCL) for one workload.
#   bash tools/run_scale.sh <workload> <graphs per GPU> <out prefix> [gpu counts...]
set -u
w=$1; per=$2; out=$3; shift 3
counts=${*:-1 2 4}
for n in $counts; do
  g=$((per * n))
  if [ "$n" = 1 ]; then
    python bench.py --workload "$w" --graphs "$g" --steps 100 --warmup 10 --no-cpu-baseline > "${out}_${n}gpu.json" 2> "${out}_${n}gpu.err"
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 --master-port $((29500 + n)) \
      bench.py --gpus "$n" --workload "$w" --graphs "$g" --steps 100 --warmup 10 > "${out}_${n}gpu.json" 2> "${out}_${n}gpu.err"
  fi
  echo "$w n=$n rc=$? $(tail -c 300 "${out}_${n}gpu.json" | head -c 0)"
done
