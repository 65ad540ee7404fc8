#!/bin/bash
# Pipeline bench logic with several ranks on ONE GPU (gloo host staging instead of NCCL).
#   tools/pp_bench_check.sh [steps] [config] [ranks]
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${3:-2} \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --pp-backend gloo --gpus ${3:-2} --steps ${1:-20} --warmup 3 ${2:+--config $2}
