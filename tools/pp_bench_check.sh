#!/bin/bash
# Pipeline bench logic with several ranks on ONE GPU (gloo host staging instead of NCCL).
#   tools/pp_bench_check.sh [steps] [config] [ranks] [extra bench args...]
steps=${1:-20}; cfg=$2; ranks=${3:-2}; shift 3 2>/dev/null || shift $#
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $ranks \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --pp-backend gloo --gpus $ranks --steps $steps --warmup 3 ${cfg:+--config $cfg} "$@"
